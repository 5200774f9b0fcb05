"""Per-step DRAM traffic of the K2 stage from per-model ncu launch lists of
tools/profile_run.py (one config-5 batch of 100 searches per model, every kernel
launched >= 2 times):

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/lt_<model>.csv python tools/profile_run.py <model> 100
    python tools/k2_traffic_models.py gpurun_out/lt_gpt-oss-120b.csv gpurun_out/lt_deepseek-v3.csv \
        > profiles/r2_ncu_k2_traffic.json

One step of the config-5 bench = one pipeline pass of each model, so the K2
stage's bytes per step are the sum over models of the per-launch means of the K2
kernels.  The per-kernel table (time, DRAM bytes per launch) is printed with it.
"""

import csv
import json
import sys
from collections import defaultdict

K2 = ("k_qtables", "k_dstables", "k_dseries", "k_ptables", "k_eval_cells", "k_expand")
SCALE = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def per_kernel(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ix = {n: i for i, n in enumerate(h)}
    acc = defaultdict(lambda: defaultdict(list))
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("<unnamed>::", "").replace("void ", "").strip()
        name = name.split("<")[0] if name.startswith(("k_qtables", "k_dstables")) else name
        v = float(r[ix["Metric Value"]].replace(",", "") or 0) * SCALE.get(r[ix["Metric Unit"]].lower(), 1.0)
        acc[name][r[ix["Metric Name"]]].append(v)
    out = {}
    for k, m in acc.items():
        t = m.get("gpu__time_duration.sum", [])
        rd, wr = m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", [])
        out[k] = {"us": sum(t) / len(t) if t else None, "launches": len(t),
                  "dram_read": sum(rd) / len(rd) if rd else None, "dram_write": sum(wr) / len(wr) if wr else None}
    return out


models = {}
for path in sys.argv[1:]:
    name = path.rsplit("/", 1)[-1].removeprefix("lt_").removesuffix(".csv")
    models[name] = per_kernel(path)
k2 = 0.0
by = defaultdict(float)
for m, ks in models.items():
    for k, v in ks.items():
        if k in K2 and v["dram_read"] is not None:
            b = v["dram_read"] + v["dram_write"]
            k2 += b
            by[k] += b
print(json.dumps({"source": sys.argv[1:], "how": "per-launch means of each model's K2 kernels, summed over the "
                  "models (one pipeline pass per model per step)", "kernels": list(K2),
                  "dram_bytes_per_step": k2, "by_kernel_per_step": dict(by), "per_model": models}, indent=1))
