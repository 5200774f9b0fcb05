"""Per-step DRAM traffic of the K2 stage from an ncu launch list of `bench.py --steps 1 --warmup 1`.

    python tools/k2_traffic.py gpurun_out/launches_vN.csv > profiles/ncu_k2_traffic.json

The launch list holds every launch of the run (the e2e warm-up, the staging
batch, the per-kernel replay, the timed replay and the e2e step).  Each model
runs the pipeline once per pass, so per-step traffic = total bytes of the K2
stage kernels / passes, with passes = launches of k_eval_cells / models.
"""

import csv
import json
import sys
from collections import defaultdict

K2 = ("k_qtables", "k_dstables", "k_dseries", "k_ptables", "k_eval_cells", "k_expand")  # k_expand: filtered path only
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
idx = {n: i for i, n in enumerate(h)}
bytes_by = defaultdict(float)
launches = defaultdict(set)
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    name = r[idx["Kernel Name"]].split("(")[0].replace("<unnamed>::", "")
    if name not in K2:
        continue
    launches[name].add(r[idx["ID"]])
    if r[idx["Metric Name"]].startswith("dram__bytes"):
        v = float(r[idx["Metric Value"]] or 0)
        unit = r[idx["Metric Unit"]].lower()
        scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(unit, 1)
        bytes_by[name] += v * scale
models = 2
passes = len(launches["k_eval_cells"]) / models
# bytes_by sums every launch of both models; one step = one pass of each model
per_step = sum(bytes_by.values()) / passes if passes else None
print(json.dumps({"source": sys.argv[1], "kernels": list(K2), "passes_per_model": passes,
                  "dram_bytes_per_step": per_step,
                  "by_kernel_per_step": {k: v / passes for k, v in bytes_by.items()}}, indent=2))
