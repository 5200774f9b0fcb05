"""Refresh the round-2 profile artifacts from one tools/gpu_r2_final.sh <tag> run:

    python tools/r2_update_profiles.py <tag>

writes profiles/r2_ncu_k2_traffic.json (per-model launch lists), r2_ncu_kernels.md/.json
(ncu --set full table), r2_ncu_launches_bench.csv/.md (the bench's own launch list),
r2_pytest_gpu_head.txt and r2_bench_final.json.
"""
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
G, PR = ROOT / "gpurun_out", ROOT / "profiles"
tag = sys.argv[1]
run = lambda *a: subprocess.run([sys.executable, *a], capture_output=True, text=True, check=True).stdout

(PR / "r2_ncu_k2_traffic.json").write_text(run(str(ROOT / "tools/k2_traffic_models.py"),
                                                str(G / "lt_gpt-oss-120b.csv"), str(G / "lt_deepseek-v3.csv")))
tmp = G / "ncu_kernels_tmp.json"
(PR / "r2_ncu_kernels.md").write_text(run(str(ROOT / "tools/ncu_table.py"), str(G / f"prof_{tag}.ncu-rep"), "6553.6",
                                          f"--json={tmp}"))
d = json.loads(tmp.read_text())
fp64 = json.loads((PR / "fp64_peak.json").read_text())
json.dump({"source": f"profiles/r2_ncu_kernels.md (gpurun_out/prof_{tag}.ncu-rep: ncu --set full, one GPT-OSS-120B batch "
                     "of 100 config-5 searches, first launch of each kernel)",
           "hbm_peak_gbs": d["hbm_peak_gbs"], "fp64_fma_peak_gflops_measured": fp64["fp64_fma_gflops"],
           "k_eval_cells": d["kernels"].get("k_eval_cells"), "kernels": d["kernels"]},
          open(PR / "r2_ncu_kernels.json", "w"), indent=1)
lb = G / f"launches_bench_{tag}.csv"
if lb.exists() and lb.stat().st_size > 1000:
    shutil.copy(lb, PR / "r2_ncu_launches_bench.csv")
    out = run(str(ROOT / "tools/kernel_times.py"), str(PR / "r2_ncu_launches_bench.csv"))
    rows = []
    for l in out.strip().splitlines()[1:]:
        p = l.split()
        rows.append((" ".join(p[:-3]).replace("void ", ""), float(p[-3]), p[-1]))
    tot = sum(r[1] for r in rows)
    k2 = sum(r[1] for r in rows if r[0].split("<")[0] in ("k_qtables", "k_dstables", "k_dseries", "k_ptables",
                                                          "k_eval_cells", "k_expand"))
    md = ["# ncu launch list of the bench's own command (round 2, HEAD)\n",
          "`LC_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
          "--clock-control none -c 400 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --north-star none` "
          "(`tools/gpu_r2_final.sh`; direct launches, the same kernels the batch graph holds; raw list in "
          "`r2_ncu_launches_bench.csv`).\n",
          "Per-launch means over both models' pipelines (cold caches, serialised: compare shares, not absolute "
          "times).\n", "| kernel | µs per launch | launches | share |", "|---|---|---|---|"]
    md += [f"| {n} | {us:.1f} | {x} | {100 * us / tot:.1f} % |" for n, us, x in rows]
    md.append(f"\nK2 stage share: {100 * k2 / tot:.0f} %.")
    (PR / "r2_ncu_launches_bench.md").write_text("\n".join(md) + "\n")
log = (G / f"pytest_gpu_{tag}.log").read_text().strip().splitlines()
(PR / "r2_pytest_gpu_head.txt").write_text("\n".join(log[-3:]) + "\n")
b = (G / f"bench_{tag}.json").read_text().strip().splitlines()[-1]
(PR / "r2_bench_final.json").write_text(b + "\n")
print("updated")
