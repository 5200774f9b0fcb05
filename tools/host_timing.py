"""Host-side breakdown of one e2e sweep step (run_batch + fetch_fronts)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2601_06288_b200.engine import Engine, fetch_fronts
from paper_2601_06288_b200.sweeps import sweep

parts = sweep("config5")
engs = {p.model_name: Engine(0) for p in parts}
for _ in range(2):
    for p in parts:
        out = engs[p.model_name].run_batch(p.db, p.model, p.space, p.workloads)
        fetch_fronts(out)
for p in parts:
    e = engs[p.model_name]
    t0 = time.perf_counter()
    out = e.run_batch(p.db, p.model, p.space, p.workloads)
    t1 = time.perf_counter()
    fetch_fronts(out)
    t2 = time.perf_counter()
    print(f"{p.model_name}: run_batch {1000*(t1-t0):.2f} ms (device {sum(out.totals.kernel_ms):.2f} ms), fetch_fronts {1000*(t2-t1):.2f} ms")
import cProfile, pstats
p = parts[0]
pr = cProfile.Profile(); pr.enable()
out = engs[p.model_name].run_batch(p.db, p.model, p.space, p.workloads); fetch_fronts(out)
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(14)

# front / plan statistics of the sweep
for p in parts:
    out = engs[p.model_name].run_batch(p.db, p.model, p.space, p.workloads)
    r = out.results
    print(p.model_name, "n_front max/mean", int(r["n_front"].max()), float(r["n_front"].mean()),
          "n_plans max", int(r["n_plans"].max()), "units/search max", int(r["n_units"].max()),
          "feasible mean", float(r["n_feasible"].mean()))
