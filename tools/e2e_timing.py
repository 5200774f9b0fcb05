"""Where the e2e step's time goes: per-model host timestamps around run_batch /
fetch_fronts with both models in flight (as bench.py's e2e leg runs them)."""
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_06288_b200.engine import Engine, fetch_fronts  # noqa: E402
from paper_2601_06288_b200.sweeps import sweep  # noqa: E402

parts = sweep("config5")
engs = {p.model_name: Engine(0) for p in parts}
pool = ThreadPoolExecutor(max_workers=2)
T0 = [0.0]


def one(p):
    e = engs[p.model_name]
    a = time.perf_counter()
    out = e.run_batch(p.db, p.model, p.space, p.workloads)
    b = time.perf_counter()
    fetch_fronts(out)
    c = time.perf_counter()
    return p.model_name, (a - T0[0]) * 1e3, (b - T0[0]) * 1e3, (c - T0[0]) * 1e3, sum(out.totals.kernel_ms)


for it in range(8):
    T0[0] = time.perf_counter()
    res = list(pool.map(one, parts))
    end = (time.perf_counter() - T0[0]) * 1e3
    if it >= 5:
        for r in res:
            print(f"{r[0]:14s} start {r[1]:.3f} run_batch done {r[2]:.3f} fetched {r[3]:.3f} (device events {r[4]:.3f})")
        print(f"step {end:.3f} ms")
