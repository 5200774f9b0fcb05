"""End-to-end single-search timing with full report JSON: object path vs columnar path.

One config-5 search (GPT-OSS-120B, ISL 4000 / OSL 500, batch 1..512, all modes).
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_06288_b200 as pkg  # noqa: E402
from paper_2601_06288_b200.sweeps import sweep  # noqa: E402

part = sweep("config5")[0]
w = part.workloads[44]
for _ in range(2):
    pkg.run_search_json(part.db, part.model, w, part.space)
t0 = time.perf_counter()
rep = pkg.run_search(part.db, part.model, w, part.space)
t1 = time.perf_counter()
slow = rep.to_json()
t2 = time.perf_counter()
fast = pkg.run_search_json(part.db, part.model, w, part.space)
t3 = time.perf_counter()
import json  # noqa: E402
a, b = json.loads(slow), json.loads(fast)
a.pop("timing"), b.pop("timing")
assert a == b
print(f"isl={w.isl} osl={w.osl}: rows={len(rep.rows)} json={len(fast) / 1e6:.1f} MB")
print(f"run_search (objects) {1000 * (t1 - t0):.1f} ms + to_json {1000 * (t2 - t1):.1f} ms; "
      f"run_search_json {1000 * (t3 - t2):.1f} ms")
