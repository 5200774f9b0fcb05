"""K4's survivor-overflow path: with more Pareto survivors than fit the sorted
front scan (2,048 in shared memory), k_front_final walks the staircase over
every row.  LC_SURVIVOR_CAP (read once per process) lowers the cap, so a
subprocess runs every golden case through that path and compares each report
with the reference's (search.py:156-208: same front, best and tie-breaks)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import json, sys
sys.path[:0] = [{root!r}, {tests!r}]
from golden_io import CASES, canonical, diff_canonical, golden_report
from product_cases import case_objects
import paper_2601_06288_b200 as pkg
bad, fronts = [], 0
for case in CASES:
    db, model, workload, space, dc = case_objects(case)
    doc = pkg.run_search(db, model, workload, space, disagg_constants=dc).to_doc()
    fronts += len(doc["frontier"])
    d = diff_canonical(canonical(doc), canonical(golden_report(case["name"])))
    if d:
        bad.append((case["name"], d[:3]))
print(json.dumps({{"bad": bad, "cases": len(CASES), "front_rows": fronts}}))
"""


@pytest.mark.parametrize("cap", [1, 3])
def test_overflow_path_matches_reference(cap):
    env = dict(os.environ, LC_SURVIVOR_CAP=str(cap))
    code = SCRIPT.format(root=str(ROOT), tests=str(ROOT / "tests"))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    import json

    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["cases"] >= 30 and res["front_rows"] > 100
    assert not res["bad"], res["bad"]
