"""Degenerate inputs through the C ABI: empty batches, searches with no
candidates, empty query lists -- the device path must return the reference's
empty answers, not fail."""

from __future__ import annotations

import pytest

from golden_io import BY_NAME
from product_cases import case_objects

pytestmark = pytest.mark.gpu


def test_empty_batch_of_searches():
    from paper_2601_06288_b200.engine import fetch_fronts, get_engine

    db, model, workload, space, dc = case_objects(BY_NAME["a1_qwen_small"])
    eng = get_engine(0)
    with eng._lock:
        out = eng.run_batch(db, model, space, [], dc)
        front, plans = fetch_fronts(out)
    assert len(out.results) == 0 and len(front) == 0 and all(len(v) == 0 for v in plans.values())


def test_search_without_consistent_candidates():
    import paper_2601_06288_b200 as pkg

    db, model, workload, _, dc = case_objects(BY_NAME["a1_qwen_small"])
    space = pkg.CandidateSpace(tp_values=(3,), pp_values=(1,), dp_values=(1,), batch_values=(1, 2))
    rep = pkg.run_search(db, model, workload, space, disagg_constants=dc)
    doc = rep.to_doc()
    assert doc["counts"] == {"enumerated": 0, "evaluated": 0, "feasible": 0, "frontier": 0, "skipped": 0}
    assert doc["best"] is None and doc["diagnostics"] is None and doc["rows"] == []


def test_batch_mixing_empty_and_full_searches():
    import paper_2601_06288_b200 as pkg
    from paper_2601_06288_b200.engine import build_report, get_engine

    db, model, workload, space, dc = case_objects(BY_NAME["a1_qwen_small"])
    huge = pkg.WorkloadSpec(isl=workload.isl, osl=workload.osl, gpu_budgets=(3,))  # no config uses 3 GPUs
    eng = get_engine(0)
    with eng._lock:
        out = eng.run_batch(db, model, space, [huge, workload, huge], dc)
        reps = [build_report(out, i, db, model, w, space, 0.0) for i, w in enumerate([huge, workload, huge])]
    full = pkg.run_search(db, model, workload, space, disagg_constants=dc).to_doc()
    mid = reps[1].to_doc()
    full.pop("timing"), mid.pop("timing")
    assert mid == full
    alone = pkg.run_search(db, model, huge, space, disagg_constants=dc).to_doc()
    alone.pop("timing")
    assert alone["counts"]["enumerated"] == 0
    for r in (reps[0], reps[2]):
        d = r.to_doc()
        d.pop("timing")
        assert d == alone


def test_empty_query_batch():
    import paper_2601_06288_b200 as pkg

    db, *_ = case_objects(BY_NAME["a1_qwen_small"])
    assert list(pkg.query_latency_batch(db, [])) == []
