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


def test_nonpositive_batch_values_are_skipped():
    """ParallelConfig(batch<1) raises and enumerate_candidates skips it (search.py:101-105,
    model.py:190-193): batch values (0, -2, 1, 8) give the report of (1, 8); (0,) gives none.
    (A workload's batch_sweep cannot hold them: WorkloadSpec rejects it, serving_modes.py:94-95.)"""
    import dataclasses

    import paper_2601_06288_b200 as pkg
    from golden_io import canonical, db_path, diff_canonical, model_doc
    from oracle import oracle

    case = BY_NAME["a1_qwen_small"]
    db, model, workload, space, dc = case_objects(case)
    space = dataclasses.replace(space, tp_values=(1, 2), pp_values=(1, 2), dp_values=(1, 2))

    def run(batches):
        return pkg.run_search(db, model, workload, dataclasses.replace(space, batch_values=batches),
                              disagg_constants=dc).to_doc()

    got, want = run((0, -2, 1, 8)), run((1, 8))
    got.pop("timing"), want.pop("timing")
    assert got == want and got["counts"]["enumerated"] > 0
    header, recs = oracle.read_db_records(db_path(case))
    ref = oracle.run_search(header, recs, model_doc(case["model"]), case["workload"],
                            {"tp_values": [1, 2], "pp_values": [1, 2], "dp_values": [1, 2], "batch_values": [1, 8]},
                            disagg=case.get("disagg"))
    assert not diff_canonical(canonical(got), canonical(ref))
    none = run((0,))
    assert none["counts"]["enumerated"] == 0 and none["rows"] == [] and none["best"] is None


def test_handle_caches_are_bounded_and_keyed_on_plan_fields():
    """Distinct spaces that share the plan fields reuse one device plan; many distinct
    plans stay under the LRU bound, evicted handles are freed, and results stay right."""
    import dataclasses

    import paper_2601_06288_b200 as pkg
    from paper_2601_06288_b200.engine import Engine, build_report

    db, model, workload, space, dc = case_objects(BY_NAME["a1_qwen_small"])
    eng = Engine(0)
    try:
        base = dataclasses.replace(space, tp_values=(1, 2), pp_values=(1,), dp_values=(1,), batch_values=(1, 8))
        out = eng.run_batch(db, model, base, [workload], dc)
        want = build_report(out, 0, db, model, workload, base, 0.0).to_doc()
        for caps in ((4, 4), (2, 8), (8, 16)):  # pool caps / batches are per search, not per plan
            sp = dataclasses.replace(base, prefill_pool_cap=caps[0], decode_pool_cap=caps[1], batch_values=(8, 1))
            eng.run_batch(db, model, sp, [workload], dc)
        assert len(eng._spaces) == 1
        for i in range(eng.MAX_SPACES + 8):
            sp = dataclasses.replace(base, dp_values=(1, 2 + i))
            eng.run_batch(db, model, sp, [workload], dc)
        assert len(eng._spaces) <= eng.MAX_SPACES
        out = eng.run_batch(db, model, base, [workload], dc)
        got = build_report(out, 0, db, model, workload, base, 0.0).to_doc()
        got.pop("timing"), want.pop("timing")
        assert got == want
        ref = pkg.run_search(db, model, workload, base, disagg_constants=dc).to_doc()
        ref.pop("timing")
        assert got == ref
    finally:
        eng.close()


@pytest.mark.parametrize("caps", [(24, 10), (32, 8), (40, 6), (64, 4), (4, 64), (17, 15)])
@pytest.mark.parametrize("name", ["a1_qwen_small", "cfg4_dsv3", "flat_ties"])
def test_large_pool_caps_match_oracle(name, caps):
    """Pool caps above 16 (the warp top-k fast path holds up to 32, larger caps take the
    per-search rounds): sorted(pool, key=_pool_rank)[:cap] (search.py:336-339) vs the oracle."""
    import dataclasses

    import paper_2601_06288_b200 as pkg
    from golden_io import canonical, db_path, diff_canonical, hw_docs, model_doc
    from oracle import oracle

    case = BY_NAME[name]
    db, model, workload, space, dc = case_objects(case)
    space = dataclasses.replace(space, prefill_pool_cap=caps[0], decode_pool_cap=caps[1])
    got = pkg.run_search(db, model, workload, space, disagg_constants=dc).to_doc()
    header, recs = oracle.read_db_records(db_path(case))
    header, recs = oracle.mutate(header, recs, case.get("mutation"), hw_docs())
    sp = dict(case.get("space", {}), prefill_pool_cap=caps[0], decode_pool_cap=caps[1])
    ref = oracle.run_search(header, recs, model_doc(case["model"]), case["workload"], sp, disagg=case.get("disagg"),
                            extrapolation=case.get("extrapolation", "default"))
    diffs = diff_canonical(canonical(got), canonical(ref))
    assert not diffs, "\n".join(diffs)
