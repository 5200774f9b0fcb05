"""CUDA engine parity: every golden case through the product path (C ABI via
ctypes), compared with the reference's own report (bit-exact floats, identical
rows / skips / fronts / best / diagnostics, byte-identical documents) and with
the CPU oracle run on this box."""

from __future__ import annotations

import json

import pytest

from golden_io import CASES, canonical, diff_canonical, golden_report, hw_docs, model_doc, db_path
from product_cases import case_objects

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2601_06288_b200 as p

    return p


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_engine_matches_reference_golden(pkg, case):
    db, model, workload, space, dc = case_objects(case)
    report = pkg.run_search(db, model, workload, space, disagg_constants=dc)
    doc = report.to_doc()
    golden = golden_report(case["name"])
    diffs = diff_canonical(canonical(doc), canonical(golden))
    assert not diffs, "\n".join(diffs)
    # whole document identical apart from timing (what the CLI / service emit)
    doc.pop("timing")
    golden.pop("_meta")
    assert json.dumps(doc, sort_keys=True) == json.dumps(golden, sort_keys=True)


@pytest.mark.parametrize("name", ["cfg4_dsv3", "moe_load_custom", "strict_long_isl", "flat_ties"])
def test_engine_matches_oracle_on_this_box(pkg, name):
    from oracle import oracle
    from golden_io import BY_NAME

    case = BY_NAME[name]
    db, model, workload, space, dc = case_objects(case)
    report = pkg.run_search(db, model, workload, space, disagg_constants=dc)
    header, recs = oracle.read_db_records(db_path(case))
    header, recs = oracle.mutate(header, recs, case.get("mutation"), hw_docs())
    ref = oracle.run_search(header, recs, model_doc(case["model"]), case["workload"], case.get("space"),
                            case.get("disagg"), case.get("extrapolation", "default"))
    diffs = diff_canonical(canonical(report.to_doc()), canonical(ref))
    assert not diffs, "\n".join(diffs)


def test_enumerate_candidates_matches_reference_counts(pkg):
    from golden_io import BY_NAME

    for name in ("cfg3_llama70b_kv50", "cfg4_dsv3", "default_big_batch"):
        case = BY_NAME[name]
        db, model, workload, space, dc = case_objects(case)
        cands = pkg.enumerate_candidates(model, space, workload, db)
        assert len(cands) == golden_report(name)["counts"]["enumerated"]


@pytest.mark.parametrize("name", ["cfg2_qwen3_disagg", "cfg4_dsv3", "missing_tp16", "unmeetable_sla", "flat_ties_moe",
                                  "gptoss_all_default"])
def test_columnar_json_matches_object_report(pkg, name):
    from golden_io import BY_NAME
    from paper_2601_06288_b200.engine import build_report, get_engine
    from paper_2601_06288_b200.fastreport import columns_from_batch, report_json

    case = BY_NAME[name]
    db, model, workload, space, dc = case_objects(case)
    eng = get_engine(0)
    with eng._lock:
        out = eng.run_batch(db, model, space, [workload], dc)
        slow = build_report(out, 0, db, model, workload, space, 7.25).to_json()
        fast = report_json(columns_from_batch(out, 0, db, model, workload, space, 7.25))
    assert fast == slow
    doc = json.loads(fast)
    doc.pop("timing")
    golden = golden_report(name)
    golden.pop("_meta")
    assert json.dumps(doc, sort_keys=True) == json.dumps(golden, sort_keys=True)
