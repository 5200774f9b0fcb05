"""Single-config seams (serving_modes.estimate_static / estimate_aggregated,
used by `llmconf estimate`, cli.py:227-228) on the device vs the CPU oracle:
same floats bit for bit, same exception type and message."""

from __future__ import annotations

import pytest

from golden_io import BY_NAME, db_path, hw_docs, model_doc
from product_cases import case_objects

pytestmark = pytest.mark.gpu

CONFIGS = [
    ("cfg4_dsv3", (8, 2, 8, 1, 128)),
    ("cfg4_dsv3", (4, 4, 2, 2, 512)),
    ("cfg4_dsv3", (1, 1, 1, 1, 4096)),       # does not fit memory: estimates still run (no filter)
    ("a1_qwen_small", (2, 2, 1, 4, 64)),
    ("moe_load_custom", (2, 1, 4, 2, 256)),
    ("missing_allreduce", (2, 1, 1, 1, 16)),  # MissingKeyError
    ("strict_long_isl", (1, 1, 1, 1, 4)),     # ExtrapolationError
    ("unsupported_quant_a100", (1, 1, 1, 1, 8)),
    ("no_chunking", (1, 1, 1, 1, 8)),         # aggregated: InfeasibleConfigError
    ("batch_too_small", (1, 1, 1, 1, 4)),
]


@pytest.mark.parametrize("name,cfg", CONFIGS, ids=[f"{n}-{'x'.join(map(str, c))}" for n, c in CONFIGS])
def test_single_config_estimates_match_oracle(name, cfg):
    import paper_2601_06288_b200 as pkg
    from oracle import oracle

    case = BY_NAME[name]
    db, model, workload, space, dc = case_objects(case)
    header, recs = oracle.read_db_records(db_path(case))
    header, recs = oracle.mutate(header, recs, case.get("mutation"), hw_docs())
    pc = space.config(*cfg, db.backend)
    for mode, fn in (("static", pkg.estimate_static), ("aggregated", pkg.estimate_aggregated)):
        ref = oracle.estimate(header, recs, model_doc(case["model"]), case["workload"], cfg, mode,
                              case.get("space"), case.get("extrapolation", "default"))
        if ref["status"]:
            kind, msg = ref["reason"].split(": ", 1)
            with pytest.raises(Exception) as ei:
                fn(db, model, pc, workload)
            assert type(ei.value).__name__ == kind
            assert str(ei.value) == msg
        else:
            est = fn(db, model, pc, workload)
            got = [est.ttft_ms, est.tpot_ms, est.speed, est.throughput_per_gpu]
            assert [x.hex() for x in got] == [float(x).hex() for x in ref["values"]]


def test_inconsistent_config_raises_parallel_config_error():
    import paper_2601_06288_b200 as pkg

    db, model, workload, space, dc = case_objects(BY_NAME["cfg4_dsv3"])
    bad = space.config(3, 1, 2, 1, 8, db.backend)
    with pytest.raises(pkg.specs.ParallelConfigError) as ei:
        pkg.estimate_static(db, model, bad, workload)
    assert "tp=3 does not divide num_heads=128" in str(ei.value)


STRIDE_CONFIGS = [("cfg4_dsv3", (8, 2, 8, 1, 128)), ("a1_qwen_small", (2, 2, 1, 4, 64)),
                  ("moe_load_custom", (2, 1, 4, 2, 256)), ("strict_long_isl", (1, 1, 1, 1, 4)),
                  ("cfg3_llama70b_kv90", (4, 2, 1, 1, 32))]


@pytest.mark.parametrize("stride", [1, 3, 7, 31, 33, 100, 10_000])
@pytest.mark.parametrize("name,cfg", STRIDE_CONFIGS, ids=[n for n, _ in STRIDE_CONFIGS])
def test_static_estimate_any_stride_matches_oracle(name, cfg, stride):
    """estimate_static(..., stride) for any stride >= 1 (serving_modes.py:236-265); stride 1 is
    acceptance A2's brute-force setting (pkg/tests/test_acceptance.py:96-135)."""
    import paper_2601_06288_b200 as pkg
    from oracle import oracle

    case = BY_NAME[name]
    db, model, workload, space, dc = case_objects(case)
    header, recs = oracle.read_db_records(db_path(case))
    header, recs = oracle.mutate(header, recs, case.get("mutation"), hw_docs())
    pc = space.config(*cfg, db.backend)
    ref = oracle.estimate(header, recs, model_doc(case["model"]), case["workload"], cfg, "static",
                          case.get("space"), case.get("extrapolation", "default"), stride=stride)
    if ref["status"]:
        kind, msg = ref["reason"].split(": ", 1)
        with pytest.raises(Exception) as ei:
            pkg.estimate_static(db, model, pc, workload, stride=stride)
        assert type(ei.value).__name__ == kind and str(ei.value) == msg
    else:
        est = pkg.estimate_static(db, model, pc, workload, stride=stride)
        got = [est.ttft_ms, est.tpot_ms, est.speed, est.throughput_per_gpu]
        assert [x.hex() for x in got] == [float(x).hex() for x in ref["values"]]


def test_stride_must_be_positive():
    import paper_2601_06288_b200 as pkg

    db, model, workload, space, dc = case_objects(BY_NAME["a1_qwen_small"])
    with pytest.raises(pkg.specs.WorkloadError):
        pkg.estimate_static(db, model, space.config(1, 1, 1, 1, 8, db.backend), workload, stride=0)
