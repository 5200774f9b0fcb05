"""get_step_latency / get_mix_latency / get_gen_latency with the per-label breakdown
(estimator.py:71-156) on the device, against 960 golden requests produced by the
unmodified reference (tests/golden/make_step_golden.py): totals and every
breakdown entry bit-exact, labels in plan order, identical exceptions.

The ParallelConfigError cases are decided on the host before any launch, so
they are checked on the CPU too."""

from __future__ import annotations

import gzip
import json
from pathlib import Path

import pytest

import paper_2601_06288_b200 as pkg
from golden_io import hw_doc, model_doc

GOLDEN = Path(__file__).resolve().parent / "golden"
_DB: dict = {}


def _requests():
    return json.loads(gzip.decompress((GOLDEN / "steps.json.gz").read_bytes()))["requests"]


def _db(model, extrapolation, mutation):
    from paper_2601_06288_b200.database import with_records

    key = (model, extrapolation, mutation)
    if key not in _DB:
        db = pkg.load_db(GOLDEN / "db" / f"db-{model}-h100-sxm-s11.jsonl.gz", extrapolation=extrapolation)
        if mutation and mutation.startswith("drop_kind:"):
            kind = mutation.split(":", 1)[1]
            db = with_records(db, [r for r in db.records if r.kind != kind])
        elif mutation and mutation.startswith("swap_hw:"):
            db = with_records(db, hardware=pkg.HardwareSpec.from_doc(hw_doc(mutation.split(":", 1)[1])))
        _DB[key] = db
    return _DB[key]


def _groups():
    groups: dict = {}
    for r in _requests():
        groups.setdefault((r["model"], r["extrapolation"], r["mutation"]), []).append(r)
    return groups


def _run(key, recs):
    from paper_2601_06288_b200.steps import StepRequest, step_latency_batch

    db = _db(*key)
    model = pkg.ModelSpec.from_doc(model_doc(key[0]))
    space = pkg.CandidateSpace()
    reqs = []
    for r in recs:
        load = pkg.PowerLawParams(**r["moe_load"]) if r["moe_load"] else None
        reqs.append(StepRequest(space.config(*r["cfg"], db.backend), r["phase"], r["n_ctx"], r["n_gen"], r["seq"],
                                load))
    return step_latency_batch(db, model, reqs)


def _assert_same(r, got):
    if "error" in r:
        assert isinstance(got, Exception), (r, got)
        assert f"{type(got).__name__}: {got}" == r["error"]
    else:
        assert not isinstance(got, Exception), (r, got)
        assert got.total_ms.hex() == r["total"], r
        assert [[k, v.hex()] for k, v in got.breakdown.items()] == r["breakdown"], r


def test_parallel_config_errors_on_host():
    from paper_2601_06288_b200.specs import ParallelConfigError
    from paper_2601_06288_b200.steps import _check

    n = 0
    for r in _requests():
        if not r.get("error", "").startswith("ParallelConfigError"):
            continue
        model = pkg.ModelSpec.from_doc(model_doc(r["model"]))
        cfg = pkg.CandidateSpace().config(*r["cfg"], "trtllm")
        with pytest.raises(ParallelConfigError) as ei:
            _check(model, cfg, r["phase"], r["n_ctx"], r["n_gen"], r["seq"])
        assert f"ParallelConfigError: {ei.value}" == r["error"]
        n += 1
    assert n > 100


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(_groups(), key=str), ids=lambda k: "-".join(str(x) for x in k))
def test_step_latency_matches_reference(key):
    recs = _groups()[key]
    for r, got in zip(recs, _run(key, recs)):
        _assert_same(r, got)


@pytest.mark.gpu
def test_mix_and_gen_wrappers_and_static_ttft():
    """get_mix/gen_latency are get_step_latency at the KV midpoint; the static
    estimate's TTFT is the prefill step's total (serving_modes.py:250-254)."""
    from paper_2601_06288_b200.steps import get_gen_latency, get_mix_latency, get_step_latency

    db = _db("deepseek-v3", "default", None)
    model = pkg.ModelSpec.from_doc(model_doc("deepseek-v3"))
    cfg = pkg.CandidateSpace().config(8, 2, 8, 1, 64, db.backend)
    mix = get_mix_latency(db, model, cfg, 2048, 63, 4000, 500)
    assert mix == get_step_latency(db, model, cfg, "mixed", n_ctx_tokens=2048, n_gen_tokens=63, seq_len=4250)
    gen = get_gen_latency(db, model, cfg, 64, 4000, 500)
    assert gen == get_step_latency(db, model, cfg, "decode", n_gen_tokens=64, seq_len=4250)
    wl = pkg.WorkloadSpec(isl=4000, osl=500)
    est = pkg.estimate_static(db, model, cfg, wl)
    pre = get_step_latency(db, model, cfg, "prefill", n_ctx_tokens=64 * 4000, seq_len=4000)
    assert est.ttft_ms == pre.total_ms
    assert abs(sum(pre.breakdown.values()) - pre.total_ms) <= 1e-9 * pre.total_ms
