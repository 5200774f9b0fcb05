"""The CPU oracle is pinned to the reference: golden reports, MoE and sum() KATs.

Goldens were produced by the unmodified reference (tests/golden/make_golden.py).
"""

from __future__ import annotations

import math

import pytest

from golden_io import CASES, canonical, db_path, diff_canonical, golden_report, hw_docs, model_doc, moe_kats, sum_kats
from oracle import oracle


def run_case(case):
    header, recs = oracle.read_db_records(db_path(case))
    header, recs = oracle.mutate(header, recs, case.get("mutation"), hw_docs())
    return oracle.run_search(header, recs, model_doc(case["model"]), case["workload"], case.get("space"),
                             case.get("disagg"), case.get("extrapolation", "default"))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference_report(case):
    doc = run_case(case)
    diffs = diff_canonical(canonical(doc), canonical(golden_report(case["name"])))
    assert not diffs, "\n".join(diffs)


def test_neumaier_sum_kats():
    for kat in sum_kats()[:1500]:
        xs = [float.fromhex(x) for x in kat["xs"]]
        assert oracle.neumaier_sum(xs).hex() == kat["sum"]


def test_moe_apportionment_kats():
    for kat in moe_kats():
        tail, counts = oracle.busiest_shard(kat["weights"], kat["total"], kat["topk"], kat["ep"])
        assert counts == kat["counts"]
        assert tail == kat["busiest"]


def test_moe_weights_match_reference_draw():
    for kat in moe_kats()[:: 12]:
        w = oracle.moe_weights({k: kat[k] for k in ("alpha", "x_min", "x_max", "seed")}, kat["num_experts"])
        assert [x.hex() for x in w] == [float(x).hex() for x in kat["weights"]]
