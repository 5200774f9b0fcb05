"""query_latency on the device (lc_query_batch / k_query) against the reference's
single-query answers (tests/golden/queries.json.gz): float bits equal, error
type and message equal.  Covers the reference's test_perfdb KATs, every query
two reference searches issue, and per-grid probes under each policy."""

from __future__ import annotations

import math

import pytest

from golden_io import BY_NAME, query_goldens, query_groups

pytestmark = pytest.mark.gpu

DOC = query_goldens()
GROUPS = query_groups(DOC)


def product_db(name: str):
    import paper_2601_06288_b200 as pkg
    from paper_2601_06288_b200.database import OperatorRecord
    from product_cases import case_db

    src = DOC["dbs"][name]
    if "inline" in src:
        doc = src["inline"]
        recs = [OperatorRecord.make(r["kind"], r["quant"], r["shape"], r["latency_us"], r["provenance"])
                for r in doc["records"]]
        return pkg.PerfDatabase.from_records(pkg.HardwareSpec.from_doc(doc["header"]["hardware"]),
                                             doc["header"]["backend"], doc["header"]["backend_version"], recs)
    return case_db(BY_NAME[src["case"]])


@pytest.mark.parametrize("group", sorted(GROUPS, key=repr), ids=lambda g: f"{g[0]}-{g[1]}")
def test_device_query_latency_matches_reference(group):
    from paper_2601_06288_b200 import queries as Q

    name, policy = group
    vecs = GROUPS[group]
    db = product_db(name)
    qs = [Q.OperatorQuery(**v["query"]) for v in vecs]
    lat = Q.query_latency_batch(db, qs, policy, errors="nan")
    for v, q, x in zip(vecs, qs, lat):
        want = v["expect"]
        if ": " in want:
            assert math.isnan(x), v["query"]
            with pytest.raises(Exception) as ei:
                Q.query_latency(db, q, policy)
            assert f"{type(ei.value).__name__}: {ei.value}" == want
        else:
            assert float(x).hex() == want, v["query"]


def test_batch_raises_first_error_in_order():
    from paper_2601_06288_b200 import queries as Q
    from paper_2601_06288_b200.specs import ExtrapolationError

    db = product_db("kat_gemm_100_400")
    q = lambda m: Q.OperatorQuery("gemm", "fp16", {"m": m, "n": 4096, "k": 4096})  # noqa: E731
    out = Q.query_latency_batch(db, [q(16), q(64), q(32)])
    assert out[0] == 100.0 and out[1] == 400.0 and out[2] == pytest.approx(200.0, rel=1e-12)
    with pytest.raises(ExtrapolationError, match="'m': 8"):
        Q.query_latency_batch(db, [q(32), q(8), q(128)], policy="strict")
    assert Q.query_latency_batch(db, []).shape == (0,)
