"""The oracle's query_latency restatement (oracle.c query_latency_p) is pinned to
the reference's own single-query answers: the unit-test KATs of
pkg/tests/test_perfdb.py, every query two reference searches issue, and seeded
probes of every grid under each extrapolation policy
(tests/golden/make_query_golden.py).  Also checks the product's host-side query
packing (paper_2601_06288_b200/queries.py) without a device."""

from __future__ import annotations

import pytest

from golden_io import BY_NAME, db_path, hw_docs, query_goldens, query_groups
from oracle import oracle

DOC = query_goldens()
GROUPS = query_groups(DOC)


def oracle_db(name: str):
    src = DOC["dbs"][name]
    if "inline" in src:
        return src["inline"]["header"], src["inline"]["records"], "default"
    case = BY_NAME[src["case"]]
    header, recs = oracle.read_db_records(db_path(case))
    header, recs = oracle.mutate(header, recs, case.get("mutation"), hw_docs())
    return header, recs, case.get("extrapolation", "default")


@pytest.mark.parametrize("group", sorted(GROUPS, key=repr), ids=lambda g: f"{g[0]}-{g[1]}")
def test_oracle_query_latency_matches_reference(group):
    name, policy = group
    vecs = [v for v in GROUPS[group] if "backend" not in v["query"]]  # backend check is host-side
    header, recs, extrap = oracle_db(name)
    got = oracle.query_batch(header, recs, [v["query"] for v in vecs], policy, extrap)
    for v, (val, msg) in zip(vecs, got):
        want = v["expect"]
        assert (val.hex() if val is not None else msg) == want, v["query"]


def test_golden_query_set_covers_policies_and_errors():
    exp = [v["expect"] for v in DOC["vectors"]]
    for kind in ("MissingKeyError", "ExtrapolationError", "UnsupportedOperatorError"):
        assert any(e.startswith(kind + ":") for e in exp), kind
    assert {v["policy"] for v in DOC["vectors"]} == {None, "default", "strict", "clamp", "sol"}
    assert sum(1 for v in DOC["vectors"] if "kv_len" in v["query"]["shape"]) >= 10
    assert len(DOC["vectors"]) > 4000


def test_query_packing_matches_canonical_dims():
    import paper_2601_06288_b200 as pkg
    from paper_2601_06288_b200 import queries as Q
    from paper_2601_06288_b200.database import flatten
    from product_cases import case_db

    db = case_db(BY_NAME["dsv3_all_default"])
    flat = flatten(db)
    qs = [Q.OperatorQuery(**v["query"]) for v in DOC["vectors"] if v["db"] == "case:dsv3_all_default"][:300]
    arr = Q._pack(flat, qs, 2)
    for q, row in zip(qs, arr):
        dims = dict(q.shape)
        assert row["grid"] == flat.index.get(q.grid_key(), -1)
        assert list(row["d"][: len(pkg.database.KIND_DIMS[q.kind][0])]) == [dims[n] for n in
                                                                            pkg.database.KIND_DIMS[q.kind][0]]
        assert row["policy"] == 2
        assert row["kv_len"] == dims.get("kv_len", -1)
