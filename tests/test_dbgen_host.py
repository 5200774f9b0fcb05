"""Host side of the device database generator (paper_2601_06288_b200/dbgen.py):
the grid harvest for a model must give exactly the grids of the reference's
generated databases (grid_spec_for_model, model.py:501-545), and GridAxes
validates like perfdb.py:594-606."""

from __future__ import annotations

import pytest

from golden_io import GOLDEN, model_doc

DBS = sorted(p.name for p in (GOLDEN / "db").glob("db-*.jsonl.gz"))


def split_name(name: str) -> tuple[str, str]:
    stem = name.removeprefix("db-").removesuffix(".jsonl.gz")
    stem = stem[: stem.rindex("-s")]
    for hw in ("h100-sxm", "b200-sxm", "a100-sxm"):
        if stem.endswith("-" + hw):
            return stem[: -len(hw) - 1], hw
    raise ValueError(name)


@pytest.mark.parametrize("name", DBS)
def test_grid_spec_matches_reference_database(name):
    import paper_2601_06288_b200 as pkg

    model_name, _ = split_name(name)
    db = pkg.load_db(GOLDEN / "db" / name)
    spec = pkg.grid_spec_for_model(pkg.ModelSpec.from_doc(model_doc(model_name)))
    assert [g.key() for g in spec] == sorted(db._grids, key=repr)
    for g in spec:
        grid = db._grids[g.key()]
        assert tuple(a for a, _ in g.axes) == tuple(grid.axes)
        assert tuple(tuple(v) for _, v in g.axes) == tuple(tuple(v) for v in grid.axis_values)


def test_grid_axes_validation():
    from paper_2601_06288_b200.dbgen import GridAxes
    from paper_2601_06288_b200.specs import DbValidationError

    with pytest.raises(DbValidationError, match="unknown kind"):
        GridAxes("conv", "fp16", (), (("m", (1, 2)),))
    with pytest.raises(DbValidationError, match="axes must be"):
        GridAxes("gemm", "fp16", (("k", 8), ("n", 8)), (("tokens", (1, 2)),))
    with pytest.raises(DbValidationError, match="empty"):
        GridAxes("gemm", "fp16", (("k", 8), ("n", 8)), (("m", ()),))
    with pytest.raises(DbValidationError, match="strictly ascending"):
        GridAxes("gemm", "fp16", (("k", 8), ("n", 8)), (("m", (4, 2)),))


def test_hash_unit_matches_reference_definition():
    import hashlib

    from paper_2601_06288_b200.dbgen import _hash_unit

    key = ("gemm", "fp16", (("k", 4096), ("n", 4096)))
    want = int.from_bytes(hashlib.blake2b(f"11|{key}|offset".encode(), digest_size=8).digest(), "big") / 2.0**64
    assert _hash_unit(11, key, "offset") == want
    assert 0.0 <= want < 1.0
