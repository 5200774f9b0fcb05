"""Binary SoA cache of a database (paper_2601_06288_b200/soa.py): the image,
records, provenance and header survive the round trip exactly; a stale cache is
rebuilt; the extrapolation policy is applied at load time."""

from __future__ import annotations

import os
import shutil

import numpy as np
import pytest

from golden_io import GOLDEN

DBS = sorted(p.name for p in (GOLDEN / "db").glob("db-*.jsonl.gz"))


def _same_flat(a, b):
    assert a.keys == b.keys and a.axes == b.axes and a.axis_values == b.axis_values and a.kinds == b.kinds
    assert a.policy == b.policy
    for f in ("grid_ndim", "grid_axis_off", "grid_axis_len", "grid_cell_off", "axis_val"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    for f in ("axis_log", "cell", "cell_log"):
        assert getattr(a, f).view(np.uint64).tolist() == getattr(b, f).view(np.uint64).tolist(), f


@pytest.mark.parametrize("name", DBS[:3])
def test_soa_round_trip_is_exact(name, tmp_path):
    import paper_2601_06288_b200 as pkg
    from paper_2601_06288_b200.database import flatten
    from paper_2601_06288_b200.soa import load_soa, save_soa

    db = pkg.load_db(GOLDEN / "db" / name)
    save_soa(db, tmp_path / "x.npz")
    back = load_soa(tmp_path / "x.npz")
    _same_flat(flatten(back), flatten(db))
    assert back.hardware == db.hardware and back.backend == db.backend
    assert back.backend_version == db.backend_version
    assert back.records == db.records  # the files are in save_db order already
    assert sorted(back._grids, key=repr) == sorted(db._grids, key=repr)


def test_provenance_survives(tmp_path):
    import paper_2601_06288_b200 as pkg
    from paper_2601_06288_b200.database import OperatorRecord, with_records
    from paper_2601_06288_b200.soa import load_soa, save_soa

    db = pkg.load_db(GOLDEN / "db" / DBS[0])
    recs = [OperatorRecord(r.kind, r.quant, r.shape, r.latency_us, "measured" if i % 3 else "synthetic")
            for i, r in enumerate(db.records)]
    db2 = with_records(db, recs)
    save_soa(db2, tmp_path / "p.npz")
    assert load_soa(tmp_path / "p.npz").records == db2.records


def test_load_db_cache_reuses_and_rebuilds(tmp_path):
    import paper_2601_06288_b200 as pkg
    from paper_2601_06288_b200.database import flatten
    from paper_2601_06288_b200.soa import FlatBackedDatabase

    src = tmp_path / "db.jsonl.gz"
    shutil.copy(GOLDEN / "db" / DBS[1], src)
    first = pkg.load_db(src, soa_cache=True)
    assert not isinstance(first, FlatBackedDatabase)
    assert (tmp_path / "db.jsonl.gz.soa.npz").exists()
    second = pkg.load_db(src, extrapolation="strict", soa_cache=True)
    assert isinstance(second, FlatBackedDatabase)
    assert second.extrapolation == "strict" and flatten(second).policy == 1
    _same_flat(flatten(pkg.load_db(src, soa_cache=True)), flatten(first))
    shutil.copy(GOLDEN / "db" / DBS[2], src)  # source changed: cache is stale
    os.utime(src, ns=(1, 1))
    third = pkg.load_db(src, soa_cache=True)
    assert not isinstance(third, FlatBackedDatabase)
    _same_flat(flatten(third), flatten(pkg.load_db(GOLDEN / "db" / DBS[2])))
