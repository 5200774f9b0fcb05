"""Binary structure-of-arrays cache of an operator-latency database.

The reference re-parses its JSON-lines file on every load
(/root/reference/pkg/src/llmconf/perfdb.py:361-407): about 10 µs per record in
Python, so seconds for measured-scale databases.  ``save_soa`` writes the
flattened grid image the device consumes (``FlatDb``, the same arrays
``lc_db_upload`` takes), plus the per-cell provenance and the header, into one
``.npz``; ``load_soa`` maps it back without touching records.  Records and the
grid index are rebuilt only if something reads them (``FlatBackedDatabase``).

``load_db(path, soa_cache=True)`` keeps ``<path>.soa.npz`` next to the source,
rebuilt whenever the source's size or mtime changes.
"""

from __future__ import annotations

import json
import os
from itertools import product
from pathlib import Path

import numpy as np

from .database import (
    EXTRAPOLATION_POLICIES,
    POLICY_CODE,
    PROVENANCES,
    FlatDb,
    OperatorRecord,
    PerfDatabase,
    _FLAT_CACHE,
    build_grids,
    flatten,
    grid_key,
)
from .specs import DbParseError, DbValidationError, HardwareSpec

SOA_VERSION = 1


class FlatBackedDatabase(PerfDatabase):
    """A database held as its flattened grid image; records and ``_grids`` are
    materialised (sorted by kind, quant, shape, perfdb.py:410-411) on first use."""

    def __init__(self, hardware, backend, backend_version, extrapolation, flat: FlatDb,
                 provenance: np.ndarray | None = None):
        if extrapolation not in EXTRAPOLATION_POLICIES:
            raise DbValidationError(f"unknown extrapolation policy {extrapolation!r}")
        self.hardware = hardware
        self.backend = backend
        self.backend_version = backend_version
        self.extrapolation = extrapolation
        self._prov = provenance
        self._recs = None
        self._grid_index = None
        if flat.policy != POLICY_CODE[extrapolation]:
            flat = FlatDb(**{**flat.__dict__, "policy": POLICY_CODE[extrapolation]})
        _FLAT_CACHE[self] = flat

    @property
    def records(self):
        if self._recs is None:
            self._recs = tuple(records_from_flat(_FLAT_CACHE[self], self._prov))
        return self._recs

    @property
    def _grids(self):
        if self._grid_index is None:
            self._grid_index = build_grids(self.records)
        return self._grid_index

    def kinds(self) -> set[str]:
        return set(_FLAT_CACHE[self].kinds)

    def grid_keys(self) -> list[tuple]:
        return list(_FLAT_CACHE[self].keys)


def records_from_flat(flat: FlatDb, provenance: np.ndarray | None = None) -> list[OperatorRecord]:
    vals = flat.cell.tolist()
    prov = None if provenance is None else provenance.tolist()
    out = []
    for g, (kind, quant, fixed) in enumerate(flat.keys):
        base = dict(fixed)
        names = flat.axes[g]
        x = int(flat.grid_cell_off[g])
        for combo in product(*flat.axis_values[g]):
            shape = dict(base)
            shape.update(zip(names, combo))
            out.append(OperatorRecord.make(kind, quant, shape, vals[x],
                                           "synthetic" if prov is None else PROVENANCES[prov[x]]))
            x += 1
    out.sort(key=lambda r: (r.kind, r.quant, r.shape))
    return out


def _provenance(db, flat: FlatDb) -> np.ndarray:
    prov = np.zeros(len(flat.cell), dtype=np.uint8)
    if isinstance(db, FlatBackedDatabase) and db._prov is not None:
        return db._prov
    for rec in db.records:
        key_shape = dict(rec.shape)
        g = flat.index[grid_key(rec.kind, rec.quant, key_shape)]
        idx = [flat.axis_values[g][a].index(int(key_shape[n])) for a, n in enumerate(flat.axes[g])]
        off = int(flat.grid_cell_off[g]) + (idx[0] * len(flat.axis_values[g][1]) + idx[1] if len(idx) == 2
                                            else idx[0])
        prov[off] = PROVENANCES.index(rec.provenance)
    return prov


def save_soa(db, path: str | os.PathLike, source_stat: tuple[int, int] | None = None) -> None:
    """Write ``db``'s flattened image, provenance and header to ``path`` (.npz)."""
    flat = flatten(db)
    meta = {
        "version": SOA_VERSION,
        "hardware": db.hardware.to_doc(),
        "backend": db.backend,
        "backend_version": db.backend_version,
        "keys": [[k[0], k[1], [list(p) for p in k[2]]] for k in flat.keys],
        "axes": [list(a) for a in flat.axes],
        "axis_values": [[list(v) for v in av] for av in flat.axis_values],
        "source": list(source_stat) if source_stat else None,
    }
    tmp = Path(str(path) + ".tmp.npz")
    np.savez(tmp, meta=np.array(json.dumps(meta)), grid_ndim=flat.grid_ndim, grid_axis_off=flat.grid_axis_off,
             grid_axis_len=flat.grid_axis_len, grid_cell_off=flat.grid_cell_off, axis_val=flat.axis_val,
             axis_log=flat.axis_log, cell=flat.cell, cell_log=flat.cell_log, provenance=_provenance(db, flat))
    os.replace(tmp, path)


def _soa_meta(path) -> dict:
    with np.load(path, allow_pickle=False) as z:
        return json.loads(str(z["meta"]))


def load_soa(path: str | os.PathLike, extrapolation: str = "default") -> FlatBackedDatabase:
    """Map a ``save_soa`` file back to a database (no record parsing)."""
    with np.load(path, allow_pickle=False) as z:
        meta = json.loads(str(z["meta"]))
        if meta.get("version") != SOA_VERSION:
            raise DbParseError(f"{path}: SoA cache version {meta.get('version')!r}, expected {SOA_VERSION}")
        arrays = {k: z[k] for k in ("grid_ndim", "grid_axis_off", "grid_axis_len", "grid_cell_off", "axis_val",
                                    "axis_log", "cell", "cell_log", "provenance")}
    keys = [(k[0], k[1], tuple(tuple(p) for p in k[2])) for k in meta["keys"]]
    flat = FlatDb(keys=keys, index={k: i for i, k in enumerate(keys)}, axes=[tuple(a) for a in meta["axes"]],
                  axis_values=[tuple(tuple(v) for v in av) for av in meta["axis_values"]],
                  kinds=sorted({k[0] for k in keys}), policy=POLICY_CODE.get(extrapolation, 0),
                  **{k: v for k, v in arrays.items() if k != "provenance"})
    return FlatBackedDatabase(HardwareSpec.from_doc(meta["hardware"]), meta["backend"], meta["backend_version"],
                              extrapolation, flat, arrays["provenance"])


def load_db_cached(path: str | os.PathLike, extrapolation: str = "default",
                   cache: str | os.PathLike | None = None) -> PerfDatabase:
    """``load_db`` through a SoA cache file (default ``<path>.soa.npz``)."""
    from .database import load_db

    path = Path(path)
    cache = Path(cache) if cache else Path(str(path) + ".soa.npz")
    st = path.stat()
    stamp = (int(st.st_size), int(st.st_mtime_ns))
    if cache.exists():
        try:
            if tuple(_soa_meta(cache).get("source") or ()) == stamp:
                return load_soa(cache, extrapolation)
        except (OSError, ValueError, KeyError, DbParseError):
            pass
    db = load_db(path, extrapolation)
    try:
        save_soa(db, cache, stamp)
    except OSError:
        pass  # read-only location: the parsed database is still returned
    return db
