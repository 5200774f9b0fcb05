"""Synthetic operator-latency databases generated on the device.

Mirrors the reference's generator (/root/reference/pkg/src/llmconf/perfdb.py:586-666)
and the grid harvest for a model (model.py:483-545).  Every cell's latency is
its roofline bound times a smooth, seeded efficiency factor; both depend only on
the cell's coordinates, so ``k_dbgen`` prices all cells in one launch:

* the host evaluates, with CPython's own ``hashlib`` / ``math`` exactly as the
  reference does, the per-grid hash constants (offset, and per axis omega and
  phase) and one sine term per axis VALUE -- O(sum of axis lengths);
* the device evaluates ``sol_estimate`` per cell, combines the terms in the
  reference's operation order, and takes ``log(latency)`` for the device image
  (glibc's ``__log_fma`` restated; the rare near-1 inputs are redone on the host).

The result is the reference's database bit for bit (tests/test_gpu_dbgen.py
compares every latency of the committed reference-generated databases), with the
flattened device image built straight from the device arrays.  ``lazy=True``
defers the per-record Python objects until someone reads ``records`` or
``_grids``, so measured-scale grids (10^6-10^8 cells) go from spec to a search
without building them.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import math
from dataclasses import dataclass
from itertools import product
from pathlib import Path
from typing import Mapping, Sequence

import numpy as np

from . import _native as N
from .database import (
    KIND_DIMS,
    OPERATOR_KINDS,
    POLICY_CODE,
    SCHEMA_ID,
    FlatDb,
    OperatorRecord,
    PerfDatabase,
    _FLAT_CACHE,
)
from .plans import KIND_CODE, _problems, _template
from .specs import QUANT_FORMATS, DbValidationError, ParallelConfig, ParallelConfigError, UnsupportedOperatorError


def _pow2(lo: int, hi: int, step: int = 1) -> tuple[int, ...]:
    return tuple(2**i for i in range(lo, hi + 1, step))


# model.py:486-498
DEFAULT_AXES: dict[str, tuple[tuple[str, tuple[int, ...]], ...]] = {
    "gemm": (("m", _pow2(0, 15)),),
    "attention_context": (("batch", _pow2(0, 6)), ("seq_len", _pow2(5, 14))),
    "attention_generation": (("batch", _pow2(0, 10)), ("seq_len", _pow2(4, 17))),
    "allreduce": (("message_bytes", _pow2(12, 30, 2)),),
    "allgather": (("message_bytes", _pow2(12, 30, 2)),),
    "alltoall": (("message_bytes", _pow2(12, 30, 2)),),
    "p2p": (("message_bytes", _pow2(12, 30, 2)),),
    "moe_dispatch": (("tokens", _pow2(0, 15)),),
    "moe_combine": (("tokens", _pow2(0, 15)),),
    "moe_gemm": (("tokens", _pow2(0, 15)),),
    "embedding": (("tokens", _pow2(0, 15, 3)),),
}


@dataclass(frozen=True)
class GridAxes:
    """One grid to synthesize (perfdb.py:586-614): fixed dims + values per interpolated axis."""

    kind: str
    quant: str
    fixed: tuple
    axes: tuple

    def __post_init__(self) -> None:
        if self.kind not in OPERATOR_KINDS:
            raise DbValidationError(f"unknown kind {self.kind!r}")
        expected = KIND_DIMS[self.kind][1]
        names = tuple(a for a, _ in self.axes)
        if names != expected:
            raise DbValidationError(f"{self.kind}: axes must be {expected}, got {names}")
        for name, values in self.axes:
            if not values:
                raise DbValidationError(f"{self.kind}: axis {name} is empty")
            if list(values) != sorted(set(values)):
                raise DbValidationError(f"{self.kind}: axis {name} must be strictly ascending")

    def key(self) -> tuple:
        return (self.kind, self.quant, self.fixed)

    def n_cells(self) -> int:
        return math.prod(len(v) for _, v in self.axes)


class _NoGrids:
    index: dict = {}


def grid_spec_for_model(model, tp_values: Sequence[int] = (1, 2, 4, 8), pp_values: Sequence[int] = (1, 2, 4),
                        ep_values: Sequence[int] | None = None, dp_values: Sequence[int] = (1, 8),
                        axes: Mapping[str, tuple] | None = None) -> list[GridAxes]:
    """Every grid a database needs to serve this model's plans (model.py:501-545).

    The reference harvests grid keys from ``decompose`` over three passes
    (prefill, decode, mixed); the union of those plans' keys is exactly the
    key set of this package's per-(tp, pp, ep) plan templates, which carry
    every entry any phase uses.
    """
    if ep_values is None:
        ep_values = (1,) if model.moe is None else (1, 2, 4, 8)
    table = dict(DEFAULT_AXES)
    if axes:
        table.update(axes)
    keys: dict[tuple, None] = {}
    seen: set = set()
    for tp, pp, ep, dp in product(tp_values, pp_values, ep_values, dp_values):
        try:
            ParallelConfig(tp=tp, pp=pp, ep=ep, dp=dp)
        except ParallelConfigError:
            continue
        if _problems(model, tp, pp, ep, dp) or (tp, pp, ep) in seen:
            continue
        seen.add((tp, pp, ep))
        _, infos = _template(model, _NoGrids, tp, pp, ep)
        for info in infos:
            keys.setdefault(info.key, None)
    return [GridAxes(kind=k[0], quant=k[1], fixed=k[2], axes=table[k[0]]) for k in sorted(keys, key=repr)]


def _hash_unit(*parts) -> float:
    """perfdb.py:617-621."""
    material = "|".join(str(p) for p in parts).encode()
    return int.from_bytes(hashlib.blake2b(material, digest_size=8).digest(), "big") / 2.0**64


def _canonical_fixed(kind: str, fixed: tuple) -> list[int]:
    req, interp = KIND_DIMS[kind]
    f = dict(fixed)
    return [0 if n in interp else int(f[n]) for n in req] + [0] * (5 - len(req))


def _device_cells(hw, spec: Sequence[GridAxes], seed: int, amplitude: float, device: int):
    from .engine import get_engine

    grids = np.zeros(len(spec), dtype=N.GEN_GRID_DTYPE)
    axv: list[int] = []
    term: list[float] = []
    off = 0
    for i, g in enumerate(spec):
        key = g.key()
        req = KIND_DIMS[g.kind][0]
        row = grids[i]
        row["kind"] = KIND_CODE[g.kind]
        row["quant"] = QUANT_FORMATS.index(g.quant)
        row["n_axes"] = len(g.axes)
        row["cell_off"] = off
        row["d"] = _canonical_fixed(g.kind, g.fixed)
        # _efficiency (perfdb.py:624-638): hash constants and one sine term per axis value
        row["offset"] = (_hash_unit(seed, key, "offset") - 0.5) * 0.3 if amplitude != 0.0 else 0.0
        for a, (name, values) in enumerate(g.axes):
            row["axis_dim"][a] = req.index(name)
            row["axis_off"][a] = len(axv)
            row["axis_len"][a] = len(values)
            if amplitude != 0.0:
                omega = 0.03 + 0.02 * _hash_unit(seed, key, name, "omega")
                phase = 2.0 * math.pi * _hash_unit(seed, key, name, "phase")
                term.extend(math.sin(omega * math.log2(x) + phase) for x in values)
            else:
                term.extend(0.0 for _ in values)
            axv.extend(int(v) for v in values)
        off += g.n_cells()
    axv_a = np.array(axv, dtype=np.int64)
    term_a = np.array(term, dtype=np.float64)
    d = N.LcDbgenDesc()
    d.n_grids = len(spec)
    d.grids = C.c_void_p(grids.ctypes.data)
    d.n_axis = len(axv)
    d.axis_val = N.ptr(axv_a, C.c_int64)
    d.axis_term = N.ptr(term_a, C.c_double)
    d.n_cells = off
    d.amplitude = float(amplitude)
    d.mem_bandwidth = float(hw.mem_bandwidth)
    d.intra_node_bandwidth = float(hw.intra_node_bandwidth)
    d.inter_node_bandwidth = float(hw.inter_node_bandwidth)
    d.gpus_per_node = int(hw.gpus_per_node)
    for i, q in enumerate(QUANT_FORMATS):
        d.compute[i] = float(hw.compute_throughput.get(q, 0.0))
    lat = np.empty(off, dtype=np.float64)
    lat_log = np.empty(off, dtype=np.float64)
    status = np.zeros(len(spec), dtype=np.int32)
    eng = get_engine(device)
    with eng._lock:
        N.check(eng.lib.lc_dbgen(eng.ctx, C.byref(d), N.ptr(lat, C.c_double), N.ptr(lat_log, C.c_double),
                                 N.ptr(status, C.c_int32)), "lc_dbgen")
    for i in np.flatnonzero(status):
        raise UnsupportedOperatorError(
            f"hardware {hw.name!r} has no compute rate for quant {spec[int(i)].quant!r}")
    bad = np.flatnonzero(np.isnan(lat_log))
    for i in bad:  # glibc's near-1 path, not restated on the device
        lat_log[i] = math.log(float(lat[i]))
    return lat, lat_log


def _flat_from_cells(spec: Sequence[GridAxes], lat: np.ndarray, lat_log: np.ndarray) -> FlatDb:
    offs = np.cumsum([0] + [g.n_cells() for g in spec])
    order = sorted(range(len(spec)), key=lambda i: repr(spec[i].key()))
    keys = [spec[i].key() for i in order]
    ndim, aoff, alen, coff = [], [], [], []
    av, al, cv, cl = [], [], [], []
    axes, axis_values = [], []
    n = 0
    for i in order:
        g = spec[i]
        names = tuple(a for a, _ in g.axes)
        vals = tuple(tuple(int(x) for x in v) for _, v in g.axes)
        axes.append(names)
        axis_values.append(vals)
        ndim.append(len(vals))
        o, ln = [0, 0], [0, 0]
        for a, v in enumerate(vals):
            o[a] = len(av)
            ln[a] = len(v)
            av.extend(v)
            al.extend(math.log(x) for x in v)
        aoff.extend(o)
        alen.extend(ln)
        coff.append(n)
        cv.append(lat[offs[i]:offs[i + 1]])
        cl.append(lat_log[offs[i]:offs[i + 1]])
        n += g.n_cells()
    return FlatDb(
        keys=keys, index={k: i for i, k in enumerate(keys)}, axes=axes, axis_values=axis_values,
        grid_ndim=np.array(ndim, dtype=np.int32), grid_axis_off=np.array(aoff, dtype=np.int32),
        grid_axis_len=np.array(alen, dtype=np.int32), grid_cell_off=np.array(coff, dtype=np.int32),
        axis_val=np.array(av, dtype=np.int64), axis_log=np.array(al, dtype=np.float64),
        cell=np.concatenate(cv) if cv else np.zeros(0), cell_log=np.concatenate(cl) if cl else np.zeros(0),
        kinds=sorted({k[0] for k in keys}), policy=POLICY_CODE["default"])


def _records(spec: Sequence[GridAxes], lat: np.ndarray) -> list[OperatorRecord]:
    out = []
    x = 0
    vals = lat.tolist()
    for g in spec:
        fixed = dict(g.fixed)
        names = [a for a, _ in g.axes]
        for combo in product(*(v for _, v in g.axes)):
            shape = dict(fixed)
            shape.update(zip(names, combo))
            out.append(OperatorRecord.make(g.kind, g.quant, shape, vals[x], "synthetic"))
            x += 1
    out.sort(key=lambda r: (r.kind, r.quant, r.shape))  # _record_sort_key (perfdb.py:410-411)
    return out


def generate_synthetic_db(hw, grid_spec: Sequence[GridAxes], seed: int, backend: str = "trtllm",
                          backend_version: str = "synthetic", efficiency_amplitude: float = 0.8, device: int = 0,
                          lazy: bool = False) -> PerfDatabase:
    """Drop-in for ``llmconf.perfdb.generate_synthetic_db`` (perfdb.py:641-666), priced on the GPU."""
    if not 0.0 <= efficiency_amplitude <= 0.8:
        raise DbValidationError("efficiency_amplitude must be in [0, 0.8]")
    spec = list(grid_spec)
    lat, lat_log = _device_cells(hw, spec, seed, float(efficiency_amplitude), device)
    unique = len({g.key() for g in spec}) == len(spec)
    if lazy and unique:
        from .soa import FlatBackedDatabase

        return FlatBackedDatabase(hw, backend, backend_version, "default", _flat_from_cells(spec, lat, lat_log))
    db = PerfDatabase.from_records(hw, backend, backend_version, _records(spec, lat))  # raises like the reference
    if unique:
        _FLAT_CACHE[db] = _flat_from_cells(spec, lat, lat_log)
    return db


def save_db(db, path: str | Path) -> None:
    """Canonical JSON-lines form (perfdb.py:414-425): sorted records, shortest float repr."""
    header = {"schema": SCHEMA_ID, "hardware": db.hardware.to_doc(), "backend": db.backend,
              "backend_version": db.backend_version}
    out = [json.dumps(header, sort_keys=True, separators=(",", ":"))]
    for rec in sorted(db.records, key=lambda r: (r.kind, r.quant, r.shape)):
        out.append(json.dumps(rec.to_doc(), sort_keys=True, separators=(",", ":")))
    Path(path).write_text("\n".join(out) + "\n", encoding="utf-8")
