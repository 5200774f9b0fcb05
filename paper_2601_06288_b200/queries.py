"""Single-operator latency queries on the device: ``query_latency`` drop-in.

Mirrors ``llmconf.perfdb.OperatorQuery`` / ``query_latency``
(/root/reference/pkg/src/llmconf/perfdb.py:175-258 and :539-580).  The host
resolves each query's grid key against the database's flattened grid index and
packs a 64-byte ``lc_query`` (include/llmconf_b200.h); ``k_query`` does the
interpolation, the extrapolation policy and the roofline scaling on the GPU with
the same glibc log/exp restatement the search kernels use, so the results equal
the reference's float for float.  Errors carry the reference's exception types
and messages; a batch raises the first failing query's error, as a Python loop
over ``query_latency`` would.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterable, Mapping

import numpy as np

from . import _native as N
from .database import ATTENTION_KINDS, EXTRAPOLATION_POLICIES, KIND_DIMS, _check_shape, flatten, grid_key
from .plans import KIND_CODE
from .specs import QUANT_FORMATS, ExtrapolationError, MissingKeyError, PerfDbError, UnsupportedOperatorError

ST_OK, ST_MISSING, ST_EXTRAP, ST_UNSUPPORTED = 0, 1, 2, 3


@dataclass(frozen=True)
class OperatorQuery:
    """One operator invocation (perfdb.py:175-258): shape stored as a sorted tuple."""

    kind: str
    quant: str
    shape: tuple
    backend: str | None = None

    def __init__(self, kind: str, quant: str, shape: Mapping, backend: str | None = None):
        object.__setattr__(self, "kind", kind)
        object.__setattr__(self, "quant", quant)
        object.__setattr__(self, "shape", tuple(sorted(dict(shape).items())))
        object.__setattr__(self, "backend", backend)
        _check_shape(kind, quant, dict(self.shape))

    def dims(self) -> dict:
        return dict(self.shape)

    def grid_key(self) -> tuple:
        return grid_key(self.kind, self.quant, dict(self.shape))

    def coords(self) -> tuple[int, ...]:
        d = dict(self.shape)
        return tuple(int(d[a]) for a in KIND_DIMS[self.kind][1])


def _pack(flat, queries: list, policy_code: int) -> np.ndarray:
    arr = np.zeros(len(queries), dtype=N.QUERY_DTYPE)
    for i, q in enumerate(queries):
        dims = dict(q.shape)
        arr[i]["grid"] = flat.index.get(grid_key(q.kind, q.quant, dims), -1)
        arr[i]["kind"] = KIND_CODE[q.kind]
        arr[i]["quant"] = QUANT_FORMATS.index(q.quant)
        arr[i]["policy"] = policy_code
        req = KIND_DIMS[q.kind][0]
        arr[i]["d"][: len(req)] = [int(dims[n]) for n in req]
        arr[i]["kv_len"] = int(dims["kv_len"]) if q.kind in ATTENTION_KINDS and "kv_len" in dims else -1
    return arr


def _error(code: int, q, flat, db) -> PerfDbError:
    key = grid_key(q.kind, q.quant, dict(q.shape))
    if code == ST_MISSING:
        return MissingKeyError(f"no grid for key {key}; database covers kinds {flat.kinds}")
    if code == ST_UNSUPPORTED:
        return UnsupportedOperatorError(f"hardware {db.hardware.name!r} has no compute rate for quant {q.quant!r}")
    g = flat.index[key]
    axes, values = flat.axes[g], flat.axis_values[g]
    dims = dict(q.shape)
    coords = tuple(int(dims[a]) for a in KIND_DIMS[q.kind][1])
    box = {a: (v[0], v[-1]) for a, v in zip(axes, values)}
    return ExtrapolationError(f"query coords {dict(zip(axes, coords))} outside grid box {box}")


def query_latency_batch(db, queries: Iterable, policy: str | None = None, device: int = 0,
                        errors: str = "raise") -> np.ndarray:
    """Latency in microseconds of every query, in one device launch.

    ``queries`` are reference or local ``OperatorQuery`` objects (anything with
    ``kind``, ``quant``, ``shape`` and ``backend``).  ``errors="raise"`` raises
    the first failing query's error (reference order: backend check, policy
    check, grid lookup, then interpolation); ``errors="nan"`` returns NaN for
    failed queries instead.
    """
    from .engine import get_engine

    queries = list(queries)
    for q in queries:
        if q.backend is not None and q.backend != db.backend:
            if errors == "raise":
                raise MissingKeyError(f"query targets backend {q.backend!r} but database is {db.backend!r}")
    policy = policy or db.extrapolation
    if policy not in EXTRAPOLATION_POLICIES:
        raise PerfDbError(f"unknown extrapolation policy {policy!r}")
    eng = get_engine(device)
    h, flat = eng.db_handle(db)
    arr = _pack(flat, queries, EXTRAPOLATION_POLICIES.index(policy))
    n = len(queries)
    lat = np.empty(n, dtype=np.float64)
    st = np.empty(n, dtype=np.int32)
    if n:
        with eng._lock:
            N.check(eng.lib.lc_query_batch(eng.ctx, h, n, C.c_void_p(arr.ctypes.data), N.ptr(lat, C.c_double),
                                           N.ptr(st, C.c_int32)), "lc_query_batch")
    bad_backend = np.array([q.backend is not None and q.backend != db.backend for q in queries], dtype=bool)
    if errors == "raise":
        for i in np.flatnonzero(st):
            raise _error(int(st[i]), queries[i], flat, db)
    elif errors == "nan":
        lat[(st != 0) | bad_backend] = np.nan
    else:
        raise ValueError(f"errors must be 'raise' or 'nan', got {errors!r}")
    return lat


def query_latency(db, query, policy: str | None = None, device: int = 0) -> float:
    """Drop-in for ``llmconf.perfdb.query_latency`` (perfdb.py:539-580)."""
    return float(query_latency_batch(db, [query], policy, device)[0])
