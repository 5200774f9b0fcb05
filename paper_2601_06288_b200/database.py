"""Operator-latency database: JSON-lines ingest and the flattened device image.

Ingest mirrors the reference format (schema ``llmconf-perfdb/1``,
/root/reference/pkg/src/llmconf/perfdb.py:358-425) and its grid index
(``_grids``: key -> axes, sorted axis values, coords -> latency; perfdb.py:283-355),
so reference ``PerfDatabase`` objects and ours flatten the same way.

``flatten(db)`` turns the grid index into the structure-of-arrays image the
kernels stage into shared memory: per-grid descriptors, axis values with their
natural logs, cell latencies with their natural logs.  The logs are taken with
CPython's ``math.log`` -- exactly the calls the reference makes per query -- so
the device only ever needs ``log(x)`` of the query coordinate and one ``exp``.
"""

from __future__ import annotations

import gzip
import json
import math
import weakref
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, Mapping

import numpy as np

from .specs import (
    QUANT_FORMATS,
    DbParseError,
    DbValidationError,
    HardwareSpec,
)

SCHEMA_ID = "llmconf-perfdb/1"
EXTRAPOLATION_POLICIES = ("default", "strict", "clamp", "sol")
OPERATOR_KINDS = ("gemm", "attention_context", "attention_generation", "allreduce", "allgather", "alltoall",
                  "p2p", "moe_dispatch", "moe_combine", "moe_gemm", "embedding")
ATTENTION_KINDS = ("attention_context", "attention_generation")
COMM_KINDS = ("allreduce", "allgather", "alltoall", "p2p")
ATTN_VARIANTS = ("MHA", "GQA", "MLA")
PROVENANCES = ("measured", "synthetic")

# (required dims in canonical order, interpolated axes)  -- perfdb.py:51-69
KIND_DIMS: dict[str, tuple[tuple[str, ...], tuple[str, ...]]] = {
    "gemm": (("m", "n", "k"), ("m",)),
    "attention_context": (("batch", "seq_len", "num_heads", "kv_heads", "head_dim"), ("batch", "seq_len")),
    "attention_generation": (("batch", "seq_len", "num_heads", "kv_heads", "head_dim"), ("batch", "seq_len")),
    "allreduce": (("message_bytes", "participant_count"), ("message_bytes",)),
    "allgather": (("message_bytes", "participant_count"), ("message_bytes",)),
    "alltoall": (("message_bytes", "participant_count"), ("message_bytes",)),
    "p2p": (("message_bytes", "participant_count"), ("message_bytes",)),
    "moe_dispatch": (("tokens", "experts", "topk", "hidden", "intermediate"), ("tokens",)),
    "moe_combine": (("tokens", "experts", "topk", "hidden", "intermediate"), ("tokens",)),
    "moe_gemm": (("tokens", "experts", "topk", "hidden", "intermediate"), ("tokens",)),
    "embedding": (("tokens", "hidden", "vocab"), ("tokens",)),
}


def grid_key(kind: str, quant: str, shape: Mapping[str, int | str]) -> tuple:
    """(kind, quant, fixed dims) exactly as OperatorQuery.grid_key (perfdb.py:239-244)."""
    skip = set(KIND_DIMS[kind][1]) | {"kv_len"}
    return (kind, quant, tuple((k, v) for k, v in sorted(shape.items()) if k not in skip))


def _check_shape(kind: str, quant: str, shape: Mapping) -> None:
    if kind not in OPERATOR_KINDS:
        raise DbParseError(f"unknown operator kind {kind!r}")
    if quant not in QUANT_FORMATS:
        raise DbParseError(f"unknown quant format {quant!r}")
    required, _ = KIND_DIMS[kind]
    is_attn = kind in ATTENTION_KINDS
    allowed = set(required) | ({"attn_kind", "kv_len"} if is_attn else set())
    if set(shape) - allowed:
        raise DbParseError(f"{kind}: unexpected shape dims {sorted(set(shape) - allowed)}")
    if set(required) - set(shape):
        raise DbParseError(f"{kind}: missing shape dims {sorted(set(required) - set(shape))}")
    for name in required:
        v = shape[name]
        if not isinstance(v, int) or v < 1:
            raise DbParseError(f"{kind}: dim {name}={v!r} must be an integer >= 1")
    if is_attn:
        if shape.get("attn_kind") not in ATTN_VARIANTS:
            raise DbParseError(f"{kind}: attn_kind must be one of {ATTN_VARIANTS}")
        kv = shape.get("kv_len", shape["seq_len"])
        if not isinstance(kv, int) or kv < 1:
            raise DbParseError(f"{kind}: kv_len={kv!r} must be an integer >= 1")
    elif "attn_kind" in shape:
        raise DbParseError(f"{kind}: attn_kind only valid on attention kinds")
    if kind in COMM_KINDS and shape["participant_count"] < 2:
        raise DbParseError(f"{kind}: participant_count must be >= 2")


@dataclass(frozen=True)
class OperatorRecord:
    """One latency sample: kind, quant, full shape, latency (perfdb.py:260-280)."""

    kind: str
    quant: str
    shape: tuple[tuple[str, int | str], ...]
    latency_us: float
    provenance: str = "measured"

    def __post_init__(self) -> None:
        _check_shape(self.kind, self.quant, dict(self.shape))
        if not (isinstance(self.latency_us, (int, float)) and math.isfinite(self.latency_us)):
            raise DbValidationError(f"latency_us={self.latency_us!r} is not a finite number")
        if self.latency_us <= 0:
            raise DbValidationError(f"latency_us must be > 0, got {self.latency_us}")
        if self.provenance not in PROVENANCES:
            raise DbValidationError(f"provenance must be one of {PROVENANCES}")

    @classmethod
    def make(cls, kind: str, quant: str, shape: Mapping, latency_us: float, provenance: str = "measured"):
        return cls(kind, quant, tuple(sorted(dict(shape).items())), latency_us, provenance)

    def to_doc(self) -> dict:
        return {"kind": self.kind, "quant": self.quant, "shape": dict(self.shape), "latency_us": self.latency_us,
                "provenance": self.provenance}


class Grid:
    """Rectangular grid of one key: axis names, sorted axis values, coords -> latency."""

    __slots__ = ("axes", "axis_values", "cells")

    def __init__(self, axes, axis_values, cells):
        self.axes = axes
        self.axis_values = axis_values
        self.cells = cells


def record_key_coords(rec) -> tuple[tuple, tuple]:
    """(grid key, interpolation coords) of a record: this package's or the reference's
    (``rec.query.grid_key()`` / ``coords()``, perfdb.py:239-248) -- only attributes are read."""
    q = getattr(rec, "query", None)
    if q is not None:
        return q.grid_key(), q.coords()
    shape = dict(rec.shape)
    return grid_key(rec.kind, rec.quant, shape), tuple(int(shape[a]) for a in KIND_DIMS[rec.kind][1])


def build_grids(records: Iterable[OperatorRecord]) -> dict:
    """_build_grids (perfdb.py:329-355): index records by grid key; duplicates and ragged grids raise."""
    per_key: dict[tuple, dict] = {}
    first: dict[tuple, dict] = {}
    for idx, rec in enumerate(records):
        key, coords = record_key_coords(rec)
        seen = first.setdefault(key, {})
        if coords in seen:
            raise DbValidationError(
                f"duplicate coordinate {coords} for key {key} (records #{seen[coords]} and #{idx})")
        seen[coords] = idx
        per_key.setdefault(key, {})[coords] = rec.latency_us
    grids = {}
    for key, cells in per_key.items():
        axes = KIND_DIMS[key[0]][1]
        values = tuple(tuple(sorted({c[i] for c in cells})) for i in range(len(axes)))
        expected = math.prod(len(v) for v in values)
        if len(cells) != expected:
            raise DbValidationError(
                f"non-rectangular grid for key {key}: {len(cells)} cells, "
                f"expected {expected} from axes {dict(zip(axes, values))}")
        grids[key] = Grid(axes, values, cells)
    return grids


@dataclass(eq=False)
class PerfDatabase:
    """Immutable indexed records of one platform/backend; hashed by identity."""

    hardware: HardwareSpec
    backend: str
    backend_version: str
    records: tuple[OperatorRecord, ...]
    extrapolation: str = "default"
    _grids: dict = field(default_factory=dict, repr=False)

    def __hash__(self) -> int:
        return id(self)

    @classmethod
    def from_records(cls, hardware, backend, backend_version, records, extrapolation="default") -> "PerfDatabase":
        if extrapolation not in EXTRAPOLATION_POLICIES:
            raise DbValidationError(f"unknown extrapolation policy {extrapolation!r}")
        records = tuple(records)
        return cls(hardware, backend, backend_version, records, extrapolation, build_grids(records))

    def grid_keys(self) -> list[tuple]:
        return sorted(self._grids, key=repr)

    def kinds(self) -> set[str]:
        return {k[0] for k in self._grids}


@dataclass
class ValidationReport:
    """validate_db's result (perfdb.py:672-683)."""

    violations: list[str] = field(default_factory=list)
    gaps: list[str] = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return not self.violations and not self.gaps

    def lines(self) -> list[str]:
        return [f"violation: {v}" for v in self.violations] + [f"gap: {g}" for g in self.gaps]


def validate_db(db, required_kinds: Iterable[str] = ()) -> ValidationReport:
    """Drop-in for perfdb.validate_db (perfdb.py:685-701): re-check every record's latency
    and provenance, the grid invariants (duplicates, rectangularity) and the required kinds.

    Accepts this package's databases and the reference's (attributes only); the
    messages are the reference's.  Host code: it runs once per database file, off
    the search path (the device image is built by ``flatten`` from the checked grids).
    """
    report = ValidationReport()
    for idx, rec in enumerate(db.records):
        lat = rec.latency_us
        if not (isinstance(lat, (int, float)) and math.isfinite(lat) and lat > 0):
            report.violations.append(f"record #{idx} {record_key_coords(rec)[0]}: latency_us={lat}")
        if rec.provenance not in PROVENANCES:
            report.violations.append(f"record #{idx}: provenance={rec.provenance!r}")
    try:
        build_grids(db.records)
    except DbValidationError as e:
        report.violations.append(str(e))
    present = db.kinds()
    for kind in sorted(set(required_kinds)):
        if kind not in present:
            report.gaps.append(f"operator kind {kind!r} required but absent")
    return report


def load_db(path: str | Path, extrapolation: str = "default", soa_cache: bool | str | Path = False) -> PerfDatabase:
    """Load a JSON-lines database (optionally gzip-compressed).

    ``soa_cache``: True (``<path>.soa.npz``) or a cache path -- reuse the binary
    structure-of-arrays image while the source file is unchanged (soa.py).
    """
    if soa_cache:
        from .soa import load_db_cached

        return load_db_cached(path, extrapolation, None if soa_cache is True else soa_cache)
    path = Path(path)
    raw = path.read_bytes()
    if path.suffix == ".gz":
        raw = gzip.decompress(raw)
    lines = raw.decode("utf-8").splitlines()
    if not lines:
        raise DbParseError(f"{path}: empty database file")
    try:
        header = json.loads(lines[0])
    except json.JSONDecodeError as e:
        raise DbParseError(f"{path}:1: bad JSON in header: {e}") from None
    known = {"schema", "hardware", "backend", "backend_version"}
    if set(header) - known:
        raise DbParseError(f"{path}:1: unknown header fields: {sorted(set(header) - known)}")
    if header.get("schema") != SCHEMA_ID:
        raise DbParseError(f"{path}:1: schema must be {SCHEMA_ID!r}, got {header.get('schema')!r}")
    hardware = HardwareSpec.from_doc(header["hardware"])
    records = []
    for lineno, line in enumerate(lines[1:], start=2):
        if not line.strip():
            continue
        try:
            doc = json.loads(line)
        except json.JSONDecodeError as e:
            raise DbParseError(f"{path}:{lineno}: bad JSON: {e}") from None
        known_rec = {"kind", "quant", "shape", "latency_us", "provenance"}
        if set(doc) - known_rec:
            raise DbParseError(f"{path}:{lineno}: unknown record fields: {sorted(set(doc) - known_rec)}")
        if known_rec - set(doc):
            raise DbParseError(f"{path}:{lineno}: missing record fields: {sorted(known_rec - set(doc))}")
        try:
            records.append(OperatorRecord.make(doc["kind"], doc["quant"], doc["shape"], doc["latency_us"],
                                               doc["provenance"]))
        except (DbParseError, DbValidationError) as e:
            raise type(e)(f"{path}:{lineno}: {e}") from None
    try:
        return PerfDatabase.from_records(hardware, header["backend"], header["backend_version"], records,
                                         extrapolation)
    except DbValidationError as e:
        raise DbValidationError(f"{path}: {e}") from None


def with_records(db, records=None, hardware=None, extrapolation=None) -> PerfDatabase:
    """A new database sharing ``db``'s metadata with some parts replaced."""
    return PerfDatabase.from_records(hardware or db.hardware, db.backend, db.backend_version,
                                     db.records if records is None else records,
                                     db.extrapolation if extrapolation is None else extrapolation)


# ----------------------------------------------------------------------------- device image
POLICY_CODE = {p: i for i, p in enumerate(EXTRAPOLATION_POLICIES)}


@dataclass
class FlatDb:
    """Structure-of-arrays image of a grid index (see include/llmconf_b200.h lc_db_desc)."""

    keys: list[tuple]           # grid id -> key
    index: dict                 # key -> grid id
    axes: list[tuple[str, ...]]
    axis_values: list[tuple[tuple[int, ...], ...]]
    grid_ndim: np.ndarray
    grid_axis_off: np.ndarray
    grid_axis_len: np.ndarray
    grid_cell_off: np.ndarray
    axis_val: np.ndarray
    axis_log: np.ndarray
    cell: np.ndarray
    cell_log: np.ndarray
    kinds: list[str]            # sorted kinds present (MissingKeyError message)
    policy: int


_FLAT_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def flatten(db) -> FlatDb:
    """Flatten ``db._grids`` (reference or local PerfDatabase); cached per object."""
    try:
        hit = _FLAT_CACHE.get(db)
    except TypeError:
        hit = None
    if hit is not None:
        return hit
    grids = db._grids
    keys = sorted(grids, key=repr)
    ndim, aoff, alen, coff = [], [], [], []
    av, al, cv, cl = [], [], [], []
    axes, axis_values = [], []
    for key in keys:
        g = grids[key]
        values = g.axis_values
        axes.append(tuple(g.axes))
        axis_values.append(tuple(tuple(v) for v in values))
        ndim.append(len(values))
        offs, lens = [0, 0], [0, 0]
        for a, vals in enumerate(values):
            offs[a] = len(av)
            lens[a] = len(vals)
            av.extend(int(v) for v in vals)
            al.extend(math.log(v) for v in vals)
        aoff.extend(offs)
        alen.extend(lens)
        coff.append(len(cv))
        if len(values) == 1:
            for v0 in values[0]:
                lat = g.cells[(v0,)]
                cv.append(lat)
                cl.append(math.log(lat))
        else:
            for v0 in values[0]:
                for v1 in values[1]:
                    lat = g.cells[(v0, v1)]
                    cv.append(lat)
                    cl.append(math.log(lat))
    flat = FlatDb(
        keys=keys,
        index={k: i for i, k in enumerate(keys)},
        axes=axes,
        axis_values=axis_values,
        grid_ndim=np.array(ndim, dtype=np.int32),
        grid_axis_off=np.array(aoff, dtype=np.int32),
        grid_axis_len=np.array(alen, dtype=np.int32),
        grid_cell_off=np.array(coff, dtype=np.int32),
        axis_val=np.array(av, dtype=np.int64),
        axis_log=np.array(al, dtype=np.float64),
        cell=np.array(cv, dtype=np.float64),
        cell_log=np.array(cl, dtype=np.float64),
        kinds=sorted({k[0] for k in grids}),
        policy=POLICY_CODE[db.extrapolation],
    )
    try:
        _FLAT_CACHE[db] = flat
    except TypeError:
        pass
    return flat
