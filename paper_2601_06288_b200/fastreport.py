"""Columnar report materialisation.

``SearchReport.to_json()`` -- like the reference's (search.py:224-264) --
builds one dict per row and runs the pure-Python indenting JSON encoder, about
20 MB/s.  ``report_json`` writes the same bytes straight from column arrays:
one preformatted template per row kind, floats through ``float.__repr__``
exactly as ``json`` does, sub-documents (workload, counts, skips, timing)
through ``json.dumps`` re-indented to their depth.

``columns_from_batch`` fills the columns from one search of an engine batch
without creating per-row objects; ``columns_from_doc`` from a report document
(used by the tests to prove byte identity against the reference's own bytes).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

from .report import REPORT_SCHEMA, REPORT_VERSION

MODES = ("static", "aggregated", "disaggregated")


@dataclass
class Columns:
    model: str
    backend: str
    workload_doc: dict
    runtime: dict                      # ctx_capacity, chunked_prefill, kv_mem_fraction, cuda_graph, backend
    mode: np.ndarray                   # int: 0 static, 1 aggregated, 2 disaggregated
    cfg: np.ndarray                    # [n, 5] tp, pp, ep, dp, batch (static / aggregated rows)
    gpus: np.ndarray
    ttft: np.ndarray
    tpot: np.ndarray
    speed: np.ndarray
    thru: np.ndarray
    feasible: np.ndarray
    frontier_rows: list                # row indices in frontier order
    pcfg: np.ndarray = None            # [n, 5] prefill worker cfg (disaggregated rows)
    dcfg: np.ndarray = None            # [n, 5] decode worker cfg
    x: np.ndarray = None
    y: np.ndarray = None
    r_sys: np.ndarray = None
    skipped: list = field(default_factory=list)
    best: int = -1
    nearest: int = -1
    violation: float = 0.0
    enumerated: int = 0
    total_ms: float = 0.0
    median_ms: float = 0.0


def _key(c) -> str:
    return f"tp{c[0]}pp{c[1]}ep{c[2]}dp{c[3]}b{c[4]}"


def _f(x: float) -> str:
    if not math.isfinite(x):
        raise ValueError("Out of range float values are not JSON compliant")
    return float.__repr__(x)


def _indent(text: str, depth: int) -> str:
    pad = "  " * depth
    return text.replace("\n", "\n" + pad)


def _runtime_block(rt: dict, depth: int) -> str:
    return _indent(json.dumps(rt, sort_keys=True, indent=2), depth)


def _parallel_block(c, depth: int) -> str:
    p = "  " * (depth + 1)
    e = "  " * depth
    return f'{{\n{p}"dp": {c[3]},\n{p}"ep": {c[2]},\n{p}"pp": {c[1]},\n{p}"tp": {c[0]}\n{e}}}'


class _Writer:
    def __init__(self, cols: Columns):
        self.c = cols
        n = len(cols.mode)
        on_front = np.zeros(n, dtype=bool)
        on_front[list(cols.frontier_rows)] = True
        self.on_front = on_front
        self.model_json = json.dumps(cols.model)
        self.rt = {d: _runtime_block(cols.runtime, d) for d in (2, 3, 4)}

    def label(self, i: int) -> str:
        c = self.c
        if c.mode[i] < 2:
            return _key(c.cfg[i])
        return f"P:{c.x[i]}x{_key(c.pcfg[i])}|D:{c.y[i]}x{_key(c.dcfg[i])}"

    def row(self, i: int, depth: int, flags: bool, extra: str = "") -> str:
        """Row document whose opening brace sits at `depth`."""
        c = self.c
        p = "  " * (depth + 1)
        e = "  " * depth
        fl = ""
        if flags:
            fl = (f'{p}"feasible": {"true" if c.feasible[i] else "false"},\n'
                  f'{p}"frontier": {"true" if self.on_front[i] else "false"},\n')
        sp = float(c.speed[i])
        speed = "null" if not math.isfinite(sp) else _f(sp)
        tail = (f'{p}"speed": {speed},\n{p}"throughput_per_gpu": {_f(float(c.thru[i]))},\n'
                f'{p}"tpot_ms": {_f(float(c.tpot[i]))},\n{p}"ttft_ms": {_f(float(c.ttft[i]))}{extra}\n{e}}}')
        if c.mode[i] < 2:
            cfg = c.cfg[i]
            return (f'{{\n{p}"batch": {cfg[4]},\n{p}"config": "{_key(cfg)}",\n{fl}{p}"gpus": {c.gpus[i]},\n'
                    f'{p}"mode": "{MODES[c.mode[i]]}",\n{p}"model": {self.model_json},\n'
                    f'{p}"parallel": {_parallel_block(cfg, depth + 1)},\n'
                    f'{p}"runtime": {self.rt[depth + 1]},\n{tail}')

        def side(cfg, reps) -> str:
            q = "  " * (depth + 2)
            return (f'{{\n{q}"batch": {cfg[4]},\n{q}"parallel": {_parallel_block(cfg, depth + 2)},\n'
                    f'{q}"replicas": {reps},\n{q}"runtime": {self.rt[depth + 2]}\n{p}}}')

        return (f'{{\n{p}"config": "{self.label(i)}",\n{p}"decode": {side(c.dcfg[i], c.y[i])},\n{fl}'
                f'{p}"gpus": {c.gpus[i]},\n{p}"mode": "disaggregated",\n{p}"prefill": {side(c.pcfg[i], c.x[i])},\n'
                f'{p}"r_sys": {_f(float(c.r_sys[i]))},\n{tail}')


def _list(items: list[str], depth: int) -> str:
    if not items:
        return "[]"
    p = "  " * (depth + 1)
    return "[\n" + ",\n".join(p + it for it in items) + "\n" + "  " * depth + "]"


class _NativeRows:
    """The "rows" / "frontier" lists written by lc_report_rows (C ABI, host code)."""

    def __init__(self, cols: Columns):
        import ctypes as C

        from . import _native as N

        self.lib = N.load_library()
        n = len(cols.mode)
        self.n = n

        def arr(a, dt, shape=None):
            if a is None:
                a = np.zeros(shape if shape is not None else max(n, 1), dtype=dt)
            return np.ascontiguousarray(a, dtype=dt)

        self.keep = {
            "mode": arr(cols.mode, np.int32), "cfg": arr(cols.cfg, np.int64, (max(n, 1), 5)),
            "gpus": arr(cols.gpus, np.int64), "ttft": arr(cols.ttft, np.float64), "tpot": arr(cols.tpot, np.float64),
            "speed": arr(cols.speed, np.float64), "thru": arr(cols.thru, np.float64),
            "feasible": arr(cols.feasible, np.uint8), "pcfg": arr(cols.pcfg, np.int64, (max(n, 1), 5)),
            "dcfg": arr(cols.dcfg, np.int64, (max(n, 1), 5)), "x": arr(cols.x, np.int64), "y": arr(cols.y, np.int64),
            "r_sys": arr(cols.r_sys, np.float64),
        }
        front = np.zeros(max(n, 1), dtype=np.uint8)
        front[list(cols.frontier_rows)] = 1
        self.keep["frontier"] = front
        rc = N.LcReportCols()
        rc.n = n
        for name, a in self.keep.items():
            ctype = {np.dtype(np.int32): C.c_int32, np.dtype(np.int64): C.c_int64, np.dtype(np.float64): C.c_double,
                     np.dtype(np.uint8): C.c_uint8}[a.dtype]
            setattr(rc, name, a.ctypes.data_as(C.POINTER(ctype)))
        self.model_json = json.dumps(cols.model).encode()
        rc.model_json = self.model_json
        self.rt = [_runtime_block(cols.runtime, d).encode() for d in range(6)]
        for d in range(6):
            rc.runtime[d] = self.rt[d]
        self.rc = rc

    def write(self, rows, depth: int, flags: bool, head: bytes = b"", tail: bytes = b"") -> str:
        """head + the JSON list of the rows + tail, decoded once from one buffer."""
        import ctypes as C

        idx = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
        n_sel = self.n if idx is None else len(idx)
        ip = None if idx is None else idx.ctypes.data_as(C.POINTER(C.c_int64))
        cap = 800 * max(n_sel, 1) + 64
        for _ in range(2):
            buf = np.empty(len(head) + cap + len(tail), dtype=np.uint8)  # no zero fill
            buf[: len(head)] = np.frombuffer(head, dtype=np.uint8)
            at = buf[len(head):].ctypes.data_as(C.c_char_p)
            got = self.lib.lc_report_rows(C.byref(self.rc), ip, n_sel, depth, int(flags), at, cap)
            if got == -2:
                raise ValueError("Out of range float values are not JSON compliant")
            if got < 0:
                raise RuntimeError(self.lib.lc_last_error().decode())
            if got <= cap:
                end = len(head) + got
                buf[end: end + len(tail)] = np.frombuffer(tail, dtype=np.uint8)
                return str(memoryview(buf)[: end + len(tail)], "ascii")
            cap = got
        raise RuntimeError("lc_report_rows: size changed between calls")

    def list(self, rows, depth: int, flags: bool) -> str:
        return self.write(rows, depth, flags)


def report_json(cols: Columns, native: bool = True) -> str:
    """Bytes of SearchReport.to_json() for these columns.

    The row lists (the bulk of a large report) are written by the native
    writer (``lc_report_rows``); ``native=False`` keeps them in Python, the
    writer the tests hold it against.
    """
    w = _Writer(cols)
    n = len(cols.mode)
    nat = None
    if native:
        nat = _NativeRows(cols)
        rows_list = None  # written straight into the output buffer below
        frontier_list = nat.list(list(cols.frontier_rows), 1, True)
    else:
        rows = [w.row(i, 2, True) for i in range(n)]
        rows_list = _list(rows, 1)
        frontier_list = _list([rows[i] for i in cols.frontier_rows], 1)
    best = w.row(cols.best, 1, False) if cols.best >= 0 else "null"
    if cols.best < 0 and cols.nearest >= 0:
        v = cols.violation
        extra = ',\n    "violation_factor": ' + (_f(v) if math.isfinite(v) else "null")
        diagnostics = w.row(cols.nearest, 1, False, extra)
    else:
        diagnostics = "null"
    counts = {"enumerated": cols.enumerated, "evaluated": n, "feasible": int(np.count_nonzero(cols.feasible)),
              "frontier": len(cols.frontier_rows), "skipped": len(cols.skipped)}
    skipped = [_indent(json.dumps(s, sort_keys=True, indent=2), 2) for s in cols.skipped]
    timing = {"per_candidate_median_ms": cols.median_ms, "total_ms": cols.total_ms}
    parts = [
        '{\n  "backend": ' + json.dumps(cols.backend),
        '  "best": ' + best,
        '  "counts": ' + _indent(json.dumps(counts, sort_keys=True, indent=2), 1),
        '  "diagnostics": ' + diagnostics,
        '  "frontier": ' + frontier_list,
        '  "model": ' + w.model_json,
        '  "rows": ' + (rows_list if rows_list is not None else ""),
        '  "schema": ' + json.dumps(REPORT_SCHEMA),
        '  "skipped": ' + _list(skipped, 1),
        '  "timing": ' + _indent(json.dumps(timing, sort_keys=True, indent=2, allow_nan=False), 1),
        '  "version": ' + json.dumps(REPORT_VERSION),
        '  "workload": ' + _indent(json.dumps(cols.workload_doc, sort_keys=True, indent=2), 1),
    ]
    if nat is None:
        return ",\n".join(parts) + "\n}\n"
    head = (",\n".join(parts[:7])).encode("ascii")  # ... '  "rows": '
    tail = (",\n" + ",\n".join(parts[7:]) + "\n}\n").encode("ascii")
    return nat.write(None, 1, True, head, tail)


# ----------------------------------------------------------------------------- builders
def _cfg_tuple(doc: dict) -> list:
    p = doc["parallel"]
    return [p["tp"], p["pp"], p["ep"], p["dp"], doc["batch"]]


def columns_from_doc(doc: dict) -> Columns:
    """Columns of an existing report document (reference or ours)."""
    rows = doc["rows"]
    n = len(rows)
    mode = np.array([MODES.index(r["mode"]) for r in rows], dtype=np.int64)
    cfg = np.zeros((n, 5), dtype=np.int64)
    pcfg = np.zeros((n, 5), dtype=np.int64)
    dcfg = np.zeros((n, 5), dtype=np.int64)
    x = np.zeros(n, dtype=np.int64)
    y = np.zeros(n, dtype=np.int64)
    r_sys = np.zeros(n)
    runtime = None
    for i, r in enumerate(rows):
        if r["mode"] == "disaggregated":
            pcfg[i] = _cfg_tuple(r["prefill"])
            dcfg[i] = _cfg_tuple(r["decode"])
            x[i], y[i], r_sys[i] = r["prefill"]["replicas"], r["decode"]["replicas"], r["r_sys"]
            runtime = runtime or r["prefill"]["runtime"]
        else:
            cfg[i] = _cfg_tuple(r)
            runtime = runtime or r["runtime"]
    labels = [r["config"] for r in rows]
    index = {}
    for i, r in enumerate(rows):
        index.setdefault((r["mode"], r["config"]), i)
    front = [index[(f["mode"], f["config"])] for f in doc["frontier"]]
    best = index[(doc["best"]["mode"], doc["best"]["config"])] if doc["best"] else -1
    diag = doc.get("diagnostics")
    nearest = index[(diag["mode"], diag["config"])] if diag else -1
    viol = diag["violation_factor"] if diag else 0.0
    timing = doc.get("timing", {"total_ms": 0.0, "per_candidate_median_ms": 0.0})
    del labels
    return Columns(
        model=doc["model"], backend=doc["backend"], workload_doc=doc["workload"],
        runtime=runtime or {}, mode=mode, cfg=cfg,
        gpus=np.array([r["gpus"] for r in rows], dtype=np.int64),
        ttft=np.array([r["ttft_ms"] for r in rows], dtype=np.float64),
        tpot=np.array([r["tpot_ms"] for r in rows], dtype=np.float64),
        speed=np.array([math.inf if r["speed"] is None else r["speed"] for r in rows], dtype=np.float64),
        thru=np.array([r["throughput_per_gpu"] for r in rows], dtype=np.float64),
        feasible=np.array([r["feasible"] for r in rows], dtype=bool),
        frontier_rows=front, pcfg=pcfg, dcfg=dcfg, x=x, y=y, r_sys=r_sys, skipped=list(doc["skipped"]),
        best=best, nearest=nearest, violation=math.inf if viol is None else viol,
        enumerated=doc["counts"]["enumerated"], total_ms=timing["total_ms"],
        median_ms=timing["per_candidate_median_ms"],
    )


def columns_from_batch(out, si: int, db, model, workload, space, wall_ms: float) -> Columns:
    """Columns of search ``si`` of an engine batch, straight from the device arrays."""
    from .engine import MODE_AGG, MODE_DISAGG, MODE_STATIC, _reason

    U = out.fetch_units()
    R = out.results[si]
    plan, flat = out.plan, out.flat
    off, n = int(R["unit_off"]), int(R["n_units"])
    sl = slice(off, off + n)
    combos = plan.combos[U["unit_combo"][sl]]
    s = out.searches[si]
    batches = out.batches[int(s["b_off"]) + U["unit_batch"][sl]]
    cfg_all = np.stack([combos["tp"], combos["pp"], combos["ep"], combos["dp"], batches], axis=1).astype(np.int64)
    gpus_all = combos["gpus"].astype(np.int64)
    inb = U["unit_in_budget"][sl].astype(bool)
    modes = int(s["modes"])
    parts = {k: [] for k in ("mode", "cfg", "gpus", "ttft", "tpot", "speed", "thru", "key")}
    skipped = []
    err0, err1 = U["err_c0"], U["err_c1"]
    for bit, mi, pre, name in ((MODE_STATIC, 0, "st", "static"), (MODE_AGG, 1, "ag", "aggregated")):
        if not modes & bit:
            continue
        st = U[f"{pre}_status"][sl]
        ok = inb & (st == 0)
        idx = np.nonzero(ok)[0]
        parts["mode"].append(np.full(len(idx), mi))
        parts["cfg"].append(cfg_all[idx])
        parts["gpus"].append(gpus_all[idx])
        for k in ("ttft", "tpot", "speed", "thru"):
            parts[k].append(U[f"{pre}_{k}"][sl][idx])
        parts["key"].append((mi << 32) | idx)
        for i in np.nonzero(inb & (st != 0))[0]:
            k = 4 * (off + int(i)) + mi
            skipped.append({"mode": name, "config": _key(cfg_all[i]),
                            "reason": _reason(int(st[i]), int(err0[k]), int(err1[k]), plan, combos[i], flat, db,
                                              workload, space, int(cfg_all[i][4]))})
    npl = 0
    if modes & MODE_DISAGG:
        pf_st, dc_st = U["pf_status"][sl], U["dc_status"][sl]
        for i in np.nonzero((pf_st != 0) | (dc_st != 0))[0]:
            for kind, st, name in ((2, pf_st, "disaggregated/prefill"), (3, dc_st, "disaggregated/decode")):
                if st[i] != 0:
                    k = 4 * (off + int(i)) + kind
                    skipped.append({"mode": name, "config": _key(cfg_all[i]),
                                    "reason": _reason(int(st[i]), int(err0[k]), int(err1[k]), plan, combos[i], flat,
                                                      db, workload, space, int(cfg_all[i][4]))})
        p0 = int(out.results["n_plans"][:si].sum())
        npl = int(R["n_plans"])
        pk = slice(p0, p0 + npl)
        up, ud = U["plan_p"][pk] - off, U["plan_d"][pk] - off
        parts["mode"].append(np.full(npl, 2))
        parts["cfg"].append(np.zeros((npl, 5), dtype=np.int64))
        parts["gpus"].append(U["plan_gpus"][pk])
        for k, src in (("ttft", "plan_ttft"), ("tpot", "plan_tpot"), ("speed", "plan_speed"), ("thru", "plan_thru")):
            parts[k].append(U[src][pk])
        parts["key"].append((2 << 32) | np.arange(npl))
    # the reference's skip order: static, aggregated, then per worker (prefill, decode)
    cat = {k: np.concatenate(v) if v else np.zeros(0) for k, v in parts.items()}
    nrow = len(cat["mode"])
    pcfg = np.zeros((nrow, 5), dtype=np.int64)
    dcfg = np.zeros((nrow, 5), dtype=np.int64)
    xs = np.zeros(nrow, dtype=np.int64)
    ys = np.zeros(nrow, dtype=np.int64)
    rs = np.zeros(nrow)
    if npl:
        base = nrow - npl
        pcfg[base:] = cfg_all[up]
        dcfg[base:] = cfg_all[ud]
        xs[base:] = U["plan_x"][pk]
        ys[base:] = U["plan_y"][pk]
        rs[base:] = U["plan_r_sys"][pk]
    keys = cat["key"].astype(np.int64)
    pos = {int(k): i for i, k in enumerate(keys.tolist())}
    f0 = int(out.results["n_front"][:si].sum())
    front = [pos[int(k)] for k in U["front"][f0: f0 + int(R["n_front"])]]
    speed = cat["speed"].astype(np.float64)
    ttft = cat["ttft"].astype(np.float64)
    feas = np.ones(nrow, dtype=bool)
    if workload.ttft_limit_ms is not None:
        feas &= ~(ttft > workload.ttft_limit_ms)
    floor = workload.speed_floor()
    if floor is not None:
        feas &= speed >= floor
    best = pos[int(R["best"])] if R["best"] >= 0 else -1
    nearest = pos[int(R["nearest"])] if (R["best"] < 0 and R["nearest"] >= 0) else -1
    n_tasks = int(np.count_nonzero(inb)) * (bool(modes & MODE_STATIC) + bool(modes & MODE_AGG))
    n_tasks += 2 * n if modes & MODE_DISAGG else 0
    kernel_ms = float(sum(out.totals.kernel_ms))
    rt = {"backend": db.backend, "chunked_prefill": space.chunked_prefill, "ctx_capacity": space.ctx_capacity,
          "cuda_graph": space.cuda_graph, "kv_mem_fraction": space.kv_mem_fraction}
    return Columns(
        model=model.name, backend=db.backend, workload_doc=workload.to_doc(), runtime=rt,
        mode=cat["mode"].astype(np.int64), cfg=cat["cfg"].astype(np.int64), gpus=cat["gpus"].astype(np.int64),
        ttft=ttft, tpot=cat["tpot"].astype(np.float64), speed=speed, thru=cat["thru"].astype(np.float64),
        feasible=feas, frontier_rows=front, pcfg=pcfg, dcfg=dcfg, x=xs, y=ys, r_sys=rs, skipped=skipped,
        best=best, nearest=nearest, violation=float(R["nearest_violation"]), enumerated=int(R["n_enumerated"]),
        total_ms=wall_ms, median_ms=(kernel_ms / n_tasks) if n_tasks else 0.0,
    )
