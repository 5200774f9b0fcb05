"""The drop-in search seam on the CUDA engine.

``run_search`` keeps the reference signature and results
(/root/reference/pkg/src/llmconf/search.py:280-358): it flattens the database
(once per object), compiles the model x space plan (once per triple), hands one
search descriptor to ``lc_search_batch`` and materialises the reference's
``SearchReport`` from the device's per-unit arrays.  ``Engine.sweep`` is the
columnar path for very large batches of searches: only per-search summaries
and Pareto fronts come back.

Inputs may be this package's spec objects or the reference's own; only
attributes are read.
"""

from __future__ import annotations

import ctypes as C
import functools
import math
import threading
import time
import weakref
from collections import OrderedDict
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as N
from .database import FlatDb, flatten
from .plans import LABELS, SpacePlan, build_space_plan
from .report import DisaggPlan, PerfEstimate, PoolCandidate, SearchReport, estimate_row, plan_row
from .specs import (
    DEFAULT_DISAGG,
    DEFAULT_MOE_LOAD,
    CandidateSpace,
    ParallelConfig,
    SearchError,
)

MODE_STATIC, MODE_AGG, MODE_DISAGG = 1, 2, 4
ST_OK, ST_MISSING, ST_EXTRAP, ST_UNSUPPORTED, ST_CHUNK_OFF, ST_NO_SLOT = range(6)


@functools.lru_cache(maxsize=64)
def _batch_list(src: tuple) -> tuple:
    """A search's batch list as the device takes it: sorted, values < 1 dropped
    (they make ParallelConfig raise, so enumerate_candidates skips them,
    search.py:101-105; model.py:190-193), duplicates kept as there.  A pure
    function of the (immutable) candidate-space tuple, cached like the plans."""
    return tuple(sorted(b for b in src if b >= 1))


@functools.lru_cache(maxsize=256)
def _moe_q(params, num_experts: int) -> np.ndarray:
    """[q_i = w_i / sum(w)] + by-weight order, numpy exactly as moe_load.py:51-57, 84, 97."""
    rng = np.random.default_rng(params.seed)
    u = rng.random(num_experts)
    e = 1.0 - params.alpha
    x = (u * (params.x_max**e - params.x_min**e) + params.x_min**e) ** (1.0 / e)
    w = np.array(tuple(float(v) for v in x))
    q = w / w.sum()
    order = np.lexsort((np.arange(num_experts), -w)).astype(np.float64)
    return np.concatenate([q, order])


@dataclass
class BatchOutput:
    """Device results of one lc_search_batch call (summaries on host, the rest on demand)."""

    engine: "Engine"
    results: np.ndarray           # SEARCH_RESULT_DTYPE per search
    totals: N.LcBatchTotals
    plan: SpacePlan
    flat: FlatDb
    batches: np.ndarray
    searches: np.ndarray
    wall_ms: float
    units: dict = field(default_factory=dict)
    h2d_bytes: int = 0
    d2h_bytes: int = 0

    def fetch_units(self) -> dict:
        if self.units:
            return self.units
        n = int(self.totals.n_units)
        nplan = int(self.totals.n_plans)
        nfront = int(self.totals.n_front)
        out = {}
        req = N.LcFetchReq()
        spec = {"unit_search": np.int32, "unit_combo": np.int32, "unit_batch": np.int32, "unit_in_budget": np.uint8,
                "st_status": np.int32, "st_ttft": np.float64, "st_tpot": np.float64, "st_speed": np.float64,
                "st_thru": np.float64, "ag_status": np.int32, "ag_ttft": np.float64, "ag_tpot": np.float64,
                "ag_speed": np.float64, "ag_thru": np.float64, "pf_status": np.int32, "pf_lat": np.float64,
                "pf_rate": np.float64, "dc_status": np.int32, "dc_lat": np.float64, "dc_rate": np.float64}
        for name, dt in spec.items():
            out[name] = np.zeros(max(n, 1), dtype=dt)
        out["err_c0"] = np.zeros(max(4 * n, 1), dtype=np.int64)
        out["err_c1"] = np.zeros(max(4 * n, 1), dtype=np.int64)
        pspec = {"plan_p": np.int32, "plan_d": np.int32, "plan_x": np.int32, "plan_y": np.int32,
                 "plan_gpus": np.int64, "plan_r_sys": np.float64, "plan_ttft": np.float64,
                 "plan_tpot": np.float64, "plan_speed": np.float64, "plan_thru": np.float64}
        for name, dt in pspec.items():
            out[name] = np.zeros(max(nplan, 1), dtype=dt)
        out["front"] = np.zeros(max(nfront, 1), dtype=np.int64)
        for name, ctype in N._FETCH_FIELDS:
            setattr(req, name, N.ptr(out[name], ctype._type_))
        self.engine._call(self.engine.lib.lc_fetch, "lc_fetch", self.engine.ctx, C.byref(req))
        self.units = out
        return out


def fetch_fronts(out: "BatchOutput") -> tuple[np.ndarray, dict]:
    """Columnar D2H for large sweeps: Pareto-front row keys and disaggregated plans only."""
    nplan, nfront = int(out.totals.n_plans), int(out.totals.n_front)
    front = np.zeros(max(nfront, 1), dtype=np.int64)
    plans = {"plan_p": np.zeros(max(nplan, 1), np.int32), "plan_d": np.zeros(max(nplan, 1), np.int32),
             "plan_x": np.zeros(max(nplan, 1), np.int32), "plan_y": np.zeros(max(nplan, 1), np.int32),
             "plan_gpus": np.zeros(max(nplan, 1), np.int64), "plan_speed": np.zeros(max(nplan, 1)),
             "plan_thru": np.zeros(max(nplan, 1))}
    req = N.LcFetchReq()
    req.front = N.ptr(front, C.c_int64)
    for name, arr in plans.items():
        setattr(req, name, N.ptr(arr, {np.dtype(np.int32): C.c_int32, np.dtype(np.int64): C.c_int64,
                                       np.dtype(np.float64): C.c_double}[arr.dtype]))
    out.engine._call(out.engine.lib.lc_fetch, "lc_fetch", out.engine.ctx, C.byref(req))
    return front[:nfront], {k: v[:nplan] for k, v in plans.items()}


class Engine:
    """One CUDA context (device + stream + workspace) with DB / plan handle caches."""

    def __init__(self, device: int = 0):
        self.lib = N.load_library()
        self.device = device
        ctx = C.c_void_p()
        N.check(self.lib.lc_open(device, C.byref(ctx)), "lc_open")
        self.ctx = ctx
        # device handle caches, LRU-bounded; evicted / stale entries free their device memory
        self._dbs: "OrderedDict[int, tuple]" = OrderedDict()
        self._spaces: "OrderedDict[tuple, tuple]" = OrderedDict()
        self._pinned: tuple = ()  # handles the last batch uses (lc_replay_* re-runs it)
        self._deferred: list = []  # evicted while pinned: freed once the next batch no longer uses them
        self._lock = threading.Lock()

    def _call(self, fn, name, *args):
        N.check(fn(*args), name)

    def close(self) -> None:
        for h, _, _ in self._spaces.values():
            self.lib.lc_space_free(h)
        for h, _, _ in self._dbs.values():
            self.lib.lc_db_free(h)
        for h, f in self._deferred:
            f(h)
        self._spaces.clear()
        self._dbs.clear()
        self._deferred = []
        self._pinned = ()
        if self.ctx:
            self.lib.lc_close(self.ctx)
            self.ctx = None

    # ------------------------------------------------------------------ handles
    MAX_DBS = 8
    MAX_SPACES = 32

    def _release(self, h, free) -> None:
        """Free a device handle now, or after the next batch when the last batch still uses it."""
        if any(h is x for x in self._pinned):
            self._deferred.append((h, free))
        else:
            free(h)

    def _free_space(self, key) -> None:
        self._release(self._spaces.pop(key)[0], self.lib.lc_space_free)

    def _free_db(self, dbid: int) -> None:
        for key in [k for k in self._spaces if k[0] == dbid]:
            self._free_space(key)
        self._release(self._dbs.pop(dbid)[0], self.lib.lc_db_free)

    def _evict(self) -> None:
        for cache, cap, free in ((self._spaces, self.MAX_SPACES, self._free_space),
                                 (self._dbs, self.MAX_DBS, self._free_db)):
            for key in list(cache):  # least recently used first
                if len(cache) <= cap:
                    break
                if key in cache:
                    free(key)

    def db_handle(self, db) -> tuple[C.c_void_p, FlatDb]:
        hit = self._dbs.get(id(db))
        if hit is not None and hit[2]() is db:
            self._dbs.move_to_end(id(db))
            return hit[0], hit[1]
        if hit is not None:  # id() reused by a new object: the old image is dead
            self._free_db(id(db))
        flat = flatten(db)
        hw = db.hardware
        d = N.LcDbDesc()
        d.n_grids = len(flat.keys)
        d.grid_ndim = N.ptr(flat.grid_ndim, C.c_int32)
        d.grid_axis_off = N.ptr(flat.grid_axis_off, C.c_int32)
        d.grid_axis_len = N.ptr(flat.grid_axis_len, C.c_int32)
        d.grid_cell_off = N.ptr(flat.grid_cell_off, C.c_int32)
        d.n_axis = len(flat.axis_val)
        d.axis_val = N.ptr(flat.axis_val, C.c_int64)
        d.axis_log = N.ptr(flat.axis_log, C.c_double)
        d.n_cells = len(flat.cell)
        d.cell = N.ptr(flat.cell, C.c_double)
        d.cell_log = N.ptr(flat.cell_log, C.c_double)
        d.mem_bandwidth = float(hw.mem_bandwidth)
        d.intra_node_bandwidth = float(hw.intra_node_bandwidth)
        d.inter_node_bandwidth = float(hw.inter_node_bandwidth)
        d.gpu_memory = float(hw.gpu_memory)
        d.gpus_per_node = int(hw.gpus_per_node)
        for i, q in enumerate(("fp16", "fp8", "int8", "int4")):
            d.compute[i] = float(hw.compute_throughput.get(q, 0.0))
        d.policy = flat.policy
        h = C.c_void_p()
        self._call(self.lib.lc_db_upload, "lc_db_upload", self.ctx, C.byref(d), C.byref(h))
        self._dbs[id(db)] = (h, flat, weakref.ref(db))
        self._evict()
        return h, flat

    @staticmethod
    def _plan_key(space) -> tuple:
        """The CandidateSpace fields build_space_plan reads (batch lists, pool caps and the
        KV fraction's value travel per search, not in the plan)."""
        return (tuple(space.tp_values), tuple(space.pp_values), tuple(space.ep_values), tuple(space.dp_values),
                space.ctx_capacity, bool(space.chunked_prefill), float(space.kv_mem_fraction),
                bool(space.cuda_graph))

    def space_handle(self, db, model, space) -> tuple[C.c_void_p, SpacePlan, FlatDb]:
        dbh, flat = self.db_handle(db)
        key = (id(db), model, self._plan_key(space))
        hit = self._spaces.get(key)
        if hit is not None and hit[2]() is db:
            self._spaces.move_to_end(key)
            return hit[0], hit[1], flat
        if hit is not None:
            self._free_space(key)
        plan = build_space_plan(model, space, flat, db.backend)
        d = N.LcSpaceDesc()
        d.hidden, d.topk, d.n_experts, d.is_moe = plan.hidden, plan.topk, plan.n_experts, int(plan.is_moe)
        d.n_combos = len(plan.combos)
        d.combos = N.vptr(plan.combos) if len(plan.combos) else None
        d.n_tmpl = len(plan.infos)
        d.tmpl_n_entries = N.ptr(plan.tmpl_n, C.c_int32)
        d.entries = N.vptr(plan.entries)
        d.n_tp, d.n_ep = len(plan.tp_values), len(plan.ep_values)
        d.n_slots = plan.n_slots
        d.slots = N.vptr(plan.slots)
        d.slot_of = N.ptr(plan.slot_of, C.c_int32)
        d.n_gen_classes = plan.n_gen
        d.gen_classes = N.vptr(plan.gen_entries)
        d.gclass_of = N.ptr(plan.gclass_of, C.c_int32)
        h = C.c_void_p()
        self._call(self.lib.lc_space_upload, "lc_space_upload", self.ctx, C.byref(d), C.byref(h))
        self._spaces[key] = (h, plan, weakref.ref(db))
        self._evict()
        return h, plan, flat

    # ------------------------------------------------------------------ batches
    def run_batch(self, db, model, space, workloads: Sequence, disagg=DEFAULT_DISAGG, mode_override=None,
                  enforce_budget: bool = True, mode_extra: int = 0, static_stride: int = 32) -> BatchOutput:
        t0 = time.perf_counter()
        sph, plan, flat = self.space_handle(db, model, space)
        dbh, _ = self.db_handle(db)
        self._pinned = (sph, dbh)
        if self._deferred:
            keep = [(h, f) for h, f in self._deferred if any(h is x for x in self._pinned)]
            for h, f in self._deferred:
                if not any(h is x for x in self._pinned):
                    f(h)
            self._deferred = keep
        n = len(workloads)
        searches = np.zeros(n, dtype=N.SEARCH_DESC_DTYPE)
        batches: list[int] = []
        b_index: dict[tuple, int] = {}  # identical batch lists share one copy
        loads: list[np.ndarray] = []
        load_ix: dict = {}
        if space.prefill_pool_cap < 0 or space.decode_pool_cap < 0:
            raise SearchError("pool caps must be >= 0")
        # one pass over the workloads collects every per-search field (runs of
        # workloads sharing the batch list / modes / load model reuse the last
        # lookup), then each column is written with one conversion
        ws = list(workloads)
        isl, osl, prefix, ttft_v, floor_v, cap_v, modes_v, b_off, n_b, load_v = ([] for _ in range(10))
        mode_of: dict = {}
        last_src = last_modes = last_params = None
        hit = m = ld = None
        is_moe = plan.is_moe
        for w in ws:
            isl.append(w.isl)
            osl.append(w.osl)
            prefix.append(w.prefix_len)
            t = w.ttft_limit_ms
            ttft_v.append(float(t) if t is not None else None)
            f = w.speed_floor()
            if f is not None:
                floor_v.append(float(f))
                cap_v.append(float(1000.0 / f))  # tpot_ceiling() = 1000 / speed_floor() (specs.py)
            else:
                floor_v.append(None)
                cap_v.append(0.0)
            if mode_override is None and w.modes is not last_modes:
                last_modes = w.modes
                m = mode_of.get(last_modes)
                if m is None:
                    m = mode_of[last_modes] = ((MODE_STATIC if "static" in last_modes else 0)
                                               | (MODE_AGG if "aggregated" in last_modes else 0)
                                               | (MODE_DISAGG if "disaggregated" in last_modes else 0) | mode_extra)
            modes_v.append(m)
            src = w.batch_sweep or space.batch_values
            if src is not last_src:
                last_src = src
                key = (id(src), len(src)) if isinstance(src, tuple) else tuple(src)
                hit = b_index.get(key)
                if hit is None:
                    bs = _batch_list(src if isinstance(src, tuple) else tuple(src))
                    hit = b_index.get(bs)
                    if hit is None:
                        hit = (len(batches), len(bs))
                        batches.extend(bs)
                        b_index[bs] = hit
                    b_index[key] = hit
            b_off.append(hit[0])
            n_b.append(hit[1])
            if is_moe:
                params = w.moe_load if w.moe_load is not None else DEFAULT_MOE_LOAD
                if params is not last_params:
                    last_params = params
                    lk = (params.alpha, params.x_min, params.x_max, params.seed)
                    ld = load_ix.get(lk)
                    if ld is None:
                        ld = load_ix[lk] = len(loads)
                        loads.append(_moe_q(params, plan.n_experts))
                load_v.append(ld)
        searches["isl"] = isl
        searches["osl"] = osl
        searches["prefix"] = prefix
        searches["has_ttft"] = [t is not None for t in ttft_v]
        searches["ttft_limit"] = [t if t is not None else 0.0 for t in ttft_v]
        searches["has_floor"] = [f is not None for f in floor_v]
        searches["speed_floor"] = [f if f is not None else 0.0 for f in floor_v]
        searches["tpot_cap"] = cap_v
        searches["modes"] = mode_override if mode_override is not None else modes_v
        if enforce_budget:
            budget_rows = searches["budgets"]
            for i, w in enumerate(ws):
                if w.gpu_budgets:
                    budgets = sorted(set(w.gpu_budgets))
                    if len(budgets) > N.LC_MAX_BUDGETS:
                        raise SearchError(f"at most {N.LC_MAX_BUDGETS} distinct gpu budgets are supported")
                    searches["n_budgets"][i] = len(budgets)
                    budget_rows[i, : len(budgets)] = budgets
        searches["b_off"], searches["n_b"] = b_off, n_b
        searches["load"] = load_v if is_moe else -1
        searches["has_ctx_capacity"] = space.ctx_capacity is not None
        searches["ctx_capacity"] = space.ctx_capacity or 0
        searches["chunked_prefill"] = int(bool(space.chunked_prefill))
        searches["kv_mem_fraction"] = float(space.kv_mem_fraction)
        searches["prefill_cap"], searches["decode_cap"] = space.prefill_pool_cap, space.decode_pool_cap
        searches["ttft_headroom"] = float(disagg.ttft_headroom)
        searches["prefill_util"] = float(disagg.prefill_utilization)
        searches["decode_util"] = float(disagg.decode_utilization)
        searches["max_x"], searches["max_y"] = disagg.max_prefill_replicas, disagg.max_decode_replicas
        searches["static_stride"] = static_stride  # estimate_static's decode stride (serving_modes.py:236)
        b_arr = np.array(batches if batches else [1], dtype=np.int64)
        l_arr = np.concatenate(loads) if loads else np.zeros(1)
        results = np.zeros(n, dtype=N.SEARCH_RESULT_DTYPE)
        totals = N.LcBatchTotals()
        self._call(self.lib.lc_search_batch, "lc_search_batch", self.ctx, dbh, sph, n, N.vptr(searches),
                   len(batches), N.ptr(b_arr, C.c_int64), len(loads), N.ptr(l_arr, C.c_double),
                   N.vptr(results), C.byref(totals))
        out = BatchOutput(self, results, totals, plan, flat, b_arr, searches, (time.perf_counter() - t0) * 1000.0)
        out.h2d_bytes = searches.nbytes + 8 * len(batches) + (l_arr.nbytes if loads else 0)
        out.d2h_bytes = results.nbytes + 4
        return out

    def set_raw_filter(self, lo: int = 0, hi: int = -1, mask: np.ndarray | None = None) -> None:
        """Restrict the raw candidate tuples of the following batches (lc_set_raw_filter); hi < 0 clears."""
        m = None
        if mask is not None:
            mask = np.ascontiguousarray(mask, dtype=np.uint8)
            if len(mask) != hi - lo:
                raise ValueError("mask length must be hi - lo")
            m = C.c_void_p(mask.ctypes.data)
        self._call(self.lib.lc_set_raw_filter, "lc_set_raw_filter", self.ctx, int(lo), int(hi), m)

    def fetch_pools(self, n_search: int) -> tuple[np.ndarray, np.ndarray]:
        """Pool selections of the last batch: units [n_search, 2, 64] and counts [n_search, 2]."""
        units = np.zeros((max(n_search, 1), 2, 64), dtype=np.int32)
        counts = np.zeros((max(n_search, 1), 2), dtype=np.int32)
        self._call(self.lib.lc_fetch_pools, "lc_fetch_pools", self.ctx, N.ptr(units, C.c_int32),
                   N.ptr(counts, C.c_int32))
        return units[:n_search], counts[:n_search]

    def unit_raw(self, units: np.ndarray) -> np.ndarray:
        """Raw tuple index of each unit of the last batch (lc_unit_raw)."""
        u = np.ascontiguousarray(units, dtype=np.int32)
        raw = np.zeros(max(len(u), 1), dtype=np.int64)
        self._call(self.lib.lc_unit_raw, "lc_unit_raw", self.ctx, len(u), N.ptr(u, C.c_int32), N.ptr(raw, C.c_int64))
        return raw[: len(u)]

    def replay_async(self) -> None:
        """Enqueue the last batch's device pipeline on this engine's stream (no sync)."""
        self._call(self.lib.lc_replay_async, "lc_replay_async", self.ctx)

    def set_priority(self, priority: int) -> None:
        """Stream priority of this engine (lc_set_priority): negative = higher, 0 = default."""
        self._call(self.lib.lc_set_priority, "lc_set_priority", self.ctx, int(priority))

    def stream_ptr(self) -> int:
        """cudaStream_t of this engine (for torch.cuda.ExternalStream)."""
        h = C.c_void_p()
        self._call(self.lib.lc_stream, "lc_stream", self.ctx, C.byref(h))
        return int(h.value or 0)

    def replay(self, iters: int = 1) -> N.LcBatchTotals:
        """Re-run the last batch's device pipeline (K0..K4) on resident inputs; per-kernel CUDA-event ms."""
        totals = N.LcBatchTotals()
        self._call(self.lib.lc_replay_last, "lc_replay_last", self.ctx, iters, C.byref(totals))
        return totals


# ------------------------------------------------------------------------------ report building
def _reason(code_word: int, c0: int, c1: int, plan: SpacePlan, combo, flat: FlatDb, db, workload, space,
            batch: int) -> str:
    code, label = code_word & 0xFF, code_word >> 8
    if code in (ST_MISSING, ST_EXTRAP, ST_UNSUPPORTED):
        info = next(e for e in plan.infos[int(combo["tmpl"])] if e.label == LABELS[label])
        if code == ST_MISSING:
            return f"MissingKeyError: no grid for key {info.key}; database covers kinds {flat.kinds}"
        if code == ST_UNSUPPORTED:
            return (f"UnsupportedOperatorError: hardware {db.hardware.name!r} has no compute rate for quant "
                    f"{info.quant!r}")
        axes = flat.axes[info.grid]
        values = flat.axis_values[info.grid]
        coords = (c0, c1)[: len(axes)]
        box = {a: (v[0], v[-1]) for a, v in zip(axes, values)}
        return f"ExtrapolationError: query coords {dict(zip(axes, coords))} outside grid box {box}"
    chunk_total = workload.isl - workload.prefix_len
    c_ctx = space.ctx_capacity if space.ctx_capacity is not None else max(chunk_total, 2048)
    if code == ST_CHUNK_OFF:
        return f"InfeasibleConfigError: context of {chunk_total} tokens exceeds capacity {c_ctx} and chunking is off"
    if code == ST_NO_SLOT:
        prefilling = math.ceil(c_ctx / chunk_total)
        return f"InfeasibleConfigError: batch {batch} too small to decode alongside {prefilling} prefilling requests"
    raise SearchError(f"unknown device status {code_word}")


def build_report(out: BatchOutput, si: int, db, model, workload, space, wall_ms: float) -> SearchReport:
    """Materialise the reference SearchReport of search ``si`` from device arrays."""
    U = out.fetch_units()
    R = out.results[si]
    plan, flat = out.plan, out.flat
    off, n = int(R["unit_off"]), int(R["n_units"])
    sl = slice(off, off + n)
    combos = plan.combos[U["unit_combo"][sl]]
    bidx = U["unit_batch"][sl]
    s = out.searches[si]
    batches = out.batches[int(s["b_off"]) + bidx]
    inb = U["unit_in_budget"][sl].astype(bool)
    modes = int(s["modes"])
    cfgs = [space.config(int(c["tp"]), int(c["pp"]), int(c["ep"]), int(c["dp"]), int(b), db.backend)
            for c, b in zip(combos, batches)]
    by_key: dict[int, object] = {}
    rows, skipped = [], []
    err0, err1 = U["err_c0"], U["err_c1"]

    def add_mode(mode_bit, mode_idx, name, prefix):
        if not modes & mode_bit:
            return
        st = U[f"{prefix}_status"][sl]
        ttft, tpot, speed, thru = (U[f"{prefix}_{k}"][sl] for k in ("ttft", "tpot", "speed", "thru"))
        for i in np.nonzero(inb)[0]:
            i = int(i)
            cfg = cfgs[i]
            if st[i] == 0:
                est = PerfEstimate(name, model.name, cfg, float(ttft[i]), float(tpot[i]), float(speed[i]),
                                   float(thru[i]), cfg.gpus(), cfg.batch)
                row = estimate_row(est)
                rows.append(row)
                by_key[(mode_idx << 32) | i] = row
            else:
                k = 4 * (off + i) + mode_idx
                skipped.append({"mode": name, "config": cfg.key(),
                                "reason": _reason(int(st[i]), int(err0[k]), int(err1[k]), plan, combos[i], flat, db,
                                                  workload, space, cfg.batch)})

    add_mode(MODE_STATIC, 0, "static", "st")
    add_mode(MODE_AGG, 1, "aggregated", "ag")
    n_tasks = (int(np.count_nonzero(inb)) * (bool(modes & MODE_STATIC) + bool(modes & MODE_AGG)))
    if modes & MODE_DISAGG:
        n_tasks += 2 * n
        pf_st, dc_st = U["pf_status"][sl], U["dc_status"][sl]
        for i in range(n):
            for kind, st, name in ((2, pf_st, "disaggregated/prefill"), (3, dc_st, "disaggregated/decode")):
                if st[i] != 0:
                    k = 4 * (off + i) + kind
                    skipped.append({"mode": name, "config": cfgs[i].key(),
                                    "reason": _reason(int(st[i]), int(err0[k]), int(err1[k]), plan, combos[i], flat,
                                                      db, workload, space, cfgs[i].batch)})
        p0 = int(out.results["n_plans"][:si].sum())
        for j in range(int(R["n_plans"])):
            k = p0 + j
            up, ud = int(U["plan_p"][k]) - off, int(U["plan_d"][k]) - off
            pc = PoolCandidate("prefill", cfgs[up], float(U["pf_lat"][off + up]), float(U["pf_rate"][off + up]),
                               cfgs[up].gpus())
            dc = PoolCandidate("decode", cfgs[ud], float(U["dc_lat"][off + ud]), float(U["dc_rate"][off + ud]),
                               cfgs[ud].gpus())
            dp = DisaggPlan(pc, dc, int(U["plan_x"][k]), int(U["plan_y"][k]), int(U["plan_gpus"][k]),
                            float(U["plan_r_sys"][k]), float(U["plan_ttft"][k]), float(U["plan_tpot"][k]),
                            float(U["plan_speed"][k]), float(U["plan_thru"][k]))
            row = plan_row(dp)
            rows.append(row)
            by_key[(2 << 32) | j] = row
    f0 = int(out.results["n_front"][:si].sum())
    frontier = [by_key[int(k)] for k in U["front"][f0: f0 + int(R["n_front"])]]
    best = by_key[int(R["best"])] if R["best"] >= 0 else None
    nearest = by_key[int(R["nearest"])] if (best is None and R["nearest"] >= 0) else None
    kernel_ms = float(sum(out.totals.kernel_ms))
    per = [kernel_ms / n_tasks] * n_tasks if n_tasks else []
    return SearchReport(model=model.name, backend=db.backend, workload=workload, rows=rows, frontier=frontier,
                        best=best, skipped=skipped, enumerated=int(R["n_enumerated"]), total_ms=wall_ms,
                        per_candidate_ms=per, nearest=nearest)


_ENGINES: dict[int, Engine] = {}
_ENGINES_LOCK = threading.Lock()


def get_engine(device: int = 0) -> Engine:
    """Process-wide engine per device (one stream; calls are serialised)."""
    with _ENGINES_LOCK:
        eng = _ENGINES.get(device)
        if eng is None:
            eng = _ENGINES[device] = Engine(device)
        return eng


def run_search(db, model, workload, space=CandidateSpace(), jobs: int = 1, disagg_constants=DEFAULT_DISAGG,
               device: int = 0) -> SearchReport:
    """Drop-in for llmconf.search.run_search (search.py:280-358) on the B200 engine.

    ``jobs`` is validated like the reference and otherwise ignored: the search
    is one batched device pass whatever its value.
    """
    if jobs < 1:
        raise SearchError("jobs must be >= 1")
    t0 = time.perf_counter()
    eng = get_engine(device)
    with eng._lock:
        out = eng.run_batch(db, model, space, [workload], disagg_constants)
        return build_report(out, 0, db, model, workload, space, (time.perf_counter() - t0) * 1000.0)


def enumerate_candidates(model, space, workload, db, enforce_budget: bool = True, device: int = 0) -> list:
    """Drop-in for llmconf.search.enumerate_candidates (search.py:82-113), K0 on the device."""
    eng = get_engine(device)
    with eng._lock:
        out = eng.run_batch(db, model, space, [workload], mode_override=0, enforce_budget=enforce_budget)
        U = out.fetch_units()
        n = int(out.results[0]["n_units"])
        combos = out.plan.combos[U["unit_combo"][:n]]
        bs = out.batches[U["unit_batch"][:n]]
        return [space.config(int(c["tp"]), int(c["pp"]), int(c["ep"]), int(c["dp"]), int(b), db.backend)
                for c, b in zip(combos, bs)]


def run_search_json(db, model, workload, space=CandidateSpace(), jobs: int = 1,
                    disagg_constants=DEFAULT_DISAGG, device: int = 0) -> str:
    """``run_search(...).to_json()`` without materialising per-row objects.

    Same bytes as the reference's report JSON (search.py:262-264); rows are
    written from the device's column arrays (fastreport.report_json).
    """
    return search_json_columns(db, model, workload, space, jobs, disagg_constants, device)[0]


def search_json_columns(db, model, workload, space=CandidateSpace(), jobs: int = 1,
                        disagg_constants=DEFAULT_DISAGG, device: int = 0):
    """(report JSON text, fastreport.Columns): run_search_json plus the columns it was written from."""
    from .fastreport import columns_from_batch, report_json

    if jobs < 1:
        raise SearchError("jobs must be >= 1")
    t0 = time.perf_counter()
    eng = get_engine(device)
    with eng._lock:
        out = eng.run_batch(db, model, space, [workload], disagg_constants)
        cols = columns_from_batch(out, 0, db, model, workload, space, 0.0)
    cols.total_ms = (time.perf_counter() - t0) * 1000.0
    return report_json(cols), cols


def count_candidates(model, space, workload, db, enforce_budget: bool = True, device: int = 0) -> int:
    """len(enumerate_candidates(...)) from K0 alone: no configs are materialised on the host."""
    eng = get_engine(device)
    with eng._lock:
        out = eng.run_batch(db, model, space, [workload], mode_override=0, enforce_budget=enforce_budget)
        return int(out.results[0]["n_units"])


MODE_FORCE = 16  # LC_MODE_FORCE: no memory-fit / budget filter


def consistency_problems(model, cfg) -> list[str]:
    """check_consistency messages (model.py:209-236)."""
    out = []
    if model.num_heads % cfg.tp:
        out.append(f"tp={cfg.tp} does not divide num_heads={model.num_heads}")
    if cfg.pp > model.num_layers:
        out.append(f"pp={cfg.pp} exceeds num_layers={model.num_layers}")
    moe = model.moe
    if moe is None:
        if cfg.ep != 1:
            out.append("ep > 1 requires a mixture-of-experts model")
        if cfg.tp <= model.intermediate_size and model.intermediate_size % cfg.tp:
            out.append(f"tp={cfg.tp} does not divide intermediate_size={model.intermediate_size}")
    else:
        if moe.num_experts % cfg.ep:
            out.append(f"ep={cfg.ep} does not divide num_experts={moe.num_experts}")
        if cfg.ep > cfg.tp * cfg.dp:
            out.append(f"ep={cfg.ep} exceeds tp*dp={cfg.tp * cfg.dp}")
        hi, lo = max(cfg.ep, cfg.tp), min(cfg.ep, cfg.tp)
        if hi % lo:
            out.append(f"ep={cfg.ep} and tp={cfg.tp} must nest (one divides the other)")
        elif cfg.tp > cfg.ep and moe.expert_intermediate % (cfg.tp // cfg.ep):
            out.append(f"tp/ep={cfg.tp // cfg.ep} does not divide expert_intermediate={moe.expert_intermediate}")
        if moe.shared_intermediate and cfg.tp <= moe.shared_intermediate and moe.shared_intermediate % cfg.tp:
            out.append(f"tp={cfg.tp} does not divide shared_intermediate={moe.shared_intermediate}")
    return out


def _estimate(mode_bit: int, name: str, db, model, cfg, workload, device: int, stride: int = 32):
    import dataclasses

    from . import specs as S

    problems = consistency_problems(model, cfg)
    if problems:
        raise S.ParallelConfigError("; ".join(problems))
    space = CandidateSpace(tp_values=(cfg.tp,), pp_values=(cfg.pp,), ep_values=(cfg.ep,), dp_values=(cfg.dp,),
                           batch_values=(cfg.batch,), ctx_capacity=cfg.ctx_capacity,
                           chunked_prefill=cfg.chunked_prefill, kv_mem_fraction=cfg.kv_mem_fraction,
                           cuda_graph=cfg.cuda_graph)
    wl = dataclasses.replace(workload, batch_sweep=())
    eng = get_engine(device)
    with eng._lock:
        out = eng.run_batch(db, model, space, [wl], mode_override=mode_bit | MODE_FORCE, enforce_budget=False,
                            static_stride=stride)
        U = out.fetch_units()
        if int(out.results[0]["n_units"]) != 1:
            raise SearchError("single-config estimate did not produce exactly one unit")
        pre = "st" if mode_bit == MODE_STATIC else "ag"
        st = int(U[f"{pre}_status"][0])
        if st:
            k = 0 if mode_bit == MODE_STATIC else 1
            msg = _reason(st, int(U["err_c0"][k]), int(U["err_c1"][k]), out.plan, out.plan.combos[U["unit_combo"][0]],
                          out.flat, db, workload, space, cfg.batch)
            kind, text = msg.split(": ", 1)
            raise getattr(S, kind)(text)
        return PerfEstimate(name, model.name, cfg, float(U[f"{pre}_ttft"][0]), float(U[f"{pre}_tpot"][0]),
                            float(U[f"{pre}_speed"][0]), float(U[f"{pre}_thru"][0]), cfg.gpus(), cfg.batch)


def estimate_static(db, model, cfg, workload, stride: int = 32, device: int = 0) -> PerfEstimate:
    """Drop-in for serving_modes.estimate_static (serving_modes.py:231-267) for one config.

    Raises like the reference (ParallelConfigError, PerfDbError subclasses).  The
    decode loop samples the KV length every ``stride`` tokens on the device (the
    decode-series table and loop take the stride per search); stride 1 is the
    reference's brute-force setting (acceptance A2, tests/test_acceptance.py:96-135).
    """
    from .specs import WorkloadError

    if stride < 1:
        raise WorkloadError("stride must be >= 1")
    if stride > 2**31 - 1:
        stride = 2**31 - 1  # any stride >= osl - 1 samples once; keep it in the descriptor's int32
    return _estimate(MODE_STATIC, "static", db, model, cfg, workload, device, int(stride))


def estimate_aggregated(db, model, cfg, workload, device: int = 0) -> PerfEstimate:
    """Drop-in for serving_modes.estimate_aggregated (serving_modes.py:279-341) for one config."""
    return _estimate(MODE_AGG, "aggregated", db, model, cfg, workload, device)
