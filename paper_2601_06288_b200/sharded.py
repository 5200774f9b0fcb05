"""One search sharded across GPUs: one process per GPU, one
exchange step.

Candidates are independent until the per-search reductions, so each rank runs
the whole device pipeline (K0 .. K4) on a contiguous block of the search's raw
(tp, pp, ep, dp, batch) tuples -- ``lc_set_raw_filter`` -- with
``LC_MODE_NO_PLANS``: pools are selected, but no disaggregated plans are built,
so the local front / best / nearest miss cover static and aggregated rows only.

Each rank then reduces its block to the candidates any global answer can
need -- its local Pareto-front rows, its local best and nearest miss, and its
local top-k prefill / decode pool members (search.py:336-339) -- identified by
raw tuple index, plus its counts.  One all-gather of those small records
(``dist.all_gather_bytes``, one fixed-size payload: NCCL over NVLink on a GPU box) gives every rank the
union S, and every rank runs one *merge pass* of the same pipeline on S
(``lc_set_raw_filter`` with a mask).  The merge pass's answers are the global
ones because, for any S with global-front ⊆ S ⊆ all rows,

* pareto_filter(S) = pareto_filter(all) (search.py:156-175): a row off the
  global front is dominated by a global-front row, which is in S;
* select_best(S) = select_best(all): the best row is on the global front;
* top-k(S) = top-k(all) for each pool, since the global top-k is inside the
  union of the local top-k lists -- so estimate_disaggregated
  (serving_modes.py:449-494) on S builds exactly the reference's plans, and
  the plans join the front and best in the same pass;
* the nearest miss (search.py:190-208) is needed only when nothing is feasible
  anywhere, and then every rank's local nearest miss is in S.

Row order is preserved: S keeps the global candidate order, so the merge
pass's front tie-breaks (speed desc, then row order) match.  Counts are sums of
the ranks' counts plus the merge pass's plan rows.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .dist import all_gather_bytes, pack_records, shard_range, unpack_records
from .engine import MODE_DISAGG, BatchOutput, build_report, fetch_fronts, get_engine
from .specs import DEFAULT_DISAGG, CandidateSpace, SearchError

MODE_NO_PLANS = 32  # LC_MODE_NO_PLANS (include/llmconf_b200.h)

COUNTS_DTYPE = np.dtype([("n_units", "<i8"), ("n_enumerated", "<i8"), ("n_rows", "<i8"), ("n_feasible", "<i8"),
                         ("n_skipped", "<i8"), ("queries_1d", "<i8"), ("queries_2d", "<i8")])
KEEP_DTYPE = np.dtype([("raw", "<i8"), ("unit", "<i8")])


@dataclass
class LocalShard:
    """One rank's reduction of its candidate block."""

    counts: np.ndarray           # COUNTS_DTYPE, one record
    keep: np.ndarray             # KEEP_DTYPE: (raw tuple index, local unit index), sorted by raw
    device_ms: float = 0.0


@dataclass
class ShardedResult:
    """Global answer of a sharded search: counts, front, best, nearest miss, plans.

    ``report`` is the merge pass's SearchReport: its frontier / best /
    diagnostics documents are the global ones (the rows it holds are the union
    set S only).  Row indices in ``front`` / ``best`` are global: static and
    aggregated rows are (mode, global unit index), plans (2, plan index).
    """

    counts: dict
    front: list
    best: tuple | None
    nearest: tuple | None
    plans: dict
    report: object
    n_union: int
    timing_ms: dict = field(default_factory=dict)

    def summary_doc(self) -> dict:
        """The reference report document minus per-row data (rows, skipped, timing)."""
        doc = self.report.to_doc()
        return {
            "schema": doc["schema"], "version": doc["version"], "model": doc["model"], "backend": doc["backend"],
            "workload": doc["workload"], "counts": dict(self.counts), "frontier": doc["frontier"],
            "best": doc["best"], "diagnostics": doc["diagnostics"],
        }


def _n_raw(plan, workload, space) -> int:
    src = workload.batch_sweep or space.batch_values
    return len(plan.combos) * sum(1 for b in src if b >= 1)  # batch values < 1 are skipped (engine.run_batch)


def _modes(workload) -> int:
    return ((1 if "static" in workload.modes else 0) | (2 if "aggregated" in workload.modes else 0)
            | (4 if "disaggregated" in workload.modes else 0))


def local_pass(eng, db, model, workload, space, disagg, lo: int, hi: int) -> LocalShard:
    """Evaluate raw tuples [lo, hi) of the search and reduce them (caller holds eng._lock)."""
    t0 = time.perf_counter()
    eng.set_raw_filter(lo, hi)
    try:
        out = eng.run_batch(db, model, space, [workload], disagg, mode_extra=MODE_NO_PLANS)
    finally:
        eng.set_raw_filter()
    R = out.results[0]
    counts = np.zeros(1, COUNTS_DTYPE)
    for name in COUNTS_DTYPE.names:
        counts[name] = int(R[name])
    units: set[int] = set()
    front, _ = fetch_fronts(out)
    for key in list(front) + [int(R["best"]), int(R["nearest"])]:
        key = int(key)
        if key >= 0 and (key >> 32) < 2:
            units.add(key & 0xFFFFFFFF)
    if _modes(workload) & MODE_DISAGG:
        sel, cnt = eng.fetch_pools(1)
        units.update(int(u) for u in sel[0, 0, : cnt[0, 0]])
        units.update(int(u) for u in sel[0, 1, : cnt[0, 1]])
    u = np.array(sorted(units), dtype=np.int32)
    keep = np.zeros(len(u), KEEP_DTYPE)
    if len(u):
        keep["raw"] = eng.unit_raw(u)
        keep["unit"] = u
        if (keep["raw"] < 0).any():
            raise SearchError("local pass referenced a unit outside the batch")
    return LocalShard(counts, keep, (time.perf_counter() - t0) * 1000.0)


def merge_pass(eng, db, model, workload, space, disagg, shards: list[LocalShard]) -> ShardedResult:
    """Global front / best / nearest / plans from every rank's LocalShard (caller holds eng._lock)."""
    t0 = time.perf_counter()
    offs = np.cumsum([0] + [int(s.counts["n_units"][0]) for s in shards])
    gunit: dict[int, int] = {}
    for r, s in enumerate(shards):
        for raw, u in zip(s.keep["raw"].tolist(), s.keep["unit"].tolist()):
            gunit[raw] = int(offs[r]) + u
    S = np.array(sorted(gunit), dtype=np.int64)
    lo, hi = (int(S[0]), int(S[-1]) + 1) if len(S) else (0, 0)
    mask = np.zeros(hi - lo, dtype=np.uint8)
    mask[S - lo] = 1
    eng.set_raw_filter(lo, hi, mask)
    try:
        out: BatchOutput = eng.run_batch(db, model, space, [workload], disagg)
    finally:
        eng.set_raw_filter()
    R = out.results[0]
    if int(R["n_units"]) != len(S):
        raise SearchError(f"merge pass kept {int(R['n_units'])} of {len(S)} union candidates")
    g_of = np.array([gunit[int(x)] for x in S], dtype=np.int64)

    def gkey(key: int) -> tuple | None:
        if key < 0:
            return None
        mode, i = key >> 32, key & 0xFFFFFFFF
        return (int(mode), int(g_of[i]) if mode < 2 else int(i))

    front, plans = fetch_fronts(out)
    plans = dict(plans)
    for k in ("plan_p", "plan_d"):
        plans[k] = g_of[plans[k]] if len(plans[k]) else plans[k].astype(np.int64)
    tot = {name: int(sum(int(s.counts[name][0]) for s in shards)) for name in COUNTS_DTYPE.names}
    report = build_report(out, 0, db, model, workload, space, 0.0)
    counts = {"enumerated": tot["n_enumerated"], "evaluated": tot["n_rows"] + int(R["n_plans"]),
              "feasible": tot["n_feasible"] + int(R["n_feasible_plans"]), "frontier": int(R["n_front"]),
              "skipped": tot["n_skipped"]}
    best = gkey(int(R["best"]))
    nearest = gkey(int(R["nearest"])) if best is None else None
    res = ShardedResult(counts, [gkey(int(k)) for k in front], best, nearest, plans, report, len(S))
    res.timing_ms["merge"] = (time.perf_counter() - t0) * 1000.0
    res.timing_ms["units"] = tot["n_units"]
    res.timing_ms["queries_1d"] = tot["queries_1d"]
    res.timing_ms["queries_2d"] = tot["queries_2d"]
    return res


def _default_exchange(payload: bytes) -> list[bytes]:
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return all_gather_bytes(payload)
    return [payload]


def run_search_sharded(db, model, workload, space=CandidateSpace(), disagg_constants=DEFAULT_DISAGG,
                       rank: int | None = None, world: int | None = None, device: int = 0,
                       exchange=None) -> ShardedResult:
    """run_search's reductions for one search split over ``world`` ranks (one process per GPU).

    Every rank calls this with the same inputs; every rank returns the same
    global result.  ``exchange(payload: bytes) -> [payload of rank 0, 1, ...]``
    is the all-gather (default: one fixed-size torch.distributed all-gather of
    the packed counts + keep set, ``dist.all_gather_bytes``; world = 1 when
    torch.distributed is not initialised).
    """
    if rank is None or world is None:
        import torch.distributed as dist

        init = dist.is_available() and dist.is_initialized()
        rank = dist.get_rank() if init else 0
        world = dist.get_world_size() if init else 1
    if not 0 <= rank < world:
        raise SearchError("rank must be in [0, world)")
    exchange = exchange or _default_exchange
    t0 = time.perf_counter()
    eng = get_engine(device)
    with eng._lock:
        _, plan, _ = eng.space_handle(db, model, space)
        lo, hi = shard_range(_n_raw(plan, workload, space), rank, world)
        mine = local_pass(eng, db, model, workload, space, disagg_constants, lo, hi)
    t1 = time.perf_counter()
    # ONE exchange per search: counts and keep set packed into a single record
    gathered = exchange(pack_records(mine.counts, mine.keep))
    shards = [LocalShard(*unpack_records(b, [COUNTS_DTYPE, KEEP_DTYPE])) for b in gathered]
    t2 = time.perf_counter()
    with eng._lock:
        res = merge_pass(eng, db, model, workload, space, disagg_constants, shards)
    res.timing_ms.update(local=(t1 - t0) * 1000.0, exchange=(t2 - t1) * 1000.0,
                         total=(time.perf_counter() - t0) * 1000.0)
    return res
