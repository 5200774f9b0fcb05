"""Step latencies with the per-operator breakdown (the reference's L3 interface).

Drop-ins for ``llmconf.estimator.get_step_latency`` / ``get_mix_latency`` /
``get_gen_latency`` (/root/reference/pkg/src/llmconf/estimator.py:71-156):
same arguments, same ``StepLatency(total_ms, breakdown)`` result (breakdown in
plan order, one entry per plan label, ``total_ms`` = CPython's float sum of the
breakdown), same exceptions (``ParallelConfigError`` from ``decompose``'s
checks, model.py:286-299; ``MissingKeyError`` / ``ExtrapolationError`` /
``UnsupportedOperatorError`` from the first failing query in plan order).

Every number comes from the device (``lc_step_latency``: one warp per step --
the busiest-EP-shard expert tokens, each plan entry's interpolated latency and
the bubble-scaled plan-order sum); the host only resolves the (tp, pp, ep)
template of the configuration and formats errors.  ``step_latency_batch``
prices many steps of one (db, model) in a single launch.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

from . import _native as N
from .plans import LABELS
from .specs import DEFAULT_MOE_LOAD, CandidateSpace, ParallelConfigError

PHASES = ("prefill", "decode", "mixed")
GEN_KV_MIDPOINT = True  # estimator.py:20


class EstimationError(RuntimeError):
    """Latency could not be estimated for this configuration (estimator.py:24-25)."""


@dataclass(frozen=True)
class StepLatency:
    """One iteration's latency in milliseconds with a per-operator breakdown (estimator.py:28-42)."""

    total_ms: float
    breakdown: Mapping[str, float]

    def __post_init__(self) -> None:
        s = sum(self.breakdown.values())
        if self.total_ms and abs(s - self.total_ms) > 1e-9 * abs(self.total_ms):
            raise EstimationError(f"breakdown sums to {s}, total is {self.total_ms}")


@dataclass(frozen=True)
class StepRequest:
    """Arguments of one get_step_latency call."""

    cfg: object
    phase: str
    n_ctx_tokens: int = 0
    n_gen_tokens: int = 0
    seq_len: int = 1
    moe_load: object = None


def _check(model, cfg, phase: str, n_ctx: int, n_gen: int, seq: int) -> None:
    """decompose's argument checks, in its order and with its messages (model.py:286-299)."""
    from .engine import consistency_problems

    if phase not in PHASES:
        raise ParallelConfigError(f"phase must be one of {PHASES}")
    problems = consistency_problems(model, cfg)
    if problems:
        raise ParallelConfigError("; ".join(problems))
    if phase == "prefill" and (n_ctx < 1 or n_gen):
        raise ParallelConfigError("prefill pass needs n_ctx_tokens >= 1 and no generation tokens")
    if phase == "decode" and (n_gen < 1 or n_ctx):
        raise ParallelConfigError("decode pass needs n_gen_tokens >= 1 and no context tokens")
    if phase == "mixed" and (n_ctx < 1 or n_gen < 0):
        raise ParallelConfigError("mixed pass needs n_ctx_tokens >= 1")
    if seq < 1:
        raise ParallelConfigError("seq_len must be >= 1")
    if phase == "prefill" and n_ctx % seq:
        raise ParallelConfigError(f"n_ctx_tokens={n_ctx} not a multiple of seq_len={seq}")


def step_latency_batch(db, model, requests: Sequence[StepRequest], device: int = 0) -> list:
    """StepLatency (or the exception instance the reference would raise) per request, one launch."""
    from . import specs as S
    from .engine import _moe_q, _reason, get_engine

    out: list = [None] * len(requests)
    live = []
    for i, r in enumerate(requests):
        try:
            _check(model, r.cfg, r.phase, r.n_ctx_tokens, r.n_gen_tokens, r.seq_len)
            live.append(i)
        except ParallelConfigError as e:
            out[i] = e
    if not live:
        return out
    eng = get_engine(device)
    with eng._lock:
        # one space plan holding a template for every requested (tp, pp, ep): the
        # cross product of the requested values (each request's own config is
        # consistent, so its combo and template are in it); one launch
        cfgs = [requests[i].cfg for i in live]
        space = CandidateSpace(tp_values=tuple(sorted({c.tp for c in cfgs})),
                               pp_values=tuple(sorted({c.pp for c in cfgs})),
                               ep_values=tuple(sorted({c.ep for c in cfgs})),
                               dp_values=tuple(sorted({c.dp for c in cfgs})))
        sph, plan, flat = eng.space_handle(db, model, space)
        tmpl_of = {(int(c["tp"]), int(c["pp"]), int(c["ep"])): int(c["tmpl"]) for c in plan.combos}
        reqs = np.zeros(len(live), dtype=N.STEP_REQ_DTYPE)
        loads: list[np.ndarray] = []
        load_ix: dict = {}
        for j, i in enumerate(live):
            r = requests[i]
            cfg = r.cfg
            reqs[j]["tmpl"] = tmpl_of[(cfg.tp, cfg.pp, cfg.ep)]
            reqs[j]["phase"] = PHASES.index(r.phase)
            reqs[j]["n_ctx"], reqs[j]["n_gen"], reqs[j]["seq"] = r.n_ctx_tokens, r.n_gen_tokens, r.seq_len
            reqs[j]["batch"] = cfg.batch
            load = -1
            if model.moe is not None:  # resolve_moe_load (estimator.py:51-55)
                params = r.moe_load if r.moe_load is not None else DEFAULT_MOE_LOAD
                lk = (params.alpha, params.x_min, params.x_max, params.seed)
                load = load_ix.get(lk)
                if load is None:
                    load = load_ix[lk] = len(loads)
                    loads.append(_moe_q(params, plan.n_experts))
            reqs[j]["load"] = load
        dbh, flat = eng.db_handle(db)
        res = np.zeros(len(live), dtype=N.STEP_OUT_DTYPE)
        l_arr = np.concatenate(loads) if loads else np.zeros(1)
        eng._call(eng.lib.lc_step_latency, "lc_step_latency", eng.ctx, dbh, sph, len(live), N.vptr(reqs),
                  len(loads), N.ptr(l_arr, C.c_double), N.vptr(res))
    for j, i in enumerate(live):
        o = res[j]
        if o["status"]:
            cfg = requests[i].cfg
            msg = _reason(int(o["status"]), int(o["c0"]), int(o["c1"]), plan, {"tmpl": int(reqs[j]["tmpl"])}, flat,
                          db, None, None, cfg.batch)
            kind, text = msg.split(": ", 1)
            out[i] = getattr(S, kind)(text)
            continue
        breakdown = {}
        for k in range(int(o["n_entries"])):
            lb = int(o["entry_label"][k])
            if lb >= 0:
                breakdown[LABELS[lb]] = float(o["entry_ms"][k])
        out[i] = StepLatency(float(o["total_ms"]), breakdown)
    return out


def get_step_latency(db, model, cfg, phase: str, n_ctx_tokens: int = 0, n_gen_tokens: int = 0, seq_len: int = 1,
                     moe_load=None, device: int = 0) -> StepLatency:
    """Drop-in for estimator.get_step_latency (estimator.py:98-110)."""
    r = step_latency_batch(db, model, [StepRequest(cfg, phase, n_ctx_tokens, n_gen_tokens, seq_len, moe_load)],
                           device)[0]
    if isinstance(r, Exception):
        raise r
    return r


def _gen_kv_len(isl: int, osl: int) -> int:
    return isl + osl // 2 if GEN_KV_MIDPOINT else isl


def get_mix_latency(db, model, cfg, chunk_tokens: int, n_gen_tokens: int, isl: int, osl: int, moe_load=None,
                    device: int = 0) -> StepLatency:
    """Drop-in for estimator.get_mix_latency (estimator.py:117-138)."""
    return get_step_latency(db, model, cfg, "mixed", n_ctx_tokens=chunk_tokens, n_gen_tokens=n_gen_tokens,
                            seq_len=_gen_kv_len(isl, osl), moe_load=moe_load, device=device)


def get_gen_latency(db, model, cfg, n_gen_tokens: int, isl: int, osl: int, moe_load=None,
                    device: int = 0) -> StepLatency:
    """Drop-in for estimator.get_gen_latency (estimator.py:141-156)."""
    return get_step_latency(db, model, cfg, "decode", n_gen_tokens=n_gen_tokens, seq_len=_gen_kv_len(isl, osl),
                            moe_load=moe_load, device=device)


__all__ = ["StepLatency", "StepRequest", "EstimationError", "get_step_latency", "get_mix_latency",
           "get_gen_latency", "step_latency_batch"]
