"""Python driver for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module.  It marshals a search (raw
database records + model / workload / space / disagg scalars as plain dicts,
the same shapes the reference's JSON documents use) into ``liboracle.so`` and
returns a report document with the fields of the reference's
``SearchReport.to_doc()`` (/root/reference/pkg/src/llmconf/search.py:224-260)
that parity is judged on.

Independence: nothing here imports the product package; DB parsing, key
handling and the MoE weight draw are restated locally.
"""

from __future__ import annotations

import ctypes as C
import gzip
import json
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "liboracle.so"

KINDS = ("gemm", "attention_context", "attention_generation", "allreduce", "allgather", "alltoall",
         "p2p", "moe_dispatch", "moe_combine", "moe_gemm", "embedding")
KIND_DIMS = {
    "gemm": ("m", "n", "k"),
    "attention_context": ("batch", "seq_len", "num_heads", "kv_heads", "head_dim"),
    "attention_generation": ("batch", "seq_len", "num_heads", "kv_heads", "head_dim"),
    "allreduce": ("message_bytes", "participant_count"),
    "allgather": ("message_bytes", "participant_count"),
    "alltoall": ("message_bytes", "participant_count"),
    "p2p": ("message_bytes", "participant_count"),
    "moe_dispatch": ("tokens", "experts", "topk", "hidden", "intermediate"),
    "moe_combine": ("tokens", "experts", "topk", "hidden", "intermediate"),
    "moe_gemm": ("tokens", "experts", "topk", "hidden", "intermediate"),
    "embedding": ("tokens", "hidden", "vocab"),
}
QUANTS = ("fp16", "fp8", "int8", "int4")
ATTN = {None: 0, "MHA": 1, "GQA": 2, "MLA": 3}
POLICIES = ("default", "strict", "clamp", "sol")
MODES = ("static", "aggregated", "disaggregated")
BACKENDS = ("trtllm", "vllm", "sglang", "dynamo")

I64P = C.POINTER(C.c_int64)
I32P = C.POINTER(C.c_int32)
F64P = C.POINTER(C.c_double)


class OrDb(C.Structure):
    _fields_ = [("n", C.c_int32), ("kind", I32P), ("quant", I32P), ("attn", I32P), ("dims", I64P),
                ("latency", F64P), ("hw_name", C.c_char_p), ("gpu_memory", C.c_double),
                ("mem_bw", C.c_double), ("intra_bw", C.c_double), ("inter_bw", C.c_double),
                ("gpus_per_node", C.c_int32), ("compute", C.c_double * 4), ("policy", C.c_int32),
                ("backend", C.c_char_p)]


class OrModel(C.Structure):
    _fields_ = [("name", C.c_char_p), ("num_layers", C.c_int64), ("hidden", C.c_int64), ("heads", C.c_int64),
                ("kv_heads", C.c_int64), ("head_dim", C.c_int64), ("inter", C.c_int64), ("vocab", C.c_int64),
                ("attn", C.c_int32), ("mla_kv_dim", C.c_int64), ("is_moe", C.c_int32),
                ("n_experts", C.c_int64), ("topk", C.c_int64), ("expert_inter", C.c_int64),
                ("shared_inter", C.c_int64), ("wq", C.c_int32), ("kq", C.c_int32), ("params", C.c_int64),
                ("moe_weights", F64P), ("moe_n_weights", C.c_int32)]


class OrSearch(C.Structure):
    _fields_ = [("isl", C.c_int64), ("osl", C.c_int64), ("prefix", C.c_int64),
                ("has_ttft", C.c_int32), ("ttft_limit", C.c_double),
                ("has_floor", C.c_int32), ("speed_floor", C.c_double),
                ("has_tpot_cap", C.c_int32), ("tpot_cap", C.c_double),
                ("n_budgets", C.c_int32), ("budgets", I64P),
                ("mode_static", C.c_int32), ("mode_agg", C.c_int32), ("mode_disagg", C.c_int32),
                ("n_tp", C.c_int32), ("tp", I64P), ("n_pp", C.c_int32), ("pp", I64P),
                ("n_ep", C.c_int32), ("ep", I64P), ("n_dp", C.c_int32), ("dp", I64P),
                ("n_b", C.c_int32), ("batch", I64P),
                ("has_ctx_capacity", C.c_int32), ("ctx_capacity", C.c_int64),
                ("chunked_prefill", C.c_int32), ("kv_mem_fraction", C.c_double),
                ("prefill_pool_cap", C.c_int32), ("decode_pool_cap", C.c_int32),
                ("ttft_headroom", C.c_double), ("prefill_util", C.c_double), ("decode_util", C.c_double),
                ("max_x", C.c_int32), ("max_y", C.c_int32), ("static_stride", C.c_int32)]


class OrRow(C.Structure):
    _fields_ = [("mode", C.c_int32), ("cand", C.c_int32), ("p_worker", C.c_int32), ("d_worker", C.c_int32),
                ("x", C.c_int32), ("y", C.c_int32), ("gpus", C.c_int64), ("ttft", C.c_double),
                ("tpot", C.c_double), ("speed", C.c_double), ("thru", C.c_double), ("r_sys", C.c_double),
                ("feasible", C.c_int32), ("frontier", C.c_int32)]


class OrSkip(C.Structure):
    _fields_ = [("mode", C.c_int32), ("cand", C.c_int32), ("reason", C.c_char * 512)]


class OrCfg(C.Structure):
    _fields_ = [("tp", C.c_int64), ("pp", C.c_int64), ("ep", C.c_int64), ("dp", C.c_int64), ("batch", C.c_int64)]


class OrResult(C.Structure):
    _fields_ = [("n_cand", C.c_int32), ("cand", C.POINTER(OrCfg)), ("n_work", C.c_int32),
                ("work", C.POINTER(OrCfg)), ("n_rows", C.c_int32), ("rows", C.POINTER(OrRow)),
                ("n_skip", C.c_int32), ("skip", C.POINTER(OrSkip)), ("n_front", C.c_int32),
                ("front", I32P), ("best", C.c_int32), ("nearest", C.c_int32),
                ("nearest_violation", C.c_double), ("n_queries", C.c_int64)]


_LIB = None


def build() -> Path:
    """Compile liboracle.so (gcc, -ffp-contract=off) if missing or stale."""
    src = [HERE / "oracle.c", HERE / "oracle.h"]
    if not LIB_PATH.exists() or any(p.stat().st_mtime > LIB_PATH.stat().st_mtime for p in src):
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _LIB
    if _LIB is None:
        build()
        _LIB = C.CDLL(str(LIB_PATH))
        _LIB.or_run_search.argtypes = [C.POINTER(OrDb), C.POINTER(OrModel), C.POINTER(OrSearch), C.POINTER(OrResult)]
        _LIB.or_free.argtypes = [C.POINTER(OrResult)]
        _LIB.or_neumaier_sum.argtypes = [F64P, C.c_int]
        _LIB.or_neumaier_sum.restype = C.c_double
        _LIB.or_busiest_shard.argtypes = [F64P, C.c_int, C.c_int64, C.c_int64, C.c_int64, I64P]
        _LIB.or_busiest_shard.restype = C.c_int64
        _LIB.or_estimate.argtypes = [C.POINTER(OrDb), C.POINTER(OrModel), C.POINTER(OrSearch), C.POINTER(OrCfg),
                                     C.c_int, F64P, C.c_char_p, C.c_int]
        _LIB.or_query_batch.argtypes = [C.POINTER(OrDb), C.c_int32, I32P, I32P, I32P, I64P, I64P, C.c_int32,
                                        F64P, I32P, C.c_char_p, C.c_int32]
    return _LIB


# ---------------------------------------------------------------------------
# inputs

def read_db_records(path: str | os.PathLike) -> tuple[dict, list[dict]]:
    """JSON-lines DB (schema llmconf-perfdb/1): header then one record per line."""
    raw = Path(path).read_bytes()
    if str(path).endswith(".gz"):
        raw = gzip.decompress(raw)
    lines = [ln for ln in raw.decode().splitlines() if ln.strip()]
    header = json.loads(lines[0])
    return header, [json.loads(ln) for ln in lines[1:]]


def mutate(header: dict, records: list[dict], mutation: str | None, hw_docs: dict) -> tuple[dict, list[dict]]:
    if not mutation:
        return header, records
    if mutation == "flat":
        return header, [dict(r, latency_us=100.0) for r in records]
    if mutation.startswith("swap_hw:"):
        return dict(header, hardware=hw_docs[mutation.split(":", 1)[1]]), records
    if mutation.startswith("drop_kind:"):
        kind = mutation.split(":", 1)[1]
        return header, [r for r in records if r["kind"] != kind]
    raise ValueError(mutation)


def model_params(m: dict) -> int:
    if m.get("param_count") is not None:
        return int(m["param_count"])
    h, hd, L = m["hidden_size"], m["head_dim"], m["num_layers"]
    mla = m.get("mla_kv_dim", 576)
    if m.get("attn_kind", "GQA") == "MLA":
        attn = h * m["num_heads"] * hd + 2 * h * mla + m["num_heads"] * hd * h
    else:
        attn = h * hd * (2 * m["num_heads"] + 2 * m["kv_heads"])
    moe = m.get("moe")
    if not moe:
        ffn = 3 * h * m["intermediate_size"]
    else:
        expert = L * moe["num_experts"] * 3 * h * moe["expert_intermediate"]
        ffn = h * moe["num_experts"] + expert // L
        if moe.get("shared_intermediate"):
            ffn += 3 * h * moe["shared_intermediate"]
    return 2 * m["vocab_size"] * h + L * (attn + ffn)


def moe_weights(load: dict | None, num_experts: int) -> np.ndarray:
    """Bounded power-law popularity by inverse CDF (moe_load.py:51-57), numpy PCG64."""
    load = load or {}
    alpha = float(load.get("alpha", 1.2))
    x_min = float(load.get("x_min", 1.0))
    x_max = float(load.get("x_max", 100.0))
    seed = int(load.get("seed", 0))
    rng = np.random.default_rng(seed)
    u = rng.random(num_experts)
    e = 1.0 - alpha
    x = (u * (x_max**e - x_min**e) + x_min**e) ** (1.0 / e)
    return np.array([float(v) for v in x], dtype=np.float64)


class _Keep:
    """Holds ctypes buffers alive for the duration of a call."""

    def __init__(self):
        self.items = []

    def arr(self, values, ctype):
        a = (ctype * max(1, len(values)))(*values)
        self.items.append(a)
        return C.cast(a, C.POINTER(ctype))


def _db(header: dict, records: list[dict], extrapolation: str, keep: "_Keep") -> OrDb:
    hw = header["hardware"]
    n = len(records)
    kinds, quants, attns, dims, lats = [], [], [], [], []
    for r in records:
        kinds.append(KINDS.index(r["kind"]))
        quants.append(QUANTS.index(r["quant"]))
        attns.append(ATTN[r["shape"].get("attn_kind")])
        d = [int(r["shape"][name]) for name in KIND_DIMS[r["kind"]]]
        dims.extend(d + [0] * (5 - len(d)))
        lats.append(float(r["latency_us"]))
    db = OrDb()
    db.n = n
    db.kind = keep.arr(kinds, C.c_int32)
    db.quant = keep.arr(quants, C.c_int32)
    db.attn = keep.arr(attns, C.c_int32)
    db.dims = keep.arr(dims, C.c_int64)
    db.latency = keep.arr(lats, C.c_double)
    db.hw_name = hw["name"].encode()
    db.gpu_memory = float(hw["gpu_memory"])
    db.mem_bw = float(hw["mem_bandwidth"])
    db.intra_bw = float(hw["intra_node_bandwidth"])
    db.inter_bw = float(hw["inter_node_bandwidth"])
    db.gpus_per_node = int(hw["gpus_per_node"])
    for i, q in enumerate(QUANTS):
        db.compute[i] = float(hw["compute_throughput"].get(q, 0.0))
    db.policy = POLICIES.index(extrapolation)
    db.backend = header["backend"].encode()
    return db


def query_batch(header: dict, records: list[dict], queries: list[dict], policy: str | None = None,
                extrapolation: str = "default") -> list[tuple[float | None, str]]:
    """query_latency (perfdb.py:539-580) of each {kind, quant, shape} query:
    (latency_us, "") or (None, "Type: message")."""
    keep = _Keep()
    db = _db(header, records, extrapolation, keep)
    n = len(queries)
    kinds, quants, attns, dims, kv = [], [], [], [], []
    for q in queries:
        kinds.append(KINDS.index(q["kind"]))
        quants.append(QUANTS.index(q["quant"]))
        attns.append(ATTN[q["shape"].get("attn_kind")])
        d = [int(q["shape"][name]) for name in KIND_DIMS[q["kind"]]]
        dims.extend(d + [0] * (5 - len(d)))
        kv.append(int(q["shape"].get("kv_len", 0)))
    out = (C.c_double * max(n, 1))()
    st = (C.c_int32 * max(n, 1))()
    msgs = C.create_string_buffer(512 * max(n, 1))
    lib().or_query_batch(C.byref(db), n, keep.arr(kinds, C.c_int32), keep.arr(quants, C.c_int32),
                         keep.arr(attns, C.c_int32), keep.arr(dims, C.c_int64), keep.arr(kv, C.c_int64),
                         -1 if policy is None else POLICIES.index(policy), out, st, msgs, 512)
    res = []
    for i in range(n):
        if st[i]:
            res.append((None, msgs.raw[i * 512:(i + 1) * 512].split(b"\0", 1)[0].decode()))
        else:
            res.append((out[i], ""))
    return res


def run_search(header: dict, records: list[dict], model: dict, workload: dict, space: dict | None = None,
               disagg: dict | None = None, extrapolation: str = "default", _estimate=None) -> dict:
    """Evaluate one search on the CPU oracle; returns a report-like document."""
    space = dict(space or {})
    disagg = dict(disagg or {})
    keep = _Keep()
    db = _db(header, records, extrapolation, keep)

    moe = model.get("moe")
    mm = OrModel()
    mm.name = model["name"].encode()
    mm.num_layers, mm.hidden = model["num_layers"], model["hidden_size"]
    mm.heads, mm.kv_heads, mm.head_dim = model["num_heads"], model["kv_heads"], model["head_dim"]
    mm.inter, mm.vocab = model["intermediate_size"], model["vocab_size"]
    mm.attn = ATTN[model.get("attn_kind", "GQA")]
    mm.mla_kv_dim = model.get("mla_kv_dim", 576)
    mm.is_moe = 1 if moe else 0
    mm.wq = QUANTS.index(model.get("weight_quant", "fp16"))
    mm.kq = QUANTS.index(model.get("kv_quant", "fp16"))
    mm.params = model_params(model)
    if moe:
        mm.n_experts, mm.topk = moe["num_experts"], moe["topk"]
        mm.expert_inter, mm.shared_inter = moe["expert_intermediate"], moe.get("shared_intermediate", 0)
        w = moe_weights(workload.get("moe_load"), moe["num_experts"])
        mm.moe_weights = keep.arr(list(w), C.c_double)
        mm.moe_n_weights = len(w)

    s = OrSearch()
    s.isl, s.osl, s.prefix = workload["isl"], workload["osl"], workload.get("prefix_len", 0)
    if workload.get("ttft_limit_ms") is not None:
        s.has_ttft, s.ttft_limit = 1, float(workload["ttft_limit_ms"])
    floor = None
    if workload.get("min_speed") is not None:
        floor = float(workload["min_speed"])
    elif workload.get("tpot_limit_ms") is not None:
        floor = 1000.0 / float(workload["tpot_limit_ms"])
    if floor is not None:
        s.has_floor, s.speed_floor = 1, floor
        s.has_tpot_cap, s.tpot_cap = 1, 1000.0 / floor
    budgets = list(workload.get("gpu_budgets", []))
    s.n_budgets, s.budgets = len(budgets), keep.arr(budgets, C.c_int64)
    modes = workload.get("modes", list(MODES))
    s.mode_static, s.mode_agg, s.mode_disagg = ("static" in modes), ("aggregated" in modes), ("disaggregated" in modes)
    tp = sorted(space.get("tp_values", (1, 2, 4, 8)))
    pp = sorted(space.get("pp_values", (1, 2, 4)))
    ep = sorted(set(space.get("ep_values", (1, 2, 4, 8)))) if moe else [1]
    dp = sorted(space.get("dp_values", (1, 2, 4, 8)))
    batches = sorted(workload.get("batch_sweep") or space.get("batch_values", tuple(2**i for i in range(10))))
    ctx_cap = space.get("ctx_capacity")
    kvf = float(space.get("kv_mem_fraction", 0.9))
    # knobs shared by every ParallelConfig: if invalid, every candidate fails construction
    shared_ok = (ctx_cap is None or ctx_cap >= 1) and 0.0 < kvf <= 1.0 and header["backend"] in BACKENDS
    if not shared_ok:
        tp = []
    s.n_tp, s.tp = len(tp), keep.arr(tp, C.c_int64)
    s.n_pp, s.pp = len(pp), keep.arr(pp, C.c_int64)
    s.n_ep, s.ep = len(ep), keep.arr(ep, C.c_int64)
    s.n_dp, s.dp = len(dp), keep.arr(dp, C.c_int64)
    s.n_b, s.batch = len(batches), keep.arr(batches, C.c_int64)
    s.has_ctx_capacity = ctx_cap is not None
    s.ctx_capacity = ctx_cap or 0
    s.chunked_prefill = bool(space.get("chunked_prefill", True))
    s.kv_mem_fraction = kvf
    s.prefill_pool_cap = space.get("prefill_pool_cap", 8)
    s.decode_pool_cap = space.get("decode_pool_cap", 16)
    s.ttft_headroom = float(disagg.get("ttft_headroom", 1.8))
    s.prefill_util = float(disagg.get("prefill_utilization", 0.90))
    s.decode_util = float(disagg.get("decode_utilization", 0.92))
    s.max_x = disagg.get("max_prefill_replicas", 32)
    s.max_y = disagg.get("max_decode_replicas", 64)

    if _estimate is not None:
        s.static_stride = _estimate[2] if len(_estimate) > 2 else 32
        cfg = OrCfg(*_estimate[0])
        out = (C.c_double * 4)()
        reason = C.create_string_buffer(512)
        st = lib().or_estimate(C.byref(db), C.byref(mm), C.byref(s), C.byref(cfg), _estimate[1], out, reason, 512)
        return {"status": st, "values": list(out), "reason": reason.value.decode()}
    res = OrResult()
    lib().or_run_search(C.byref(db), C.byref(mm), C.byref(s), C.byref(res))
    try:
        return _to_doc(res, model["name"], header["backend"], space)
    finally:
        lib().or_free(C.byref(res))


def _key(c) -> str:
    return f"tp{c.tp}pp{c.pp}ep{c.ep}dp{c.dp}b{c.batch}"


def _to_doc(res: OrResult, model_name: str, backend: str, space: dict) -> dict:
    cand = [res.cand[i] for i in range(res.n_cand)]
    work = [res.work[i] for i in range(res.n_work)]
    rows = []
    for i in range(res.n_rows):
        r = res.rows[i]
        speed = r.speed if math.isfinite(r.speed) else None
        doc = {"mode": MODES[r.mode], "gpus": r.gpus, "ttft_ms": r.ttft, "tpot_ms": r.tpot, "speed": speed,
               "throughput_per_gpu": r.thru, "feasible": bool(r.feasible), "frontier": bool(r.frontier)}
        if r.mode < 2:
            c = cand[r.cand]
            doc.update(config=_key(c), batch=c.batch, model=model_name,
                       parallel={"tp": c.tp, "pp": c.pp, "ep": c.ep, "dp": c.dp})
        else:
            p, d = work[r.p_worker], work[r.d_worker]
            doc.update(config=f"P:{r.x}x{_key(p)}|D:{r.y}x{_key(d)}", r_sys=r.r_sys,
                       prefill={"replicas": r.x, "batch": p.batch,
                                "parallel": {"tp": p.tp, "pp": p.pp, "ep": p.ep, "dp": p.dp}},
                       decode={"replicas": r.y, "batch": d.batch,
                               "parallel": {"tp": d.tp, "pp": d.pp, "ep": d.ep, "dp": d.dp}})
        rows.append(doc)
    skip_modes = ("static", "aggregated", "disaggregated/prefill", "disaggregated/decode")
    skipped = []
    for i in range(res.n_skip):
        sk = res.skip[i]
        c = cand[sk.cand] if sk.mode < 2 else work[sk.cand]
        skipped.append({"mode": skip_modes[sk.mode], "config": _key(c), "reason": sk.reason.decode()})
    frontier = [rows[res.front[i]] for i in range(res.n_front)]
    best = rows[res.best] if res.best >= 0 else None
    diagnostics = None
    if res.best < 0 and res.nearest >= 0:
        diagnostics = dict(rows[res.nearest])
        v = res.nearest_violation
        diagnostics["violation_factor"] = v if math.isfinite(v) else None
    return {
        "model": model_name,
        "backend": backend,
        "counts": {"enumerated": res.n_cand, "evaluated": len(rows),
                   "feasible": sum(r["feasible"] for r in rows), "frontier": len(frontier),
                   "skipped": len(skipped)},
        "rows": rows,
        "frontier": frontier,
        "best": best,
        "diagnostics": diagnostics,
        "skipped": skipped,
        "n_queries": res.n_queries,
    }


def neumaier_sum(xs: list[float]) -> float:
    a = (C.c_double * max(1, len(xs)))(*xs)
    return lib().or_neumaier_sum(a, len(xs))


def busiest_shard(weights, total: int, topk: int, ep: int) -> tuple[int, list[int]]:
    w = (C.c_double * len(weights))(*weights)
    out = (C.c_int64 * len(weights))()
    tail = lib().or_busiest_shard(w, len(weights), total, topk, ep, out)
    return tail, list(out)


def estimate(header: dict, records: list[dict], model: dict, workload: dict, cfg: tuple, mode: str,
             space: dict | None = None, extrapolation: str = "default", stride: int = 32) -> dict:
    """estimate_static (with its decode ``stride``, serving_modes.py:231-267) / estimate_aggregated
    of one (tp, pp, ep, dp, batch) config."""
    return run_search(header, records, model, workload, space, None, extrapolation,
                      _estimate=(cfg, 0 if mode == "static" else 1, stride))
