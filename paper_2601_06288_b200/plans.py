"""Host-compiled plan templates and parallel-mapping combos for one model x space.

The reference lowers every (config, phase, tokens) to an operator list on every
call (``decompose``, /root/reference/pkg/src/llmconf/model.py:271-406).  The
list's *structure* -- which labels appear, their kinds, quantizations, fixed
dims, repeat counts and therefore which database grid each entry lands in --
depends only on (model, tp, pp, ep); only the interpolated coordinates depend
on the token counts.  So the host builds one template per (tp, pp, ep) here,
resolving every grid key once, and the device fills coordinates per step
(``LC_COORD_*`` recipes).

Combos are the consistent (tp, pp, ep, dp) tuples in the reference's nested
enumeration order (search.py:97-101) with the batch-independent parts of the
memory model (model.py:440-456) precomputed in Python float arithmetic.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .database import FlatDb, grid_key
from .specs import QUANT_BYTES, QUANT_FORMATS, ParallelConfig, ParallelConfigError

KIND_CODE = {k: i for i, k in enumerate(("gemm", "attention_context", "attention_generation", "allreduce",
                                         "allgather", "alltoall", "p2p", "moe_dispatch", "moe_combine",
                                         "moe_gemm", "embedding"))}
LABELS = ("embedding", "qkv_proj", "context_attention", "generation_attention", "attn_out_proj", "mlp_up",
          "mlp_down", "moe_router", "shared_expert_up", "shared_expert_down", "expert_ffn", "expert_dispatch",
          "expert_combine", "attn_allreduce", "mlp_allreduce", "stage_boundary")
LABEL_CODE = {name: i for i, name in enumerate(LABELS)}
COORD_TOKENS, COORD_MSG, COORD_CTX, COORD_GEN, COORD_EXPERT = range(5)
MAX_ENTRIES = 16

ENTRY_DTYPE = np.dtype([("label", "<i4"), ("kind", "<i4"), ("quant", "<i4"), ("grid", "<i4"), ("coord", "<i4"),
                        ("_pad", "<i4"), ("repeat", "<i8"), ("d", "<i8", (5,))])
SLOT_DTYPE = np.dtype([("e", ENTRY_DTYPE), ("step", "<i4"), ("pair", "<i4")])
STEP_P, STEP_G, STEP_M = 0, 1, 2  # prefill (b*chunk), decode at kv midpoint (b), mixed chunk
COMBO_DTYPE = np.dtype([("tp", "<i8"), ("pp", "<i8"), ("ep", "<i8"), ("dp", "<i8"), ("gpus", "<i8"),
                        ("tp_i", "<i4"), ("ep_i", "<i4"), ("tmpl", "<i4"), ("_pad", "<i4"),
                        ("weight_bytes", "<f8"), ("kv_token_bytes", "<f8")])


@dataclass
class EntryInfo:
    """Host-side facts about one template entry (for skip-reason messages)."""

    label: str
    kind: str
    quant: str
    key: tuple
    grid: int


def _problems(model, tp: int, pp: int, ep: int, dp: int) -> bool:
    """True when check_consistency (model.py:209-236) reports any problem."""
    if model.num_heads % tp or pp > model.num_layers:
        return True
    moe = model.moe
    if moe is None:
        return ep != 1 or (tp <= model.intermediate_size and model.intermediate_size % tp != 0)
    if moe.num_experts % ep or ep > tp * dp:
        return True
    hi, lo = max(ep, tp), min(ep, tp)
    if hi % lo:
        return True
    if tp > ep and moe.expert_intermediate % (tp // ep):
        return True
    return bool(moe.shared_intermediate and tp <= moe.shared_intermediate and moe.shared_intermediate % tp)


def _template(model, flat: FlatDb, tp: int, pp: int, ep: int) -> tuple[np.ndarray, list[EntryInfo]]:
    h = model.hidden_size
    heads = model.num_heads // tp
    if model.attn_kind == "MLA":
        kvh, hd = 1, model.mla_kv_dim
        qkv_n = heads * model.head_dim + model.mla_kv_dim
    else:
        kvh, hd = max(1, model.kv_heads // tp), model.head_dim
        qkv_n = (heads + 2 * kvh) * model.head_dim
    wq, kq = model.weight_quant, model.kv_quant
    layers = math.ceil(model.num_layers / pp)
    rows: list[tuple] = []

    def add(label, kind, quant, coord, repeat, dims: dict, extra: dict | None = None):
        shape = dict(dims)
        if extra:
            shape.update(extra)
        key = grid_key(kind, quant, shape)
        gid = flat.index.get(key, -1)
        names = {"gemm": ("m", "n", "k"), "embedding": ("tokens", "hidden", "vocab")}.get(kind)
        if names is None:
            if kind.startswith("attention"):
                names = ("batch", "seq_len", "num_heads", "kv_heads", "head_dim")
            elif kind in ("allreduce", "allgather", "alltoall", "p2p"):
                names = ("message_bytes", "participant_count")
            else:
                names = ("tokens", "experts", "topk", "hidden", "intermediate")
        d = [int(dims.get(n, 0)) for n in names] + [0] * (5 - len(names))
        rows.append(((LABEL_CODE[label], KIND_CODE[kind], QUANT_FORMATS.index(quant), gid, coord, 0, repeat, d),
                     EntryInfo(label, kind, quant, key, gid)))

    add("embedding", "embedding", wq, COORD_TOKENS, 1, {"tokens": 1, "hidden": h, "vocab": model.vocab_size})
    add("qkv_proj", "gemm", wq, COORD_TOKENS, layers, {"m": 1, "n": qkv_n, "k": h})
    attn = {"batch": 1, "seq_len": 1, "num_heads": heads, "kv_heads": kvh, "head_dim": hd}
    add("context_attention", "attention_context", kq, COORD_CTX, layers, attn, {"attn_kind": model.attn_kind})
    add("generation_attention", "attention_generation", kq, COORD_GEN, layers, attn, {"attn_kind": model.attn_kind})
    add("attn_out_proj", "gemm", wq, COORD_TOKENS, layers, {"m": 1, "n": h, "k": heads * model.head_dim})
    if model.moe is None:
        inter = max(1, model.intermediate_size // tp)
        add("mlp_up", "gemm", wq, COORD_TOKENS, layers, {"m": 1, "n": 2 * inter, "k": h})
        add("mlp_down", "gemm", wq, COORD_TOKENS, layers, {"m": 1, "n": h, "k": inter})
    else:
        moe = model.moe
        add("moe_router", "gemm", wq, COORD_TOKENS, layers, {"m": 1, "n": moe.num_experts, "k": h})
        if moe.shared_intermediate:
            shared = max(1, moe.shared_intermediate // tp)
            add("shared_expert_up", "gemm", wq, COORD_TOKENS, layers, {"m": 1, "n": 2 * shared, "k": h})
            add("shared_expert_down", "gemm", wq, COORD_TOKENS, layers, {"m": 1, "n": h, "k": shared})
        inter = moe.expert_intermediate // max(1, tp // ep)
        add("expert_ffn", "moe_gemm", wq, COORD_EXPERT, layers,
            {"tokens": 1, "experts": moe.num_experts // ep, "topk": moe.topk, "hidden": h, "intermediate": inter})
        if ep > 1:
            xfer = {"tokens": 1, "experts": moe.num_experts, "topk": moe.topk, "hidden": h,
                    "intermediate": moe.expert_intermediate}
            add("expert_dispatch", "moe_dispatch", "fp16", COORD_TOKENS, layers, xfer)
            add("expert_combine", "moe_combine", "fp16", COORD_TOKENS, layers, xfer)
    if tp > 1:
        msg = {"message_bytes": 1, "participant_count": tp}
        add("attn_allreduce", "allreduce", "fp16", COORD_MSG, layers, msg)
        add("mlp_allreduce", "allreduce", "fp16", COORD_MSG, layers, msg)
    if pp > 1:
        add("stage_boundary", "p2p", "fp16", COORD_MSG, pp - 1, {"message_bytes": 1, "participant_count": 2})
    arr = np.zeros(MAX_ENTRIES, dtype=ENTRY_DTYPE)
    for i, (row, _) in enumerate(rows):
        arr[i] = row
    return arr[: len(rows)], [info for _, info in rows]


def _present(coord: int, step: int) -> bool:
    """Static presence of an entry in a step's plan (context attention needs n_ctx,
    generation attention n_gen; the mixed step's n_gen can still be 0 at batch 1)."""
    if coord == COORD_CTX:
        return step != STEP_G
    if coord == COORD_GEN:
        return step != STEP_P
    return True


def build_slots(entries: np.ndarray, tmpl_n: np.ndarray, combos: np.ndarray, n_ep: int):
    """Distinct (step, grid, coordinate recipe[, expert (tp,ep) pair]) query families.

    Latency is a pure function of (grid, coordinates) (the grid key fixes kind,
    quant and every fixed dim), so one slot serves every template entry that
    shares it; the device prices each slot once per (search, batch).
    Returns (slots, slot_of[n_tmpl, 16, 3], gen_classes, gclass_of[n_tmpl]).
    """
    n_tmpl = len(tmpl_n)
    pair_of = {}
    for c in combos:
        pair_of[int(c["tmpl"])] = (int(c["tp_i"]), int(c["ep_i"]))
    slots, index = [], {}
    slot_of = np.full((max(n_tmpl, 1), MAX_ENTRIES, 3), -1, dtype=np.int32)
    gen, gindex = [], {}
    gclass_of = np.full(max(n_tmpl, 1), -1, dtype=np.int32)
    for t in range(n_tmpl):
        tp_i, ep_i = pair_of.get(t, (0, 0))
        for i in range(int(tmpl_n[t])):
            e = entries[t * MAX_ENTRIES + i]
            coord, grid = int(e["coord"]), int(e["grid"])
            pair = tp_i * n_ep + ep_i if coord == COORD_EXPERT else -1
            for step in (STEP_P, STEP_G, STEP_M):
                if not _present(coord, step):
                    continue
                key = (step, grid, coord, pair) if grid >= 0 else (step, -1, coord, pair)
                if key not in index:
                    index[key] = len(slots)
                    slots.append((e, step, pair))
                slot_of[t, i, step] = index[key]
            if coord == COORD_GEN:
                gk = grid
                if gk not in gindex:
                    gindex[gk] = len(gen)
                    gen.append(e)
                gclass_of[t] = gindex[gk]
    arr = np.zeros(max(len(slots), 1), dtype=SLOT_DTYPE)
    for k, (e, step, pair) in enumerate(slots):
        arr[k]["e"] = e
        arr[k]["step"] = step
        arr[k]["pair"] = pair
    garr = np.zeros(max(len(gen), 1), dtype=ENTRY_DTYPE)
    for k, e in enumerate(gen):
        garr[k] = e
    return arr[: max(len(slots), 1)], len(slots), slot_of, garr, len(gen), gclass_of


@dataclass
class SpacePlan:
    """Everything lc_space_upload needs, plus host lookups for report building."""

    tp_values: list[int]
    pp_values: list[int]
    ep_values: list[int]
    dp_values: list[int]
    combos: np.ndarray            # COMBO_DTYPE
    tmpl_n: np.ndarray            # int32 per template
    entries: np.ndarray           # ENTRY_DTYPE [n_tmpl * MAX_ENTRIES]
    infos: list[list[EntryInfo]]  # per template
    is_moe: bool
    hidden: int
    topk: int
    n_experts: int
    slots: np.ndarray = None
    n_slots: int = 0
    slot_of: np.ndarray = None
    gen_entries: np.ndarray = None
    n_gen: int = 0
    gclass_of: np.ndarray = None


def build_space_plan(model, space, flat: FlatDb, backend: str) -> SpacePlan:
    tp_values = sorted(space.tp_values)
    pp_values = sorted(space.pp_values)
    ep_values = sorted(set(space.ep_values)) if model.moe else [1]
    dp_values = sorted(space.dp_values)
    # knobs shared by every candidate: when they are invalid, every config fails construction
    try:
        ParallelConfig(ctx_capacity=space.ctx_capacity, chunked_prefill=space.chunked_prefill,
                       kv_mem_fraction=space.kv_mem_fraction, cuda_graph=space.cuda_graph, backend=backend)
        shared_ok = True
    except ParallelConfigError:
        shared_ok = False
    bw = QUANT_BYTES[model.weight_quant]
    bkv = QUANT_BYTES[model.kv_quant]
    expert = model.expert_params()
    dense = max(0, model.params() - expert)
    templates: dict[tuple[int, int, int], int] = {}
    entries, tmpl_n, infos = [], [], []
    combos = []
    for ti, tp in enumerate(tp_values):
        for pi, pp in enumerate(pp_values):
            for ei, ep in enumerate(ep_values):
                for dp in dp_values:
                    if not shared_ok or min(tp, pp, ep, dp) < 1 or _problems(model, tp, pp, ep, dp):
                        continue
                    tkey = (tp, pp, ep)
                    if tkey not in templates:
                        arr, info = _template(model, flat, tp, pp, ep)
                        templates[tkey] = len(tmpl_n)
                        padded = np.zeros(MAX_ENTRIES, dtype=ENTRY_DTYPE)
                        padded[: len(arr)] = arr
                        entries.append(padded)
                        tmpl_n.append(len(arr))
                        infos.append(info)
                    weight = bw * (dense / tp + expert / max(ep, tp)) / pp
                    layers = math.ceil(model.num_layers / pp)
                    if model.attn_kind == "MLA":
                        kv_token = layers * model.mla_kv_dim * bkv
                    else:
                        kv_token = 2 * layers * max(1, model.kv_heads // tp) * model.head_dim * bkv
                    combos.append((tp, pp, ep, dp, tp * pp * dp, ti, ei, templates[tkey], 0, weight, kv_token))
    combo_arr = np.array(combos, dtype=COMBO_DTYPE) if combos else np.zeros(0, dtype=COMBO_DTYPE)
    ent = np.concatenate(entries) if entries else np.zeros(MAX_ENTRIES, dtype=ENTRY_DTYPE)
    moe = model.moe
    tmpl_arr = np.array(tmpl_n if tmpl_n else [0], dtype=np.int32)
    slots, n_slots, slot_of, gen, n_gen, gclass_of = build_slots(ent, np.array(tmpl_n, dtype=np.int32), combo_arr, len(ep_values))
    return SpacePlan(tp_values, pp_values, ep_values, dp_values, combo_arr, tmpl_arr, ent, infos, moe is not None,
                     model.hidden_size, moe.topk if moe else 0, moe.num_experts if moe else 0,
                     slots, n_slots, slot_of, gen, n_gen, gclass_of)
