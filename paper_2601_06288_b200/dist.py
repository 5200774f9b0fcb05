"""Multi-GPU plumbing for sharded searches (one process per GPU, torch.distributed).

The candidate space of a sweep is independent until the per-search reductions
(SURVEY.md §8e), so sharding needs one exchange step: an all-gather of packed
fixed-size records.  Two granularities:

* whole searches per rank (``shard_range``) -- what ``bench.py`` uses; the
  gathered records are the per-search summaries (``lc_search_result``), one
  fixed-size all-gather (``all_gather_bytes``);
* one search split across ranks -- each rank reduces its candidate block to a
  local Pareto front, local best and local pool top-k; after the all-gather
  ``merge_fronts`` / ``merge_best`` / ``merge_topk`` give exactly the global
  answer because front(union of local fronts) = front(all),
  best = min(local bests) and top-k(union of local top-k) = top-k(all).

The merge functions restate the reference rules on plain arrays
(pareto_filter / select_best / _pool_rank, search.py:156-187, 276-277).
"""

from __future__ import annotations

import math

import numpy as np

FRONT_DTYPE = np.dtype([("speed", "<f8"), ("thru", "<f8"), ("key", "<i8")])


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items owned by ``rank``."""
    return n * rank // world, n * (rank + 1) // world


def _collective_device(device: str | None) -> str:
    import torch.distributed as dist

    if device is not None:
        return device
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


# Counter of collectives issued by this module (tests assert "one all-gather per search").
COLLECTIVES = {"all_gather": 0}


def all_gather_bytes(payload: bytes, cap: int = 64 * 1024, device: str | None = None) -> list[bytes]:
    """All-gather one variable-length byte payload per rank with ONE collective.

    Every rank contributes a fixed-size ``8 + cap`` byte buffer (an int64
    length header, then the payload zero-padded).  The payloads of this path
    are small (per-search summaries, local fronts and pool top-k: a few KB), so
    one fixed-size all-gather is latency-bound and the size exchange of a
    two-collective protocol is saved.  If some rank's payload exceeds ``cap``
    every rank sees it in the gathered headers and all of them issue one more
    all-gather sized to the largest payload (the same decision everywhere).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    if world == 1:
        return [payload]
    device = _collective_device(device)
    raw = np.frombuffer(payload, dtype=np.uint8)
    buf = np.zeros(8 + cap, dtype=np.uint8)
    buf[:8] = np.frombuffer(np.int64(raw.size).tobytes(), dtype=np.uint8)
    fits = raw.size <= cap
    if fits:
        buf[8: 8 + raw.size] = raw
    t = torch.from_numpy(buf).to(device)
    outs = torch.empty(world * (8 + cap), dtype=torch.uint8, device=device)
    dist.all_gather_into_tensor(outs, t)
    COLLECTIVES["all_gather"] += 1
    got = outs.cpu().numpy().reshape(world, 8 + cap)
    sizes = [int(np.frombuffer(got[r, :8].tobytes(), dtype=np.int64)[0]) for r in range(world)]
    if max(sizes) <= cap:
        return [got[r, 8: 8 + sizes[r]].tobytes() for r in range(world)]
    # overflow (rare): one more all-gather sized to the largest payload
    mx = max(sizes)
    big = np.zeros(mx, dtype=np.uint8)
    big[: raw.size] = raw
    outs2 = torch.empty(world * mx, dtype=torch.uint8, device=device)
    dist.all_gather_into_tensor(outs2, torch.from_numpy(big).to(device))
    COLLECTIVES["all_gather"] += 1
    got2 = outs2.cpu().numpy().reshape(world, mx)
    return [got2[r, : sizes[r]].tobytes() for r in range(world)]


def gather_records(records: np.ndarray, device: str | None = None, cap: int = 64 * 1024) -> list[np.ndarray]:
    """All-gather a structured array of any length from every rank (one collective
    in the common case, see ``all_gather_bytes``); returns the per-rank arrays."""
    parts = all_gather_bytes(records.tobytes(), cap=cap, device=device)
    return [np.frombuffer(b, dtype=records.dtype).copy() for b in parts]


def pack_records(*arrays: np.ndarray) -> bytes:
    """Several structured arrays as one payload: [n_arrays][len_0 .. len_k][bytes ...]."""
    head = np.array([len(arrays)] + [a.size for a in arrays], dtype=np.int64)
    return head.tobytes() + b"".join(np.ascontiguousarray(a).tobytes() for a in arrays)


def unpack_records(payload: bytes, dtypes: list) -> list[np.ndarray]:
    """Inverse of ``pack_records`` given each array's dtype."""
    k = int(np.frombuffer(payload[:8], dtype=np.int64)[0])
    if k != len(dtypes):
        raise ValueError(f"packed payload holds {k} arrays, expected {len(dtypes)}")
    lens = np.frombuffer(payload[8: 8 + 8 * k], dtype=np.int64)
    off = 8 + 8 * k
    out = []
    for n, dt in zip(lens, dtypes):
        nb = int(n) * np.dtype(dt).itemsize
        out.append(np.frombuffer(payload[off: off + nb], dtype=dt).copy())
        off += nb
    return out


def pareto_front(rows: np.ndarray) -> np.ndarray:
    """Front of FRONT_DTYPE rows by the reference rule, in speed-desc / key order."""
    if len(rows) == 0:
        return rows[:0]
    order = np.lexsort((rows["key"], -rows["speed"]))
    r = rows[order]
    out = []
    best = -math.inf
    i = 0
    while i < len(r):
        j = i
        while j < len(r) and r["speed"][j] == r["speed"][i]:
            j += 1
        top = r["thru"][i:j].max()
        if top > best:
            out.extend(k for k in range(i, j) if r["thru"][k] == top)
            best = top
        i = j
    return r[out]


def merge_fronts(local_fronts: list[np.ndarray]) -> np.ndarray:
    """Global front from the ranks' local fronts (exact, see module docstring)."""
    allrows = np.concatenate(local_fronts) if local_fronts else np.zeros(0, FRONT_DTYPE)
    return pareto_front(allrows)


def merge_best(candidates: list[tuple]) -> tuple | None:
    """min over the ranks' local best keys (tuples ordered like select_best's key)."""
    cands = [c for c in candidates if c is not None]
    return min(cands) if cands else None


def merge_topk(local: list[list[tuple]], k: int) -> list[tuple]:
    """top-k of the union of the ranks' local top-k lists ((-rate/gpus, key) tuples)."""
    return sorted(x for lst in local for x in lst)[:k]
