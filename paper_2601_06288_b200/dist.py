"""Multi-GPU plumbing for sharded searches (one process per GPU, torch.distributed).

The candidate space of a sweep is independent until the per-search reductions
(SURVEY.md §8e), so sharding needs one exchange step: an all-gather of packed
fixed-size records.  Two granularities:

* whole searches per rank (``shard_range``) -- what ``bench.py`` uses; the
  gathered records are the per-search summaries (``lc_search_result``);
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


def gather_records(records: np.ndarray, device: str | None = None) -> list[np.ndarray]:
    """All-gather a structured array of any length from every rank (one collective
    for the sizes, one for the padded payload); returns the per-rank arrays."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    if world == 1:
        return [records]
    if device is None:
        device = "cuda" if dist.get_backend() == "nccl" else "cpu"
    raw = np.frombuffer(records.tobytes(), dtype=np.uint8)
    n = torch.tensor([raw.size], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    mx = max(int(s.item()) for s in sizes)
    buf = torch.zeros(max(mx, 1), dtype=torch.uint8, device=device)
    if raw.size:
        buf[: raw.size] = torch.from_numpy(raw.copy()).to(device)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    res = []
    for o, s in zip(outs, sizes):
        b = o[: int(s.item())].cpu().numpy().tobytes()
        res.append(np.frombuffer(b, dtype=records.dtype).copy())
    return res


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
