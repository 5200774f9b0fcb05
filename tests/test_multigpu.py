"""Multi-process (gloo, world size 2, CPU) coverage of the sharded path.

* the rank blocks of a sweep cover every search exactly once;
* the all-gather of packed records returns every rank's bytes unchanged;
* merging local reductions gives the global answer: on the CPU oracle's rows
  of real searches, front(union of local fronts) == front(all rows),
  min(local bests) == best, top-k(union of local top-k) == top-k.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_06288_b200.dist import (
    COLLECTIVES,
    FRONT_DTYPE,
    all_gather_bytes,
    gather_records,
    pack_records,
    unpack_records,
    merge_best,
    merge_fronts,
    merge_topk,
    pareto_front,
    shard_range,
)


def test_shard_ranges_partition():
    for n in (0, 1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(n, r, world)
                seen.extend(range(lo, hi))
            assert seen == list(range(n))


def _rows_from_doc(doc):
    feas = [(i, r) for i, r in enumerate(doc["rows"]) if r["feasible"]]
    arr = np.zeros(len(feas), FRONT_DTYPE)
    for j, (i, r) in enumerate(feas):
        arr[j] = (r["speed"] if r["speed"] is not None else np.inf, r["throughput_per_gpu"], i)
    return arr


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, rows, topk_src, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(len(rows), rank, world)
        mine = rows[lo:hi]
        local_front = pareto_front(mine)
        gathered = gather_records(local_front, device="cpu")
        merged = merge_fronts(gathered)
        # local best by (-thru, -speed, key) and local pool top-k
        best = None
        if len(mine):
            i = np.lexsort((mine["key"], -mine["speed"], -mine["thru"]))[0]
            best = (-mine["thru"][i], -mine["speed"][i], int(mine["key"][i]))
        bests = gather_records(np.array([best if best else (np.inf, np.inf, -1)],
                                        dtype=[("a", "<f8"), ("b", "<f8"), ("k", "<i8")]), device="cpu")
        gbest = merge_best([tuple(b[0]) if b[0]["k"] >= 0 else None for b in bests])
        tk_lo, tk_hi = shard_range(len(topk_src), rank, world)
        local_tk = sorted(topk_src[tk_lo:tk_hi])[:4]
        tk = gather_records(np.array(local_tk, dtype=[("r", "<f8"), ("k", "<i8")]), device="cpu")
        gtk = merge_topk([[tuple(x) for x in t] for t in tk], 4)
        if rank == 0:
            q.put((merged["key"].tolist(), gbest, gtk))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case_name", ["a1_qwen_small", "flat_ties", "cfg4_dsv3"])
def test_gloo_world2_merge_matches_global(case_name):
    from golden_io import golden_report

    doc = golden_report(case_name)
    rows = _rows_from_doc(doc)
    rng = np.random.default_rng(3)
    rows = rows[rng.permutation(len(rows))]  # ranks see arbitrary subsets
    topk_src = [(float(-r["throughput_per_gpu"]), i) for i, r in enumerate(doc["rows"])]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rows, topk_src, q)) for r in range(2)]
    for p in procs:
        p.start()
    keys, gbest, gtk = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # global answers computed without sharding
    assert keys == pareto_front(rows)["key"].tolist()
    front_rows = [doc["rows"][k]["config"] + doc["rows"][k]["mode"] for k in keys]
    assert front_rows == [r["config"] + r["mode"] for r in doc["frontier"]]
    i = np.lexsort((rows["key"], -rows["speed"], -rows["thru"]))[0]
    assert gbest == (-rows["thru"][i], -rows["speed"][i], int(rows["key"][i]))
    assert gtk == sorted(topk_src)[:4]


def _bytes_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = np.arange(rank * 3, dtype=np.int64)
        b = np.zeros(rank + 1, dtype=[("x", "<f8"), ("k", "<i4")])
        b["x"] = rank + 0.5
        n0 = COLLECTIVES["all_gather"]
        small = all_gather_bytes(pack_records(a, b), device="cpu")
        n_small = COLLECTIVES["all_gather"] - n0
        # rank 1's payload overflows a tiny cap: every rank takes the second gather
        n0 = COLLECTIVES["all_gather"]
        big = all_gather_bytes(bytes(range(rank * 40 % 256)) * (1 + rank), cap=16, device="cpu")
        n_big = COLLECTIVES["all_gather"] - n0
        if rank == 0:
            q.put(([[x.tolist() for x in unpack_records(p, [np.int64, b.dtype])] for p in small], n_small,
                   [len(x) for x in big], n_big))
    finally:
        dist.destroy_process_group()


def test_gloo_packed_gather_one_collective():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bytes_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    small, n_small, big_lens, n_big = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert n_small == 1 and n_big == 2
    assert small[0][0] == [] and small[1][0] == [0, 1, 2]
    assert small[0][1] == [(0.5, 0)] and small[1][1] == [(1.5, 0), (1.5, 0)]
    assert big_lens == [0, 80]


def test_pack_roundtrip():
    a = np.array([3, 1, 2], dtype=np.int64)
    b = np.zeros(0, dtype=FRONT_DTYPE)
    got = unpack_records(pack_records(a, b), [np.int64, FRONT_DTYPE])
    assert got[0].tolist() == [3, 1, 2] and len(got[1]) == 0
    with pytest.raises(ValueError):
        unpack_records(pack_records(a), [np.int64, FRONT_DTYPE])
