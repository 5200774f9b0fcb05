"""NCCL data plane (one process per GPU): the packed all-gather and a sharded
search over real NCCL ranks.  Needs >= 2 GPUs; skipped otherwise (the
gloo-backed tests in test_multigpu.py / test_gpu_sharded.py cover the same
host logic with ranks sharing one device).
"""

from __future__ import annotations

import json
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _n_gpus() -> int:
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from golden_io import BY_NAME as cases
    from paper_2601_06288_b200.dist import COLLECTIVES, all_gather_bytes
    from paper_2601_06288_b200.sharded import run_search_sharded
    from product_cases import case_objects as objs

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        assert dist.get_backend() == "nccl"
        echoed = all_gather_bytes(bytes([rank + 1]) * (rank + 2))
        db, model, workload, space, dc = objs(cases[name])
        before = COLLECTIVES["all_gather"]
        res = run_search_sharded(db, model, workload, space, dc, device=rank)
        q.put((rank, [len(e) for e in echoed], json.dumps(res.summary_doc(), sort_keys=True),
               COLLECTIVES["all_gather"] - before))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(_n_gpus() < 2, reason="NCCL test needs >= 2 GPUs")
@pytest.mark.parametrize("name", ["cfg4_dsv3"])
def test_nccl_two_gpus_sharded_search(name):
    import torch.multiprocessing as mp

    from test_gpu_sharded import _golden_summary

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = json.dumps(_golden_summary(name), sort_keys=True)
    for rank, lens, doc, n_coll in got:
        assert lens == [2, 3]
        assert doc == want
        assert n_coll == 1
