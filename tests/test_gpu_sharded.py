"""One search split across ranks on the product path.

Each rank evaluates a contiguous block of the search's raw candidate tuples
with the device pipeline (lc_set_raw_filter + LC_MODE_NO_PLANS) and reduces it
to its local front / best / nearest miss / pool top-k; the merge pass re-runs
the pipeline on the union.  Checked here:

* in-process, ranks simulated sequentially on one GPU for world sizes 2, 3, 7:
  counts, frontier, best and diagnostics documents equal the reference's golden
  report for every golden case, and the front / best / plans equal the
  unsharded device run index for index;
* two real processes (gloo all-gather, both on cuda:0): every rank returns the
  golden answer.
"""

from __future__ import annotations

import json
import os
import socket

import numpy as np
import pytest

from golden_io import BY_NAME, CASES, golden_report
from product_cases import case_objects

pytestmark = pytest.mark.gpu

SMALL = [c for c in CASES if not c.get("large")]


def _golden_summary(name: str) -> dict:
    g = golden_report(name)
    return {k: g[k] for k in ("schema", "version", "model", "backend", "workload", "counts", "frontier", "best",
                              "diagnostics")}


def _simulate(case, world: int):
    from paper_2601_06288_b200.dist import shard_range
    from paper_2601_06288_b200.engine import get_engine
    from paper_2601_06288_b200.sharded import _n_raw, local_pass, merge_pass

    db, model, workload, space, dc = case_objects(case)
    eng = get_engine(0)
    with eng._lock:
        _, plan, _ = eng.space_handle(db, model, space)
        n_raw = _n_raw(plan, workload, space)
        shards = [local_pass(eng, db, model, workload, space, dc, *shard_range(n_raw, r, world))
                  for r in range(world)]
        return merge_pass(eng, db, model, workload, space, dc, shards)


@pytest.mark.parametrize("world", [2, 3, 7])
@pytest.mark.parametrize("case", SMALL, ids=[c["name"] for c in SMALL])
def test_sharded_summary_matches_golden(case, world):
    res = _simulate(case, world)
    got = res.summary_doc()
    want = _golden_summary(case["name"])
    assert json.dumps(got, sort_keys=True) == json.dumps(want, sort_keys=True)


@pytest.mark.parametrize("name", ["cfg3_llama70b_kv70", "cfg4_dsv3", "dsv3_all_default", "flat_ties_moe",
                                  "gptoss_all_default"])
def test_sharded_matches_unsharded_by_index(name):
    from paper_2601_06288_b200.engine import fetch_fronts, get_engine

    case = BY_NAME[name]
    db, model, workload, space, dc = case_objects(case)
    eng = get_engine(0)
    with eng._lock:
        out = eng.run_batch(db, model, space, [workload], dc)
        R = out.results[0]
        front, plans = fetch_fronts(out)
    want_front = [(int(k) >> 32, int(k) & 0xFFFFFFFF) for k in front]
    want_best = (int(R["best"]) >> 32, int(R["best"]) & 0xFFFFFFFF) if R["best"] >= 0 else None
    for world in (2, 5):
        res = _simulate(case, world)
        assert res.front == want_front
        assert res.best == want_best
        assert res.timing_ms["units"] == int(R["n_units"])
        assert res.timing_ms["queries_1d"] == int(R["queries_1d"])
        assert res.timing_ms["queries_2d"] == int(R["queries_2d"])
        assert res.counts["evaluated"] == int(R["n_rows"])
        assert res.counts["feasible"] == int(R["n_feasible"])
        assert res.counts["skipped"] == int(R["n_skipped"])
        for k, v in plans.items():
            np.testing.assert_array_equal(res.plans[k], v, err_msg=k)
        assert res.n_union < int(R["n_units"]) or int(R["n_units"]) < 64


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
    import torch.distributed as dist

    from golden_io import BY_NAME as cases
    from paper_2601_06288_b200.sharded import run_search_sharded
    from product_cases import case_objects as objs

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        db, model, workload, space, dc = objs(cases[name])
        from paper_2601_06288_b200.dist import COLLECTIVES

        before = COLLECTIVES["all_gather"]
        res = run_search_sharded(db, model, workload, space, dc)
        n_coll = COLLECTIVES["all_gather"] - before
        q.put((rank, json.dumps(res.summary_doc(), sort_keys=True), res.front, res.best, n_coll))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg4_dsv3", "cfg3_llama70b_kv90"])
def test_two_processes_gloo_match_golden(name):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = json.dumps(_golden_summary(name), sort_keys=True)
    assert got[0][1] == want and got[1][1] == want
    assert got[0][2] == got[1][2] and got[0][3] == got[1][3]
    # one collective per sharded search (counts + keep set in one fixed-size record)
    assert got[0][4] == 1 and got[1][4] == 1
