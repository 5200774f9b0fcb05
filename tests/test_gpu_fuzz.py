"""Randomised parity: seeded random searches through the product path against
the CPU oracle (itself pinned to the reference by the golden reports).

Each case draws a model and its database, an extrapolation policy, a workload
(ISL / OSL / prefix, TTFT / speed / TPOT objectives, GPU budgets, modes,
batch sweep, MoE load), a candidate space (parallelism lists, batch sizes,
context capacity, chunking, KV fraction, pool caps) and disaggregation
constants.  Reports must agree bit for bit (rows, skip reasons, fronts, best,
diagnostics).  The batched variant evaluates several random workloads of one
(model, space) in one device pass -- the table-sharing path -- and checks each
search against the oracle.
"""

from __future__ import annotations

import json
import os
import random

import pytest

from golden_io import canonical, diff_canonical

pytestmark = pytest.mark.gpu

MODELS = ["qwen-small", "moe-small", "qwen3-32b", "llama-3.1-70b", "deepseek-v3", "gpt-oss-120b"]
_DB_CACHE: dict = {}


def _inputs(model: str, hw: str, extrapolation: str):
    import paper_2601_06288_b200 as pkg
    from oracle import oracle
    from paper_2601_06288_b200.sweeps import GOLDEN

    key = (model, hw, extrapolation)
    if key not in _DB_CACHE:
        path = GOLDEN / "db" / f"db-{model}-{hw}-s11.jsonl.gz"
        header, recs = oracle.read_db_records(path)
        mdoc = json.loads((GOLDEN / "specs" / f"model-{model}.json").read_text())
        _DB_CACHE[key] = (pkg.load_db(path, extrapolation=extrapolation), header, recs, mdoc)
    return _DB_CACHE[key]


def _subset(rng, values, k_min=1):
    k = rng.randint(k_min, len(values))
    return sorted(rng.sample(values, k))


def _workload(rng, moe: bool) -> dict:
    isl = int(round(10 ** rng.uniform(1.3, 4.3)))
    osl = rng.choice([1, 2, 3, 31, 32, 33, 64, 97, 500, 1024, int(round(10 ** rng.uniform(0, 3.4)))])
    w = {"isl": isl, "osl": osl}
    if rng.random() < 0.2:
        w["prefix_len"] = rng.randint(0, isl - 1)
    if rng.random() < 0.7:
        w["ttft_limit_ms"] = float(round(10 ** rng.uniform(1.5, 4.5), 3))
    r = rng.random()
    if r < 0.45:
        w["min_speed"] = float(round(10 ** rng.uniform(0, 2.5), 3))
    elif r < 0.7:
        w["tpot_limit_ms"] = float(round(10 ** rng.uniform(0.5, 2.5), 3))
    if rng.random() < 0.5:
        w["gpu_budgets"] = _subset(rng, [1, 2, 4, 8, 16, 32, 64])
    if rng.random() < 0.5:
        w["modes"] = _subset(rng, ["static", "aggregated", "disaggregated"])
        order = ["static", "aggregated", "disaggregated"]
        w["modes"] = [m for m in order if m in w["modes"]]
    if rng.random() < 0.15:
        w["batch_sweep"] = _subset(rng, [1, 2, 3, 5, 8, 16, 24, 64, 100, 256, 1000])
    if moe and rng.random() < 0.3:
        alpha = rng.choice([0.6, 0.9, 1.2, 1.5, 1.9])
        w["moe_load"] = {"alpha": alpha, "x_min": 1.0, "x_max": rng.choice([10.0, 100.0]), "seed": rng.randint(0, 9)}
    return w


def _space(rng) -> dict:
    sp = {}
    if rng.random() < 0.7:
        sp["tp_values"] = _subset(rng, [1, 2, 4, 8, 16])
    if rng.random() < 0.7:
        sp["pp_values"] = _subset(rng, [1, 2, 3, 4, 8])
    if rng.random() < 0.7:
        sp["ep_values"] = _subset(rng, [1, 2, 4, 8, 16])
    if rng.random() < 0.7:
        sp["dp_values"] = _subset(rng, [1, 2, 3, 4, 8])
    if rng.random() < 0.8:
        sp["batch_values"] = _subset(rng, [1, 2, 3, 4, 6, 8, 12, 16, 32, 48, 64, 96, 128, 200, 256, 512, 1024, 2048])
    if rng.random() < 0.25:
        sp["ctx_capacity"] = rng.choice([512, 1000, 2048, 4096, 8192, 16384])
    if rng.random() < 0.2:
        sp["chunked_prefill"] = False
    if rng.random() < 0.4:
        sp["kv_mem_fraction"] = rng.choice([0.3, 0.5, 0.75, 0.9, 1.0])
    if rng.random() < 0.3:
        sp["prefill_pool_cap"] = rng.randint(0, 16)
        sp["decode_pool_cap"] = rng.randint(1, 16)
    return sp


def _disagg(rng) -> dict | None:
    if rng.random() < 0.75:
        return None
    return {"ttft_headroom": rng.choice([1.0, 1.5, 2.2]), "prefill_utilization": rng.choice([0.7, 1.0]),
            "decode_utilization": rng.choice([0.8, 0.95]), "max_prefill_replicas": rng.randint(1, 32),
            "max_decode_replicas": rng.randint(1, 64)}


def _case(seed: int):
    rng = random.Random(seed)
    model = rng.choice(MODELS)
    hw = "b200-sxm" if model == "deepseek-v3" and rng.random() < 0.3 else "h100-sxm"
    extrapolation = rng.choice(["default"] * 5 + ["clamp", "sol", "strict"])
    db, header, recs, mdoc = _inputs(model, hw, extrapolation)
    return rng, model, extrapolation, db, header, recs, mdoc


def _objects(mdoc, wdoc, sdoc, ddoc):
    import paper_2601_06288_b200 as pkg

    model = pkg.ModelSpec.from_doc(mdoc)
    workload = pkg.WorkloadSpec.from_doc(dict(wdoc))
    space = pkg.CandidateSpace(**{k: tuple(v) if isinstance(v, list) else v for k, v in sdoc.items()})
    dc = pkg.DisaggConstants(**ddoc) if ddoc else pkg.DEFAULT_DISAGG
    return model, workload, space, dc


N_SINGLE = int(os.environ.get("LC_FUZZ_N", "200"))      # LC_FUZZ_N=3000 for a long campaign
N_BATCH = int(os.environ.get("LC_FUZZ_BATCHES", "30"))


@pytest.mark.parametrize("seed", range(N_SINGLE))
def test_random_search_matches_oracle(seed):
    import paper_2601_06288_b200 as pkg
    from oracle import oracle

    rng, model_name, extrapolation, db, header, recs, mdoc = _case(seed)
    wdoc = _workload(rng, mdoc.get("moe") is not None)
    sdoc = _space(rng)
    ddoc = _disagg(rng)
    model, workload, space, dc = _objects(mdoc, wdoc, sdoc, ddoc)
    report = pkg.run_search(db, model, workload, space, disagg_constants=dc)
    ref = oracle.run_search(header, recs, mdoc, wdoc, sdoc, ddoc, extrapolation)
    diffs = diff_canonical(canonical(report.to_doc()), canonical(ref))
    assert not diffs, f"{model_name} {extrapolation} {wdoc} {sdoc} {ddoc}\n" + "\n".join(diffs)


@pytest.mark.parametrize("seed", range(100_000, 100_000 + N_BATCH))
def test_random_batch_matches_oracle(seed):
    from oracle import oracle
    from paper_2601_06288_b200.engine import build_report, get_engine

    rng, model_name, extrapolation, db, header, recs, mdoc = _case(seed)
    sdoc = _space(rng)
    ddoc = _disagg(rng)
    wdocs = [_workload(rng, mdoc.get("moe") is not None) for _ in range(rng.randint(2, 7))]
    if rng.random() < 0.5:  # repeat some inputs: searches that share every table
        wdocs.append(dict(wdocs[0], osl=wdocs[0]["osl"] + 40))
    objs = [_objects(mdoc, w, sdoc, ddoc) for w in wdocs]
    model, _, space, dc = objs[0]
    workloads = [o[1] for o in objs]
    eng = get_engine(0)
    with eng._lock:
        out = eng.run_batch(db, model, space, workloads, dc)
        reports = [build_report(out, i, db, model, w, space, 0.0) for i, w in enumerate(workloads)]
    for w, rep in zip(wdocs, reports):
        ref = oracle.run_search(header, recs, mdoc, w, sdoc, ddoc, extrapolation)
        diffs = diff_canonical(canonical(rep.to_doc()), canonical(ref))
        assert not diffs, f"{model_name} {extrapolation} {w} {sdoc} {ddoc}\n" + "\n".join(diffs)
