"""Generate single-query golden vectors from the UNMODIFIED reference (survey container only).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_query_golden.py

Writes ``queries.json.gz`` next to this file: reference ``query_latency``
(/root/reference/pkg/src/llmconf/perfdb.py:539-580) on

  * the reference's own unit-test known answers (pkg/tests/test_perfdb.py:
    TestInterpolation / TestExtrapolation), on inline databases;
  * every query the reference estimator issues during the ``a1_qwen_small`` and
    ``dsv3_all_default`` searches (harvested by wrapping
    ``llmconf.estimator.query_latency``), de-duplicated and capped;
  * seeded random probes of every grid of four case databases under each
    extrapolation policy: on-grid, inside, below, above, mixed 2-D, generation
    attention with an explicit kv_len, missing keys and backend mismatches.

Each vector is ``{db, policy, query, expect}``, ``expect`` a float hex string or
``"Type: message"``.
"""

from __future__ import annotations

import json
import math
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from cases import BY_NAME  # noqa: E402
from make_golden import case_objects, load_case_db, model, write_gz  # noqa: E402

from llmconf import estimator, moe_load  # noqa: E402
from llmconf.perfdb import HardwareSpec, OperatorQuery, OperatorRecord, PerfDatabase, query_latency  # noqa: E402
from llmconf.search import run_search  # noqa: E402

POLICIES = (None, "default", "strict", "clamp", "sol")
KAT_HW = {"name": "testgpu", "gpu_memory": 80 * 2**30, "mem_bandwidth": 3e12,
          "compute_throughput": {"fp16": 1e15, "fp8": 2e15}, "intra_node_bandwidth": 400e9,
          "inter_node_bandwidth": 50e9, "gpus_per_node": 8}
ATTN_FIXED = {"num_heads": 8, "kv_heads": 8, "head_dim": 64, "attn_kind": "MHA"}


def qdoc(q: OperatorQuery) -> dict:
    d = {"kind": q.kind, "quant": q.quant, "shape": dict(q.shape)}
    if q.backend is not None:
        d["backend"] = q.backend
    return d


def run(db, q, policy):
    try:
        return query_latency(db, q, policy).hex()
    except Exception as e:  # noqa: BLE001 - the reference's exception type and text are the expectation
        return f"{type(e).__name__}: {e}"


def inline_db(name: str, records: list[tuple[OperatorQuery, float]]) -> tuple[dict, PerfDatabase]:
    hw = HardwareSpec.from_doc(KAT_HW)
    recs = [OperatorRecord(q, lat) for q, lat in records]
    db = PerfDatabase.from_records(hw, "trtllm", "1.0", recs)
    doc = {"header": {"schema": "llmconf-perfdb/1", "hardware": KAT_HW, "backend": "trtllm",
                      "backend_version": "1.0"},
           "records": [{"kind": q.kind, "quant": q.quant, "shape": dict(q.shape), "latency_us": lat,
                        "provenance": "measured"} for q, lat in records]}
    return doc, db


def gemm_q(m: int, n: int = 4096, k: int = 4096) -> OperatorQuery:
    return OperatorQuery("gemm", "fp16", {"m": m, "n": n, "k": k})


def kat_vectors(dbs: dict, vectors: list) -> None:
    def add(name, records, probes):
        doc, db = inline_db(name, records)
        dbs[name] = {"inline": doc}
        for q, policy in probes:
            vectors.append({"db": name, "policy": policy, "query": qdoc(q), "expect": run(db, q, policy)})

    g = lambda pts: [(gemm_q(m), lat) for m, lat in pts.items()]  # noqa: E731
    add("kat_gemm_exact", g({16: 103.7, 64: 411.9}), [(gemm_q(16), None), (gemm_q(64), None)])
    probes = [(gemm_q(m), None) for m in (32, 17, 23, 40, 63, 2, 4096)]
    probes += [(gemm_q(m), "strict") for m in (8, 128)]
    probes += [(gemm_q(m), "clamp") for m in (8, 1024)]
    probes += [(gemm_q(m), "sol") for m in (1024, 8)]
    probes += [(OperatorQuery("embedding", "fp16", {"tokens": 4, "hidden": 64, "vocab": 1000}), None),
               (OperatorQuery("gemm", "fp16", {"m": 16, "n": 4096, "k": 4096}, backend="vllm"), None),
               (OperatorQuery("gemm", "int4", {"m": 16, "n": 4096, "k": 4096}), None)]
    add("kat_gemm_100_400", g({16: 100.0, 64: 400.0}), probes)
    lats = {(1, 128): 50.0, (1, 512): 200.0, (4, 128): 180.0, (4, 512): 720.0}
    recs = [(OperatorQuery("attention_context", "fp16", {"batch": b, "seq_len": s, **ATTN_FIXED}), lat)
            for (b, s), lat in lats.items()]
    aq = lambda b, s: OperatorQuery("attention_context", "fp16", {"batch": b, "seq_len": s, **ATTN_FIXED})  # noqa
    add("kat_attn_2d", recs, [(aq(2, 256), None), (aq(4, 128), None), (aq(8, 64), None), (aq(8, 1024), "sol"),
                              (aq(2, 1024), None), (aq(1, 64), "clamp")])
    q1 = OperatorQuery("attention_generation", "fp16", {"batch": 2, "seq_len": 128, **ATTN_FIXED})
    gq = lambda b, s, kv: OperatorQuery("attention_generation", "fp16",  # noqa: E731
                                        {"batch": b, "seq_len": s, **({"kv_len": kv} if kv else {}), **ATTN_FIXED})
    add("kat_kv_len", [(q1, 42.0)], [(gq(2, 128, 128), None), (gq(2, 128, 0), None), (gq(4, 256, 4096), None),
                                     (gq(4, 256, 0), None), (gq(4, 64, 9), "sol"), (gq(1, 1, 0), "sol")])
    # hypothesis-style bracketing / monotone grids (test_perfdb.py:96-128), seeded
    rng = random.Random(11)
    for i in range(12):
        grid_ms = [16, 32, 64, 128, 256]
        if i % 2:
            cur, lats5 = 10.0, []
            for s in [0.0] + [rng.uniform(0.0, 2.0) for _ in range(4)]:
                cur *= 1.0 + s
                lats5.append(cur)
        else:
            lats5 = [rng.uniform(1.0, 1e6) for _ in range(5)]
        add(f"kat_gemm_rand{i}", g(dict(zip(grid_ms, lats5))),
            [(gemm_q(rng.randint(16, 256)), None) for _ in range(12)] + [(gemm_q(m), None) for m in grid_ms])


def harvest(case_name: str, cap: int, rng: random.Random) -> list[OperatorQuery]:
    case = BY_NAME[case_name]
    db = load_case_db(case)
    wl, space, dc = case_objects(case)
    seen: dict = {}
    orig = estimator.query_latency

    def wrapped(d, q, policy=None):
        seen.setdefault(q, None)
        return orig(d, q, policy)

    estimator.query_latency = wrapped
    try:
        estimator.clear_caches()
        moe_load._cached_weights.cache_clear()
        run_search(db, model(case["model"]), wl, space, jobs=1, disagg_constants=dc)
    finally:
        estimator.query_latency = orig
    qs = list(seen)
    rng.shuffle(qs)
    return qs[:cap]


def log_uniform(rng: random.Random, lo: int, hi: int) -> int:
    return max(1, int(round(math.exp(rng.uniform(math.log(lo), math.log(hi))))))


def probe_grid(db, key, grid, rng: random.Random) -> list[OperatorQuery]:
    kind, quant, fixed = key
    fixed = dict(fixed)
    axes, vals = grid.axes, grid.axis_values
    out = []

    def mk(coords, extra=None):
        shape = dict(fixed)
        shape.update(dict(zip(axes, coords)))
        if extra:
            shape.update(extra)
        return OperatorQuery(kind, quant, shape)

    def pick(v, where):
        lo, hi = v[0], v[-1]
        if where == "grid":
            return rng.choice(v)
        if where == "in":
            return log_uniform(rng, lo, hi) if hi > lo else lo
        if where == "below":
            return max(1, rng.randint(max(1, lo // 8), lo)) if lo > 1 else None
        return rng.randint(hi + 1, hi * 8 + 1)

    wheres = ("grid", "in", "below", "above")
    for _ in range(6):
        for w0 in wheres:
            if len(axes) == 1:
                c = pick(vals[0], w0)
                if c is not None:
                    out.append(mk((c,)))
            else:
                w1 = rng.choice(wheres)
                c0, c1 = pick(vals[0], w0), pick(vals[1], w1)
                if c0 is not None and c1 is not None:
                    out.append(mk((c0, c1)))
    if kind == "attention_generation":
        for _ in range(4):
            c = (pick(vals[0], "in"), pick(vals[1], rng.choice(("in", "above"))))
            out.append(mk(c, {"kv_len": rng.randint(1, 4 * vals[1][-1])}))
    return out


def main() -> None:
    rng = random.Random(20260117)
    dbs: dict = {}
    vectors: list = []
    kat_vectors(dbs, vectors)
    n_kat = len(vectors)

    for case_name, cap in (("a1_qwen_small", 1500), ("dsv3_all_default", 1500)):
        case = BY_NAME[case_name]
        db = load_case_db(case)
        name = f"case:{case_name}"
        dbs[name] = {"case": case_name}
        for q in harvest(case_name, cap, rng):
            vectors.append({"db": name, "policy": None, "query": qdoc(q), "expect": run(db, q, None)})
    n_harvest = len(vectors) - n_kat

    for case_name in ("a1_qwen_small", "unsupported_quant_a100", "dsv3_all_default", "gptoss_all_default"):
        case = BY_NAME[case_name]
        db = load_case_db(case)
        name = f"case:{case_name}"
        dbs[name] = {"case": case_name}
        for key in sorted(db._grids, key=repr):
            for q in probe_grid(db, key, db._grids[key], rng):
                policy = rng.choice(POLICIES)
                vectors.append({"db": name, "policy": policy, "query": qdoc(q), "expect": run(db, q, policy)})
        # missing keys (an n no gemm grid has) and a backend mismatch
        for m in (1, 77, 4096):
            q = OperatorQuery("gemm", "fp16", {"m": m, "n": 12345, "k": 678})
            vectors.append({"db": name, "policy": None, "query": qdoc(q), "expect": run(db, q, None)})
        q = OperatorQuery("gemm", "fp16", {"m": 8, "n": 12345, "k": 678}, backend="sglang")
        vectors.append({"db": name, "policy": None, "query": qdoc(q), "expect": run(db, q, None)})

    doc = {"dbs": dbs, "vectors": vectors}
    write_gz(HERE / "queries.json.gz", json.dumps(doc, sort_keys=True) + "\n")
    errs = sum(1 for v in vectors if ":" in v["expect"])
    print(f"{len(vectors)} vectors ({n_kat} KAT, {n_harvest} harvested, {errs} errors) over {len(dbs)} databases")


if __name__ == "__main__":
    main()
