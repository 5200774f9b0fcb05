"""Sweep-scale parity: real config-5 searches (batch 1..512, default space, all
modes) evaluated together in one multi-search batch -- the path bench.py
times -- and each search's full report compared with the CPU oracle run on
this box (bit-exact floats, identical rows / skips / fronts / best).

Both named sweeps are covered (sweeps.py): ``config5`` (GPT-OSS-120B +
DeepSeek-V3) and the north-star target ``config5_qwen`` (Qwen3-32B +
DeepSeek-V3, with the extended OSL list 96 ... 6144).  Per (sweep, model) a
stratified pick of >= 20 workloads covers every ISL of the grid at least twice
and every OSL at least once (twice on the 10 x 10 grid), including the
extremes ISL 512 / 16384 and OSL 64 / 4096 / 6144.  The picked searches run
in ONE shared-table batch and every one of them is checked against the oracle.

A second test runs each model's FULL workload list (the bench's exact batch:
100 or 220 searches, ~10^7 candidates over both models) and checks that the
picked searches' summaries (counts, query totals, best / nearest row keys,
Pareto front row keys, disaggregated plans) are identical to the ones of the
picks-only batch, so sharing tables across the whole sweep changes nothing.

This covers what the per-search golden cases cannot: tail tables shared
between searches, the dense mixed-token tail region, query tables at full
batch width, and the split Pareto / pool kernels on ~10^5-row searches.
"""

from __future__ import annotations

import json
import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from golden_io import canonical, diff_canonical

pytestmark = pytest.mark.gpu


def stratified_picks(n_isl: int, n_osl: int) -> list[int]:
    """Workload indices (ISL-major grid) covering every ISL >= 2x and every OSL >= 1x (>= 20 picks)."""
    picks = set()
    if n_osl <= n_isl:
        for i in range(n_isl):
            picks.add(i * n_osl + (3 * i) % n_osl)
            picks.add(i * n_osl + (7 * i + 5) % n_osl)
    else:
        for j in range(n_osl):
            picks.add((j % n_isl) * n_osl + j)
        for i in range(n_isl):  # second ISL coverage on the other diagonal
            picks.add(i * n_osl + (n_osl - 1 - (3 * i) % n_osl))
    return sorted(picks)


_ORACLE: dict = {}
_ORACLE_LOCK = threading.Lock()


def _oracle_doc(model_name: str, batch_values: tuple, workload):
    from oracle import oracle
    from paper_2601_06288_b200.sweeps import GOLDEN

    header, recs = oracle.read_db_records(GOLDEN / "db" / f"db-{model_name}-h100-sxm-s11.jsonl.gz")
    mdoc = json.loads((GOLDEN / "specs" / f"model-{model_name}.json").read_text())
    return oracle.run_search(header, recs, mdoc, workload.to_doc(), {"batch_values": list(batch_values)})


def _oracle_docs(model_name, batch_values, workloads):
    """Oracle reports (cached across tests: DeepSeek-V3 appears in both sweeps), all host threads."""
    keys = [(model_name, w.isl, w.osl) for w in workloads]
    with _ORACLE_LOCK:
        todo = [(k, w) for k, w in zip(keys, workloads) if k not in _ORACLE]
        # longest jobs first (static decode cost grows with the OSL) for a short tail
        todo.sort(key=lambda kw: -kw[1].osl)
        with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            docs = list(ex.map(lambda kw: _oracle_doc(model_name, batch_values, kw[1]), todo))
        for (k, _), d in zip(todo, docs):
            _ORACLE[k] = d
        return [_ORACLE[k] for k in keys]


CASES = [("config5", "gpt-oss-120b"), ("config5", "deepseek-v3"),
         ("config5_qwen", "qwen3-32b"), ("config5_qwen", "deepseek-v3")]


def _part(sweep_name, model_name):
    from paper_2601_06288_b200.sweeps import ISL, OSL, OSL_QWEN, sweep

    part = next(p for p in sweep(sweep_name) if p.model_name == model_name)
    n_osl = len(OSL_QWEN if sweep_name == "config5_qwen" else OSL)
    picks = stratified_picks(len(ISL), n_osl)
    assert len(part.workloads) == len(ISL) * n_osl
    return part, picks


def test_stratified_picks_cover_grid():
    from paper_2601_06288_b200.sweeps import ISL, OSL, OSL_QWEN

    for osl in (OSL, OSL_QWEN):
        picks = stratified_picks(len(ISL), len(osl))
        assert len(picks) >= 20
        isl_hits = np.bincount([p // len(osl) for p in picks], minlength=len(ISL))
        osl_hits = np.bincount([p % len(osl) for p in picks], minlength=len(osl))
        assert isl_hits.min() >= 2 and osl_hits.min() >= 1


@pytest.mark.parametrize("sweep_name,model_name", CASES)
def test_sweep_batch_matches_oracle(sweep_name, model_name):
    from paper_2601_06288_b200.engine import build_report, get_engine

    part, picks = _part(sweep_name, model_name)
    workloads = [part.workloads[i] for i in picks]
    eng = get_engine(0)
    with eng._lock:
        out = eng.run_batch(part.db, part.model, part.space, workloads)
        reports = [build_report(out, i, part.db, part.model, w, part.space, 0.0) for i, w in enumerate(workloads)]
    refs = _oracle_docs(model_name, part.space.batch_values, workloads)
    total = 0
    for w, rep, ref in zip(workloads, reports, refs):
        diffs = diff_canonical(canonical(rep.to_doc()), canonical(ref))
        assert not diffs, f"{sweep_name} {model_name} isl={w.isl} osl={w.osl}:\n" + "\n".join(diffs)
        total += ref["counts"]["enumerated"]
    assert total > 300_000


SUMMARY_FIELDS = ("n_units", "n_enumerated", "n_rows", "n_feasible", "n_skipped", "n_front", "n_plans", "best",
                  "nearest", "nearest_violation", "best_thru", "best_speed", "queries_1d", "queries_2d",
                  "n_feasible_plans")


def _summaries(eng, part, workloads):
    from paper_2601_06288_b200.engine import fetch_fronts

    out = eng.run_batch(part.db, part.model, part.space, workloads)
    front, plans = fetch_fronts(out)
    res = out.results.copy()
    f_off = np.concatenate([[0], np.cumsum(res["n_front"])])
    p_off = np.concatenate([[0], np.cumsum(res["n_plans"])])
    per = []
    for i in range(len(workloads)):
        per.append((res[i], front[f_off[i]:f_off[i + 1]].copy(),
                    {k: v[p_off[i]:p_off[i + 1]].copy() for k, v in plans.items()}))
    return per


@pytest.mark.parametrize("sweep_name,model_name", CASES)
def test_full_sweep_batch_equals_picks_batch(sweep_name, model_name):
    from paper_2601_06288_b200.engine import get_engine

    part, picks = _part(sweep_name, model_name)
    eng = get_engine(0)
    with eng._lock:
        full = _summaries(eng, part, part.workloads)
        small = _summaries(eng, part, [part.workloads[i] for i in picks])
    for j, i in enumerate(picks):
        (rf, ff, pf), (rs, fs, ps) = full[i], small[j]
        for f in SUMMARY_FIELDS:
            a, b = rf[f], rs[f]
            assert a == b or (isinstance(a, float) and np.isnan(a) and np.isnan(b)), (i, f, a, b)
        assert np.array_equal(ff, fs), i
        for k in pf:
            # plan_p / plan_d are unit indices of the batch: compare them relative to the search's offset
            if k in ("plan_p", "plan_d"):
                assert np.array_equal(pf[k] - rf["unit_off"], ps[k] - rs["unit_off"]), (i, k)
            else:
                assert np.array_equal(pf[k], ps[k]), (i, k)
    total = sum(int(r["n_enumerated"]) for r, _, _ in full)
    assert total > 2_000_000  # DeepSeek-V3 config5: 2.58M; GPT-OSS 7.7M; Qwen3-32B 4.2M
