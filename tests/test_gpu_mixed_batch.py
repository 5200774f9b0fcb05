"""Heterogeneous searches in one device batch.

The engine shares query tables, decode-series tables and MoE tail tables
between the searches of a batch whenever their inputs agree (context length,
batch list, MoE load, KV midpoint).  Here one batch mixes workloads that agree
on some of those inputs and differ on others -- modes, budgets, prefix reuse,
batch sweeps, MoE loads, SLAs, repeated ISLs with different OSLs -- and every
search's report must equal the CPU oracle's for that search alone.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import pytest

from golden_io import canonical, db_path, diff_canonical, model_doc

pytestmark = pytest.mark.gpu

WORKLOADS = [
    dict(isl=1024, osl=128, ttft_limit_ms=2000.0, tpot_limit_ms=50.0),
    dict(isl=1024, osl=512, ttft_limit_ms=2000.0, min_speed=5.0),                       # same isl, other osl
    dict(isl=1024, osl=128, prefix_len=512, min_speed=5.0),                             # same isl, prefix
    dict(isl=512, osl=128, ttft_limit_ms=2000.0, min_speed=5.0, gpu_budgets=[2, 8]),   # budgets
    dict(isl=700, osl=50, min_speed=3.0, moe_load=dict(alpha=0.0, x_min=1.0, x_max=2.0, seed=9)),
    dict(isl=700, osl=50, min_speed=3.0),                                               # same, default load
    dict(isl=3000, osl=40, batch_sweep=[1, 3, 100, 1500], ttft_limit_ms=60000.0, min_speed=1.0),
    dict(isl=2048, osl=300, modes=["static"], min_speed=2.0),
    dict(isl=2048, osl=300, modes=["aggregated", "disaggregated"], min_speed=2.0),
    dict(isl=2048, osl=1, ttft_limit_ms=10000.0),
    dict(isl=4096, osl=64, ttft_limit_ms=0.001, min_speed=1.0),                         # nothing feasible
    dict(isl=1500, osl=90, ttft_limit_ms=5000.0, min_speed=5.0,
         moe_load=dict(alpha=0.5, x_min=1.0, x_max=1000.0, seed=3)),
]


def test_mixed_batch_matches_oracle_per_search():
    import paper_2601_06288_b200 as pkg
    from oracle import oracle
    from paper_2601_06288_b200.engine import build_report, get_engine

    case = {"model": "moe-small"}
    db = pkg.load_db(db_path(case))
    model = pkg.ModelSpec.from_doc(model_doc("moe-small"))
    space = pkg.CandidateSpace()
    workloads = [pkg.WorkloadSpec.from_doc(dict(w)) for w in WORKLOADS]
    eng = get_engine(0)
    with eng._lock:
        out = eng.run_batch(db, model, space, workloads)
        reports = [build_report(out, i, db, model, w, space, 0.0) for i, w in enumerate(workloads)]
    header, recs = oracle.read_db_records(db_path(case))

    def ref(w):
        return oracle.run_search(header, recs, model_doc("moe-small"), w, {})

    with ThreadPoolExecutor(max_workers=8) as ex:
        refs = list(ex.map(ref, WORKLOADS))
    for w, rep, r in zip(WORKLOADS, reports, refs):
        diffs = diff_canonical(canonical(rep.to_doc()), canonical(r))
        assert not diffs, f"{w}:\n" + "\n".join(diffs)
