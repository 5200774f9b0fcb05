"""Sweep-scale parity: real config-5 searches (batch 1..512, default space, all
modes) evaluated together in one multi-search batch -- the path bench.py
times -- and each search's full report compared with the CPU oracle run on
this box (bit-exact floats, identical rows / skips / fronts / best).

This covers what the per-search golden cases cannot: tail tables shared
between searches, the dense mixed-token tail region, query tables at full
batch width, and the split Pareto / pool kernels on ~10^5-row searches.
"""

from __future__ import annotations

import json
from concurrent.futures import ThreadPoolExecutor

import pytest

from golden_io import canonical, diff_canonical

pytestmark = pytest.mark.gpu

ROOT_SPECS = None


def _oracle_doc(part, workload):
    from oracle import oracle
    from paper_2601_06288_b200.sweeps import GOLDEN

    header, recs = oracle.read_db_records(GOLDEN / "db" / f"db-{part.model_name}-h100-sxm-s11.jsonl.gz")
    mdoc = json.loads((GOLDEN / "specs" / f"model-{part.model_name}.json").read_text())
    return oracle.run_search(header, recs, mdoc, workload.to_doc(), {"batch_values": list(part.space.batch_values)})


@pytest.mark.parametrize("model_name", ["gpt-oss-120b", "deepseek-v3"])
def test_sweep_batch_matches_oracle(model_name):
    from paper_2601_06288_b200.engine import build_report, get_engine
    from paper_2601_06288_b200.sweeps import sweep

    part = next(p for p in sweep("config5") if p.model_name == model_name)
    # a spread of workloads incl. the extremes (isl 512 / 16384, osl 64 / 4096)
    picks = [0, 9, 37, 54, 90, 99]
    workloads = [part.workloads[i] for i in picks]
    eng = get_engine(0)
    with eng._lock:
        out = eng.run_batch(part.db, part.model, part.space, workloads)
        reports = [build_report(out, i, part.db, part.model, w, part.space, 0.0) for i, w in enumerate(workloads)]
    with ThreadPoolExecutor(max_workers=6) as ex:
        refs = list(ex.map(lambda w: _oracle_doc(part, w), workloads))
    total = 0
    for w, rep, ref in zip(workloads, reports, refs):
        diffs = diff_canonical(canonical(rep.to_doc()), canonical(ref))
        assert not diffs, f"isl={w.isl} osl={w.osl}:\n" + "\n".join(diffs)
        total += ref["counts"]["enumerated"]
    assert total > 100_000
