"""bench.py host logic (no GPU): how the fixed config-5 sweep is split into
pipelines (--streams) and across ranks (strong scaling), so that every
workload is evaluated exactly once, in ISL-major contiguous blocks."""

from __future__ import annotations

import importlib.util
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def bench():
    sys.path.insert(0, str(ROOT))
    spec = importlib.util.spec_from_file_location("bench_under_test", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.fixture(scope="module")
def parts():
    from paper_2601_06288_b200.sweeps import sweep

    return sweep("config5")


@pytest.mark.parametrize("spec", ["*:1", "*:2", "*:3", "gpt-oss-120b:2", "gpt-oss-120b:3,deepseek-v3:2"])
@pytest.mark.parametrize("ws", [1, 2, 3, 8])
def test_pipelines_cover_the_sweep_once(bench, parts, spec, ws):
    bench._STREAMS.clear()
    for item in spec.split(","):
        name, _, k = item.partition(":")
        bench._STREAMS[name] = int(k)
    seen = {p.model_name: [] for p in parts}
    for rank in range(ws):
        jobs = bench._my_workloads(parts, ws, rank, "strong")
        keys = [k for k, _, _ in jobs]
        assert len(keys) == len(set(keys))
        for key, p, wls in jobs:
            assert key.split("#")[0] == p.model_name
            # a contiguous block of the model's ISL-major workload list
            i0 = p.workloads.index(wls[0])
            assert p.workloads[i0:i0 + len(wls)] == wls
            seen[p.model_name].extend(wls)
    for p in parts:
        assert seen[p.model_name] == list(p.workloads)
    bench._STREAMS.clear()


def test_weak_scaling_offsets_the_isl_grid(bench, parts):
    bench._STREAMS.clear()
    j0 = bench._my_workloads(parts, 2, 0, "weak")
    j1 = bench._my_workloads(parts, 2, 1, "weak")
    for (k0, p0, w0), (k1, p1, w1) in zip(j0, j1):
        assert k0 == k1 and len(w0) == len(w1) == len(p0.workloads)
        assert all(b.isl == a.isl + 1 and b.osl == a.osl for a, b in zip(w0, w1))
