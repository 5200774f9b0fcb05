"""The drop-in boundary accepts the reference's own objects.

CPU-only; needs the reference importable from /root/reference/pkg/src (the
builder container), so every test here skips on the GPU box, where the same
host logic is exercised through this package's objects.

* ``database.flatten`` of a reference ``PerfDatabase`` equals the image of this
  package's database loaded from the same file, array for array;
* ``plans.build_space_plan`` from reference ``ModelSpec`` / ``CandidateSpace``
  objects equals the plan from this package's objects (combos, templates, slot
  tables, generation classes);
* the ``Engine`` host side builds identical search descriptors from reference
  ``WorkloadSpec`` objects;
* ``validate_db`` gives the reference's report on clean and corrupted databases;
* the INTEGRATION.md patch block imports cleanly into the reference modules and
  rebinds their seams to this package.
"""

from __future__ import annotations

import dataclasses
import gzip
import json
import re
import sys
from pathlib import Path

import numpy as np
import pytest

REF_SRC = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"

pytestmark = pytest.mark.skipif(not (REF_SRC / "llmconf").exists(), reason="reference not importable here")


@pytest.fixture(scope="module")
def ref():
    sys.dont_write_bytecode = True  # /root/reference is read-only
    if str(REF_SRC) not in sys.path:
        sys.path.append(str(REF_SRC))
    import llmconf.model
    import llmconf.perfdb
    import llmconf.search
    import llmconf.serving_modes

    return llmconf


def _db_file(name):
    return GOLDEN / "db" / f"db-{name}-h100-sxm-s11.jsonl.gz"


@pytest.fixture(scope="module")
def dbs(ref, tmp_path_factory):
    import paper_2601_06288_b200 as pkg

    out = {}
    for name in ("qwen-small", "deepseek-v3", "gpt-oss-120b"):
        tmp = tmp_path_factory.mktemp("db") / f"{name}.jsonl"
        tmp.write_bytes(gzip.decompress(_db_file(name).read_bytes()))
        out[name] = (ref.perfdb.load_db(str(tmp)), pkg.load_db(_db_file(name)))
    return out


def _arrays_equal(a, b):
    for f in dataclasses.fields(a):
        x, y = getattr(a, f.name), getattr(b, f.name)
        if isinstance(x, np.ndarray):
            assert x.dtype == y.dtype and np.array_equal(x, y), f.name
        else:
            assert x == y, f.name


@pytest.mark.parametrize("name", ["qwen-small", "deepseek-v3", "gpt-oss-120b"])
def test_flatten_reference_db_equals_own(dbs, name):
    from paper_2601_06288_b200.database import flatten

    ref_db, own_db = dbs[name]
    _arrays_equal(flatten(ref_db), flatten(own_db))


@pytest.mark.parametrize("name,space_kw", [
    ("qwen-small", {}),
    ("deepseek-v3", {}),
    ("gpt-oss-120b", {"tp_values": (8, 2, 1), "pp_values": (1, 4), "ep_values": (8, 4, 4), "dp_values": (1, 2)}),
    ("deepseek-v3", {"kv_mem_fraction": 0.5, "ctx_capacity": 4096, "chunked_prefill": False}),
    ("qwen-small", {"kv_mem_fraction": 1.5}),  # invalid shared knob: no combos on either side
])
def test_space_plan_from_reference_objects(ref, dbs, name, space_kw):
    import paper_2601_06288_b200 as pkg
    from paper_2601_06288_b200.database import flatten
    from paper_2601_06288_b200.plans import build_space_plan

    ref_db, own_db = dbs[name]
    mdoc = json.loads((GOLDEN / "specs" / f"model-{name}.json").read_text())
    ref_plan = build_space_plan(ref.model.ModelSpec.from_doc(mdoc), ref.search.CandidateSpace(**space_kw),
                                flatten(ref_db), ref_db.backend)
    own_plan = build_space_plan(pkg.ModelSpec.from_doc(mdoc), pkg.CandidateSpace(**space_kw),
                                flatten(own_db), own_db.backend)
    for f in dataclasses.fields(ref_plan):
        x, y = getattr(ref_plan, f.name), getattr(own_plan, f.name)
        if isinstance(x, np.ndarray):
            assert np.array_equal(x, y), f.name
        elif f.name == "infos":
            assert [[(e.label, e.key, e.quant, e.grid) for e in t] for t in x] == \
                   [[(e.label, e.key, e.quant, e.grid) for e in t] for t in y]
        else:
            assert x == y, f.name
    if space_kw.get("kv_mem_fraction", 0.9) > 1:
        assert len(own_plan.combos) == 0


def test_workload_descriptors_from_reference_objects(ref, dbs, monkeypatch):
    """Engine.run_batch's host side (descriptor building) from reference WorkloadSpec /
    CandidateSpace / DisaggConstants objects: the lc_search_batch arguments are identical."""
    import paper_2601_06288_b200 as pkg
    from paper_2601_06288_b200 import engine as E

    import types

    monkeypatch.setattr(E.Engine, "_call", lambda self, fn, name, *args: None)  # no device call
    eng = E.Engine.__new__(E.Engine)
    eng.lib = types.SimpleNamespace(lc_search_batch=None)
    eng.ctx = None
    eng._pinned, eng._deferred = (), []
    eng.space_handle = lambda db, model, space: (None, E.build_space_plan(model, space, E.flatten(db), db.backend),
                                                   E.flatten(db))
    eng.db_handle = lambda db: (None, E.flatten(db))
    ref_db, own_db = dbs["deepseek-v3"]
    mdoc = json.loads((GOLDEN / "specs" / "model-deepseek-v3.json").read_text())
    wdocs = [dict(isl=4000, osl=500, ttft_limit_ms=5000.0, min_speed=20.0),
             dict(isl=512, osl=64, tpot_limit_ms=40.0, gpu_budgets=[8, 16], modes=["aggregated", "disaggregated"],
                  batch_sweep=[4, 1, 64], moe_load={"alpha": 1.5, "x_min": 1.0, "x_max": 50.0, "seed": 3})]
    outs = []
    for mod_model, mod_wl, mod_space, mod_dc, db in (
            (ref.model.ModelSpec, ref.serving_modes.WorkloadSpec, ref.search.CandidateSpace,
             ref.serving_modes.DisaggConstants, ref_db),
            (pkg.ModelSpec, pkg.WorkloadSpec, pkg.CandidateSpace, pkg.DisaggConstants, own_db)):
        model = mod_model.from_doc(mdoc)
        wls = [mod_wl.from_doc(dict(d)) for d in wdocs]
        space = mod_space(batch_values=(1, 2, 8, 32), prefill_pool_cap=4)
        out = eng.run_batch(db, model, space, wls, mod_dc(ttft_headroom=2.0))
        outs.append((out.searches.tobytes(), out.batches.tolist()))
    assert outs[0] == outs[1]


def _corrupt(records, kind):
    recs = list(records)
    if kind == "latency":
        object.__setattr__(recs[3], "latency_us", -1.0)
        object.__setattr__(recs[7], "latency_us", float("nan"))
    elif kind == "provenance":
        object.__setattr__(recs[2], "provenance", "guessed")
    elif kind == "duplicate":
        recs.append(recs[5])
    elif kind == "ragged":  # drop one cell of a 2-D (attention) grid
        kinds = [getattr(getattr(r, "query", r), "kind") for r in recs]
        recs.pop(next(i for i, k in enumerate(kinds) if k.startswith("attention")) + 1)
    return recs


@pytest.mark.parametrize("corruption", [None, "latency", "provenance", "duplicate", "ragged"])
@pytest.mark.parametrize("required", [(), ("gemm", "embedding"), ("alltoall", "gemm", "moe_gemm")])
def test_validate_db_matches_reference(ref, dbs, corruption, required):
    import copy

    from paper_2601_06288_b200.database import validate_db

    ref_db, own_db = dbs["deepseek-v3"]
    ref_db, own_db = copy.copy(ref_db), copy.copy(own_db)
    ref_recs = [copy.copy(r) for r in ref_db.records]
    own_recs = [copy.copy(r) for r in own_db.records]
    object.__setattr__(ref_db, "records", tuple(_corrupt(ref_recs, corruption)))
    object.__setattr__(own_db, "records", tuple(_corrupt(own_recs, corruption)))
    want = ref.perfdb.validate_db(ref_db, required_kinds=required)
    got = validate_db(own_db, required_kinds=required)
    assert got.lines() == want.lines() and got.ok == want.ok
    # the reference's own database objects through this package's validate_db
    assert validate_db(ref_db, required_kinds=required).lines() == want.lines()
    if corruption:
        assert not got.ok


def test_integration_patch_imports_cleanly(ref, monkeypatch):
    """Execute INTEGRATION.md's patch block in the reference modules' namespaces."""
    import paper_2601_06288_b200 as pkg

    text = (ROOT / "INTEGRATION.md").read_text()
    block = re.search(r"## 1\. Python drop-in.*?```python\n(.*?)```", text, re.S).group(1)
    parts = [p for p in re.split(r"\n(?=# llmconf/)", "\n" + block.strip()) if p.strip()]
    monkeypatch.setenv("LLMCONF_ENGINE", "b200")
    import llmconf.estimator

    targets = {"search.py": ref.search, "perfdb.py": ref.perfdb, "serving_modes.py": ref.serving_modes,
               "estimator.py": llmconf.estimator}
    done = set()
    saved = {m: dict(vars(m)) for m in targets.values()}
    try:
        for part in parts:
            head = part.strip().splitlines()[0]
            fname = re.match(r"# llmconf/(\w+\.py)", head).group(1)
            mod = targets[fname]
            code = part if "import os" in part else "import os\n" + part
            exec(compile(code, f"INTEGRATION.md:{fname}", "exec"), vars(mod))
            done.add(fname)
        assert done == set(targets)
        assert ref.search.run_search is pkg.run_search
        assert ref.search.enumerate_candidates is pkg.enumerate_candidates
        assert ref.perfdb.query_latency is pkg.query_latency
        assert ref.serving_modes.estimate_static is pkg.estimate_static
        assert ref.serving_modes.estimate_aggregated is pkg.estimate_aggregated
        assert llmconf.estimator.get_step_latency is pkg.get_step_latency
        assert llmconf.estimator.get_gen_latency is pkg.get_gen_latency
    finally:
        for m, d in saved.items():
            vars(m).clear()
            vars(m).update(d)


@pytest.mark.parametrize("stride", [1, 5, 32, 77, 5000])
@pytest.mark.parametrize("name,cfg,wl", [
    ("deepseek-v3", (8, 2, 8, 1, 128), dict(isl=5000, osl=1000)),
    ("qwen3-32b", (2, 1, 1, 4, 64), dict(isl=4000, osl=500, prefix_len=1000)),
    ("gpt-oss-120b", (4, 1, 4, 1, 512), dict(isl=512, osl=97)),
])
def test_oracle_static_stride_matches_reference(ref, name, cfg, wl, stride, tmp_path):
    """The oracle's estimate_static at any stride equals the reference's (serving_modes.py:231-267)
    bit for bit: the oracle that pins the device's stride path (tests/test_gpu_estimate.py)."""
    from oracle import oracle

    header, recs = oracle.read_db_records(_db_file(name))
    mdoc = json.loads((GOLDEN / "specs" / f"model-{name}.json").read_text())
    tmp = tmp_path / "db.jsonl"
    tmp.write_bytes(gzip.decompress(_db_file(name).read_bytes()))
    rdb = ref.perfdb.load_db(str(tmp))
    rmodel = ref.model.ModelSpec.from_doc(mdoc)
    rwl = ref.serving_modes.WorkloadSpec.from_doc(dict(wl))
    rcfg = ref.search.CandidateSpace().config(*cfg, rdb.backend)
    from llmconf import estimator

    estimator.clear_caches()
    est = ref.serving_modes.estimate_static(rdb, rmodel, rcfg, rwl, stride=stride)
    got = oracle.estimate(header, recs, mdoc, dict(wl), cfg, "static", stride=stride)
    assert got["status"] == 0
    want = [est.ttft_ms, est.tpot_ms, est.speed, est.throughput_per_gpu]
    assert [float(x).hex() for x in got["values"]] == [x.hex() for x in want]
