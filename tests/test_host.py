"""Host-side logic that needs no GPU: DB ingest, the device image, plan
templates, skip-reason formatting and report documents."""

from __future__ import annotations

import json
import math

import numpy as np
import pytest

import paper_2601_06288_b200 as pkg
from golden_io import BY_NAME, CASES, db_path, golden_report, model_doc
from paper_2601_06288_b200.database import KIND_DIMS, flatten, grid_key
from paper_2601_06288_b200.engine import _reason
from paper_2601_06288_b200.plans import LABEL_CODE, build_space_plan
from product_cases import case_objects


def test_load_db_rebuilds_reference_grids():
    from oracle import oracle

    header, recs = oracle.read_db_records(db_path(BY_NAME["cfg4_dsv3"]))
    db = pkg.load_db(db_path(BY_NAME["cfg4_dsv3"]))
    assert len(db.records) == len(recs) == 1390
    assert len(db._grids) == 41
    for r in recs[:200]:
        key = grid_key(r["kind"], r["quant"], r["shape"])
        g = db._grids[key]
        coords = tuple(int(r["shape"][a]) for a in KIND_DIMS[r["kind"]][1])
        assert g.cells[coords] == r["latency_us"]


def test_flat_image_matches_grid_index():
    db = pkg.load_db(db_path(BY_NAME["a1_qwen_small"]))
    flat = flatten(db)
    assert flatten(db) is flat  # cached per object
    for gid, key in enumerate(flat.keys):
        g = db._grids[key]
        off, n = flat.grid_axis_off[2 * gid], flat.grid_axis_len[2 * gid]
        assert tuple(flat.axis_val[off: off + n]) == g.axis_values[0]
        assert all(flat.axis_log[off + i] == math.log(v) for i, v in enumerate(g.axis_values[0]))
        c0 = flat.grid_cell_off[gid]
        first = tuple(v[0] for v in g.axis_values)
        assert flat.cell[c0] == g.cells[first]
        assert flat.cell_log[c0] == math.log(g.cells[first])


@pytest.mark.parametrize("name", ["cfg4_dsv3", "gptoss_all_default", "a1_qwen_small", "moe_small_all"])
def test_templates_resolve_every_grid_of_a_complete_db(name):
    db, model, workload, space, dc = case_objects(BY_NAME[name])
    plan = build_space_plan(model, space, flatten(db), db.backend)
    assert all(e.grid >= 0 for infos in plan.infos for e in infos)
    # one template per distinct (tp, pp, ep); slots cover every present entry of every step
    assert len({(int(c["tp"]), int(c["pp"]), int(c["ep"])) for c in plan.combos}) == len(plan.infos)
    for t, n in enumerate(plan.tmpl_n):
        for i in range(int(n)):
            coord = int(plan.entries[t * 16 + i]["coord"])
            steps = [s for s in range(3) if plan.slot_of[t, i, s] >= 0]
            assert steps == ([0, 2] if coord == 2 else [1, 2] if coord == 3 else [0, 1, 2])


def _combo_for(plan, cfg_key):
    for c in plan.combos:
        tp, pp, ep, dp = (int(c[k]) for k in ("tp", "pp", "ep", "dp"))
        if cfg_key.startswith(f"tp{tp}pp{pp}ep{ep}dp{dp}b"):
            return c
    raise KeyError(cfg_key)


@pytest.mark.parametrize("name", ["missing_allreduce", "missing_tp16", "unsupported_quant_a100", "strict_long_isl",
                                  "no_chunking", "batch_too_small"])
def test_skip_reasons_format_like_the_reference(name):
    """Rebuild each golden skip reason from the status word the device emits."""
    case = BY_NAME[name]
    db, model, workload, space, dc = case_objects(case)
    flat = flatten(db)
    plan = build_space_plan(model, space, flat, db.backend)
    golden = golden_report(name)["skipped"]
    assert golden
    for sk in golden:
        reason = sk["reason"]
        combo = _combo_for(plan, sk["config"])
        batch = int(sk["config"].rsplit("b", 1)[1])
        kind = reason.split(":", 1)[0]
        if kind == "InfeasibleConfigError":
            code = 4 if "chunking is off" in reason else 5
            got = _reason(code, 0, 0, plan, combo, flat, db, workload, space, batch)
            assert got == reason
            continue
        code = {"MissingKeyError": 1, "ExtrapolationError": 2, "UnsupportedOperatorError": 3}[kind]
        # find the entry whose message matches (labels are unique per template)
        ok = False
        for info in plan.infos[int(combo["tmpl"])]:
            c0 = c1 = 0
            if code == 2:
                coords = reason.split("{", 1)[1].split("}", 1)[0]
                vals = [int(x.split(":")[1]) for x in coords.split(",")]
                c0, c1 = (vals + [0])[:2]
            got = _reason(code | (LABEL_CODE[info.label] << 8), c0, c1, plan, combo, flat, db, workload, space,
                          batch)
            ok |= got == reason
        assert ok, reason


def test_report_document_shape():
    from paper_2601_06288_b200.report import PerfEstimate, SearchReport, estimate_row

    w = pkg.WorkloadSpec(isl=100, osl=10, ttft_limit_ms=50.0, min_speed=1.0)
    cfg = pkg.ParallelConfig(tp=2, batch=4)
    est = PerfEstimate("static", "m", cfg, 10.0, 2.0, 500.0, 123.0, cfg.gpus(), 4)
    row = estimate_row(est)
    rep = SearchReport("m", "trtllm", w, [row], [row], row, [], 1, 1.0, [1.0])
    doc = json.loads(rep.to_json())
    assert doc["counts"] == {"enumerated": 1, "evaluated": 1, "feasible": 1, "frontier": 1, "skipped": 0}
    assert doc["best"]["config"] == "tp2pp1ep1dp1b4"
    assert doc["schema"] == "llmconf-report/1" and doc["version"] == "0.1.0"
    assert set(doc["rows"][0]) == {"mode", "model", "parallel", "batch", "runtime", "gpus", "ttft_ms", "tpot_ms",
                                   "speed", "throughput_per_gpu", "config", "feasible", "frontier"}


def test_spec_validation_mirrors_reference():
    with pytest.raises(pkg.specs.WorkloadError):
        pkg.WorkloadSpec(isl=10, osl=1, min_speed=1.0, tpot_limit_ms=1.0)
    with pytest.raises(pkg.specs.ParallelConfigError):
        pkg.ParallelConfig(tp=0)
    with pytest.raises(pkg.specs.ModelConfigError):
        pkg.ModelSpec.from_doc(dict(model_doc("qwen-small"), kv_heads=7))
    with pytest.raises(pkg.specs.SearchError):
        pkg.run_search(None, None, None, jobs=0)


def test_power_of_two_division_is_an_exact_multiply():
    """The device divides by power-of-two gpu counts (and ceil_div_f divisors) with
    a multiply by 2^-k (GpuDiv, lc_eval.cuh ceil_div_f): both are one correctly
    rounded operation on the same exact value, subnormal results included."""
    import numpy as np

    rng = np.random.default_rng(7)
    bits = rng.integers(0, 2**63 - 1, size=200_000, dtype=np.int64)
    x = bits.view(np.float64)
    x = np.concatenate([x[np.isfinite(x)], -x[np.isfinite(x)][:1000],
                        np.array([0.0, -0.0, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308])])
    for k in (0, 1, 2, 3, 5, 8, 10, 20, 40, 51):
        g = float(2**k)
        inv = float(2.0**-k)
        a = x / g
        b = x * inv
        assert np.array_equal(a.view(np.int64), b.view(np.int64)), k


def test_search_descriptors_one_pass_matches_per_field():
    """Engine.run_batch's one-pass descriptor builder (reusing the last batch-list /
    modes / load lookup across runs of workloads) equals a per-field restatement on
    interleaved workloads: batch lists, modes and MoE load models alternating, limits
    unset or set, duplicated and out-of-order batch sweeps."""
    import types

    from paper_2601_06288_b200 import _native as N
    from paper_2601_06288_b200 import engine as E
    from paper_2601_06288_b200.specs import DEFAULT_MOE_LOAD

    model, space, db = None, pkg.CandidateSpace(batch_values=(8, 1, 32, 0, 2)), None
    L1 = pkg.PowerLawParams(alpha=1.5, x_min=1.0, x_max=50.0, seed=3)
    L2 = pkg.PowerLawParams()
    sw = (64, 4, 4, 1)
    wls = [pkg.WorkloadSpec(isl=4000, osl=500, ttft_limit_ms=5000.0, min_speed=20.0),
           pkg.WorkloadSpec(isl=512, osl=64, tpot_limit_ms=40.0, batch_sweep=sw, moe_load=L1,
                            modes=("aggregated", "disaggregated"), gpu_budgets=(16, 8, 8)),
           pkg.WorkloadSpec(isl=300, osl=7, prefix_len=10),
           pkg.WorkloadSpec(isl=512, osl=64, min_speed=3, batch_sweep=sw, moe_load=L1, modes=("static",)),
           pkg.WorkloadSpec(isl=100, osl=9, batch_sweep=(2, 1), moe_load=L2, modes=("static",)),
           pkg.WorkloadSpec(isl=100, osl=9, ttft_limit_ms=7, batch_sweep=(64, 4, 4, 1), moe_load=L1)]

    class Plan:
        is_moe, n_experts = True, 16

    eng = E.Engine.__new__(E.Engine)
    eng.lib = types.SimpleNamespace(lc_search_batch=None)
    eng.ctx, eng._pinned, eng._deferred = None, (), []
    eng._call = lambda *a: None
    eng.space_handle = lambda d, m, s: (None, Plan, None)
    eng.db_handle = lambda d: (None, None)
    out = eng.run_batch(db, model, space, wls)
    s, batches = out.searches, out.batches.tolist()
    loads_seen: list = []
    for i, w in enumerate(wls):
        bl = tuple(sorted(b for b in (w.batch_sweep or space.batch_values) if b >= 1))
        assert tuple(batches[s["b_off"][i]: s["b_off"][i] + s["n_b"][i]]) == bl
        f = w.speed_floor()
        assert (s["isl"][i], s["osl"][i], s["prefix"][i]) == (w.isl, w.osl, w.prefix_len)
        assert bool(s["has_ttft"][i]) == (w.ttft_limit_ms is not None)
        assert s["ttft_limit"][i] == (float(w.ttft_limit_ms) if w.ttft_limit_ms is not None else 0.0)
        assert bool(s["has_floor"][i]) == (f is not None)
        assert s["speed_floor"][i] == (float(f) if f is not None else 0.0)
        assert s["tpot_cap"][i] == (w.tpot_ceiling() if f is not None else 0.0)
        modes = ((E.MODE_STATIC if "static" in w.modes else 0) | (E.MODE_AGG if "aggregated" in w.modes else 0)
                 | (E.MODE_DISAGG if "disaggregated" in w.modes else 0))
        assert s["modes"][i] == modes
        bud = sorted(set(w.gpu_budgets))
        assert s["n_budgets"][i] == len(bud) and list(s["budgets"][i][: len(bud)]) == bud
        p = w.moe_load if w.moe_load is not None else DEFAULT_MOE_LOAD
        key = (p.alpha, p.x_min, p.x_max, p.seed)
        if key not in loads_seen:
            loads_seen.append(key)
        assert s["load"][i] == loads_seen.index(key)
    # equal batch lists share one copy: (1, 2, 8, 32), (1, 4, 4, 64), (1, 2)
    assert len(batches) == 4 + 4 + 2
    assert s.dtype == N.SEARCH_DESC_DTYPE
