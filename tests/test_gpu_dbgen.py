"""Device database generation (lc_dbgen / k_dbgen) against the reference's
generate_synthetic_db output, and searches over generated databases, including
one too large for shared-memory staging (global-memory path)."""

from __future__ import annotations

import gzip
import json

import numpy as np
import pytest

from golden_io import BY_NAME, GOLDEN, canonical, diff_canonical, golden_report, hw_doc, model_doc
from test_dbgen_host import DBS, split_name

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2601_06288_b200 as pkg

    return pkg


@pytest.mark.parametrize("name", DBS)
def test_generated_database_bytes_equal_reference_file(name, tmp_path):
    pkg = _pkg()
    model_name, hw_name = split_name(name)
    spec = pkg.grid_spec_for_model(pkg.ModelSpec.from_doc(model_doc(model_name)))
    db = pkg.generate_synthetic_db(pkg.HardwareSpec.from_doc(hw_doc(hw_name)), spec, seed=11)
    pkg.save_db(db, tmp_path / "out.jsonl")
    want = gzip.decompress((GOLDEN / "db" / name).read_bytes())
    assert (tmp_path / "out.jsonl").read_bytes() == want


def test_device_image_equals_host_flatten():
    pkg = _pkg()
    from paper_2601_06288_b200.database import flatten

    spec = pkg.grid_spec_for_model(pkg.ModelSpec.from_doc(model_doc("deepseek-v3")))
    hw = pkg.HardwareSpec.from_doc(hw_doc("b200-sxm"))
    gen = pkg.generate_synthetic_db(hw, spec, seed=11, lazy=True)
    dev = flatten(gen)
    host = flatten(pkg.PerfDatabase.from_records(hw, "trtllm", "synthetic", gen.records))
    assert dev.keys == host.keys and dev.axes == host.axes and dev.axis_values == host.axis_values
    for f in ("grid_ndim", "grid_axis_off", "grid_axis_len", "grid_cell_off", "axis_val"):
        assert np.array_equal(getattr(dev, f), getattr(host, f)), f
    for f in ("axis_log", "cell", "cell_log"):
        assert getattr(dev, f).view(np.uint64).tolist() == getattr(host, f).view(np.uint64).tolist(), f


def _golden_cases():
    return json.loads(gzip.decompress((GOLDEN / "dbgen.json.gz").read_bytes()))


@pytest.mark.parametrize("case", [c["name"] for c in _golden_cases()["cases"]])
def test_generator_options_match_reference(case):
    pkg = _pkg()
    from paper_2601_06288_b200.specs import UnsupportedOperatorError

    doc = _golden_cases()
    c = next(x for x in doc["cases"] if x["name"] == case)
    axes = None
    if c.get("axes") == "dense":
        axes = {k: tuple((a, tuple(v)) for a, v in ax) for k, ax in doc["dense_axes"].items()}
    spec = pkg.grid_spec_for_model(pkg.ModelSpec.from_doc(model_doc(c["model"])), axes=axes)
    hw = pkg.HardwareSpec.from_doc(hw_doc(c["hw"]))
    if "error" in c:
        with pytest.raises(UnsupportedOperatorError) as ei:
            pkg.generate_synthetic_db(hw, spec, seed=c["seed"], efficiency_amplitude=c["amplitude"])
        assert f"UnsupportedOperatorError: {ei.value}" == c["error"]
        return
    db = pkg.generate_synthetic_db(hw, spec, seed=c["seed"], efficiency_amplitude=c["amplitude"])
    assert [r.latency_us.hex() for r in db.records] == c["latency"]
    assert len(db._grids) == c["n_grids"]


def test_search_over_lazy_generated_database_matches_golden_report():
    pkg = _pkg()
    from product_cases import case_objects

    case = BY_NAME["a1_qwen_small"]
    _, model, workload, space, dc = case_objects(case)
    spec = pkg.grid_spec_for_model(model)
    db = pkg.generate_synthetic_db(pkg.HardwareSpec.from_doc(hw_doc("h100-sxm")), spec, seed=11, lazy=True)
    doc = pkg.run_search(db, model, workload, space, disagg_constants=dc).to_doc()
    doc.pop("timing", None)
    diffs = diff_canonical(canonical(doc), canonical(golden_report(case["name"])))
    assert not diffs, "\n".join(diffs[:20])


def test_search_over_database_too_large_for_shared_memory():
    """Denser axes than the defaults push the image past the 200 KB staging budget;
    the table kernels then read it from global memory.  Checked against the oracle."""
    pkg = _pkg()
    from oracle import oracle
    from paper_2601_06288_b200.database import flatten

    model = pkg.ModelSpec.from_doc(model_doc("qwen-small"))
    axes = {"attention_generation": (("batch", tuple(range(1, 1025, 24))), ("seq_len", tuple(range(16, 140000, 2048)))),
            "gemm": (("m", tuple(range(1, 40000, 97))),)}
    spec = pkg.grid_spec_for_model(model, axes=axes)
    hw = pkg.HardwareSpec.from_doc(hw_doc("h100-sxm"))
    db = pkg.generate_synthetic_db(hw, spec, seed=3, lazy=True)
    flat = flatten(db)
    assert len(flat.cell) * 16 > 200 * 1024, len(flat.cell)
    workload = pkg.WorkloadSpec.from_doc({"isl": 3000, "osl": 700, "ttft_limit_ms": 4000.0, "min_speed": 15.0})
    space = pkg.CandidateSpace(batch_values=(1, 3, 8, 24, 64, 200, 512))
    doc = pkg.run_search(db, model, workload, space).to_doc()
    header = {"schema": "llmconf-perfdb/1", "hardware": hw.to_doc(), "backend": db.backend,
              "backend_version": db.backend_version}
    recs = [r.to_doc() for r in db.records]
    ref = oracle.run_search(header, recs, model_doc("qwen-small"), workload.to_doc(),
                            {"batch_values": list(space.batch_values)})
    doc.pop("timing", None)
    diffs = diff_canonical(canonical(doc), canonical(ref))
    assert not diffs, "\n".join(diffs[:20])


def test_search_over_soa_loaded_database_matches_golden_report(tmp_path):
    """A database mapped from the binary cache searches without materialising records."""
    pkg = _pkg()
    from paper_2601_06288_b200.soa import FlatBackedDatabase, load_soa, save_soa
    from product_cases import case_db, case_objects

    case = BY_NAME["cfg4_dsv3"]
    _, model, workload, space, dc = case_objects(case)
    save_soa(case_db(case), tmp_path / "db.npz")
    db = load_soa(tmp_path / "db.npz", extrapolation=case.get("extrapolation", "default"))
    assert isinstance(db, FlatBackedDatabase)
    doc = pkg.run_search(db, model, workload, space, disagg_constants=dc).to_doc()
    assert db._recs is None  # the search never built per-record objects
    diffs = diff_canonical(canonical(doc), canonical(golden_report(case["name"])))
    assert not diffs, "\n".join(diffs[:20])
