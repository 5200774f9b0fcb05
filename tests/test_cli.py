"""CLI entry points (reference cli.py): argument handling, exit codes and
output bytes.  CPU tests cover what is decided before the device runs; -m gpu
tests compare `search` output with the reference's golden reports (all but
`timing`) and `estimate` with the single-config drop-ins."""

from __future__ import annotations

import gzip
import json
import subprocess
import sys
from pathlib import Path

import pytest

from golden_io import BY_NAME, db_path, golden_report

ROOT = Path(__file__).resolve().parents[1]
SPECS = ROOT / "tests" / "golden" / "specs"


def _run(*args, stdin=None):
    return subprocess.run([sys.executable, "-m", "paper_2601_06288_b200", *args], capture_output=True, text=True,
                          cwd=ROOT, input=stdin, timeout=600)


def test_workload_and_space_from_flags():
    from paper_2601_06288_b200.cli import build_parser, space_from_args, workload_from_args
    from paper_2601_06288_b200.specs import CandidateSpace, WorkloadSpec

    args = build_parser().parse_args(
        ["search", "--db", "x", "--model", "m", "--isl", "4000", "--osl", "500", "--ttft-limit", "1200",
         "--min-speed", "60", "--budgets", "8", "--modes", "aggregated", "--pp", "1", "--batches", "1,8",
         "--set", "prefix_len=100", "--kv-mem-fraction", "0.7"])
    assert workload_from_args(args) == WorkloadSpec(isl=4000, osl=500, prefix_len=100, ttft_limit_ms=1200.0,
                                                    min_speed=60.0, gpu_budgets=(8,), modes=("aggregated",),
                                                    batch_sweep=(1, 8))
    assert space_from_args(args) == CandidateSpace(pp_values=(1,), kv_mem_fraction=0.7)


def test_usage_errors_exit_2():
    r = _run("search", "--db", str(db_path(BY_NAME["a1_qwen_small"])), "--model", "nope.json", "--isl", "1",
             "--osl", "1")
    assert r.returncode == 2 and "usage error" in r.stderr
    r = _run("search", "--db", str(db_path(BY_NAME["a1_qwen_small"])), "--model",
             str(SPECS / "model-qwen-small.json"))
    assert r.returncode == 2 and "isl and osl are required" in r.stderr
    r = _run("search", "--model", "m", "--isl", "1", "--osl", "1")
    assert r.returncode == 2 and "--db is required" in r.stderr
    r = _run("search", "--db", "x", "--model", "m", "--tpot-limit", "1", "--min-speed", "2")
    assert r.returncode == 2  # argparse: mutually exclusive


def test_export_csv_and_json(tmp_path):
    from paper_2601_06288_b200.report import csv_from_doc

    doc = golden_report("cfg2_qwen3_disagg")
    doc.pop("_meta")
    p = tmp_path / "r.json"
    p.write_text(json.dumps(doc))
    r = _run("export", "--report", str(p))
    assert r.returncode == 0 and r.stdout == csv_from_doc(doc)
    r = _run("export", "--report", "-", "--format", "json", stdin=json.dumps(doc))
    assert r.returncode == 0 and json.loads(r.stdout) == doc
    p.write_text(json.dumps({"schema": "other"}))
    assert _run("export", "--report", str(p)).returncode == 2


# ------------------------------------------------------------------ on the GPU
CLI_CASES = {
    "cfg1_qwen3_agg": ["--isl", "4000", "--osl", "500", "--ttft-limit", "1200", "--min-speed", "60",
                       "--budgets", "8", "--modes", "aggregated", "--pp", "1"],
    "cfg3_llama70b_kv50": ["--isl", "4000", "--osl", "500", "--ttft-limit", "1200", "--min-speed", "60",
                           "--budgets", "8,16", "--modes", "aggregated,disaggregated", "--kv-mem-fraction", "0.5"],
    "cfg4_dsv3": ["--isl", "5000", "--osl", "1000", "--ttft-limit", "5000", "--min-speed", "20", "--budgets", "8,16"],
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CLI_CASES))
def test_search_stdout_matches_reference_report(name, tmp_path):
    case = BY_NAME[name]
    csv_path = tmp_path / "rows.csv"
    r = _run("search", "--db", str(db_path(case)), "--model", str(SPECS / f"model-{case['model']}.json"),
             *CLI_CASES[name], "--csv", str(csv_path))
    assert r.returncode == 0, r.stderr
    doc = json.loads(r.stdout)
    doc.pop("timing")
    golden = golden_report(name)
    golden.pop("_meta")
    assert json.dumps(doc, sort_keys=True) == json.dumps(golden, sort_keys=True)
    from paper_2601_06288_b200.report import csv_from_doc

    assert csv_path.read_text() == csv_from_doc(golden)


@pytest.mark.gpu
def test_search_without_feasible_config_exits_1():
    case = BY_NAME["a1_qwen_small"]
    r = _run("search", "--db", str(db_path(case)), "--model", str(SPECS / "model-qwen-small.json"),
             "--isl", "512", "--osl", "64", "--min-speed", "1e9", "--tp", "1", "--pp", "1", "--dp", "1")
    assert r.returncode == 1
    assert json.loads(r.stdout)["diagnostics"]["violation_factor"] > 1


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["static", "aggregated"])
def test_estimate_matches_drop_in(mode):
    import paper_2601_06288_b200 as pkg

    case = BY_NAME["cfg4_dsv3"]
    r = _run("estimate", "--db", str(db_path(case)), "--model", str(SPECS / "model-deepseek-v3.json"),
             "--mode", mode, "--isl", "5000", "--osl", "1000", "--tp", "8", "--ep", "8", "--pp", "2",
             "--batch", "64")
    assert r.returncode == 0, r.stderr
    db = pkg.load_db(db_path(case))
    model = pkg.load_model_spec(SPECS / "model-deepseek-v3.json")
    cfg = pkg.ParallelConfig(tp=8, pp=2, ep=8, batch=64, backend=db.backend)
    wl = pkg.WorkloadSpec(isl=5000, osl=1000)
    fn = pkg.estimate_static if mode == "static" else pkg.estimate_aggregated
    want = fn(db, model, cfg, wl).to_doc()
    want["config"] = cfg.key()
    assert json.loads(r.stdout) == want


@pytest.mark.gpu
def test_dbgen_writes_the_reference_database(tmp_path):
    out = tmp_path / "db.jsonl"
    r = _run("dbgen", "--model", str(SPECS / "model-qwen3-32b.json"), "--hardware", str(SPECS / "hw-h100-sxm.json"),
             "--seed", "11", "-o", str(out))
    assert r.returncode == 0, r.stderr
    want = gzip.decompress((ROOT / "tests" / "golden" / "db" / "db-qwen3-32b-h100-sxm-s11.jsonl.gz").read_bytes())
    assert out.read_bytes() == want


@pytest.mark.gpu
def test_estimate_reports_infeasible_config_with_exit_1():
    case = BY_NAME["a1_qwen_small"]
    r = _run("estimate", "--db", str(db_path(case)), "--model", str(SPECS / "model-qwen-small.json"),
             "--isl", "512", "--osl", "64", "--tp", "3", "--batch", "4")
    assert r.returncode == 1 and "does not divide" in r.stderr
