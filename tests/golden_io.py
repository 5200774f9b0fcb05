"""Fixture loading and report canonicalisation shared by the parity tests."""

from __future__ import annotations

import gzip
import json
import math
import sys
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLDEN))

from cases import BY_NAME, CASES, case_db_key, db_file  # noqa: E402,F401

SPECS = GOLDEN / "specs"


def read_json(name: str) -> dict:
    return json.loads((SPECS / name).read_text())


def model_doc(name: str) -> dict:
    return read_json(f"model-{name}.json")


def hw_doc(name: str) -> dict:
    return read_json(f"hw-{name}.json")


def hw_docs() -> dict:
    return {p.stem.removeprefix("hw-"): json.loads(p.read_text()) for p in SPECS.glob("hw-*.json")}


def db_path(case: dict) -> Path:
    m, h = case_db_key(case)
    return GOLDEN / "db" / db_file(m, h)


def golden_report(name: str) -> dict:
    return json.loads(gzip.decompress((GOLDEN / "reports" / f"{name}.json.gz").read_bytes()))


def moe_kats() -> list[dict]:
    return json.loads(gzip.decompress((GOLDEN / "moe" / "apportion.json.gz").read_bytes()))


def sum_kats() -> list[dict]:
    return json.loads(gzip.decompress((GOLDEN / "sums.json.gz").read_bytes()))


def _f(x):
    """Exact float identity (hex), None for null (infinite speed)."""
    if x is None:
        return None
    return float(x).hex()


def _row(r: dict) -> tuple:
    base = (r["mode"], r["config"], r["gpus"], _f(r["ttft_ms"]), _f(r["tpot_ms"]), _f(r["speed"]),
            _f(r["throughput_per_gpu"]), r["feasible"], r["frontier"])
    if r["mode"] == "disaggregated":
        base += (_f(r["r_sys"]), r["prefill"]["replicas"], r["decode"]["replicas"])
    else:
        base += (r["batch"], r["parallel"]["tp"], r["parallel"]["pp"], r["parallel"]["ep"], r["parallel"]["dp"])
    return base


def canonical(doc: dict) -> dict:
    """The parity-relevant content of a report document, floats as exact hex."""
    best = doc["best"]
    diag = doc.get("diagnostics")
    return {
        "counts": doc["counts"],
        "rows": [_row(r) for r in doc["rows"]],
        "frontier": [(r["mode"], r["config"]) for r in doc["frontier"]],
        "best": None if best is None else (best["mode"], best["config"]),
        "diagnostics": None if diag is None else (diag["mode"], diag["config"], _f(diag["violation_factor"])),
        "skipped": [(s["mode"], s["config"], s["reason"]) for s in doc["skipped"]],
    }


def diff_canonical(a: dict, b: dict, limit: int = 8) -> list[str]:
    out = []
    for key in ("counts", "best", "diagnostics"):
        if a[key] != b[key]:
            out.append(f"{key}: {a[key]} != {b[key]}")
    for key in ("rows", "frontier", "skipped"):
        xa, xb = a[key], b[key]
        if len(xa) != len(xb):
            out.append(f"{key}: length {len(xa)} != {len(xb)}")
        for i, (u, v) in enumerate(zip(xa, xb)):
            if u != v:
                out.append(f"{key}[{i}]: {u} != {v}")
                if len(out) >= limit:
                    return out
    return out


def max_rel_err(a: dict, b: dict) -> float:
    """Largest relative difference over the per-row latencies/metrics of two docs."""
    worst = 0.0
    for ra, rb in zip(a["rows"], b["rows"]):
        for k in ("ttft_ms", "tpot_ms", "speed", "throughput_per_gpu"):
            x, y = ra[k], rb[k]
            if x is None or y is None:
                if x != y:
                    return math.inf
                continue
            if x != y:
                worst = max(worst, abs(x - y) / max(abs(x), abs(y)))
    return worst


def query_goldens() -> dict:
    """Single-query vectors from the reference (tests/golden/make_query_golden.py)."""
    return json.loads(gzip.decompress((GOLDEN / "queries.json.gz").read_bytes()))


def query_groups(doc: dict) -> dict:
    """Vectors grouped by (database, policy), in file order."""
    groups: dict = {}
    for v in doc["vectors"]:
        groups.setdefault((v["db"], v["policy"]), []).append(v)
    return groups
