"""How much faster the C restatement (oracle/oracle.c) is than the pure-Python reference.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tools/python_vs_port.py \
        > profiles/r2_python_vs_port.json

Runs in the builder container only (the Python reference does not travel to
the GPU box).  For a few config-5 sweep searches restricted to a slice of batch
sizes it times, on ONE thread of the same host:
  * the unmodified reference: ``llmconf.search.run_search(..., jobs=1)`` with
    ``estimator.clear_caches()`` and ``moe_load._cached_weights.cache_clear()``
    before each search, and
  * the oracle's ``run_search`` on the same inputs,
checks that both produce the same counts, and reports the time ratio.
bench.py quotes the median ratio beside its ``cpu_baseline`` (which times the
oracle) so the figure for the real reference can be read off.
"""

from __future__ import annotations

import gzip
import json
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

from llmconf import estimator, moe_load  # noqa: E402
from llmconf.model import ModelSpec  # noqa: E402
from llmconf.perfdb import load_db  # noqa: E402
from llmconf.search import CandidateSpace, run_search  # noqa: E402
from llmconf.serving_modes import WorkloadSpec  # noqa: E402

from oracle import oracle  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"
PICKS = [  # (model, isl, osl, batch slice)
    ("gpt-oss-120b", 4000, 500, (1, 17)),
    ("deepseek-v3", 4000, 500, (1, 17)),
    ("qwen3-32b", 4000, 500, (1, 33)),
    ("gpt-oss-120b", 1024, 128, (100, 132)),
    ("deepseek-v3", 8192, 1000, (40, 56)),
]


def main() -> None:
    oracle.build()
    rows = []
    for name, isl, osl, (b0, b1) in PICKS:
        dbfile = GOLDEN / "db" / f"db-{name}-h100-sxm-s11.jsonl.gz"
        with tempfile.NamedTemporaryFile("wb", suffix=".jsonl", delete=False) as f:
            f.write(gzip.decompress(dbfile.read_bytes()))
        db = load_db(f.name)
        mdoc = json.loads((GOLDEN / "specs" / f"model-{name}.json").read_text())
        model = ModelSpec.from_doc(mdoc)
        wl = WorkloadSpec(isl=isl, osl=osl, ttft_limit_ms=5000.0, min_speed=20.0)
        batches = tuple(range(b0, b1))
        estimator.clear_caches()
        moe_load._cached_weights.cache_clear()
        t0 = time.perf_counter()
        rep = run_search(db, model, wl, CandidateSpace(batch_values=batches), jobs=1)
        t_py = time.perf_counter() - t0
        header, recs = oracle.read_db_records(dbfile)
        t0 = time.perf_counter()
        doc = oracle.run_search(header, recs, mdoc, wl.to_doc(), {"batch_values": list(batches)})
        t_c = time.perf_counter() - t0
        ref_counts = rep.to_doc()["counts"]
        assert ref_counts == doc["counts"], (ref_counts, doc["counts"])
        rows.append({"model": name, "isl": isl, "osl": osl, "batches": [b0, b1 - 1],
                     "candidates": ref_counts["enumerated"], "python_s": t_py, "port_s": t_c,
                     "factor": t_py / t_c})
        print(rows[-1], file=sys.stderr)
    factors = sorted(r["factor"] for r in rows)
    cpu = "unknown"
    for line in Path("/proc/cpuinfo").read_text().splitlines():
        if line.startswith("model name"):
            cpu = line.split(":", 1)[1].strip()
            break
    print(json.dumps({"how": "same host, one thread each: unmodified Python reference run_search (caches cleared) "
                             "vs oracle/oracle.c on the same searches; counts checked equal",
                      "cpu_model": cpu, "factor_median": factors[len(factors) // 2],
                      "factor_min": factors[0], "factor_max": factors[-1], "searches": rows}, indent=2))


if __name__ == "__main__":
    main()
