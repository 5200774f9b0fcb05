"""Generate the golden fixtures from the UNMODIFIED reference (survey container only).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes, next to this file:
  db/db-<model>-<hw>-s11.jsonl.gz   reference ``generate_synthetic_db`` + ``save_db``
                                    (/root/reference/pkg/src/llmconf/perfdb.py:414-425, 641-666)
  reports/<case>.json.gz            reference ``run_search(...).to_doc()`` minus ``timing``
                                    (/root/reference/pkg/src/llmconf/search.py:224-264, 280-358)
  moe/apportion.json.gz             reference ``tokens_per_expert`` / ``busiest_shard_tokens`` KATs
                                    (/root/reference/pkg/src/llmconf/moe_load.py:67-147)
  sums.json.gz                      CPython 3.12 ``sum()`` of float lists (Neumaier) KATs

The reference cannot travel to the GPU box, so these committed files are what
the oracle and the CUDA path are pinned against there.  Floats survive the
JSON round trip exactly (``repr`` is shortest round-trip).
"""

from __future__ import annotations

import gzip
import io
import json
import random
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from cases import CASES, DB_SEED, case_db_key, db_file  # noqa: E402

from llmconf import estimator, moe_load  # noqa: E402
from llmconf.model import ModelSpec, grid_spec_for_model  # noqa: E402
from llmconf.perfdb import (  # noqa: E402
    HardwareSpec,
    OperatorRecord,
    PerfDatabase,
    generate_synthetic_db,
    load_db,
    save_db,
)
from llmconf.search import CandidateSpace, run_search  # noqa: E402
from llmconf.serving_modes import DisaggConstants, WorkloadSpec  # noqa: E402

SPECS = HERE / "specs"


def write_gz(path: Path, text: str) -> None:
    path.parent.mkdir(parents=True, exist_ok=True)
    buf = io.BytesIO()
    with gzip.GzipFile(fileobj=buf, mode="wb", mtime=0) as f:
        f.write(text.encode())
    path.write_bytes(buf.getvalue())


def model(name: str) -> ModelSpec:
    return ModelSpec.from_doc(json.loads((SPECS / f"model-{name}.json").read_text()))


def hw(name: str) -> HardwareSpec:
    return HardwareSpec.from_doc(json.loads((SPECS / f"hw-{name}.json").read_text()))


def make_dbs() -> None:
    keys = sorted({case_db_key(c) for c in CASES})
    for m, h in keys:
        out = HERE / "db" / db_file(m, h)
        db = generate_synthetic_db(hw(h), grid_spec_for_model(model(m)), seed=DB_SEED)
        tmp = Path("/tmp") / db_file(m, h).removesuffix(".gz")
        save_db(db, tmp)
        write_gz(out, tmp.read_text())
        print(f"db {out.name}: {len(db.records)} records, {len(db._grids)} grids")


def load_case_db(case: dict) -> PerfDatabase:
    m, h = case_db_key(case)
    tmp = Path("/tmp") / db_file(m, h).removesuffix(".gz")
    tmp.write_bytes(gzip.decompress((HERE / "db" / db_file(m, h)).read_bytes()))
    db = load_db(tmp, extrapolation=case.get("extrapolation", "default"))
    mut = case.get("mutation")
    if mut is None:
        return db
    records = list(db.records)
    hardware = db.hardware
    if mut == "flat":
        records = [OperatorRecord(r.query, 100.0, "synthetic") for r in records]
    elif mut.startswith("swap_hw:"):
        hardware = hw(mut.split(":", 1)[1])
    elif mut.startswith("drop_kind:"):
        kind = mut.split(":", 1)[1]
        records = [r for r in records if r.query.kind != kind]
    else:
        raise ValueError(mut)
    return PerfDatabase.from_records(hardware, db.backend, db.backend_version, records, db.extrapolation)


def case_objects(case: dict):
    wl = WorkloadSpec.from_doc(dict(case["workload"]))
    sp = {k: tuple(v) if isinstance(v, list) else v for k, v in case.get("space", {}).items()}
    space = CandidateSpace(**sp)
    dc = DisaggConstants(**case["disagg"]) if case.get("disagg") else DisaggConstants()
    return wl, space, dc


def make_reports() -> None:
    for case in CASES:
        db = load_case_db(case)
        wl, space, dc = case_objects(case)
        estimator.clear_caches()
        moe_load._cached_weights.cache_clear()
        t0 = time.perf_counter()
        report = run_search(db, model(case["model"]), wl, space, jobs=1, disagg_constants=dc)
        dt = time.perf_counter() - t0
        doc = report.to_doc()
        doc.pop("timing")
        doc["_meta"] = {"case": case["name"], "reference_wall_s": round(dt, 4)}
        write_gz(HERE / "reports" / f"{case['name']}.json.gz",
                 json.dumps(doc, sort_keys=True, allow_nan=False) + "\n")
        c = doc["counts"]
        best = doc["best"]["config"] if doc["best"] else None
        print(f"{case['name']}: {c} best={best} {dt:.3f}s")


def make_moe_kats() -> None:
    rng = random.Random(5)
    kats = []
    for params in (moe_load.PowerLawParams(), moe_load.PowerLawParams(alpha=0.5, x_max=1000.0, seed=3),
                   moe_load.PowerLawParams(alpha=1.9, seed=17), moe_load.PowerLawParams(alpha=0.0, x_max=2.0, seed=9)):
        for num in (8, 32, 128, 256):
            w = moe_load.sample_weights(params, num)
            for _ in range(12):
                topk = rng.choice([1, 2, 4, 8, num])
                topk = min(topk, num)
                total = rng.choice([0, 1, 2, 3, 7, 64, 513, 4096, 123457, 8 * 4000 * 64, rng.randint(1, 10**7)])
                eps = [e for e in (1, 2, 4, 8, 16, 32) if num % e == 0]
                ep = rng.choice(eps)
                counts = moe_load.tokens_per_expert(w, total, topk)
                kats.append({
                    "alpha": params.alpha, "x_min": params.x_min, "x_max": params.x_max, "seed": params.seed,
                    "num_experts": num, "total": total, "topk": topk, "ep": ep,
                    "weights": [float(x) for x in w], "counts": [int(x) for x in counts],
                    "busiest": moe_load.busiest_shard_tokens(params, num, total, topk, ep),
                })
    write_gz(HERE / "moe" / "apportion.json.gz", json.dumps(kats) + "\n")
    print(f"moe kats: {len(kats)}")


def make_sum_kats() -> None:
    rng = random.Random(9)
    kats = []
    for _ in range(4000):
        n = rng.randint(1, 20)
        kind = rng.random()
        if kind < 0.3:
            xs = [rng.uniform(0.0, 10.0) * 10 ** rng.randint(-6, 6) for _ in range(n)]
        elif kind < 0.6:
            xs = [rng.uniform(-1.0, 1.0) * 10 ** rng.randint(-3, 3) for _ in range(n)]
        else:
            xs = [rng.choice([1e16, -1e16, 1.0, 0.1, -0.3, 3.0e-17, 1e308]) for _ in range(n)]
        s = sum(xs)
        kats.append({"xs": [x.hex() for x in xs], "sum": s.hex()})
    write_gz(HERE / "sums.json.gz", json.dumps(kats) + "\n")
    print(f"sum kats: {len(kats)}")


if __name__ == "__main__":
    what = sys.argv[1:] or ["dbs", "reports", "moe", "sums"]
    if "dbs" in what:
        make_dbs()
    if "reports" in what:
        make_reports()
    if "moe" in what:
        make_moe_kats()
    if "sums" in what:
        make_sum_kats()
