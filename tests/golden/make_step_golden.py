"""Golden vectors for the step-latency breakdown (builder container only).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_step_golden.py

Runs the UNMODIFIED reference ``llmconf.estimator.get_step_latency``
(/root/reference/pkg/src/llmconf/estimator.py:71-110) over seeded requests --
every model, prefill / decode / mixed steps, consistent and inconsistent
configs, default and custom MoE loads, extrapolation policies, a database
missing a kind and one whose hardware lacks a quant rate -- and writes
``steps.json.gz`` next to this file: per request the total and the per-label
breakdown as exact float hex, or the exception ``"Type: message"``.
"""

from __future__ import annotations

import gzip
import io
import json
import random
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from llmconf import estimator  # noqa: E402
from llmconf.model import ModelSpec  # noqa: E402
from llmconf.moe_load import PowerLawParams  # noqa: E402
from llmconf.perfdb import HardwareSpec, PerfDatabase, load_db  # noqa: E402
from llmconf.search import CandidateSpace  # noqa: E402

MODELS = ("qwen-small", "moe-small", "qwen3-32b", "deepseek-v3", "gpt-oss-120b", "llama-3.1-70b")
DBS = [  # (model, extrapolation, mutation)
    *[(m, "default", None) for m in MODELS],
    ("qwen-small", "strict", None), ("qwen-small", "clamp", None), ("qwen-small", "sol", None),
    ("deepseek-v3", "strict", None), ("gpt-oss-120b", "sol", None),
    ("qwen3-32b", "default", "drop_kind:allreduce"), ("deepseek-v3", "default", "drop_kind:moe_dispatch"),
    ("gpt-oss-120b", "default", "swap_hw:a100-sxm"),
]


def write_gz(path: Path, text: str) -> None:
    buf = io.BytesIO()
    with gzip.GzipFile(fileobj=buf, mode="wb", mtime=0) as f:
        f.write(text.encode())
    path.write_bytes(buf.getvalue())


def load(model: str, extrapolation: str, mutation: str | None) -> PerfDatabase:
    src = HERE / "db" / f"db-{model}-h100-sxm-s11.jsonl.gz"
    with tempfile.NamedTemporaryFile("wb", suffix=".jsonl", delete=False) as f:
        f.write(gzip.decompress(src.read_bytes()))
    db = load_db(f.name, extrapolation=extrapolation)
    if mutation is None:
        return db
    records, hardware = list(db.records), db.hardware
    if mutation.startswith("drop_kind:"):
        kind = mutation.split(":", 1)[1]
        records = [r for r in records if r.query.kind != kind]
    elif mutation.startswith("swap_hw:"):
        hardware = HardwareSpec.from_doc(json.loads((HERE / "specs" / f"hw-{mutation.split(':', 1)[1]}.json")
                                                    .read_text()))
    return PerfDatabase.from_records(hardware, db.backend, db.backend_version, records, db.extrapolation)


def main() -> None:
    rng = random.Random(20260117)
    out = []
    for model_name, extrapolation, mutation in DBS:
        db = load(model_name, extrapolation, mutation)
        mdoc = json.loads((HERE / "specs" / f"model-{model_name}.json").read_text())
        model = ModelSpec.from_doc(mdoc)
        space = CandidateSpace()
        n = 120 if mutation is None and extrapolation == "default" else 30
        for _ in range(n):
            tp = rng.choice([1, 2, 4, 8, 3])
            pp = rng.choice([1, 2, 4])
            ep = rng.choice([1, 2, 4, 8]) if model.moe else 1
            dp = rng.choice([1, 2, 4, 8])
            batch = rng.choice([1, 2, 7, 32, 64, 256, 512])
            cfg = space.config(tp, pp, ep, dp, batch, db.backend)
            phase = rng.choice(["prefill", "decode", "mixed", "mixed", "decode", "bogus"] if rng.random() < 0.03
                               else ["prefill", "decode", "mixed"])
            seq = rng.choice([1, 7, 128, 512, 4000, 5250, 16384, 70000, 200000])
            if phase == "prefill":
                n_ctx, n_gen = batch * seq, 0
                if rng.random() < 0.05:
                    n_ctx += 1  # not a multiple of seq_len
            elif phase == "decode":
                n_ctx, n_gen = 0, rng.choice([batch, 1, 3, 97])
            else:
                n_ctx, n_gen = rng.choice([1, 512, 2048, 4000, 8192]), rng.choice([0, 1, batch, 63])
            load_params = None
            if model.moe and rng.random() < 0.3:
                load_params = PowerLawParams(alpha=rng.choice([0.5, 1.2, 1.9]), x_max=rng.choice([50.0, 100.0]),
                                             seed=rng.randint(0, 9))
            rec = {"model": model_name, "extrapolation": extrapolation, "mutation": mutation,
                   "cfg": [tp, pp, ep, dp, batch], "phase": phase, "n_ctx": n_ctx, "n_gen": n_gen, "seq": seq,
                   "moe_load": None if load_params is None else
                   {"alpha": load_params.alpha, "x_min": load_params.x_min, "x_max": load_params.x_max,
                    "seed": load_params.seed}}
            estimator.clear_caches()
            try:
                st = estimator.get_step_latency(db, model, cfg, phase, n_ctx_tokens=n_ctx, n_gen_tokens=n_gen,
                                                seq_len=seq, moe_load=load_params)
                rec["total"] = st.total_ms.hex()
                rec["breakdown"] = [[k, v.hex()] for k, v in st.breakdown.items()]
            except Exception as e:  # noqa: BLE001 -- the reference's exception is the expected answer
                rec["error"] = f"{type(e).__name__}: {e}"
            out.append(rec)
    write_gz(HERE / "steps.json.gz", json.dumps({"requests": out}, sort_keys=True) + "\n")
    errs = sum("error" in r for r in out)
    print(f"{len(out)} step requests, {errs} raise")


if __name__ == "__main__":
    main()
