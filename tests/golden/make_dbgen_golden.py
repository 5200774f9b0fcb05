"""Generate synthetic-database golden vectors from the UNMODIFIED reference (survey container only).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_dbgen_golden.py

The committed db/*.jsonl.gz files already pin the default generator settings
(seed 11, amplitude 0.8, default axes).  This adds ``dbgen.json.gz``: reference
``generate_synthetic_db`` (/root/reference/pkg/src/llmconf/perfdb.py:641-666)
latencies for other seeds / amplitudes / custom axes, and the error raised for
hardware that lacks a quant's compute rate.  Latencies are float hex strings in
the reference's record order (sorted by kind, quant, shape).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from make_golden import hw, model, write_gz  # noqa: E402

from llmconf.model import grid_spec_for_model  # noqa: E402
from llmconf.perfdb import generate_synthetic_db  # noqa: E402

DENSE = {"gemm": (("m", tuple(sorted({round(2 ** (i / 4)) for i in range(0, 61)}))),),
         "attention_generation": (("batch", (1, 2, 3, 5, 8, 13, 21, 34, 55, 89, 144, 233, 377, 610, 987)),
                                  ("seq_len", tuple(range(16, 131073, 4096)) + (131072,)))}

CASES = [
    dict(name="qwen_seed5_amp0", model="qwen-small", hw="h100-sxm", seed=5, amplitude=0.0),
    dict(name="moe_seed123_amp037", model="moe-small", hw="h100-sxm", seed=123, amplitude=0.37),
    dict(name="llama_b200_seed7", model="llama-3.1-70b", hw="b200-sxm", seed=7, amplitude=0.8),
    dict(name="qwen_dense_axes", model="qwen-small", hw="h100-sxm", seed=11, amplitude=0.8, axes="dense"),
    dict(name="qwen_a100_unsupported", model="qwen-small", hw="a100-sxm", seed=11, amplitude=0.8),
]


def main() -> None:
    out = []
    for c in CASES:
        kw = {"axes": DENSE} if c.get("axes") == "dense" else {}
        spec = grid_spec_for_model(model(c["model"]), **kw)
        rec = dict(c)
        try:
            db = generate_synthetic_db(hw(c["hw"]), spec, seed=c["seed"], efficiency_amplitude=c["amplitude"])
            rec["latency"] = [r.latency_us.hex() for r in db.records]
            rec["n_grids"] = len(db._grids)
        except Exception as e:  # noqa: BLE001 - the reference's error is the expectation
            rec["error"] = f"{type(e).__name__}: {e}"
        out.append(rec)
        print(c["name"], rec.get("n_grids"), len(rec.get("latency", [])), rec.get("error", ""))
    doc = {"dense_axes": {k: [[a, list(v)] for a, v in axes] for k, axes in DENSE.items()}, "cases": out}
    write_gz(HERE / "dbgen.json.gz", json.dumps(doc, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
