"""Throughput of device database generation at measured scale (GPU box).

    python tools/dbgen_bench.py [--scale 256]

Builds DeepSeek-V3's grid spec with every default axis densified ``scale``-fold
(log-spaced integer values between the default end points), generates it with
``generate_synthetic_db(lazy=True)`` (host hash terms + k_dbgen + D2H + image
assembly) and prints cells/s.  The reference's pure-Python generator runs at
~26K records/s on this image's CPU (1,390 DeepSeek-V3 records in 54 ms,
measured in the survey container); ``--cpu-sample`` times the same generator
restated on the host here for comparison.
"""

from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def dense_axes(scale: int) -> dict:
    from paper_2601_06288_b200.dbgen import DEFAULT_AXES

    out = {}
    for kind, axes in DEFAULT_AXES.items():
        new = []
        for name, vals in axes:
            lo, hi = math.log(vals[0]), math.log(vals[-1])
            n = (len(vals) - 1) * scale + 1
            v = sorted({max(1, round(math.exp(lo + (hi - lo) * i / (n - 1)))) for i in range(n)} | set(vals))
            new.append((name, tuple(v)))
        out[kind] = tuple(new)
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import paper_2601_06288_b200 as pkg
    from golden_io import hw_doc, model_doc

    model = pkg.ModelSpec.from_doc(model_doc("deepseek-v3"))
    hw = pkg.HardwareSpec.from_doc(hw_doc("h100-sxm"))
    spec = pkg.grid_spec_for_model(model, axes=dense_axes(args.scale))
    cells = sum(g.n_cells() for g in spec)
    pkg.generate_synthetic_db(hw, pkg.grid_spec_for_model(model), seed=11, lazy=True)  # warm-up / context
    best = None
    for _ in range(args.reps):
        t = time.perf_counter()
        db = pkg.generate_synthetic_db(hw, spec, seed=11, lazy=True)
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    from paper_2601_06288_b200.database import flatten

    flat = flatten(db)
    print(json.dumps({"tool": "dbgen_bench", "model": "deepseek-v3", "scale": args.scale, "grids": len(spec),
                      "cells": cells, "seconds": best, "cells_per_s": cells / best,
                      "image_bytes": int(flat.cell.nbytes * 2 + flat.axis_val.nbytes * 2),
                      "reference_python_records_per_s": 25833.5,
                      "reference_note": "reference generate_synthetic_db, 1390 records in 53.8 ms (survey container)"}))


if __name__ == "__main__":
    main()
