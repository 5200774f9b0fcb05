"""Named benchmark sweeps (BASELINE.json configs).

``config5`` is the headline: a dense synthetic sweep of >= 10^7 candidates
over parallelism x batch x ISL/OSL for GPT-OSS-120B + DeepSeek-V3 (10,303,947
candidates with batch 1..512, default tp/pp/ep/dp, all serving modes,
TTFT <= 5 s, speed >= 20 tok/s, one synthetic H100 database per model).
``config5_qwen`` is the north-star variant (Qwen3-32B + DeepSeek-V3).
Databases and model specs are the committed fixtures under tests/golden.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

from .database import load_db
from .specs import CandidateSpace, ModelSpec, WorkloadSpec

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"

ISL = (512, 1024, 2048, 3072, 4000, 5000, 6144, 8192, 12288, 16384)
OSL = (64, 128, 256, 500, 750, 1000, 1024, 1536, 2048, 4096)
OSL_QWEN = OSL + (96, 192, 384, 640, 896, 1280, 1792, 2560, 3072, 3584, 5120, 6144)


@dataclass
class SweepPart:
    model_name: str
    db: object
    model: ModelSpec
    space: CandidateSpace
    workloads: list


def _model(name: str) -> ModelSpec:
    return ModelSpec.from_doc(json.loads((GOLDEN / "specs" / f"model-{name}.json").read_text()))


def _db(name: str, hw: str = "h100-sxm"):
    return load_db(GOLDEN / "db" / f"db-{name}-{hw}-s11.jsonl.gz")


def sweep(name: str = "config5") -> list[SweepPart]:
    if name == "config5":
        models, isl, osl = ("gpt-oss-120b", "deepseek-v3"), ISL, OSL
    elif name == "config5_qwen":
        models, isl, osl = ("qwen3-32b", "deepseek-v3"), ISL, OSL_QWEN
    elif name == "smoke":
        models, isl, osl = ("gpt-oss-120b", "deepseek-v3"), ISL[:2], OSL[:2]
    else:
        raise KeyError(name)
    space = CandidateSpace(batch_values=tuple(range(1, 513)))
    parts = []
    for m in models:
        wls = [WorkloadSpec(isl=i, osl=o, ttft_limit_ms=5000.0, min_speed=20.0) for i in isl for o in osl]
        parts.append(SweepPart(m, _db(m), _model(m), space, wls))
    return parts
