"""Result objects of a search and their canonical documents.

The document forms (field names, order-insensitive JSON with ``sort_keys``,
``indent=2``, ``allow_nan=False``) reproduce the reference byte for byte:
PerfEstimate / DisaggPlan / ResultRow / SearchReport at
/root/reference/pkg/src/llmconf/serving_modes.py:175-218, 384-426 and
search.py:116-153, 211-264, 361-390.  Values come from the device; nothing
here recomputes the model.
"""

from __future__ import annotations

import json
import math
import statistics
from dataclasses import dataclass
from typing import Mapping, Sequence

REPORT_SCHEMA = "llmconf-report/1"
# version field of the report document; matches the reference package's __version__
# (/root/reference/pkg/src/llmconf/__init__.py:3) so reports stay byte-identical
REPORT_VERSION = "0.1.0"


def _runtime_doc(cfg) -> dict:
    return {"ctx_capacity": cfg.ctx_capacity, "chunked_prefill": cfg.chunked_prefill,
            "kv_mem_fraction": cfg.kv_mem_fraction, "cuda_graph": cfg.cuda_graph, "backend": cfg.backend}


def _parallel_doc(cfg) -> dict:
    return {"tp": cfg.tp, "pp": cfg.pp, "ep": cfg.ep, "dp": cfg.dp}


@dataclass(frozen=True)
class PerfEstimate:
    mode: str
    model_name: str
    cfg: object
    ttft_ms: float
    tpot_ms: float
    speed: float
    throughput_per_gpu: float
    gpus: int
    batch: int

    def meets_sla(self, workload) -> bool:
        return _meets(workload, self.ttft_ms, self.speed)

    def to_doc(self) -> dict:
        return {
            "mode": self.mode, "model": self.model_name, "parallel": _parallel_doc(self.cfg), "batch": self.batch,
            "runtime": _runtime_doc(self.cfg), "gpus": self.gpus, "ttft_ms": self.ttft_ms, "tpot_ms": self.tpot_ms,
            "speed": self.speed if math.isfinite(self.speed) else None,
            "throughput_per_gpu": self.throughput_per_gpu,
        }


@dataclass(frozen=True)
class PoolCandidate:
    role: str
    cfg: object
    latency_ms: float
    seq_rate: float
    gpus: int


@dataclass(frozen=True)
class DisaggPlan:
    prefill: PoolCandidate
    decode: PoolCandidate
    x: int
    y: int
    gpus: int
    r_sys: float
    ttft_ms: float
    tpot_ms: float
    speed: float
    throughput_per_gpu: float

    def to_doc(self) -> dict:
        def side(c: PoolCandidate, n: int) -> dict:
            return {"replicas": n, "parallel": _parallel_doc(c.cfg), "batch": c.cfg.batch,
                    "runtime": _runtime_doc(c.cfg)}

        return {
            "mode": "disaggregated", "prefill": side(self.prefill, self.x), "decode": side(self.decode, self.y),
            "gpus": self.gpus, "r_sys": self.r_sys, "ttft_ms": self.ttft_ms, "tpot_ms": self.tpot_ms,
            "speed": self.speed if math.isfinite(self.speed) else None,
            "throughput_per_gpu": self.throughput_per_gpu,
        }


def _meets(workload, ttft: float, speed: float) -> bool:
    if workload.ttft_limit_ms is not None and ttft > workload.ttft_limit_ms:
        return False
    floor = workload.speed_floor()
    return floor is None or speed >= floor


@dataclass(frozen=True)
class ResultRow:
    mode: str
    config_label: str
    speed: float
    throughput_per_gpu: float
    ttft_ms: float
    tpot_ms: float
    gpus: int
    detail: object

    def meets_sla(self, workload) -> bool:
        return _meets(workload, self.ttft_ms, self.speed)

    def to_doc(self) -> dict:
        doc = self.detail.to_doc()
        doc["config"] = self.config_label
        return doc


def estimate_row(est: PerfEstimate) -> ResultRow:
    return ResultRow(est.mode, est.cfg.key(), est.speed, est.throughput_per_gpu, est.ttft_ms, est.tpot_ms,
                     est.gpus, est)


def plan_row(plan: DisaggPlan) -> ResultRow:
    label = f"P:{plan.x}x{plan.prefill.cfg.key()}|D:{plan.y}x{plan.decode.cfg.key()}"
    return ResultRow("disaggregated", label, plan.speed, plan.throughput_per_gpu, plan.ttft_ms, plan.tpot_ms,
                     plan.gpus, plan)


def violation(row, workload) -> float:
    worst = 1.0
    if workload.ttft_limit_ms is not None and row.ttft_ms > workload.ttft_limit_ms:
        worst = max(worst, row.ttft_ms / workload.ttft_limit_ms)
    floor = workload.speed_floor()
    if floor is not None and row.speed < floor:
        worst = max(worst, math.inf if row.speed == 0 else floor / row.speed)
    return worst


def nearest_miss_doc(row, workload) -> dict | None:
    if row is None:
        return None
    doc = row.to_doc()
    worst = violation(row, workload)
    doc["violation_factor"] = worst if math.isfinite(worst) else None
    return doc


@dataclass
class SearchReport:
    model: str
    backend: str
    workload: object
    rows: list
    frontier: list
    best: object
    skipped: list
    enumerated: int
    total_ms: float
    per_candidate_ms: list
    nearest: object = None  # row chosen by the device's nearest-miss reduction (when best is None)

    def to_doc(self) -> dict:
        on_front = {id(r) for r in self.frontier}
        by_id = {}
        rows = []
        feasible = 0
        for r in self.rows:
            doc = r.to_doc()
            doc["feasible"] = r.meets_sla(self.workload)
            doc["frontier"] = id(r) in on_front
            feasible += doc["feasible"]
            by_id[id(r)] = doc
            rows.append(doc)
        return {
            "schema": REPORT_SCHEMA,
            "version": REPORT_VERSION,
            "model": self.model,
            "backend": self.backend,
            "workload": self.workload.to_doc(),
            "counts": {"enumerated": self.enumerated, "evaluated": len(self.rows), "feasible": feasible,
                       "frontier": len(self.frontier), "skipped": len(self.skipped)},
            "rows": rows,
            "frontier": [by_id[id(r)] for r in self.frontier],
            "best": self.best.to_doc() if self.best else None,
            "diagnostics": None if self.best else nearest_miss_doc(self.nearest, self.workload),
            "skipped": self.skipped,
            "timing": {"total_ms": self.total_ms,
                       "per_candidate_median_ms": statistics.median(self.per_candidate_ms)
                       if self.per_candidate_ms else 0.0},
        }

    def to_json(self) -> str:
        return json.dumps(self.to_doc(), sort_keys=True, indent=2, allow_nan=False) + "\n"


CSV_COLUMNS = ("mode", "config", "gpus", "batch", "ttft_ms", "tpot_ms", "speed", "throughput_per_gpu", "feasible",
               "frontier")


def csv_from_doc(doc: Mapping) -> str:
    lines = [",".join(CSV_COLUMNS)]
    for row in doc["rows"]:
        batch = row["decode"]["batch"] if row["mode"] == "disaggregated" else row["batch"]
        speed = row["speed"]
        lines.append(",".join([
            row["mode"], row["config"], str(row["gpus"]), str(batch), f"{row['ttft_ms']:.6g}",
            f"{row['tpot_ms']:.6g}", "inf" if speed is None or math.isinf(speed) else f"{speed:.6g}",
            f"{row['throughput_per_gpu']:.6g}", "yes" if row["feasible"] else "no",
            "yes" if row["frontier"] else "no",
        ]))
    return "\n".join(lines) + "\n"


def export_csv(report: SearchReport) -> str:
    return csv_from_doc(report.to_doc())
