"""Input types of the search seam, mirroring the reference's public dataclasses.

Field names, defaults, validation messages and document forms follow
/root/reference/pkg/src/llmconf/{perfdb,model,moe_load,serving_modes,search}.py
so that reports built from these objects are byte-identical and so that the
reference's own objects can be passed in instead (everything downstream reads
attributes only).  These are plain host-side records: no arithmetic of the
search path lives here.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path
from typing import Mapping

QUANT_FORMATS = ("fp16", "fp8", "int8", "int4")
QUANT_BYTES = {"fp16": 2.0, "fp8": 1.0, "int8": 1.0, "int4": 0.5}  # perfdb.py:25
ATTENTION_VARIANTS = ("MHA", "GQA", "MLA")
BACKENDS = ("trtllm", "vllm", "sglang", "dynamo")
SERVING_MODES = ("static", "aggregated", "disaggregated")
MLA_KV_DIM = 576
DEFAULT_BATCHES = tuple(2**i for i in range(10))


# ----------------------------------------------------------------------------- errors
class PerfDbError(Exception):
    """Base class for database failures (perfdb.py:80)."""


class DbParseError(PerfDbError):
    pass


class DbValidationError(PerfDbError):
    pass


class MissingKeyError(PerfDbError):
    pass


class ExtrapolationError(PerfDbError):
    pass


class UnsupportedOperatorError(PerfDbError):
    pass


class ModelConfigError(ValueError):
    pass


class ParallelConfigError(ValueError):
    pass


class WorkloadError(ValueError):
    pass


class InfeasibleConfigError(RuntimeError):
    pass


class MoELoadError(ValueError):
    pass


class SearchError(RuntimeError):
    pass


# ----------------------------------------------------------------------------- hardware
@dataclass(frozen=True)
class HardwareSpec:
    name: str
    gpu_memory: int
    mem_bandwidth: float
    compute_throughput: Mapping[str, float]
    intra_node_bandwidth: float
    inter_node_bandwidth: float
    gpus_per_node: int

    def __post_init__(self) -> None:
        if not self.compute_throughput:
            raise DbValidationError("compute_throughput must not be empty")
        for fmt, rate in self.compute_throughput.items():
            if fmt not in QUANT_FORMATS:
                raise DbValidationError(f"unknown numeric format {fmt!r}")
            if rate <= 0:
                raise DbValidationError(f"compute_throughput[{fmt}] must be positive")
        for attr in ("gpu_memory", "mem_bandwidth", "intra_node_bandwidth", "inter_node_bandwidth"):
            if getattr(self, attr) <= 0:
                raise DbValidationError(f"{attr} must be positive")
        if self.gpus_per_node < 1:
            raise DbValidationError("gpus_per_node must be >= 1")

    _FIELDS = ("name", "gpu_memory", "mem_bandwidth", "compute_throughput", "intra_node_bandwidth",
               "inter_node_bandwidth", "gpus_per_node")

    def to_doc(self) -> dict:
        doc = {k: getattr(self, k) for k in self._FIELDS}
        doc["compute_throughput"] = dict(sorted(self.compute_throughput.items()))
        return doc

    @classmethod
    def from_doc(cls, doc: Mapping) -> "HardwareSpec":
        known = set(cls._FIELDS)
        if set(doc) - known:
            raise DbParseError(f"unknown hardware fields: {sorted(set(doc) - known)}")
        if known - set(doc):
            raise DbParseError(f"missing hardware fields: {sorted(known - set(doc))}")
        return cls(
            name=doc["name"],
            gpu_memory=int(doc["gpu_memory"]),
            mem_bandwidth=float(doc["mem_bandwidth"]),
            compute_throughput={k: float(v) for k, v in doc["compute_throughput"].items()},
            intra_node_bandwidth=float(doc["intra_node_bandwidth"]),
            inter_node_bandwidth=float(doc["inter_node_bandwidth"]),
            gpus_per_node=int(doc["gpus_per_node"]),
        )


def load_hardware_spec(path: str | Path) -> HardwareSpec:
    return HardwareSpec.from_doc(json.loads(Path(path).read_text(encoding="utf-8")))


# ----------------------------------------------------------------------------- model
@dataclass(frozen=True)
class MoESpec:
    num_experts: int
    topk: int
    expert_intermediate: int
    shared_intermediate: int = 0

    def __post_init__(self) -> None:
        if self.num_experts < 2:
            raise ModelConfigError("num_experts must be >= 2")
        if not 1 <= self.topk <= self.num_experts:
            raise ModelConfigError("topk must be in [1, num_experts]")
        if self.expert_intermediate < 1:
            raise ModelConfigError("expert_intermediate must be >= 1")
        if self.shared_intermediate < 0:
            raise ModelConfigError("shared_intermediate must be >= 0")


@dataclass(frozen=True)
class ModelSpec:
    name: str
    num_layers: int
    hidden_size: int
    num_heads: int
    kv_heads: int
    head_dim: int
    intermediate_size: int
    vocab_size: int
    attn_kind: str = "GQA"
    moe: MoESpec | None = None
    weight_quant: str = "fp16"
    kv_quant: str = "fp16"
    param_count: int | None = None
    mla_kv_dim: int = MLA_KV_DIM

    def __post_init__(self) -> None:
        for attr in ("num_layers", "hidden_size", "num_heads", "kv_heads", "head_dim", "vocab_size"):
            if getattr(self, attr) < 1:
                raise ModelConfigError(f"{attr} must be >= 1")
        if self.intermediate_size < 0:
            raise ModelConfigError("intermediate_size must be >= 0")
        if self.attn_kind not in ATTENTION_VARIANTS:
            raise ModelConfigError(f"attn_kind must be one of {ATTENTION_VARIANTS}")
        if self.kv_heads > self.num_heads or self.num_heads % self.kv_heads:
            raise ModelConfigError("kv_heads must divide num_heads")
        if self.weight_quant not in QUANT_FORMATS or self.kv_quant not in QUANT_FORMATS:
            raise ModelConfigError(f"quant formats must be from {QUANT_FORMATS}")
        if self.moe is None and self.intermediate_size < 1:
            raise ModelConfigError("dense models need intermediate_size >= 1")
        if self.param_count is not None and self.param_count < 1:
            raise ModelConfigError("param_count must be positive")

    def expert_params(self) -> int:
        if self.moe is None:
            return 0
        return self.num_layers * self.moe.num_experts * 3 * self.hidden_size * self.moe.expert_intermediate

    def params(self) -> int:
        if self.param_count is not None:
            return self.param_count
        h, hd = self.hidden_size, self.head_dim
        if self.attn_kind == "MLA":
            attn = h * self.num_heads * hd + 2 * h * self.mla_kv_dim + self.num_heads * hd * h
        else:
            attn = h * hd * (2 * self.num_heads + 2 * self.kv_heads)
        if self.moe is None:
            ffn = 3 * h * self.intermediate_size
        else:
            ffn = h * self.moe.num_experts + self.expert_params() // self.num_layers
            if self.moe.shared_intermediate:
                ffn += 3 * h * self.moe.shared_intermediate
        return 2 * self.vocab_size * h + self.num_layers * (attn + ffn)

    @classmethod
    def from_doc(cls, doc: Mapping) -> "ModelSpec":
        known = {"name", "num_layers", "hidden_size", "num_heads", "kv_heads", "head_dim", "intermediate_size",
                 "vocab_size", "attn_kind", "moe", "weight_quant", "kv_quant", "param_count", "mla_kv_dim"}
        if set(doc) - known:
            raise ModelConfigError(f"unknown model fields: {sorted(set(doc) - known)}")
        kwargs = {k: v for k, v in doc.items() if k != "moe"}
        moe = MoESpec(**doc["moe"]) if doc.get("moe") is not None else None
        return cls(moe=moe, **kwargs)


def load_model_spec(path: str | Path) -> ModelSpec:
    return ModelSpec.from_doc(json.loads(Path(path).read_text(encoding="utf-8")))


# ----------------------------------------------------------------------------- parallel config
@dataclass(frozen=True)
class ParallelConfig:
    tp: int = 1
    pp: int = 1
    ep: int = 1
    dp: int = 1
    batch: int = 1
    ctx_capacity: int | None = None
    chunked_prefill: bool = True
    kv_mem_fraction: float = 0.9
    cuda_graph: bool = True
    backend: str = "trtllm"

    def __post_init__(self) -> None:
        for attr in ("tp", "pp", "ep", "dp", "batch"):
            if getattr(self, attr) < 1:
                raise ParallelConfigError(f"{attr} must be >= 1")
        if self.ctx_capacity is not None and self.ctx_capacity < 1:
            raise ParallelConfigError("ctx_capacity must be >= 1 when set")
        if not 0.0 < self.kv_mem_fraction <= 1.0:
            raise ParallelConfigError("kv_mem_fraction must be in (0, 1]")
        if self.backend not in BACKENDS:
            raise ParallelConfigError(f"backend must be one of {BACKENDS}")

    def gpus(self) -> int:
        return self.tp * self.pp * self.dp

    def key(self) -> str:
        return f"tp{self.tp}pp{self.pp}ep{self.ep}dp{self.dp}b{self.batch}"


# ----------------------------------------------------------------------------- MoE load
@dataclass(frozen=True)
class PowerLawParams:
    alpha: float = 1.2
    x_min: float = 1.0
    x_max: float = 100.0
    seed: int = 0

    def __post_init__(self) -> None:
        if not 0.0 <= self.alpha <= 2.0:
            raise MoELoadError(f"alpha={self.alpha} outside [0, 2]")
        if self.alpha == 1.0:
            raise MoELoadError("alpha=1 has a singular inverse CDF; use a nearby value")
        if not 0 < self.x_min < self.x_max:
            raise MoELoadError(f"need 0 < x_min < x_max, got [{self.x_min}, {self.x_max}]")


DEFAULT_MOE_LOAD = PowerLawParams()


# ----------------------------------------------------------------------------- workload
@dataclass(frozen=True)
class WorkloadSpec:
    isl: int
    osl: int
    prefix_len: int = 0
    ttft_limit_ms: float | None = None
    tpot_limit_ms: float | None = None
    min_speed: float | None = None
    gpu_budgets: tuple[int, ...] = ()
    modes: tuple[str, ...] = SERVING_MODES
    batch_sweep: tuple[int, ...] = ()
    moe_load: PowerLawParams | None = None

    def __post_init__(self) -> None:
        if self.isl < 1 or self.osl < 1:
            raise WorkloadError("isl and osl must be >= 1")
        if not 0 <= self.prefix_len < self.isl:
            raise WorkloadError("prefix_len must be in [0, isl)")
        for name in ("ttft_limit_ms", "tpot_limit_ms", "min_speed"):
            v = getattr(self, name)
            if v is not None and v <= 0:
                raise WorkloadError(f"{name} must be positive when set")
        if self.tpot_limit_ms is not None and self.min_speed is not None:
            raise WorkloadError("set either tpot_limit_ms or min_speed, not both")
        if set(self.modes) - set(SERVING_MODES):
            raise WorkloadError(f"unknown serving modes: {sorted(set(self.modes) - set(SERVING_MODES))}")
        if any(b < 1 for b in self.gpu_budgets):
            raise WorkloadError("gpu budgets must be positive")
        if any(b < 1 for b in self.batch_sweep):
            raise WorkloadError("batch sizes must be positive")

    def effective_isl(self) -> int:
        return self.isl - self.prefix_len

    def speed_floor(self) -> float | None:
        if self.min_speed is not None:
            return self.min_speed
        if self.tpot_limit_ms is not None:
            return 1000.0 / self.tpot_limit_ms
        return None

    def tpot_ceiling(self) -> float | None:
        floor = self.speed_floor()
        return None if floor is None else 1000.0 / floor

    def to_doc(self) -> dict:
        doc: dict = {"isl": self.isl, "osl": self.osl, "prefix_len": self.prefix_len}
        for name in ("ttft_limit_ms", "tpot_limit_ms", "min_speed"):
            if getattr(self, name) is not None:
                doc[name] = getattr(self, name)
        if self.gpu_budgets:
            doc["gpu_budgets"] = list(self.gpu_budgets)
        doc["modes"] = list(self.modes)
        if self.batch_sweep:
            doc["batch_sweep"] = list(self.batch_sweep)
        if self.moe_load is not None:
            m = self.moe_load
            doc["moe_load"] = {"alpha": m.alpha, "x_min": m.x_min, "x_max": m.x_max, "seed": m.seed}
        return doc

    @classmethod
    def from_doc(cls, doc: dict) -> "WorkloadSpec":
        known = {"isl", "osl", "prefix_len", "ttft_limit_ms", "tpot_limit_ms", "min_speed", "gpu_budgets", "modes",
                 "batch_sweep", "moe_load"}
        if set(doc) - known:
            raise WorkloadError(f"unknown workload fields: {sorted(set(doc) - known)}")
        kwargs = dict(doc)
        for name in ("gpu_budgets", "modes", "batch_sweep"):
            if name in kwargs:
                kwargs[name] = tuple(kwargs[name])
        if kwargs.get("moe_load") is not None:
            kwargs["moe_load"] = PowerLawParams(**kwargs["moe_load"])
        return cls(**kwargs)


# ----------------------------------------------------------------------------- space / disagg
@dataclass(frozen=True)
class CandidateSpace:
    tp_values: tuple[int, ...] = (1, 2, 4, 8)
    pp_values: tuple[int, ...] = (1, 2, 4)
    ep_values: tuple[int, ...] = (1, 2, 4, 8)
    dp_values: tuple[int, ...] = (1, 2, 4, 8)
    batch_values: tuple[int, ...] = DEFAULT_BATCHES
    ctx_capacity: int | None = None
    chunked_prefill: bool = True
    kv_mem_fraction: float = 0.9
    cuda_graph: bool = True
    prefill_pool_cap: int = 8
    decode_pool_cap: int = 16

    def config(self, tp: int, pp: int, ep: int, dp: int, batch: int, backend: str) -> ParallelConfig:
        return ParallelConfig(tp=tp, pp=pp, ep=ep, dp=dp, batch=batch, ctx_capacity=self.ctx_capacity,
                              chunked_prefill=self.chunked_prefill, kv_mem_fraction=self.kv_mem_fraction,
                              cuda_graph=self.cuda_graph, backend=backend)


@dataclass(frozen=True)
class DisaggConstants:
    ttft_headroom: float = 1.8
    prefill_utilization: float = 0.90
    decode_utilization: float = 0.92
    max_prefill_replicas: int = 32
    max_decode_replicas: int = 64


DEFAULT_DISAGG = DisaggConstants()
