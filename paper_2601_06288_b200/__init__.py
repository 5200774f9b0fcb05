"""B200-native configuration-search engine for the llmconf (AIConfigurator) hot path.

Public seam: ``run_search`` -- a drop-in for ``llmconf.search.run_search``
(/root/reference/pkg/src/llmconf/search.py:280-358) whose arithmetic runs in
hand-written sm_100a kernels behind the C ABI in include/llmconf_b200.h.
"""

from .database import PerfDatabase, ValidationReport, load_db, validate_db
from .engine import (
    Engine,
    enumerate_candidates,
    estimate_aggregated,
    estimate_static,
    get_engine,
    run_search,
    run_search_json,
)
from .dbgen import GridAxes, generate_synthetic_db, grid_spec_for_model, save_db
from .sharded import ShardedResult, run_search_sharded
from .soa import load_soa, save_soa
from .steps import StepLatency, get_gen_latency, get_mix_latency, get_step_latency, step_latency_batch
from .queries import OperatorQuery, query_latency, query_latency_batch
from .report import SearchReport, csv_from_doc, export_csv
from .specs import (
    DEFAULT_DISAGG,
    CandidateSpace,
    DisaggConstants,
    HardwareSpec,
    ModelSpec,
    MoESpec,
    ParallelConfig,
    PowerLawParams,
    WorkloadSpec,
    load_hardware_spec,
    load_model_spec,
)

__all__ = [
    "CandidateSpace", "DEFAULT_DISAGG", "DisaggConstants", "Engine", "HardwareSpec", "ModelSpec", "MoESpec",
    "ParallelConfig", "PerfDatabase", "PowerLawParams", "SearchReport", "WorkloadSpec", "csv_from_doc",
    "ValidationReport", "validate_db", "enumerate_candidates", "estimate_aggregated", "estimate_static",
    "export_csv", "get_engine", "load_db", "load_hardware_spec", "load_model_spec",
    "StepLatency", "get_step_latency", "get_mix_latency", "get_gen_latency", "step_latency_batch",
    "GridAxes", "generate_synthetic_db", "load_soa", "save_soa", "grid_spec_for_model", "save_db",
    "OperatorQuery", "query_latency", "query_latency_batch", "run_search", "run_search_json",
    "ShardedResult", "run_search_sharded",
]
