"""ctypes binding of the in-tree CUDA library ``_lc_b200.so`` (include/llmconf_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .plans import COMBO_DTYPE, ENTRY_DTYPE

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "_lc_b200.so"
LC_MAX_BUDGETS = 16

I32P, I64P, F64P, U8P = (C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_double),
                         C.POINTER(C.c_uint8))


class NativeUnavailable(RuntimeError):
    """The CUDA engine cannot run here (library not built or no device), or a CUDA call failed."""


class EngineLimitError(ValueError):
    """The C ABI rejected its arguments (LC_ERR_ARG): a request beyond the device path's
    documented limits or a malformed call -- not an unavailable engine."""


LC_ERR_ARG = -1


class LcDbDesc(C.Structure):
    _fields_ = [("n_grids", C.c_int32), ("grid_ndim", I32P), ("grid_axis_off", I32P), ("grid_axis_len", I32P),
                ("grid_cell_off", I32P), ("n_axis", C.c_int32), ("axis_val", I64P), ("axis_log", F64P),
                ("n_cells", C.c_int32), ("cell", F64P), ("cell_log", F64P), ("mem_bandwidth", C.c_double),
                ("intra_node_bandwidth", C.c_double), ("inter_node_bandwidth", C.c_double),
                ("gpu_memory", C.c_double), ("gpus_per_node", C.c_int32), ("compute", C.c_double * 4),
                ("policy", C.c_int32)]


class LcSpaceDesc(C.Structure):
    _fields_ = [("hidden", C.c_int64), ("topk", C.c_int64), ("n_experts", C.c_int64), ("is_moe", C.c_int32),
                ("n_combos", C.c_int32), ("combos", C.c_void_p), ("n_tmpl", C.c_int32),
                ("tmpl_n_entries", I32P), ("entries", C.c_void_p), ("n_tp", C.c_int32), ("n_ep", C.c_int32),
                ("n_slots", C.c_int32), ("slots", C.c_void_p), ("slot_of", I32P), ("n_gen_classes", C.c_int32),
                ("gen_classes", C.c_void_p), ("gclass_of", I32P)]


class LcSearchDesc(C.Structure):
    _fields_ = [("isl", C.c_int64), ("osl", C.c_int64), ("prefix", C.c_int64), ("has_ttft", C.c_int32),
                ("has_floor", C.c_int32), ("ttft_limit", C.c_double), ("speed_floor", C.c_double),
                ("tpot_cap", C.c_double), ("modes", C.c_int32), ("n_budgets", C.c_int32),
                ("budgets", C.c_int64 * LC_MAX_BUDGETS), ("b_off", C.c_int32), ("n_b", C.c_int32),
                ("has_ctx_capacity", C.c_int32), ("chunked_prefill", C.c_int32), ("ctx_capacity", C.c_int64),
                ("kv_mem_fraction", C.c_double), ("prefill_cap", C.c_int32), ("decode_cap", C.c_int32),
                ("ttft_headroom", C.c_double), ("prefill_util", C.c_double), ("decode_util", C.c_double),
                ("max_x", C.c_int32), ("max_y", C.c_int32), ("load", C.c_int32), ("static_stride", C.c_int32)]


class LcSearchResult(C.Structure):
    _fields_ = [("n_units", C.c_int32), ("unit_off", C.c_int32), ("n_enumerated", C.c_int32),
                ("n_rows", C.c_int32), ("n_feasible", C.c_int32), ("n_skipped", C.c_int32),
                ("n_front", C.c_int32), ("front_off", C.c_int32), ("n_plans", C.c_int32), ("plan_off", C.c_int32),
                ("best", C.c_int64), ("nearest", C.c_int64), ("nearest_violation", C.c_double),
                ("best_thru", C.c_double), ("best_speed", C.c_double), ("queries_1d", C.c_int64),
                ("queries_2d", C.c_int64), ("n_survivors", C.c_int32), ("n_feasible_plans", C.c_int32)]


class LcBatchTotals(C.Structure):
    _fields_ = [("n_units", C.c_int64), ("n_plans", C.c_int64), ("n_front", C.c_int64),
                ("kernel_ms", C.c_float * 6), ("n_raw", C.c_int64), ("n_launches", C.c_int64),
                ("n_table_queries", C.c_int64), ("n_table_queries_2d", C.c_int64), ("n_cells", C.c_int64)]


_FETCH_FIELDS = [
    ("unit_search", I32P), ("unit_combo", I32P), ("unit_batch", I32P), ("unit_in_budget", U8P),
    ("st_status", I32P), ("st_ttft", F64P), ("st_tpot", F64P), ("st_speed", F64P), ("st_thru", F64P),
    ("ag_status", I32P), ("ag_ttft", F64P), ("ag_tpot", F64P), ("ag_speed", F64P), ("ag_thru", F64P),
    ("pf_status", I32P), ("pf_lat", F64P), ("pf_rate", F64P),
    ("dc_status", I32P), ("dc_lat", F64P), ("dc_rate", F64P),
    ("err_c0", I64P), ("err_c1", I64P),
    ("plan_p", I32P), ("plan_d", I32P), ("plan_x", I32P), ("plan_y", I32P), ("plan_gpus", I64P),
    ("plan_r_sys", F64P), ("plan_ttft", F64P), ("plan_tpot", F64P), ("plan_speed", F64P), ("plan_thru", F64P),
    ("front", I64P),
]


class LcFetchReq(C.Structure):
    _fields_ = _FETCH_FIELDS


SEARCH_RESULT_DTYPE = np.dtype([(n, {C.c_int32: "<i4", C.c_int64: "<i8", C.c_double: "<f8"}[t])
                                for n, t in LcSearchResult._fields_])
assert SEARCH_RESULT_DTYPE.itemsize == C.sizeof(LcSearchResult)

SEARCH_DESC_DTYPE = np.dtype([("isl", "<i8"), ("osl", "<i8"), ("prefix", "<i8"), ("has_ttft", "<i4"),
                              ("has_floor", "<i4"), ("ttft_limit", "<f8"), ("speed_floor", "<f8"),
                              ("tpot_cap", "<f8"), ("modes", "<i4"), ("n_budgets", "<i4"),
                              ("budgets", "<i8", (LC_MAX_BUDGETS,)), ("b_off", "<i4"), ("n_b", "<i4"),
                              ("has_ctx_capacity", "<i4"), ("chunked_prefill", "<i4"), ("ctx_capacity", "<i8"),
                              ("kv_mem_fraction", "<f8"), ("prefill_cap", "<i4"), ("decode_cap", "<i4"),
                              ("ttft_headroom", "<f8"), ("prefill_util", "<f8"), ("decode_util", "<f8"),
                              ("max_x", "<i4"), ("max_y", "<i4"), ("load", "<i4"), ("static_stride", "<i4")])
assert SEARCH_DESC_DTYPE.itemsize == C.sizeof(LcSearchDesc), (SEARCH_DESC_DTYPE.itemsize, C.sizeof(LcSearchDesc))

GEN_GRID_DTYPE = np.dtype([("kind", "<i4"), ("quant", "<i4"), ("n_axes", "<i4"), ("_pad", "<i4"),
                           ("axis_dim", "<i4", (2,)), ("axis_off", "<i4", (2,)), ("axis_len", "<i4", (2,)),
                           ("cell_off", "<i8"), ("d", "<i8", (5,)), ("offset", "<f8")])
assert GEN_GRID_DTYPE.itemsize == 96


class LcDbgenDesc(C.Structure):
    _fields_ = [("n_grids", C.c_int32), ("grids", C.c_void_p), ("n_axis", C.c_int32), ("axis_val", I64P),
                ("axis_term", F64P), ("n_cells", C.c_int64), ("amplitude", C.c_double),
                ("mem_bandwidth", C.c_double), ("intra_node_bandwidth", C.c_double),
                ("inter_node_bandwidth", C.c_double), ("gpus_per_node", C.c_int32), ("compute", C.c_double * 4)]


class LcReportCols(C.Structure):
    _fields_ = [("n", C.c_int64), ("mode", I32P), ("cfg", I64P), ("gpus", I64P), ("ttft", F64P), ("tpot", F64P),
                ("speed", F64P), ("thru", F64P), ("feasible", C.POINTER(C.c_uint8)),
                ("frontier", C.POINTER(C.c_uint8)), ("pcfg", I64P), ("dcfg", I64P), ("x", I64P), ("y", I64P),
                ("r_sys", F64P), ("model_json", C.c_char_p), ("runtime", C.c_char_p * 6)]


LC_MAX_ENTRIES = 16
STEP_REQ_DTYPE = np.dtype([("tmpl", "<i4"), ("phase", "<i4"), ("n_ctx", "<i8"), ("n_gen", "<i8"), ("seq", "<i8"),
                           ("batch", "<i8"), ("load", "<i4"), ("_pad", "<i4")])
assert STEP_REQ_DTYPE.itemsize == 48
STEP_OUT_DTYPE = np.dtype([("total_ms", "<f8"), ("status", "<i4"), ("n_entries", "<i4"), ("c0", "<i8"),
                           ("c1", "<i8"), ("entry_ms", "<f8", (LC_MAX_ENTRIES,)),
                           ("entry_label", "<i4", (LC_MAX_ENTRIES,))])
assert STEP_OUT_DTYPE.itemsize == 224

QUERY_DTYPE = np.dtype([("grid", "<i4"), ("kind", "<i4"), ("quant", "<i4"), ("policy", "<i4"), ("d", "<i8", (5,)),
                        ("kv_len", "<i8")])
assert QUERY_DTYPE.itemsize == 64

EXPORTED = ("lc_abi_version", "lc_last_error", "lc_open", "lc_close", "lc_db_upload", "lc_db_free",
            "lc_space_upload", "lc_space_free", "lc_search_batch", "lc_fetch", "lc_replay_last", "lc_replay_async",
            "lc_stream", "lc_query_batch", "lc_dbgen", "lc_set_raw_filter", "lc_fetch_pools",
            "lc_unit_raw", "lc_report_rows", "lc_step_latency", "lc_set_priority")

_LIB = None


def load_library(path: str | os.PathLike | None = None):
    """Load and type the shared library (no device needed)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path else Path(os.environ.get("LC_B200_LIB", LIB_PATH))
    if not p.exists():
        raise NativeUnavailable(f"{p} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(p))
    lib.lc_abi_version.restype = C.c_int
    lib.lc_last_error.restype = C.c_char_p
    lib.lc_open.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    lib.lc_close.argtypes = [C.c_void_p]
    lib.lc_db_upload.argtypes = [C.c_void_p, C.POINTER(LcDbDesc), C.POINTER(C.c_void_p)]
    lib.lc_db_free.argtypes = [C.c_void_p]
    lib.lc_space_upload.argtypes = [C.c_void_p, C.POINTER(LcSpaceDesc), C.POINTER(C.c_void_p)]
    lib.lc_space_free.argtypes = [C.c_void_p]
    lib.lc_search_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, I64P,
                                    C.c_int32, F64P, C.c_void_p, C.POINTER(LcBatchTotals)]
    lib.lc_fetch.argtypes = [C.c_void_p, C.POINTER(LcFetchReq)]
    lib.lc_replay_last.argtypes = [C.c_void_p, C.c_int32, C.POINTER(LcBatchTotals)]
    lib.lc_replay_async.argtypes = [C.c_void_p]
    lib.lc_stream.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    lib.lc_set_priority.argtypes = [C.c_void_p, C.c_int]
    lib.lc_dbgen.argtypes = [C.c_void_p, C.POINTER(LcDbgenDesc), F64P, F64P, I32P]
    lib.lc_query_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, F64P, I32P]
    lib.lc_set_raw_filter.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
    lib.lc_fetch_pools.argtypes = [C.c_void_p, I32P, I32P]
    lib.lc_unit_raw.argtypes = [C.c_void_p, C.c_int32, I32P, I64P]
    lib.lc_report_rows.argtypes = [C.POINTER(LcReportCols), I64P, C.c_int64, C.c_int32, C.c_int32, C.c_char_p,
                                   C.c_int64]
    lib.lc_report_rows.restype = C.c_int64
    lib.lc_step_latency.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, F64P,
                                    C.c_void_p]
    if path is None:
        _LIB = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load_library().lc_last_error().decode(errors="replace")
        if rc == LC_ERR_ARG:
            raise EngineLimitError(f"{what}: {msg}")
        raise NativeUnavailable(f"{what} failed ({rc}): {msg}")


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def vptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


assert ENTRY_DTYPE.itemsize == 72 and COMBO_DTYPE.itemsize == 72
