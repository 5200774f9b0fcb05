"""The C-ABI library loads without a GPU and exports every symbol of include/llmconf_b200.h."""

import ctypes
import re
from pathlib import Path

from paper_2601_06288_b200 import _native

HEADER = Path(__file__).resolve().parents[1] / "include" / "llmconf_b200.h"


def test_library_exports_header_symbols():
    lib = _native.load_library()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(lc_\w+)\(", HEADER.read_text(), flags=re.M))
    assert declared == set(_native.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.lc_abi_version() == 3


def test_struct_layouts_match_header_sizes():
    # sizes fixed by the header's field lists (no implicit padding by construction)
    assert ctypes.sizeof(_native.LcSearchDesc) == 272
    assert ctypes.sizeof(_native.LcSearchResult) == 104
    assert ctypes.sizeof(_native.LcBatchTotals) == 88
    assert _native.SEARCH_DESC_DTYPE.itemsize == 272


def test_open_without_device_fails_loudly():
    lib = _native.load_library()
    ctx = ctypes.c_void_p()
    rc = lib.lc_open(0, ctypes.byref(ctx))
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        assert rc == 0
        lib.lc_close(ctx)
    else:
        assert rc != 0
        assert lib.lc_last_error()


def test_ctypes_and_numpy_layouts_match_the_c_compiler(tmp_path):
    """Compile a probe against include/llmconf_b200.h with gcc and compare every
    struct size and key field offset with the ctypes / numpy mirrors."""
    import json
    import subprocess

    import numpy as np

    from paper_2601_06288_b200.plans import COMBO_DTYPE, ENTRY_DTYPE, SLOT_DTYPE

    exe = tmp_path / "abi_layout"
    src = Path(__file__).resolve().parent / "native" / "abi_layout.c"
    subprocess.run(["gcc", "-O0", "-o", str(exe), str(src)], check=True)
    c = json.loads(subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout)

    def off(dt: np.dtype, name: str) -> int:
        return dt.fields[name][1]

    N = _native
    sizes = {"lc_db_desc": ctypes.sizeof(N.LcDbDesc), "lc_space_desc": ctypes.sizeof(N.LcSpaceDesc),
             "lc_search_desc": N.SEARCH_DESC_DTYPE.itemsize, "lc_search_result": ctypes.sizeof(N.LcSearchResult),
             "lc_batch_totals": ctypes.sizeof(N.LcBatchTotals), "lc_fetch_req": ctypes.sizeof(N.LcFetchReq),
             "lc_entry": ENTRY_DTYPE.itemsize, "lc_combo": COMBO_DTYPE.itemsize, "lc_slot": SLOT_DTYPE.itemsize,
             "lc_query": N.QUERY_DTYPE.itemsize, "lc_gen_grid": N.GEN_GRID_DTYPE.itemsize,
             "lc_dbgen_desc": ctypes.sizeof(N.LcDbgenDesc), "lc_step_req": N.STEP_REQ_DTYPE.itemsize,
             "lc_step_out": N.STEP_OUT_DTYPE.itemsize}
    for k, v in sizes.items():
        assert c[k] == v, (k, c[k], v)
    fields = {
        "lc_entry.repeat": off(ENTRY_DTYPE, "repeat"), "lc_entry.d": off(ENTRY_DTYPE, "d"),
        "lc_combo.weight_bytes": off(COMBO_DTYPE, "weight_bytes"), "lc_slot.step": off(SLOT_DTYPE, "step"),
        "lc_slot.pair": off(SLOT_DTYPE, "pair"), "lc_search_desc.budgets": off(N.SEARCH_DESC_DTYPE, "budgets"),
        "lc_search_desc.ctx_capacity": off(N.SEARCH_DESC_DTYPE, "ctx_capacity"),
        "lc_search_desc.load": off(N.SEARCH_DESC_DTYPE, "load"),
        "lc_search_result.best": N.LcSearchResult.best.offset,
        "lc_search_result.n_survivors": N.LcSearchResult.n_survivors.offset,
        "lc_search_result.n_feasible_plans": N.LcSearchResult.n_feasible_plans.offset,
        "lc_batch_totals.kernel_ms": N.LcBatchTotals.kernel_ms.offset,
        "lc_batch_totals.n_cells": N.LcBatchTotals.n_cells.offset,
        "lc_query.d": off(N.QUERY_DTYPE, "d"), "lc_query.kv_len": off(N.QUERY_DTYPE, "kv_len"),
        "lc_gen_grid.cell_off": off(N.GEN_GRID_DTYPE, "cell_off"), "lc_gen_grid.d": off(N.GEN_GRID_DTYPE, "d"),
        "lc_gen_grid.offset": off(N.GEN_GRID_DTYPE, "offset"),
        "lc_dbgen_desc.amplitude": N.LcDbgenDesc.amplitude.offset,
        "lc_dbgen_desc.compute": N.LcDbgenDesc.compute.offset,
        "lc_db_desc.compute": N.LcDbDesc.compute.offset, "lc_db_desc.policy": N.LcDbDesc.policy.offset,
        "lc_space_desc.gclass_of": N.LcSpaceDesc.gclass_of.offset,
        "lc_search_desc.static_stride": off(N.SEARCH_DESC_DTYPE, "static_stride"),
        "lc_step_req.batch": off(N.STEP_REQ_DTYPE, "batch"), "lc_step_req.load": off(N.STEP_REQ_DTYPE, "load"),
        "lc_step_out.c1": off(N.STEP_OUT_DTYPE, "c1"), "lc_step_out.entry_ms": off(N.STEP_OUT_DTYPE, "entry_ms"),
        "lc_step_out.entry_label": off(N.STEP_OUT_DTYPE, "entry_label"),
    }
    for k, v in fields.items():
        assert c[k] == v, (k, c[k], v)


def test_config_key_integer_codes_sort_like_python_strings(tmp_path):
    """csrc/lc_keys.h: (combo code, batch code) order == ParallelConfig.key() string order
    (the pool-rank tie break, search.py:276-277), on random configs with many shared prefixes."""
    import random
    import subprocess

    exe = tmp_path / "key_order"
    src = Path(__file__).resolve().parent / "native" / "key_order.c"
    subprocess.run(["gcc", "-O1", "-o", str(exe), str(src)], check=True)
    rng = random.Random(7)
    pool = [1, 2, 3, 4, 5, 8, 9, 10, 11, 12, 16, 19, 20, 32, 64, 99, 100, 101, 128, 256, 512, 999, 1000, 1024, 4096,
            9999]
    bpool = pool + [10000, 65536, 99999, 123456, 1000000, 9999999999]
    cfgs = [tuple(rng.choice(pool) for _ in range(4)) + (rng.choice(bpool),) for _ in range(20000)]
    cfgs += [(1, 1, 1, 1, b) for b in (1, 10, 100, 2, 20, 9, 99)] + [(t, 1, 1, 1, 8) for t in (1, 10, 16, 2, 100)]
    text = "\n".join(" ".join(map(str, c)) for c in cfgs) + "\n"
    out = subprocess.run([str(exe)], input=text, capture_output=True, text=True, check=True).stdout.split("\n")
    codes = [tuple(int(x) for x in line.split()) for line in out if line]
    assert len(codes) == len(cfgs)
    key = [f"tp{a}pp{b}ep{c}dp{d}b{e}" for a, b, c, d, e in cfgs]
    by_str = sorted(range(len(cfgs)), key=lambda i: (key[i], i))
    by_code = sorted(range(len(cfgs)), key=lambda i: (codes[i], i))
    assert [key[i] for i in by_str] == [key[i] for i in by_code]
    # equal strings <=> equal codes
    assert len(set(key)) == len(set(codes))
