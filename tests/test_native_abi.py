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
    assert lib.lc_abi_version() == 1


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
