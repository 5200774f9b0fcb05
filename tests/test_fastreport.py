"""The columnar report writer emits exactly the bytes of SearchReport.to_json()
(reference search.py:262-264): checked on every reference golden report."""

import json
import time

import pytest

from golden_io import CASES, golden_report
from paper_2601_06288_b200.fastreport import columns_from_doc, report_json


@pytest.mark.parametrize("native", [True, False], ids=["native", "python"])
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_columnar_json_is_byte_identical(case, native):
    doc = golden_report(case["name"])
    doc.pop("_meta")
    doc["timing"] = {"total_ms": 12.345, "per_candidate_median_ms": 0.001}
    ref = json.dumps(doc, sort_keys=True, indent=2, allow_nan=False) + "\n"
    assert report_json(columns_from_doc(doc), native=native) == ref


def test_native_float_repr_matches_cpython():
    """lc_report_rows prints floats exactly as CPython's repr: random values over
    the whole exponent range and the fixed / scientific switch points."""
    import numpy as np

    doc = golden_report("qwen3_all_default")  # static, aggregated and disaggregated rows
    doc.pop("_meta")
    doc["timing"] = {"total_ms": 1.0, "per_candidate_median_ms": 0.5}
    cols = columns_from_doc(doc)
    assert cols.r_sys is not None and (cols.mode == 2).any()
    rng = np.random.default_rng(7)
    n = len(cols.mode)
    edges = np.array([1e-5, 9.999999999999999e-05, 1e-4, 0.1, 1.0, 5000.0, 1e15, 9.999999999999998e15, 1e16,
                      1.2345678901234567e16, 2.0 ** -1074, 2.0 ** 1023, 0.0, 123456789.0, 0.30000000000000004])
    for trial in range(20):
        vals = np.exp(rng.uniform(-60, 60, size=(4, n)))
        vals[:, : min(n, len(edges))] = edges[: min(n, len(edges))]
        rng.shuffle(vals, axis=1)
        cols.ttft, cols.tpot, cols.thru = vals[0].copy(), vals[1].copy(), vals[2].copy()
        cols.speed = np.where(rng.random(n) < 0.1, np.inf, vals[3])
        if cols.r_sys is not None:
            cols.r_sys = np.exp(rng.uniform(-40, 40, size=n))
        assert report_json(cols, native=True) == report_json(cols, native=False)


def test_columnar_json_is_faster_than_the_dict_encoder():
    doc = golden_report("gptoss_all_default")
    doc.pop("_meta")
    doc["timing"] = {"total_ms": 1.0, "per_candidate_median_ms": 0.5}
    cols = columns_from_doc(doc)
    t0 = time.perf_counter()
    fast = report_json(cols)
    t1 = time.perf_counter()
    slow = json.dumps(doc, sort_keys=True, indent=2, allow_nan=False) + "\n"
    t2 = time.perf_counter()
    assert fast == slow
    assert (t1 - t0) < (t2 - t1)
