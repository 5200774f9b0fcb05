"""The columnar report writer emits exactly the bytes of SearchReport.to_json()
(reference search.py:262-264): checked on every reference golden report."""

import json
import time

import pytest

from golden_io import CASES, golden_report
from paper_2601_06288_b200.fastreport import columns_from_doc, report_json


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_columnar_json_is_byte_identical(case):
    doc = golden_report(case["name"])
    doc.pop("_meta")
    doc["timing"] = {"total_ms": 12.345, "per_candidate_median_ms": 0.001}
    ref = json.dumps(doc, sort_keys=True, indent=2, allow_nan=False) + "\n"
    assert report_json(columns_from_doc(doc)) == ref


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
