"""K3's general path (any number of ep values, no key packing): the default
deduplicated K3 (k_tails_keys / k_tails_jobs / k_tails_put) is taken whenever
the (load, pooled tokens) keys pack into 64 bits and there are at most 64 ep
values.  LC_TAILS_GENERAL (read once per process) forces the general
k_tails<PER> instead, so a subprocess runs every golden case through it and
compares each report with the reference's (moe_load.py:67-147 via
estimator.py:51-68)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

from test_gpu_front_overflow import SCRIPT

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_general_tails_path_matches_reference():
    env = dict(os.environ, LC_TAILS_GENERAL="1")
    code = SCRIPT.format(root=str(ROOT), tests=str(ROOT / "tests"))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["bad"] == [], res["bad"]
    assert res["cases"] >= 30
