"""The device restatement of glibc log/exp (csrc/glibc_libm.cuh), compiled for
the host, equals this machine's libm bit for bit on every integer coordinate
below 2^22, a strided sweep to 2^34, and millions of random arguments.

This is what lets the CUDA interpolation reproduce CPython's math.log/math.exp
(/root/reference/pkg/src/llmconf/perfdb.py:505, 535-536) exactly.
"""

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_glibc_log_exp_restatement_is_bit_exact(tmp_path):
    exe = tmp_path / "libm_check"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-mfma", "-o", str(exe),
                    str(ROOT / "tests" / "native" / "libm_check.cpp")], check=True)
    out = subprocess.run([str(exe), "3000000", "11"], capture_output=True, text=True)
    checked, bad = map(int, out.stdout.split())
    assert checked > 10_000_000
    assert bad == 0, out.stderr


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_div1000_is_correctly_rounded(tmp_path):
    """lc::div1000 (the step sums' `lat * repeat / 1000.0`, estimator.py:93) is IEEE division."""
    exe = tmp_path / "div_check"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-mfma", "-o", str(exe),
                    str(ROOT / "tests" / "native" / "div_check.cpp")], check=True)
    out = subprocess.run([str(exe), "40000000", "7"], capture_output=True, text=True)
    checked, bad = map(int, out.stdout.split())
    assert checked > 40_000_000
    assert bad == 0, out.stderr
