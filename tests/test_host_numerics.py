"""Host logic of libpint on CPU (no GPU): the 1-D spatial factorisation of I - s A into
tridiagonal factors (host_numerics.cpp) for every operator of the paper (DESIGN.md
reading R14), checked by tests/host/factor_check.cpp against the operator's symbol."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2103_12571_b200", "csrc")


def test_factorisation_reproduces_symbol(tmp_path):
    exe = str(tmp_path / "factor_check")
    cmd = ["g++", "-O2", "-std=c++17", "-o", exe, os.path.join(ROOT, "tests", "host", "factor_check.cpp"),
           os.path.join(CSRC, "host_numerics.cpp"), "-I", CSRC, "-I", os.path.join(ROOT, "include")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        pytest.fail(r.stderr[-3000:])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout[-3000:]
