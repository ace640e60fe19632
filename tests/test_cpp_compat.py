"""Runs the C++ drop-in test (tests/cpp/test_compat.cpp): the reference's
operator API names over the C ABI, checked against known answers and the
oracle.  Built by __graft_entry__.build() (or here if missing)."""
import os
import subprocess

import pytest

from conftest import ROOT

HERE = os.path.join(ROOT, "tests", "cpp")


def _build():
    subprocess.check_call(["make", "-C", HERE], stdout=subprocess.DEVNULL)
    return os.path.join(HERE, "test_compat.bin")


def test_compat_header_compiles():
    """CPU-side: the header + test compile and link against the C ABI."""
    assert os.path.exists(_build())


@pytest.mark.gpu
def test_compat_runs_on_gpu(cuda):
    r = subprocess.run([_build()], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "compat OK" in r.stdout
