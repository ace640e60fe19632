"""Runs the C++ drop-in test (tests/cpp/test_compat.cpp): the reference's
operator API names over the C ABI, checked against known answers and the
oracle.  Built by __graft_entry__.build() (or here if missing)."""
import os
import subprocess

import pytest

from conftest import ROOT

HERE = os.path.join(ROOT, "tests", "cpp")


def _build(name="test_compat.bin"):
    subprocess.check_call(["make", "-C", HERE], stdout=subprocess.DEVNULL)
    return os.path.join(HERE, name)


def _ref_variant():
    path = _build("test_compat_ref.bin")
    if not os.path.exists(path):
        pytest.skip("reference headers (baseline/_ref/include) or oracle/_ref not built here")
    return path


def test_compat_header_compiles():
    """CPU-side: the header + test compile and link against the C ABI."""
    assert os.path.exists(_build())


def test_compat_compiles_against_reference_headers():
    """The drop-in compiled with the reference's own sparsegnn:: types and
    error classes (SGNN_B200_ERROR_NS=sparsegnn)."""
    assert os.path.exists(_ref_variant())


@pytest.mark.gpu
def test_compat_runs_on_gpu(cuda):
    r = subprocess.run([_build()], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "compat OK" in r.stdout


@pytest.mark.gpu
def test_compat_reference_types_run_on_gpu(cuda):
    """Reference CsrMatrix / DenseMatrix objects through the drop-in on the
    GPU, checked against the reference's own CPU spmm / transpose in the same
    process; the reference's load_report reads the drop-in's report."""
    r = subprocess.run([_ref_variant()], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "compat-ref OK" in r.stdout
