"""CPU-side checks: the C-ABI library loads and exports every symbol the
headers declare (no compute calls without a GPU), the ABI structs match the
header layout, the host generators are deterministic and match their spec,
and the host partitioner equals the reference's balanced_row_partition."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, rand_csr
from oracle import port


def _declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sgnn_\w+)\s*\(", src)))


def test_cuda_library_exports_every_declared_symbol():
    from paper_2403_14853_b200 import _lib
    lib = _lib.lib()
    declared = _declared("sgnn_b200.h")
    assert len(declared) >= 24
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_lib.SIGNATURES), set(declared) ^ set(_lib.SIGNATURES)
    assert lib.sgnn_abi_version() == 1


def test_host_library_exports_every_declared_symbol():
    from paper_2403_14853_b200 import _lib
    h = _lib.host()
    declared = _declared("sgnn_host.h")
    assert [s for s in declared if not hasattr(h, s)] == []
    assert set(declared) == set(_lib.HOST_SIGNATURES)


def test_struct_layout_matches_header():
    from paper_2403_14853_b200 import _lib
    assert C.sizeof(_lib.Csr) == 40
    assert C.sizeof(_lib.PlanParams) == 36


def test_dispatch_state_is_host_only():
    """resolve_kernel / set_dispatch need no device (dispatch.cpp:21-28)."""
    from paper_2403_14853_b200 import _lib
    lib = _lib.lib()
    sk = C.c_uint32()
    assert lib.sgnn_resolve_kernel(32, 0, C.byref(sk)) == 1 and sk.value == 32
    assert lib.sgnn_resolve_kernel(48, 0, C.byref(sk)) == 0 and sk.value == 0
    assert lib.sgnn_resolve_kernel(32, 3, C.byref(sk)) == 0
    lib.sgnn_set_dispatch(0)
    try:
        assert lib.sgnn_get_dispatch() == 0
        assert lib.sgnn_resolve_kernel(32, 0, C.byref(sk)) == 0
    finally:
        lib.sgnn_set_dispatch(1)
    from oracle import ref
    if ref.available():
        for k in (16, 32, 48, 1024, 2048):
            for r in range(4):
                for en in (0, 1):
                    lib.sgnn_set_dispatch(en)
                    tag = lib.sgnn_resolve_kernel(k, r, C.byref(sk))
                    assert (("specialized" if tag else "trusted"), sk.value) == ref.resolve_kernel(k, r, en)
        lib.sgnn_set_dispatch(1)


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2403_14853_b200 import _lib
    lib = _lib.lib()
    a = _lib.Csr(1, 1, 0, 0, 0, 0)
    ci = C.c_int()
    assert lib.sgnn_device_info(C.byref(ci), None, None, None) == 8
    rp = (C.c_uint64 * 2)(0, 0)
    a.row_ptr = C.cast(rp, C.c_void_p)
    st = lib.sgnn_spmm_f32(C.byref(a), None, 1, 4, None, 0, None, None)
    assert st == 8  # SGNN_ERR_CUDA: no silent CPU fallback


def test_er_generator():
    from paper_2403_14853_b200 import graphs
    rp, ci = graphs.er(1000, 500, 16, seed=3)
    assert rp[-1] == 16000 and (np.diff(rp) == 16).all()
    rows = ci.reshape(1000, 16)
    assert (np.diff(rows.astype(np.int64), axis=1) > 0).all() and ci.max() < 500
    rp2, ci2 = graphs.er(1000, 500, 16, seed=3, threads=1)
    assert np.array_equal(ci, ci2)
    assert not np.array_equal(ci, graphs.er(1000, 500, 16, seed=4)[1])


def test_rmat_generator_properties():
    from paper_2403_14853_b200 import graphs
    rp, ci = graphs.rmat(12, 4096 * 16, seed=5)
    n = 4096
    assert len(rp) == n + 1 and rp[-1] == len(ci)
    deg = np.diff(rp.astype(np.int64))
    for i in np.nonzero(deg)[0][:200]:
        row = ci[rp[i]:rp[i + 1]]
        assert (np.diff(row.astype(np.int64)) > 0).all()
    assert deg[:64].sum() > deg[-64:].sum()  # skew towards low ids (no permutation)
    rp1, ci1 = graphs.rmat(12, 4096 * 16, seed=5, threads=1)
    assert np.array_equal(rp, rp1) and np.array_equal(ci, ci1)
    # symmetrised + self loops is structurally symmetric with a full diagonal
    rp, ci = graphs.rmat(10, 1024 * 8, seed=2, symmetrize=True, self_loops=True)
    assert port.is_symmetric(rp, ci, np.ones(len(ci), np.float32), 1024)
    for i in range(1024):
        assert i in set(ci[rp[i]:rp[i + 1]].tolist())


def test_value_generators():
    from paper_2403_14853_b200 import graphs
    u = graphs.uniform(200000, -1, 1, seed=1)
    assert u.min() >= -1 and u.max() < 1 and abs(u.mean()) < 0.01
    z = graphs.normal(200000, 0, 1, seed=1)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01
    assert np.array_equal(z, graphs.normal(200000, 0, 1, seed=1, threads=1))


def test_host_partition_matches_reference_rule():
    from paper_2403_14853_b200 import graphs
    rng = np.random.default_rng(1)
    for m, n in ((1, 1), (50, 50), (1000, 300)):
        rp, _, _ = rand_csr(rng, m, n, 0.05, hub_rows=(0,) if m > 1 else (), empty_frac=0.2)
        for chunks in (1, 2, 3, 4, 8):
            np.testing.assert_array_equal(graphs.balanced_row_partition(rp, chunks),
                                          port.balanced_row_partition(rp, chunks))
