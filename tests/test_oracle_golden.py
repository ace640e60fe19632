"""Pins the oracle (oracle/sgnn_oracle.c via oracle/port.py) against
(i) the SPEC.md known-answer examples on the hot path and (ii) the golden
fixtures the reference itself produced (tests/golden/make_golden.py, run on
oracle/_ref built from /root/reference/proj).  fp32 results must match the
reference fp32 (no-FMA) build bit for bit; fp64 likewise (same loop order)."""
import numpy as np
import pytest

from conftest import golden_cases, load_golden
from oracle import port


def _bits(a):
    a = np.asarray(a)
    return a.view(np.uint8)


# ---- SPEC known answers ---------------------------------------------------------
def test_kat_spmm():
    rp, ci, v = np.array([0, 1, 2], np.uint64), np.array([1, 0], np.uint32), np.array([2, 3], np.float32)
    np.testing.assert_array_equal(port.spmm(rp, ci, v, np.array([[1, 1], [2, 2]]), 0), [[4, 4], [3, 3]])
    rp, ci, v = np.array([0, 2], np.uint64), np.array([0, 1], np.uint32), np.ones(2, np.float32)
    b = np.array([[2, 8], [4, 2]])
    assert port.spmm(rp, ci, v, b, port.MIN).tolist() == [[2, 2]]
    assert port.spmm(rp, ci, v, b, port.MAX).tolist() == [[4, 8]]
    assert port.spmm(rp, ci, v, b, port.MEAN).tolist() == [[3, 5]]


def test_kat_sddmm_fusedmm():
    ident = (np.arange(3, dtype=np.uint64), np.arange(2, dtype=np.uint32), np.ones(2))
    x = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert port.sddmm(*ident, x, x).tolist() == [5, 25]
    assert port.fusedmm(*ident, x, x).tolist() == [[5, 10], [75, 100]]


def test_kat_transpose_normalize_partition():
    trp, tci, tv = port.transpose(np.array([0, 1, 1], np.uint64), np.array([1], np.uint32), np.array([2.0], np.float32), 2)
    assert trp.tolist() == [0, 0, 1] and tci.tolist() == [0] and tv.tolist() == [2.0]
    # single undirected edge with self loops -> all four entries 0.5
    rp, ci, v = port.normalize_adjacency(np.array([0, 1, 2], np.uint64), np.array([1, 0], np.uint32), np.ones(2, np.float32))
    assert rp.tolist() == [0, 2, 4] and ci.tolist() == [0, 1, 0, 1] and v.tolist() == [0.5] * 4
    # zeros(2x2) with self loops -> identity
    rp, ci, v = port.normalize_adjacency(np.zeros(3, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32))
    assert rp.tolist() == [0, 1, 2] and ci.tolist() == [0, 1] and v.tolist() == [1.0, 1.0]
    assert port.row_degrees(np.array([0, 2, 2], np.uint64)).tolist() == [2, 0]


# ---- reference golden fixtures ----------------------------------------------------
@pytest.mark.parametrize("name", golden_cases())
def test_oracle_matches_reference(name):
    g = load_golden(name)
    rp, ci, v, n = g["row_ptr"], g["col_idx"], g["values"], int(g["n_cols"])
    for a, b in zip(port.transpose(rp, ci, v, n), (g["t_row_ptr"], g["t_col_idx"], g["t_values"])):
        np.testing.assert_array_equal(_bits(a), _bits(b))
    assert port.is_symmetric(rp, ci, v, n) == bool(g["is_symmetric"])
    np.testing.assert_array_equal(port.balanced_row_partition(rp, 7), g["partition7"])
    for k in g["ks"]:
        x, xi = g[f"x_{k}"], g[f"xi_{k}"]
        for r in range(4):
            np.testing.assert_array_equal(_bits(port.spmm(rp, ci, v, x, r, np.float32)), _bits(g[f"spmm32_{k}_{r}"]))
            np.testing.assert_array_equal(_bits(port.spmm(rp, ci, v, x.astype(np.float64), r)), _bits(g[f"spmm64_{k}_{r}"]))
            for eo in (0, 1):
                np.testing.assert_array_equal(_bits(port.fusedmm(rp, ci, v, xi, x, eo, r, np.float32)),
                                              _bits(g[f"fused32_{k}_{eo}_{r}"]))
                np.testing.assert_array_equal(_bits(port.fusedmm(rp, ci, v, xi, x, eo, r)),
                                              _bits(g[f"fused64_{k}_{eo}_{r}"]))
        if f"spmm32spec_{k}" in g:  # specialised == trusted bitwise
            np.testing.assert_array_equal(_bits(g[f"spmm32spec_{k}"]), _bits(g[f"spmm32_{k}_0"]))
        np.testing.assert_array_equal(_bits(port.sddmm(rp, ci, v, xi, x, np.float32)), _bits(g[f"sddmm32_{k}"]))
        np.testing.assert_array_equal(_bits(port.sddmm(rp, ci, v, xi, x)), _bits(g[f"sddmm64_{k}"]))
    if f"cache_mean_1_v" in g:
        sym = bool(g["is_symmetric"])
        for a, b in zip(port.mean_operand(rp, ci, v, n, sym), (g["cache_mean_1_rp"], g["cache_mean_1_ci"], g["cache_mean_1_v"])):
            np.testing.assert_array_equal(_bits(a), _bits(b))
        for a, b in zip(port.mean_operand(rp, ci, v, n, False), (g["cache_mean_0_rp"], g["cache_mean_0_ci"], g["cache_mean_0_v"])):
            np.testing.assert_array_equal(_bits(a), _bits(b))
    if "norm_values" in g:
        for a, b in zip(port.normalize_adjacency(rp, ci, v), (g["norm_row_ptr"], g["norm_col_idx"], g["norm_values"])):
            np.testing.assert_array_equal(_bits(a), _bits(b))


def test_oracle_vs_live_reference():
    """When the compiled reference is present (oracle/_ref), compare on fresh
    random inputs too (this container; the GPU box has the .so as well)."""
    from oracle import ref
    if not ref.available("O2"):
        pytest.skip("oracle/_ref not built")
    from conftest import rand_csr
    rng = np.random.default_rng(77)
    rp, ci, v = rand_csr(rng, 200, 150, 0.05, hub_rows=(2,), empty_frac=0.2)
    x = rng.uniform(-1, 1, (150, 24)).astype(np.float32)
    for r in range(4):
        np.testing.assert_array_equal(_bits(port.spmm(rp, ci, v, x, r, np.float32)), _bits(ref.spmm_f32(rp, ci, v, x, 150, r)))
    for a, b in zip(port.transpose(rp, ci, v, 150), ref.transpose_f32(rp, ci, v, 150)):
        np.testing.assert_array_equal(_bits(a), _bits(b))
