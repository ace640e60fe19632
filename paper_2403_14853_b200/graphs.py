"""Deterministic synthetic inputs for the BASELINE configs (host C++ generators,
include/sgnn_host.h).  The paper's datasets are not available offline; seeded
synthetic graphs with BASELINE.json's shapes and value distributions stand in
(SURVEY 6, 8d, Appendix A).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib


def _h():
    return _lib.host()


def uniform(n: int, lo: float, hi: float, seed: int, stream: int = 0, threads: int = 0) -> np.ndarray:
    out = np.empty(int(n), np.float32)
    _h().sgnn_host_fill_uniform(out.ctypes.data, out.size, lo, hi, seed, stream, threads)
    return out


def normal(n: int, mean: float, std: float, seed: int, stream: int = 0, threads: int = 0) -> np.ndarray:
    out = np.empty(int(n), np.float32)
    _h().sgnn_host_fill_normal(out.ctypes.data, out.size, mean, std, seed, stream, threads)
    return out


def er(n_rows: int, n_cols: int, deg: int, seed: int, threads: int = 0):
    """Exactly `deg` distinct uniform columns per row (BASELINE cfg1)."""
    rp = np.empty(n_rows + 1, np.uint64)
    ci = np.empty(n_rows * deg, np.uint32)
    st = _h().sgnn_host_er(n_rows, n_cols, deg, seed, rp.ctypes.data, ci.ctypes.data, threads)
    if st:
        raise _lib.ConfigError("er: deg exceeds n_cols")
    return rp, ci


def rmat(scale: int, n_samples: int, a=0.57, b=0.19, c=0.19, seed=1, symmetrize=False,
         self_loops=False, threads: int = 0):
    """R-MAT on 2^scale nodes, duplicates removed, no vertex permutation."""
    h = _h().sgnn_host_rmat_build(scale, n_samples, a, b, c, seed, int(symmetrize), int(self_loops), threads)
    if not h:
        raise _lib.ConfigError("rmat: bad scale")
    try:
        nnz = _h().sgnn_host_rmat_nnz(h)
        rp = np.empty((1 << scale) + 1, np.uint64)
        ci = np.empty(nnz, np.uint32)
        _h().sgnn_host_rmat_export(h, rp.ctypes.data, ci.ctypes.data)
    finally:
        _h().sgnn_host_rmat_free(h)
    return rp, ci


def balanced_row_partition(rp: np.ndarray, n_chunks: int) -> np.ndarray:
    """balanced_row_partition (parallel.hpp:28-41) in the host library."""
    rp = np.ascontiguousarray(rp, np.uint64)
    out = np.empty(n_chunks + 1, np.uint32)
    _h().sgnn_host_balanced_row_partition(rp.ctypes.data, len(rp) - 1, n_chunks, out.ctypes.data)
    return out


@dataclass
class Workload:
    name: str
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    n_cols: int
    k: int
    seed: int
    notes: dict = field(default_factory=dict)

    @property
    def n_rows(self):
        return len(self.row_ptr) - 1

    @property
    def nnz(self):
        return int(self.row_ptr[-1])


def cfg1(seed: int = 1) -> Workload:
    """SpMM, ER 16384^2 with exactly 16 distinct cols/row, vals U[-1,1], K=32."""
    n, deg = 16384, 16
    rp, ci = er(n, n, deg, seed)
    v = uniform(len(ci), -1.0, 1.0, seed, stream=11)
    return Workload("cfg1_er16384_d16_k32", rp, ci, v, n, 32, seed,
                    {"graph": "ER, 16 distinct uniform cols/row", "values": "U[-1,1]", "X": "U[-1,1]"})


def cfg2(seed: int = 1) -> Workload:
    """SpMM fwd+bwd, R-MAT 2^18 with N*256 samples (a,b,c,d)=(.57,.19,.19,.05),
    duplicates removed (~50.07M nnz, not the pre-dedup 67M), values 1.0, K=128."""
    scale = 18
    rp, ci = rmat(scale, (1 << scale) * 256, seed=seed)
    v = np.ones(len(ci), np.float32)
    return Workload("cfg2_rmat18_d256_k128", rp, ci, v, 1 << scale, 128, seed,
                    {"graph": "R-MAT scale 18, N*256 samples, dedup, no permutation", "values": "1.0",
                     "X": "N(0,1)", "samples": (1 << scale) * 256})


def cfg4(seed: int = 1) -> Workload:
    """SDDMM/FusedMM, R-MAT 2^20 with N*32 samples, dedup; a_ij U[0,1]; K=64."""
    scale = 20
    rp, ci = rmat(scale, (1 << scale) * 32, seed=seed)
    v = uniform(len(ci), 0.0, 1.0, seed, stream=41)
    return Workload("cfg4_rmat20_d32_k64", rp, ci, v, 1 << scale, 64, seed,
                    {"graph": "R-MAT scale 20, N*32 samples, dedup", "values": "U[0,1]", "X,Y": "N(0,0.1)"})


def cfg3_graph(seed: int = 1):
    """GCN layer: R-MAT 2^20, N*25 samples, symmetrised, dedup (A before normalisation)."""
    scale = 20
    return rmat(scale, (1 << scale) * 25, seed=seed, symmetrize=True)


def gcn_normalize_ones(rp_a, ci_a, rp_t, ci_t):
    """A_hat = D^-1/2 (A + I) D^-1/2 for a 0/1 matrix A (structure rp_a/ci_a),
    given the structure of A+I (rp_t/ci_t, duplicates removed).  Follows
    normalize_adjacency (sparse.hpp:116-174): a diagonal already present in A
    gets value 1+1, degrees are value sums in double, entries are
    v * (s_i * s_j) in double, then rounded to fp32."""
    n = len(rp_t) - 1
    rows_a = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp_a.astype(np.int64)))
    has_diag = np.zeros(n, np.float64)
    has_diag[rows_a[ci_a.astype(np.int64) == rows_a]] = 1.0
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp_t.astype(np.int64)))
    ci64 = ci_t.astype(np.int64)
    val = np.ones(len(ci_t), np.float64)
    diag = ci64 == rows
    val[diag] += has_diag[rows[diag]]
    d = np.bincount(rows, weights=val, minlength=n)
    inv = np.where(d > 0, 1.0 / np.sqrt(np.maximum(d, 1e-300)), 0.0)
    return (val * (inv[rows] * inv[ci64])).astype(np.float32)


def cfg3(seed: int = 1) -> Workload:
    """GCN layer operand: A_hat = D^-1/2 (A+I) D^-1/2 of the symmetrised
    R-MAT 2^20 (N*25 samples) graph; K=256 (H W is 2^20 x 256)."""
    scale = 20
    rp_a, ci_a = cfg3_graph(seed)
    rp, ci = rmat(scale, (1 << scale) * 25, seed=seed, symmetrize=True, self_loops=True)
    v = gcn_normalize_ones(rp_a, ci_a, rp, ci)
    return Workload("cfg3_gcn_rmat20_sym_k256", rp, ci, v, 1 << scale, 256, seed,
                    {"graph": "R-MAT scale 20, N*25 samples, symmetrised, A_hat = D^-1/2(A+I)D^-1/2",
                     "H": "N(0,1)"})


def cfg5(seed: int = 1) -> Workload:
    """GraphSAGE-mean: R-MAT 2^22, N*25 samples, symmetrised + self loops, dedup, values 1, K=128."""
    scale = 22
    rp, ci = rmat(scale, (1 << scale) * 25, seed=seed, symmetrize=True, self_loops=True)
    v = np.ones(len(ci), np.float32)
    return Workload("cfg5_rmat22_sym_self_k128", rp, ci, v, 1 << scale, 128, seed,
                    {"graph": "R-MAT scale 22, N*25 samples, symmetrised, self loops, dedup", "values": "1.0"})
