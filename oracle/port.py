"""numpy front-end to liboracle.so (oracle/sgnn_oracle.c).

TEST INFRASTRUCTURE ONLY -- the checker, never the product.  Each wrapper
names the reference function it restates; see sgnn_oracle.c for file:line.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

SUM, MIN, MAX, MEAN = 0, 1, 2, 3
EDGE_MUL, EDGE_SIGMOID_MUL = 0, 1


def build() -> str:
    path = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "sgnn_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.check_call(["make", "-C", _HERE, "oracle"], stdout=subprocess.DEVNULL)
    return path


def lib():
    global _LIB
    if _LIB is None:
        L = C.CDLL(build())
        for suf, fp in (("f64", f64p), ("f32", f32p)):
            getattr(L, f"orc_spmm_{suf}").argtypes = [C.c_uint32, u64p, u32p, fp, fp, C.c_uint32, C.c_int, fp]
            getattr(L, f"orc_transpose_{suf}").argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, fp, u64p, u32p, fp]
            getattr(L, f"orc_sddmm_{suf}").argtypes = [C.c_uint32, u64p, u32p, fp, fp, fp, C.c_uint32, fp]
            getattr(L, f"orc_fusedmm_{suf}").argtypes = [C.c_uint32, u64p, u32p, fp, fp, fp, C.c_uint32, C.c_int, C.c_int, fp]
        L.orc_spmm_absdenom_f64.argtypes = [C.c_uint32, u64p, u32p, f64p, f64p, C.c_uint32, C.c_int, f64p]
        L.orc_sddmm_absdenom_f64.argtypes = [C.c_uint32, u64p, u32p, f64p, f64p, f64p, C.c_uint32, f64p]
        L.orc_fusedmm_absdenom_f64.argtypes = [C.c_uint32, u64p, u32p, f64p, f64p, f64p, C.c_uint32, C.c_int, C.c_int, f64p]
        L.orc_row_degrees.argtypes = [C.c_uint32, u64p, u32p]
        L.orc_is_symmetric_f32.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f32p]
        L.orc_is_symmetric_f32.restype = C.c_int
        L.orc_mean_scale_f32.argtypes = [C.c_uint64, u32p, u32p, f32p]
        L.orc_balanced_row_partition.argtypes = [u64p, C.c_uint32, C.c_int, u32p]
        L.orc_normalize_adjacency_f32.argtypes = [C.c_uint32, u64p, u32p, f32p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_normalize_adjacency_f32.restype = C.c_uint64
        _LIB = L
    return _LIB


def _csr(rp, ci, v, dt):
    return (np.ascontiguousarray(rp, np.uint64), np.ascontiguousarray(ci, np.uint32),
            np.ascontiguousarray(v, dt))


def spmm(rp, ci, v, x, reduce=SUM, dtype=np.float64):
    """spmm / spmm_rows_trusted (kernels.hpp:45-91,179-182)."""
    rp, ci, v = _csr(rp, ci, v, dtype)
    x = np.ascontiguousarray(x, dtype)
    m, k = len(rp) - 1, x.shape[1]
    out = np.empty((m, k), dtype)
    getattr(lib(), "orc_spmm_" + ("f64" if dtype == np.float64 else "f32"))(m, rp, ci, v, x, k, reduce, out)
    return out


def spmm_absdenom(rp, ci, v, x, reduce=SUM):
    """sum_j |a_ij x_jk| in fp64 (the parity tolerance denominator)."""
    rp, ci, v = _csr(rp, ci, v, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    m, k = len(rp) - 1, x.shape[1]
    out = np.empty((m, k), np.float64)
    lib().orc_spmm_absdenom_f64(m, rp, ci, v, x, k, reduce, out)
    return out


def transpose(rp, ci, v, n_cols, dtype=np.float32):
    """transpose (sparse.hpp:72-89): stable counting sort by column."""
    rp, ci, v = _csr(rp, ci, v, dtype)
    m, nnz = len(rp) - 1, int(rp[-1])
    trp = np.empty(n_cols + 1, np.uint64)
    tci = np.empty(nnz, np.uint32)
    tv = np.empty(nnz, dtype)
    getattr(lib(), "orc_transpose_" + ("f64" if dtype == np.float64 else "f32"))(m, n_cols, rp, ci, v, trp, tci, tv)
    return trp, tci, tv


def sddmm(rp, ci, v, x, y, dtype=np.float64):
    """sddmm (kernels.hpp:187-210): values only; the pattern is P's."""
    rp, ci, v = _csr(rp, ci, v, dtype)
    x = np.ascontiguousarray(x, dtype)
    y = np.ascontiguousarray(y, dtype)
    out = np.empty(int(rp[-1]), dtype)
    getattr(lib(), "orc_sddmm_" + ("f64" if dtype == np.float64 else "f32"))(len(rp) - 1, rp, ci, v, x, y, x.shape[1], out)
    return out


def sddmm_absdenom(rp, ci, v, x, y):
    rp, ci, v = _csr(rp, ci, v, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    out = np.empty(int(rp[-1]), np.float64)
    lib().orc_sddmm_absdenom_f64(len(rp) - 1, rp, ci, v, x, y, x.shape[1], out)
    return out


def fusedmm(rp, ci, v, x, y, edge_op=EDGE_MUL, reduce=SUM, dtype=np.float64):
    """fusedmm (kernels.hpp:216-270)."""
    rp, ci, v = _csr(rp, ci, v, dtype)
    x = np.ascontiguousarray(x, dtype)
    y = np.ascontiguousarray(y, dtype)
    m, k = len(rp) - 1, x.shape[1]
    out = np.empty((m, k), dtype)
    getattr(lib(), "orc_fusedmm_" + ("f64" if dtype == np.float64 else "f32"))(m, rp, ci, v, x, y, k, edge_op, reduce, out)
    return out


def fusedmm_absdenom(rp, ci, v, x, y, edge_op=EDGE_MUL, reduce=SUM):
    rp, ci, v = _csr(rp, ci, v, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    m, k = len(rp) - 1, x.shape[1]
    out = np.empty((m, k), np.float64)
    lib().orc_fusedmm_absdenom_f64(m, rp, ci, v, x, y, k, edge_op, reduce, out)
    return out


def row_degrees(rp):
    """row_degrees (sparse.hpp:105-109)."""
    rp = np.ascontiguousarray(rp, np.uint64)
    out = np.empty(len(rp) - 1, np.uint32)
    lib().orc_row_degrees(len(rp) - 1, rp, out)
    return out


def is_symmetric(rp, ci, v, n_cols):
    """is_symmetric (sparse.hpp:179-192)."""
    rp, ci, v = _csr(rp, ci, v, np.float32)
    return bool(lib().orc_is_symmetric_f32(len(rp) - 1, n_cols, rp, ci, v))


def mean_operand(rp, ci, v, n_cols, symmetric):
    """TrainingCache::mean_operand (gnn.hpp:149-172): (transpose unless
    symmetric) then values[e] /= deg_A[col_idx[e]]."""
    if symmetric:
        trp, tci, tv = (np.array(rp, np.uint64), np.array(ci, np.uint32), np.array(v, np.float32))
    else:
        trp, tci, tv = transpose(rp, ci, v, n_cols, np.float32)
    deg = row_degrees(rp)
    lib().orc_mean_scale_f32(len(tv), tci, deg, tv)
    return trp, tci, tv


def balanced_row_partition(rp, n_chunks):
    """balanced_row_partition (parallel.hpp:28-41)."""
    rp = np.ascontiguousarray(rp, np.uint64)
    out = np.empty(n_chunks + 1, np.uint32)
    lib().orc_balanced_row_partition(rp, len(rp) - 1, n_chunks, out)
    return out


def normalize_adjacency(rp, ci, v, add_self_loops=True):
    """normalize_adjacency (sparse.hpp:116-174)."""
    rp, ci, v = _csr(rp, ci, v, np.float32)
    n = len(rp) - 1
    nnz = lib().orc_normalize_adjacency_f32(n, rp, ci, v, int(add_self_loops), None, None, None)
    trp = np.empty(n + 1, np.uint64)
    tci = np.empty(nnz, np.uint32)
    tv = np.empty(nnz, np.float32)
    lib().orc_normalize_adjacency_f32(n, rp, ci, v, int(add_self_loops), trp.ctypes.data,
                                      tci.ctypes.data, tv.ctypes.data)
    return trp, tci, tv
