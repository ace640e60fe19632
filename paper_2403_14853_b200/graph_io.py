"""On-disk formats either side of the hot path (io.hpp:80-262), over the
native host library (include/sgnn_host.h, csrc/host/mtx.cpp):

  load_mtx / save_mtx   Matrix Market coordinate files  (io.hpp:80-185)
  load_features         "n k" dense text                (io.hpp:187-205)
  load_labels/load_mask "n" integer columns             (io.hpp:243-262)

Same acceptance rules, messages and 1-based line numbers as the reference:
failures raise IoError / ParseError (``.line``) from error.hpp's hierarchy.
The entry lines are parsed by all host cores; `load_mtx(..., device=...)`
uploads the result as an ops.CsrMatrix for the B200 kernels.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import ConfigError, IoError, ParseError

_ERR_LEN = 4096


@dataclass
class HostCsr:
    """CsrMatrix<float> on the host (types.hpp:26-79)."""
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray  # u64[n_rows + 1]
    col_idx: np.ndarray  # u32[nnz]
    values: np.ndarray   # f32[nnz]

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def to_device(self, device="cuda"):
        from . import ops
        return ops.CsrMatrix.from_numpy(self.row_ptr, self.col_idx, self.values, self.n_cols, device=device)


def _raise(status: int, err, line) -> None:
    msg = err.value.decode(errors="replace")
    if status == 6:
        raise ParseError(msg, int(line.value))
    if status == 5:
        raise IoError(msg)
    raise ConfigError(msg)


def load_mtx(path, threads: int = 0, device=None):
    """load_mtx<float> (io.hpp:80-165).  Returns a HostCsr, or an
    ops.CsrMatrix on `device` when given."""
    h = _lib.host()
    handle = C.c_void_p()
    err = C.create_string_buffer(_ERR_LEN)
    line = C.c_long(0)
    st = h.sgnn_host_mtx_load(os.fsencode(path), int(threads), C.byref(handle), err, _ERR_LEN, C.byref(line))
    if st != 0:
        _raise(st, err, line)
    try:
        m, n, nnz = C.c_uint32(), C.c_uint32(), C.c_uint64()
        h.sgnn_host_csr_dims(handle, C.byref(m), C.byref(n), C.byref(nnz))
        rp = np.empty(m.value + 1, np.uint64)
        ci = np.empty(nnz.value, np.uint32)
        v = np.empty(nnz.value, np.float32)
        h.sgnn_host_csr_export(handle, rp.ctypes.data, ci.ctypes.data, v.ctypes.data)
    finally:
        h.sgnn_host_csr_free(handle)
    a = HostCsr(m.value, n.value, rp, ci, v)
    return a.to_device(device) if device is not None else a


def save_mtx(a, path, threads: int = 0) -> None:
    """save_mtx (io.hpp:168-185): coordinate real general, %.9g values.
    `a` is a HostCsr, an ops.CsrMatrix, or (n_rows, n_cols, row_ptr, col_idx, values)."""
    if isinstance(a, tuple):
        m, n, rp, ci, v = a
    elif isinstance(a, HostCsr):
        m, n, rp, ci, v = a.n_rows, a.n_cols, a.row_ptr, a.col_idx, a.values
    else:  # ops.CsrMatrix
        rp, ci, v = a.to_numpy()
        m, n = a.n_rows, a.n_cols
    rp = np.ascontiguousarray(rp, np.uint64)
    ci = np.ascontiguousarray(ci, np.uint32)
    v = np.ascontiguousarray(v, np.float32)
    if rp.shape[0] != m + 1 or ci.shape[0] != int(rp[m]) or v.shape[0] != ci.shape[0]:
        raise ConfigError("save_mtx: row_ptr / col_idx / values sizes do not match")
    err = C.create_string_buffer(_ERR_LEN)
    st = _lib.host().sgnn_host_mtx_save(os.fsencode(path), int(m), int(n), rp.ctypes.data, ci.ctypes.data,
                                        v.ctypes.data, int(threads), err, _ERR_LEN)
    if st != 0:
        _raise(st, err, C.c_long(0))


def load_features(path, threads: int = 0) -> np.ndarray:
    """load_features<float> (io.hpp:187-205) -> f32[n, k]."""
    h = _lib.host()
    handle = C.c_void_p()
    err = C.create_string_buffer(_ERR_LEN)
    line = C.c_long(0)
    st = h.sgnn_host_features_load(os.fsencode(path), int(threads), C.byref(handle), err, _ERR_LEN,
                                   C.byref(line))
    if st != 0:
        _raise(st, err, line)
    try:
        r, c = C.c_uint32(), C.c_uint32()
        h.sgnn_host_dense_dims(handle, C.byref(r), C.byref(c))
        out = np.empty((r.value, c.value), np.float32)
        h.sgnn_host_dense_export(handle, out.ctypes.data)
    finally:
        h.sgnn_host_dense_free(handle)
    return out


def _int_column(path, kind: int) -> np.ndarray:
    h = _lib.host()
    err = C.create_string_buffer(_ERR_LEN)
    line = C.c_long(0)
    n = C.c_uint64()
    st = h.sgnn_host_int_column_load(os.fsencode(path), kind, 0, None, C.byref(n), err, _ERR_LEN, C.byref(line))
    if st != 0:
        _raise(st, err, line)
    out = np.empty(n.value, np.uint32)
    st = h.sgnn_host_int_column_load(os.fsencode(path), kind, n.value, out.ctypes.data, C.byref(n), err,
                                     _ERR_LEN, C.byref(line))
    if st != 0:
        _raise(st, err, line)
    return out


def load_labels(path) -> np.ndarray:
    """load_labels (io.hpp:243-251) -> u32[n]."""
    return _int_column(path, 0)


def load_mask(path) -> np.ndarray:
    """load_mask (io.hpp:254-262) -> u8[n] of 0/1."""
    return _int_column(path, 1).astype(np.uint8)
