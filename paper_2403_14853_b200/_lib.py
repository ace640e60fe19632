"""ctypes binding of the C ABI (include/sgnn_b200.h, include/sgnn_host.h).

The CUDA library is built in-tree (``paper_2403_14853_b200/libsgnn_b200.so``,
see ``build.py``).  There is no CPU fallback: if the library or a B200 is
missing, the compute entry points raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SGNN_B200_LIB") or os.path.join(_HERE, "libsgnn_b200.so")
HOST_LIB_PATH = os.path.join(_HERE, "libsgnn_host.so")

# ---- status codes <-> reference exception classes (error.hpp:9-61) ----------


class Error(RuntimeError):
    """sparsegnn::Error (error.hpp:9-12)."""


class ShapeError(Error):
    """error.hpp:15-18"""


class DispatchError(Error):
    """error.hpp:22-25"""


class ConfigError(Error):
    """error.hpp:28-31"""


class TapeError(Error):
    """error.hpp:34-37"""


class IoError(Error):
    """error.hpp:40-43"""


class ParseError(Error):
    """error.hpp:46-55: what() is "line N: <message>", .line is N."""

    def __init__(self, what: str, line: int = 0):
        super().__init__(f"line {line}: {what}")
        self.line = line


class InternalError(Error):
    """error.hpp:58-61"""


class CudaError(Error):
    """CUDA runtime/device failure (no reference analogue)."""


class UnsupportedError(Error):
    """A configuration this build does not implement."""


_STATUS = {1: ShapeError, 2: DispatchError, 3: ConfigError, 4: TapeError, 5: IoError,
           6: ParseError, 7: InternalError, 8: CudaError, 9: CudaError, 10: UnsupportedError}

SUM, MIN, MAX, MEAN = 0, 1, 2, 3
REDUCE = {"sum": SUM, "min": MIN, "max": MAX, "mean": MEAN}
EDGE_MUL, EDGE_SIGMOID_MUL = 0, 1
TRUSTED, SPECIALIZED = 0, 1
SEGMENT = 256


class Csr(C.Structure):
    _fields_ = [("n_rows", C.c_uint32), ("n_cols", C.c_uint32), ("nnz", C.c_uint64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p)]


class PlanParams(C.Structure):
    _fields_ = [("lanes", C.c_uint32), ("vec", C.c_uint32), ("unroll", C.c_uint32),
                ("path_items", C.c_uint32), ("split_rows_over", C.c_uint32),
                ("k_tile", C.c_uint32), ("block", C.c_uint32), ("scalar", C.c_uint32),
                ("occupancy", C.c_uint32)]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


class TuneEntry(C.Structure):
    _fields_ = [("params", PlanParams), ("ms", C.c_float), ("reserved", C.c_float)]


# Every symbol include/sgnn_b200.h declares, with (restype, argtypes).
P = C.c_void_p
u32, u64, i32 = C.c_uint32, C.c_uint64, C.c_int
CsrP = C.POINTER(Csr)
SIGNATURES = {
    "sgnn_abi_version": (i32, []),
    "sgnn_last_error": (C.c_char_p, []),
    "sgnn_device_info": (i32, [C.POINTER(i32)] * 4),
    "sgnn_release_scratch": (i32, [C.c_size_t]),
    "sgnn_plan_create": (i32, [CsrP, u32, C.POINTER(PlanParams), C.POINTER(P), P]),
    "sgnn_plan_destroy": (i32, [P]),
    "sgnn_plan_get_params": (i32, [P, C.POINTER(PlanParams)]),
    "sgnn_plan_stats": (i32, [P, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)]),
    "sgnn_spmm_f32": (i32, [CsrP, P, u32, u32, P, i32, P, P]),
    "sgnn_spmm_with_f32": (i32, [CsrP, P, u32, u32, P, i32, i32, u32, P, P]),
    "sgnn_tune_spmm": (i32, [CsrP, P, u32, i32, i32, C.POINTER(P), C.POINTER(TuneEntry), i32,
                             C.POINTER(i32), P]),
    "sgnn_spmm_peer_f32": (i32, [CsrP, C.POINTER(P), u32, u32, u32, P, i32, P, P]),
    "sgnn_peer_alloc": (i32, [C.c_size_t, C.POINTER(P)]),
    "sgnn_peer_free": (i32, [P]),
    "sgnn_ipc_get_handle": (i32, [P, P]),
    "sgnn_ipc_open_handle": (i32, [P, C.POINTER(P)]),
    "sgnn_ipc_close_handle": (i32, [P]),
    "sgnn_resolve_kernel": (i32, [u32, i32, C.POINTER(u32)]),
    "sgnn_set_dispatch": (None, [i32]),
    "sgnn_get_dispatch": (i32, []),
    "sgnn_selftest_count_division": (i32, [u64, u64, u32, u64, C.POINTER(u64), C.POINTER(u64), C.POINTER(u32)]),
    "sgnn_transpose_workspace": (i32, [CsrP, C.POINTER(C.c_size_t)]),
    "sgnn_csr_transpose": (i32, [CsrP, P, P, P, P, C.c_size_t, P]),
    "sgnn_row_degrees": (i32, [CsrP, P, P]),
    "sgnn_is_symmetric": (i32, [CsrP, C.POINTER(i32), P]),
    "sgnn_cache_create": (i32, [CsrP, i32, C.POINTER(P), P]),
    "sgnn_cache_create_model": (i32, [CsrP, i32, i32, i32, C.POINTER(P), P]),
    "sgnn_cache_a_hat": (i32, [P, CsrP]),
    "sgnn_normalize_adjacency": (i32, [CsrP, i32, C.POINTER(u64), P, P, P, P]),
    "sgnn_cache_destroy": (i32, [P]),
    "sgnn_cache_sum_operand": (i32, [P, CsrP, P]),
    "sgnn_cache_mean_operand": (i32, [P, CsrP, P]),
    "sgnn_cache_counters": (i32, [P, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64), C.POINTER(i32)]),
    "sgnn_spmm_backward_f32": (i32, [P, P, u32, u32, P, i32, P]),
    "sgnn_sddmm_f32": (i32, [CsrP, P, u32, P, u32, u32, P, P]),
    "sgnn_sddmm_plan_f32": (i32, [CsrP, P, u32, P, u32, u32, P, P, P]),
    "sgnn_fusedmm_f32": (i32, [CsrP, P, u32, P, u32, u32, i32, i32, P, P]),
    "sgnn_fusedmm_plan_f32": (i32, [CsrP, P, u32, P, u32, u32, i32, i32, P, P, P]),
    "sgnn_gnn_create": (i32, [CsrP, i32, u32, u32, u32, P, P, P, i32, i32, u32, C.POINTER(P), P]),
    "sgnn_gnn_set_weights": (i32, [P, P, P, P, P, C.c_float, P]),
    "sgnn_gnn_get_weights": (i32, [P, P, P, P, P, C.POINTER(C.c_float), P]),
    "sgnn_gnn_train": (i32, [P, u32, C.c_float, i32, P, P, P, P]),
    "sgnn_gnn_counters": (i32, [P, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64), C.POINTER(i32)]),
    "sgnn_gnn_destroy": (i32, [P]),
    "sgnn_comm_get_unique_id": (i32, [P]),
    "sgnn_comm_init_rank": (i32, [P, i32, i32, C.POINTER(P)]),
    "sgnn_comm_init_loopback": (i32, [i32, C.POINTER(P)]),
    "sgnn_comm_info": (i32, [P, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
    "sgnn_comm_destroy": (i32, [P]),
    "sgnn_dist_create": (i32, [P, i32, P, CsrP, CsrP, i32, u32, u32, u32, P, P, P, u32, C.POINTER(P), P]),
    "sgnn_dist_set_weights": (i32, [P, P, P, P, P, P]),
    "sgnn_dist_get_weights": (i32, [P, P, P, P, P, P]),
    "sgnn_dist_set_features": (i32, [P, P, i32, P]),
    "sgnn_dist_epochs": (i32, [P, i32, u32, C.c_float, P]),
    "sgnn_dist_stats": (i32, [P, u32, u32, P, P, P, P]),
    "sgnn_dist_stats_copy": (i32, [P, u32, u32, P, P]),
    "sgnn_dist_reset": (i32, [P]),
    "sgnn_dist_info": (i32, [P, C.POINTER(u32), C.POINTER(u32), C.POINTER(u64), C.POINTER(u64), C.POINTER(P)]),
    "sgnn_dist_destroy": (i32, [P]),
    "sgnn_dense_mm_f32": (i32, [i32, u32, u32, u32, P, P, P, P]),
    "sgnn_add_relu_f32": (i32, [P, P, u64, P, P]),
    "sgnn_sage_logits_f32": (i32, [P, P, P, P, u32, u32, u32, P, P]),
    "sgnn_softmax_xent_f32": (i32, [P, u32, u32, P, P, C.c_double, P, P, P, P]),
    "sgnn_sage_wgrad_f32": (i32, [P, P, P, u32, u32, u32, P, P, P]),
    "sgnn_sage_grad_wt_f32": (i32, [P, P, u32, u32, u32, P, P, P, P]),
}

HOST_SIGNATURES = {
    "sgnn_host_fill_uniform": (None, [P, u64, C.c_double, C.c_double, u64, u64, i32]),
    "sgnn_host_fill_normal": (None, [P, u64, C.c_double, C.c_double, u64, u64, i32]),
    "sgnn_host_er": (i32, [u32, u32, u32, u64, P, P, i32]),
    "sgnn_host_rmat_build": (P, [u32, u64, C.c_double, C.c_double, C.c_double, u64, i32, i32, i32]),
    "sgnn_host_rmat_nnz": (u64, [P]),
    "sgnn_host_rmat_export": (None, [P, P, P]),
    "sgnn_host_rmat_free": (None, [P]),
    "sgnn_host_balanced_row_partition": (None, [P, u32, i32, P]),
    "sgnn_host_weighted_row_partition": (None, [P, u32, i32, u32, P]),
    "sgnn_host_partition_block": (u64, [P, P, P, P, i32, i32, u32, P, P, P, i32]),
    "sgnn_host_mtx_load": (i32, [C.c_char_p, i32, C.POINTER(P), C.c_char_p, C.c_size_t, C.POINTER(C.c_long)]),
    "sgnn_host_csr_dims": (None, [P, C.POINTER(u32), C.POINTER(u32), C.POINTER(u64)]),
    "sgnn_host_csr_export": (None, [P, P, P, P]),
    "sgnn_host_csr_free": (None, [P]),
    "sgnn_host_mtx_save": (i32, [C.c_char_p, u32, u32, P, P, P, i32, C.c_char_p, C.c_size_t]),
    "sgnn_host_features_load": (i32, [C.c_char_p, i32, C.POINTER(P), C.c_char_p, C.c_size_t,
                                      C.POINTER(C.c_long)]),
    "sgnn_host_dense_dims": (None, [P, C.POINTER(u32), C.POINTER(u32)]),
    "sgnn_host_dense_export": (None, [P, P]),
    "sgnn_host_dense_free": (None, [P]),
    "sgnn_host_int_column_load": (i32, [C.c_char_p, i32, u64, P, C.POINTER(u64), C.c_char_p, C.c_size_t,
                                        C.POINTER(C.c_long)]),
}

_lock = threading.Lock()
_lib = None
_host = None


def _bind(path, sigs):
    if not os.path.exists(path):
        raise ImportError(
            f"{os.path.basename(path)} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the sparse hot path)")
    lib = C.CDLL(path)
    lib.missing_symbols = []
    for name, (res, args) in sigs.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            lib.missing_symbols.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The CUDA library (loads it on first use)."""
    global _lib
    with _lock:
        if _lib is None:
            _lib = _bind(LIB_PATH, SIGNATURES)
    return _lib


def host():
    global _host
    with _lock:
        if _host is None:
            _host = _bind(HOST_LIB_PATH, HOST_SIGNATURES)
    return _host


_cudart = None


def memcpy_d2h(dst: int, src: int, nbytes: int) -> None:
    """cudaMemcpy device->host (for views onto library-owned device arrays)."""
    global _cudart
    if _cudart is None:
        lib()  # make sure the runtime the library links is loaded
        for name in ("libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so"):
            try:
                _cudart = C.CDLL(name)
                break
            except OSError:
                continue
        _cudart.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    st = _cudart.cudaMemcpy(dst, src, nbytes, 2)
    if st != 0:
        raise CudaError(f"cudaMemcpy failed ({st})")


def check(status: int, what: str = "") -> None:
    if status != 0:
        msg = lib().sgnn_last_error().decode(errors="replace")
        raise _STATUS.get(status, Error)(f"{what}: {msg}" if what else msg)
