"""numpy front-end to the reference itself, compiled by oracle/Makefile from
/root/reference/proj into oracle/_ref/libsgnn_ref_<flags>.so.

TEST / BASELINE INFRASTRUCTURE ONLY.  Used to pin oracle/port.py, to make
tests/golden/ fixtures (make_golden.py) and as bench.py's CPU reference arm.
The .so files are built here (where /root/reference exists) and travel to the
GPU box with the repo snapshot; nothing at run time reads /root/reference.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")
FLAVOURS = {  # name -> (file, flags, required cpu flags)
    "O2": ("libsgnn_ref_O2.so", "-O2", ()),
    "O3v3": ("libsgnn_ref_O3v3.so", "-O3 -march=x86-64-v3", ("avx2", "fma", "bmi2")),
    "O3v4": ("libsgnn_ref_O3v4.so", "-O3 -march=x86-64-v4", ("avx512f", "avx512bw", "avx512vl", "avx512dq")),
}

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_LIBS: dict = {}


def cpu_flags() -> set:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def available(flavour: str = "O2") -> bool:
    fn, _, need = FLAVOURS[flavour]
    return os.path.exists(os.path.join(REF_DIR, fn)) and set(need) <= cpu_flags()


def flavours() -> list:
    return [f for f in FLAVOURS if available(f)]


def lib(flavour: str = "O2"):
    if flavour in _LIBS:
        return _LIBS[flavour]
    if not available(flavour):
        raise FileNotFoundError(f"oracle/_ref flavour {flavour} not built or not runnable on this CPU")
    L = C.CDLL(os.path.join(REF_DIR, FLAVOURS[flavour][0]))
    L.ref_spmm_f32.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f32p, f32p, C.c_uint32, C.c_int, C.c_int, C.c_uint32, C.c_int, f32p]
    L.ref_spmm_f64.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f64p, f64p, C.c_uint32, C.c_int, C.c_int, f64p]
    L.ref_transpose_f32.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f32p, u64p, u32p, f32p]
    L.ref_sddmm_f32.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f32p, f32p, f32p, C.c_uint32, C.c_int, f32p]
    L.ref_sddmm_f64.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f64p, f64p, f64p, C.c_uint32, C.c_int, f64p]
    L.ref_fusedmm_f32.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f32p, f32p, f32p, C.c_uint32, C.c_int, C.c_int, C.c_int, f32p]
    L.ref_fusedmm_f64.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f64p, f64p, f64p, C.c_uint32, C.c_int, C.c_int, C.c_int, f64p]
    L.ref_is_symmetric_f32.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f32p]
    L.ref_normalize_adjacency_f32.argtypes = [C.c_uint32, u64p, u32p, f32p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ref_normalize_adjacency_f32.restype = C.c_int64
    L.ref_balanced_row_partition.argtypes = [u64p, C.c_uint32, C.c_int, u32p]
    L.ref_resolve_kernel.argtypes = [C.c_uint32, C.c_int, C.c_int]
    L.ref_cache_operand_f32.argtypes = [C.c_uint32, u64p, u32p, f32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p, C.c_void_p,
                                        np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")]
    L.ref_bench_create.argtypes = [C.c_uint32, C.c_uint32, u64p, u32p, f32p, f32p, f32p, C.c_uint32, C.c_int]
    L.ref_bench_create.restype = C.c_void_p
    L.ref_bench_step.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
    L.ref_bench_out.argtypes = [C.c_void_p, C.c_int]
    L.ref_bench_out.restype = C.POINTER(C.c_float)
    L.ref_bench_free.argtypes = [C.c_void_p]
    L.ref_hw_cores.restype = C.c_int
    L.ref_trainer_create.argtypes = [C.c_int, C.c_uint32, u64p, u32p, f32p, C.c_uint32, f32p, u32p,
                                     np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS"), C.c_uint32,
                                     C.c_uint32, f32p, C.c_double, C.c_int]
    L.ref_trainer_create.restype = C.c_void_p
    L.ref_trainer_epoch.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.ref_trainer_free.argtypes = [C.c_void_p]
    L.ref_sage_sample_create.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, u64p, u32p, f32p, u64p, u32p,
                                         f32p, f32p, f32p, f32p, u32p,
                                         np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS"), C.c_uint32,
                                         C.c_uint32, f32p, C.c_double, C.c_int]
    L.ref_sage_sample_create.restype = C.c_void_p
    L.ref_sage_sample_epoch.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    L.ref_sage_sample_free.argtypes = [C.c_void_p]
    _LIBS[flavour] = L
    return L


def _csr(rp, ci, v, dt):
    return (np.ascontiguousarray(rp, np.uint64), np.ascontiguousarray(ci, np.uint32),
            np.ascontiguousarray(v, dt))


def _check(st):
    if st != 0:
        raise RuntimeError(f"reference raised status {st}")


def spmm_f32(rp, ci, v, x, n_cols, reduce=0, specialized=False, threads=0, flavour="O2"):
    rp, ci, v = _csr(rp, ci, v, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    m, k = len(rp) - 1, x.shape[1]
    out = np.empty((m, k), np.float32)
    _check(lib(flavour).ref_spmm_f32(m, n_cols, rp, ci, v, x, k, reduce, int(specialized), k, threads, out))
    return out


def spmm_f64(rp, ci, v, x, n_cols, reduce=0, threads=0):
    rp, ci, v = _csr(rp, ci, v, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    m, k = len(rp) - 1, x.shape[1]
    out = np.empty((m, k), np.float64)
    _check(lib().ref_spmm_f64(m, n_cols, rp, ci, v, x, k, reduce, threads, out))
    return out


def transpose_f32(rp, ci, v, n_cols):
    rp, ci, v = _csr(rp, ci, v, np.float32)
    nnz = int(rp[-1])
    trp, tci, tv = np.empty(n_cols + 1, np.uint64), np.empty(nnz, np.uint32), np.empty(nnz, np.float32)
    _check(lib().ref_transpose_f32(len(rp) - 1, n_cols, rp, ci, v, trp, tci, tv))
    return trp, tci, tv


def sddmm(rp, ci, v, x, y, n_cols, dtype=np.float64, threads=0):
    rp, ci, v = _csr(rp, ci, v, dtype)
    x, y = np.ascontiguousarray(x, dtype), np.ascontiguousarray(y, dtype)
    out = np.empty(int(rp[-1]), dtype)
    f = lib().ref_sddmm_f64 if dtype == np.float64 else lib().ref_sddmm_f32
    _check(f(len(rp) - 1, n_cols, rp, ci, v, x, y, x.shape[1], threads, out))
    return out


def fusedmm(rp, ci, v, x, y, n_cols, edge_op=0, reduce=0, dtype=np.float64, threads=0):
    rp, ci, v = _csr(rp, ci, v, dtype)
    x, y = np.ascontiguousarray(x, dtype), np.ascontiguousarray(y, dtype)
    m, k = len(rp) - 1, x.shape[1]
    out = np.empty((m, k), dtype)
    f = lib().ref_fusedmm_f64 if dtype == np.float64 else lib().ref_fusedmm_f32
    _check(f(m, n_cols, rp, ci, v, x, y, k, edge_op, reduce, threads, out))
    return out


def is_symmetric(rp, ci, v, n_cols):
    rp, ci, v = _csr(rp, ci, v, np.float32)
    return bool(lib().ref_is_symmetric_f32(len(rp) - 1, n_cols, rp, ci, v))


def normalize_adjacency(rp, ci, v, add_self_loops=True):
    rp, ci, v = _csr(rp, ci, v, np.float32)
    n = len(rp) - 1
    nnz = lib().ref_normalize_adjacency_f32(n, rp, ci, v, int(add_self_loops), None, None, None)
    if nnz < 0:
        raise RuntimeError(f"reference raised status {-nnz}")
    trp, tci, tv = np.empty(n + 1, np.uint64), np.empty(nnz, np.uint32), np.empty(nnz, np.float32)
    lib().ref_normalize_adjacency_f32(n, rp, ci, v, int(add_self_loops), trp.ctypes.data, tci.ctypes.data, tv.ctypes.data)
    return trp, tci, tv


def balanced_row_partition(rp, n_chunks):
    rp = np.ascontiguousarray(rp, np.uint64)
    out = np.empty(n_chunks + 1, np.uint32)
    lib().ref_balanced_row_partition(rp, len(rp) - 1, n_chunks, out)
    return out


def resolve_kernel(k, reduce, tuned_enabled):
    r = lib().ref_resolve_kernel(k, reduce, int(tuned_enabled))
    return ("specialized" if r >= 65536 else "trusted", r % 65536)


def cache_operand(rp, ci, v, model_kind, use_cache, which, n_fetches):
    """build_cache + sum_operand/mean_operand fetched n_fetches times (gnn.hpp:113-196).
    Returns (row_ptr, col_idx, values, counters{transpose_builds, normalize_builds, cache_hits, symmetric})."""
    rp, ci, v = _csr(rp, ci, v, np.float32)
    n = len(rp) - 1
    nnz = C.c_uint64(0)
    cnt = np.zeros(4, np.uint64)
    _check(lib().ref_cache_operand_f32(n, rp, ci, v, model_kind, int(use_cache), which, n_fetches,
                                       C.byref(nnz), None, None, None, cnt))
    trp, tci, tv = np.empty(n + 1, np.uint64), np.empty(nnz.value, np.uint32), np.empty(nnz.value, np.float32)
    _check(lib().ref_cache_operand_f32(n, rp, ci, v, model_kind, int(use_cache), which, n_fetches,
                                       C.byref(nnz), trp.ctypes.data, tci.ctypes.data, tv.ctypes.data, cnt))
    return trp, tci, tv, dict(zip(("transpose_builds", "normalize_builds", "cache_hits", "symmetric"),
                                  (int(c) for c in cnt)))


MODEL_KINDS = {"gcn": 0, "sage-sum": 1, "sage-mean": 2, "gin": 3}


def _gnn_sigs(L):
    if getattr(L, "_gnn_bound", False):
        return
    L.ref_init_model.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, f32p]
    L.ref_train.argtypes = [C.c_int, C.c_uint32, u64p, u32p, f32p, C.c_uint32, f32p, u32p,
                            np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS"), C.c_uint32, C.c_uint32,
                            f32p, C.c_int, C.c_double, C.c_int, C.c_int, f64p, f64p, f32p,
                            np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")]
    L.ref_synth_planted.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_uint32, C.c_double, C.c_uint64]
    L.ref_synth_planted.restype = C.c_void_p
    L.ref_dataset_nnz.argtypes = [C.c_void_p]
    L.ref_dataset_nnz.restype = C.c_uint64
    L.ref_dataset_export.argtypes = [C.c_void_p, u64p, u32p, f32p, f32p, u32p,
                                     np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")]
    L.ref_dataset_free.argtypes = [C.c_void_p]
    L._gnn_bound = True


def _n_weights(kind, in_f, hidden, classes):
    n = in_f * hidden + hidden * classes
    return 2 * n if kind in ("sage-sum", "sage-mean") else n


def init_model(kind, in_f, hidden, classes, seed):
    """init_model (gnn.hpp:75-99): packed w1|w2|(w1_self|w2_self)."""
    L = lib()
    _gnn_sigs(L)
    out = np.empty(_n_weights(kind, in_f, hidden, classes), np.float32)
    _check(L.ref_init_model(MODEL_KINDS[kind], in_f, hidden, classes, seed, out))
    return out


def synth_planted(n, classes, p_intra, p_inter, feat_dim, noise, seed):
    """synth_planted (io.hpp:315-378) -> (rp, ci, v, x, labels, mask)."""
    L = lib()
    _gnn_sigs(L)
    h = L.ref_synth_planted(n, classes, p_intra, p_inter, feat_dim, noise, seed)
    if not h:
        raise RuntimeError("synth_planted failed")
    try:
        nnz = L.ref_dataset_nnz(h)
        rp, ci, v = np.empty(n + 1, np.uint64), np.empty(nnz, np.uint32), np.empty(nnz, np.float32)
        x, lab, mask = np.empty((n, feat_dim), np.float32), np.empty(n, np.uint32), np.empty(n, np.uint8)
        L.ref_dataset_export(h, rp, ci, v, x, lab, mask)
    finally:
        L.ref_dataset_free(h)
    return rp, ci, v, x, lab, mask


def train(kind, rp, ci, v, x, labels, mask, hidden, classes, w_init, epochs, lr, use_cache=True,
          threads=0):
    """train (gnn.hpp:414-438) from w_init; returns (losses, accs, w_final, counters)."""
    L = lib()
    _gnn_sigs(L)
    rp, ci, v = _csr(rp, ci, v, np.float32)
    n, in_f = x.shape
    losses, accs = np.empty(epochs), np.empty(epochs)
    w_out = np.empty_like(np.asarray(w_init, np.float32))
    cnt = np.zeros(3, np.uint64)
    _check(L.ref_train(MODEL_KINDS[kind], n, rp, ci, v, in_f, np.ascontiguousarray(x, np.float32),
                       np.ascontiguousarray(labels, np.uint32), np.ascontiguousarray(mask, np.uint8),
                       hidden, classes, np.ascontiguousarray(w_init, np.float32), epochs, lr,
                       int(use_cache), threads, losses, accs, w_out, cnt))
    return losses, accs, w_out, dict(zip(("transpose_builds", "normalize_builds", "cache_hits"), (int(c) for c in cnt)))


class Trainer:
    """The reference's train() (gnn.hpp:414-438), one epoch-loop iteration per
    `epoch()` call (bench.py's GNN-epoch reference arm).  build_cache runs in
    the constructor, outside any timed region."""

    def __init__(self, kind, rp, ci, v, x, labels, mask, hidden, classes, w_init, lr=0.05, threads=0,
                 flavour="O2"):
        self.L = lib(flavour)
        rp, ci, v = _csr(rp, ci, v, np.float32)
        n, in_f = x.shape
        self.h = self.L.ref_trainer_create(MODEL_KINDS[kind], n, rp, ci, v, in_f, np.ascontiguousarray(x, np.float32),
                                           np.ascontiguousarray(labels, np.uint32),
                                           np.ascontiguousarray(mask, np.uint8), hidden, classes,
                                           np.ascontiguousarray(w_init, np.float32), lr, threads)
        if not self.h:
            raise RuntimeError("ref_trainer_create failed")

    def epoch(self):
        loss, acc = C.c_double(), C.c_double()
        _check(self.L.ref_trainer_epoch(self.h, C.byref(loss), C.byref(acc)))
        return loss.value, acc.value

    def close(self):
        if getattr(self, "h", None):
            self.L.ref_trainer_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


class SageSample:
    """A row sample R of the SAGE epoch on the reference's own functions
    (ref_shim.cpp ref_sage_sample_*): rows R of A_hat and of the backward
    operand (|R| x n), full-height X and stand-in operands, |R|-row dense work."""

    def __init__(self, kind, n, a_r, m_r, x, x_r, stand_in, labels_r, mask_r, hidden, classes, w_init, lr=0.05,
                 threads=0, flavour="O2"):
        self.L = lib(flavour)
        rpa, cia, va = _csr(*a_r, np.float32)
        rpm, cim, vm = _csr(*m_r, np.float32)
        self.rows = len(rpa) - 1
        self.h = self.L.ref_sage_sample_create(
            MODEL_KINDS[kind], n, x.shape[1], self.rows, rpa, cia, va, rpm, cim, vm,
            np.ascontiguousarray(x, np.float32), np.ascontiguousarray(x_r, np.float32),
            np.ascontiguousarray(stand_in, np.float32), np.ascontiguousarray(labels_r, np.uint32),
            np.ascontiguousarray(mask_r, np.uint8), hidden, classes, np.ascontiguousarray(w_init, np.float32), lr,
            threads)
        if not self.h:
            raise RuntimeError("ref_sage_sample_create failed")

    def epoch(self):
        loss = C.c_double()
        _check(self.L.ref_sage_sample_epoch(self.h, C.byref(loss)))
        return loss.value

    def close(self):
        if getattr(self, "h", None):
            self.L.ref_sage_sample_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


class Bench:
    """SpMM fwd + cached-transpose bwd on the reference CPU path (bench.py arm)."""

    def __init__(self, rp, ci, v, n_cols, x, g, reduce=0, flavour="O2"):
        self.L = lib(flavour)
        rp, ci, v = _csr(rp, ci, v, np.float32)
        self.m, self.k = len(rp) - 1, x.shape[1]
        self.n = n_cols
        self.h = self.L.ref_bench_create(self.m, n_cols, rp, ci, v, np.ascontiguousarray(x, np.float32),
                                         np.ascontiguousarray(g, np.float32), self.k, reduce)

    def step(self, specialized=False, threads=0, which=3):
        _check(self.L.ref_bench_step(self.h, int(specialized), threads, which))

    def out(self, which=1):
        rows = self.m if which == 1 else self.n
        p = self.L.ref_bench_out(self.h, which)
        return np.ctypeslib.as_array(p, shape=(rows, self.k)).copy()

    def close(self):
        if self.h:
            self.L.ref_bench_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


# ---- on-disk formats (io.hpp:80-262) through the reference's own loaders ----
class RefError(Exception):
    """A reference exception: .status (5 IoError, 6 ParseError), .what, .line."""

    def __init__(self, status, what, line):
        super().__init__(f"[{status}] {what}")
        self.status, self.what, self.line = status, what, line


def _io_sigs(L):
    if getattr(L, "_io_ready", False):
        return L
    P, s, cp, sz, lp = C.c_void_p, C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_long)
    L.ref_load_mtx.argtypes = [s, C.POINTER(P), cp, sz, lp]
    L.ref_csr_dims.argtypes = [P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)]
    L.ref_csr_export.argtypes = [P, P, P, P]
    L.ref_csr_free.argtypes = [P]
    L.ref_save_mtx.argtypes = [s, C.c_uint32, C.c_uint32, P, P, P, cp, sz]
    L.ref_load_features.argtypes = [s, C.POINTER(P), cp, sz, lp]
    L.ref_dense_dims.argtypes = [P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
    L.ref_dense_export.argtypes = [P, P]
    L.ref_dense_free.argtypes = [P]
    L.ref_load_int_column.argtypes = [s, C.c_int, P, C.POINTER(C.c_uint64), cp, sz, lp]
    L._io_ready = True
    return L


def _fail(st, err, line):
    raise RefError(st, err.value.decode(errors="replace"), int(line.value))


def load_mtx(path):
    """(n_rows, n_cols, rp, ci, v) from the reference's load_mtx<float>."""
    L = _io_sigs(lib())
    h, err, line = C.c_void_p(), C.create_string_buffer(4096), C.c_long(0)
    st = L.ref_load_mtx(os.fsencode(path), C.byref(h), err, 4096, C.byref(line))
    if st:
        _fail(st, err, line)
    m, n, nnz = C.c_uint32(), C.c_uint32(), C.c_uint64()
    L.ref_csr_dims(h, C.byref(m), C.byref(n), C.byref(nnz))
    rp = np.empty(m.value + 1, np.uint64)
    ci = np.empty(nnz.value, np.uint32)
    v = np.empty(nnz.value, np.float32)
    L.ref_csr_export(h, rp.ctypes.data, ci.ctypes.data, v.ctypes.data)
    L.ref_csr_free(h)
    return m.value, n.value, rp, ci, v


def save_mtx(path, n_rows, n_cols, rp, ci, v):
    L = _io_sigs(lib())
    rp, ci, v = _csr(rp, ci, v, np.float32)
    err = C.create_string_buffer(4096)
    st = L.ref_save_mtx(os.fsencode(path), n_rows, n_cols, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, err, 4096)
    if st:
        _fail(st, err, C.c_long(0))


def load_features(path):
    L = _io_sigs(lib())
    h, err, line = C.c_void_p(), C.create_string_buffer(4096), C.c_long(0)
    st = L.ref_load_features(os.fsencode(path), C.byref(h), err, 4096, C.byref(line))
    if st:
        _fail(st, err, line)
    r, c = C.c_uint32(), C.c_uint32()
    L.ref_dense_dims(h, C.byref(r), C.byref(c))
    out = np.empty((r.value, c.value), np.float32)
    L.ref_dense_export(h, out.ctypes.data)
    L.ref_dense_free(h)
    return out


def load_int_column(path, kind):
    L = _io_sigs(lib())
    err, line, n = C.create_string_buffer(4096), C.c_long(0), C.c_uint64()
    st = L.ref_load_int_column(os.fsencode(path), kind, None, C.byref(n), err, 4096, C.byref(line))
    if st:
        _fail(st, err, line)
    out = np.empty(n.value, np.uint32)
    L.ref_load_int_column(os.fsencode(path), kind, out.ctypes.data, C.byref(n), err, 4096, C.byref(line))
    return out
