"""Python mirror of the reference operator API over device tensors.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/sparsegnn/ (kernels.hpp, sparse.hpp, gnn.hpp,
autotune.hpp); every call goes through the C ABI of libsgnn_b200.so
(include/sgnn_b200.h).  torch supplies device memory and the stream only.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import (ConfigError, DispatchError, Error, InternalError, ShapeError,  # noqa: F401
                   TapeError, check, lib)

__all__ = [
    "CsrMatrix", "KernelKind", "Plan", "TrainingCache", "DispatchGuard", "spmm", "spmm_with",
    "spmm_into", "resolve_kernel", "set_dispatch", "get_dispatch", "transpose", "row_degrees",
    "is_symmetric", "sddmm", "fusedmm", "specialization_sweep", "spmm_plan", "spmm_peer", "release_scratch",
]

specialization_sweep = (16, 32, 64, 128, 256, 512, 1024)  # kernels.hpp:27


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


_NAMES = {0: "sum", 1: "min", 2: "max", 3: "mean"}


def _reduce(r) -> int:
    if isinstance(r, str):
        if r not in _lib.REDUCE:  # types.hpp:129-135 parse_reduce_op
            raise ConfigError(f"unknown reduce op '{r}' (expected sum|min|max|mean)")
        return _lib.REDUCE[r]
    return int(r)


def _dense(t: torch.Tensor, what: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ConfigError(f"{what}: expected a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.float32 or t.dim() != 2:
        raise ConfigError(f"{what}: expected a 2-D float32 tensor")
    if not t.is_contiguous():
        raise ConfigError(f"{what}: expected a row-major contiguous tensor")
    return t


def _on(a: "CsrMatrix", what: str, *ts: torch.Tensor) -> None:
    """Every dense operand on the sparse operand's device (a kernel would
    otherwise read another device's pointers)."""
    rp = getattr(a, "row_ptr", None)  # (a TrainingCache view holds raw device pointers only)
    if rp is None:
        return
    dev = rp.device
    for t in ts:
        if t.device != dev:
            raise ConfigError(f"{what}: operand on {t.device}, sparse operand on {dev}")


def _out(out: torch.Tensor, shape, what: str) -> torch.Tensor:
    _dense(out, f"{what} out")
    if tuple(out.shape) != tuple(shape):
        raise ShapeError(f"{what}: output is {tuple(out.shape)}, expected {tuple(shape)}")
    return out


class CsrMatrix:
    """CsrMatrix<float> on the device (types.hpp:26-79): row_ptr u64 (stored
    as int64), col_idx u32 (stored as int32), values f32."""

    def __init__(self, n_rows: int, n_cols: int, row_ptr: torch.Tensor, col_idx: torch.Tensor,
                 values: torch.Tensor):
        if row_ptr.numel() != n_rows + 1:
            raise ConfigError(f"csr: row_ptr has length {row_ptr.numel()}, expected n_rows+1 = {n_rows + 1}")
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_ptr = row_ptr.contiguous()
        self.col_idx = col_idx.contiguous()
        self.values = values.contiguous()
        self._cstruct = None
        self._plans = {}  # (kind, K) -> Plan; the structure is immutable once wrapped

    def plan(self, k: int, kind: str = "default") -> "Plan":
        """Cached work split for this matrix: "default" (trusted), "tuned"
        (registered by run_tuning / register_plan, else default) or "fused"
        (register layout holding all of K, for FusedMM)."""
        if kind == "tuned":
            return self._plans.get(("tuned", int(k))) or self.plan(k)
        key = (kind, int(k))
        if key not in self._plans:
            if kind == "fused":
                self._plans[key] = Plan(self, k, **_fused_layout(int(k)))
            else:
                self._plans[key] = Plan(self, k)
        return self._plans[key]

    def register_plan(self, k: int, plan: "Plan") -> None:
        self._plans[("tuned", int(k))] = plan

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    @classmethod
    def from_numpy(cls, row_ptr, col_idx, values, n_cols, device="cuda"):
        rp = torch.from_numpy(np.ascontiguousarray(row_ptr, np.uint64).view(np.int64)).to(device)
        ci = torch.from_numpy(np.ascontiguousarray(col_idx, np.uint32).view(np.int32)).to(device)
        v = torch.from_numpy(np.ascontiguousarray(values, np.float32)).to(device)
        return cls(len(row_ptr) - 1, n_cols, rp, ci, v)

    def to_numpy(self):
        return (self.row_ptr.cpu().numpy().view(np.uint64), self.col_idx.cpu().numpy().view(np.uint32),
                self.values.cpu().numpy())

    def c(self) -> _lib.Csr:
        if self._cstruct is None:
            self._cstruct = _lib.Csr(self.n_rows, self.n_cols, self.nnz, self.row_ptr.data_ptr(),
                                     self.col_idx.data_ptr() if self.nnz else 0,
                                     self.values.data_ptr() if self.nnz else 0)
        return self._cstruct

    def with_values(self, values: torch.Tensor) -> "CsrMatrix":
        return CsrMatrix(self.n_rows, self.n_cols, self.row_ptr, self.col_idx, values)


def _fused_layout(k: int) -> dict:
    """Register layout holding all of K (csrc/fused.cu full_k_layout)."""
    if k % 4:
        v = 1 if k <= 32 else 2 if k <= 64 else 4 if k <= 128 else 8
        return {"lanes": 32, "vec": v, "unroll": 4 if v <= 2 else 2, "scalar": 1}
    for lim, lanes, vec, unroll in ((16, 4, 1, 8), (32, 8, 1, 8), (64, 16, 1, 8), (128, 32, 1, 8),
                                    (256, 32, 2, 4), (512, 32, 4, 4), (1024, 32, 8, 2)):
        if k <= lim:
            return {"lanes": lanes, "vec": vec, "unroll": unroll}
    raise _lib.UnsupportedError(f"fusedmm: K={k} exceeds the register-resident width")


@dataclass(frozen=True)
class KernelKind:
    """KernelKind (kernels.hpp:14-25)."""
    tag: str = "trusted"
    k: int = 0

    @staticmethod
    def trusted():
        return KernelKind("trusted", 0)

    @staticmethod
    def specialized(k: int):
        return KernelKind("specialized", int(k))

    def is_specialized(self) -> bool:
        return self.tag == "specialized"


class Plan:
    """A tuned/untuned SpMM work split for (A, K) (sgnn_plan_create)."""

    def __init__(self, a: CsrMatrix, k: int, **params):
        self.a, self.k = a, int(k)
        pp = _lib.PlanParams(**{k_: int(v) for k_, v in params.items()})
        h = C.c_void_p()
        check(lib().sgnn_plan_create(C.byref(a.c()), self.k, C.byref(pp), C.byref(h), _stream()),
              "plan_create")
        self.handle = h

    @property
    def params(self) -> dict:
        pp = _lib.PlanParams()
        check(lib().sgnn_plan_get_params(self.handle, C.byref(pp)))
        return pp.as_dict()

    @property
    def stats(self) -> dict:
        w, f, s = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().sgnn_plan_stats(self.handle, C.byref(w), C.byref(f), C.byref(s)))
        return {"workers": w.value, "split_rows": f.value, "slots": s.value}

    def close(self):
        if getattr(self, "handle", None):
            lib().sgnn_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def spmm_into(a: CsrMatrix, b: torch.Tensor, reduce, kind: KernelKind, out: torch.Tensor,
              plan: Plan | None = None) -> torch.Tensor:
    """detail::spmm_into (kernels.hpp:141-149) plus spmm_with's checks (:157-169)."""
    _dense(b, "spmm")
    _out(out, (a.n_rows, b.shape[1]), "spmm")
    _on(a, "spmm", b, out)
    red = _reduce(reduce)
    if a.n_cols != b.shape[0]:  # check_spmm_shapes, kernels.hpp:131-136
        raise ShapeError(f"spmm: sparse operand is {a.n_rows}x{a.n_cols} but dense operand is "
                         f"{b.shape[0]}x{b.shape[1]}")
    if kind.is_specialized():  # kernels.hpp:159-169 (same rule as sgnn_spmm_with_f32)
        if red != _lib.SUM:
            raise DispatchError(f"specialized kernels support sum only, got {_NAMES[red]}")
        if kind.k not in specialization_sweep:
            raise DispatchError(f"K={kind.k} is not in the specialization set")
        if b.shape[1] != kind.k:
            raise DispatchError(f"kernel is fixed at K={kind.k} but dense operand has K={b.shape[1]}")
    if b.shape[1] == 0 or a.n_rows == 0:
        return out
    if plan is None:
        plan = a.plan(b.shape[1], "tuned" if kind.is_specialized() else "default")
    return spmm_plan(a, b, red, plan, out)


def spmm_with(a: CsrMatrix, b: torch.Tensor, reduce, kind: KernelKind, plan: Plan | None = None):
    """spmm_with (kernels.hpp:157-173)."""
    _dense(b, "spmm")
    out = torch.empty((a.n_rows, b.shape[1]), dtype=torch.float32, device=b.device)
    return spmm_into(a, b, reduce, kind, out, plan)


def spmm(a: CsrMatrix, b: torch.Tensor, reduce="sum", plan: Plan | None = None,
         out: torch.Tensor | None = None):
    """spmm (kernels.hpp:179-182): kernel picked by the dispatch state."""
    _dense(b, "spmm")
    kind = resolve_kernel(b.shape[1], reduce)
    if out is None:
        out = torch.empty((a.n_rows, b.shape[1]), dtype=torch.float32, device=b.device)
    return spmm_into(a, b, reduce, kind, out, plan if kind.is_specialized() else None)


def spmm_plan(a: CsrMatrix, b: torch.Tensor, reduce="sum", plan: Plan | None = None,
              out: torch.Tensor | None = None) -> torch.Tensor:
    """sgnn_spmm_f32: SpMM with an explicit plan for any reduce/K (the plan's
    launch parameters never change the result)."""
    _dense(b, "spmm")
    if out is None:
        out = torch.empty((a.n_rows, b.shape[1]), dtype=torch.float32, device=b.device)
    _out(out, (a.n_rows, b.shape[1]), "spmm")
    _on(a, "spmm", b, out)
    check(lib().sgnn_spmm_f32(C.byref(a.c()), b.data_ptr(), b.shape[0], b.shape[1], out.data_ptr(),
                              _reduce(reduce), plan.handle if plan is not None else None, _stream()), "spmm")
    return out


def spmm_peer(a: CsrMatrix, parts, part_shift: int, k: int, reduce="sum", plan: Plan | None = None,
              out: torch.Tensor | None = None, device=None) -> torch.Tensor:
    """sgnn_spmm_peer_f32: SpMM whose X is the row partition's blocks, read in
    place.  `parts` are device pointers (ints) or [2**part_shift, k] tensors,
    one per partition, possibly mapped from peer GPUs; column c of `a` is row
    (c & (2**part_shift - 1)) of block c >> part_shift.  Sum and mean only."""
    ptrs = []
    for p in parts:
        if isinstance(p, torch.Tensor):
            _dense(p, "spmm_peer block")
            if p.shape[1] != k:
                raise _lib.ShapeError(f"spmm_peer: block has {p.shape[1]} columns, K={k}")
            if p.shape[0] < (1 << part_shift):
                raise _lib.ShapeError("spmm_peer: block shorter than 2**part_shift rows")
            ptrs.append(p.data_ptr())
        else:
            ptrs.append(int(p))
    arr = (C.c_void_p * max(1, len(ptrs)))(*ptrs)
    if out is None:
        dev = device if device is not None else a.row_ptr.device
        out = torch.empty((a.n_rows, k), dtype=torch.float32, device=dev)
    check(lib().sgnn_spmm_peer_f32(C.byref(a.c()), arr, len(ptrs), int(part_shift), int(k), out.data_ptr(),
                                   _reduce(reduce), plan.handle if plan is not None else None, _stream()),
          "spmm_peer")
    return out


class _TunedPlan(Plan):
    def __init__(self, a, k, handle):  # noqa: D401 - wraps a plan made by the tuner
        self.a, self.k, self.handle = a, int(k), handle


def tune_spmm(a: CsrMatrix, k: int, reduce="sum", reps: int = 5, x: torch.Tensor | None = None,
              max_entries: int = 256):
    """On-device autotuner (sgnn_tune_spmm): returns (best Plan, [{params, ms}])."""
    if x is not None:
        _dense(x, "tune X")
    ents = (_lib.TuneEntry * max_entries)()
    n = C.c_int()
    h = C.c_void_p()
    check(lib().sgnn_tune_spmm(C.byref(a.c()), x.data_ptr() if x is not None else None, int(k),
                               _reduce(reduce), int(reps), C.byref(h), ents, max_entries, C.byref(n),
                               _stream()), "run_tuning")
    table = [{"params": ents[i].params.as_dict(), "ms": float(ents[i].ms)} for i in range(min(n.value, max_entries))]
    return _TunedPlan(a, k, h), table


@dataclass
class TuningEntry:
    """TuningEntry (autotune.hpp:54-59): default-plan vs tuned-plan time."""
    k: int
    t_trusted_ms: float
    t_specialized_ms: float
    speedup: float


@dataclass
class TuningReport:
    """TuningReport (autotune.hpp:63-70); profile = the device query."""
    entries: list
    best_k: int
    profile: dict
    graph_id: str
    skipped: list
    plans: dict


def run_tuning(a: CsrMatrix, ks, reps: int = 5, seed: int = 42, graph_id: str = "") -> TuningReport:
    """run_tuning (autotune.hpp:99-164) on the B200: for each K in the sweep,
    time the default ("trusted") plan against the on-device-tuned
    ("specialized") plan, both on a seeded uniform operand; the tuner asserts
    bitwise equality of the two outputs (InternalError otherwise).  best_k =
    argmax speedup, ties to the smaller K."""
    ks = list(ks)
    if not ks:
        raise ConfigError("run_tuning: candidate list is empty")
    if reps < 3:
        raise ConfigError("run_tuning: reps must be >= 3")
    sm, l2, ma, mi = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    check(lib().sgnn_device_info(C.byref(sm), C.byref(l2), C.byref(ma), C.byref(mi)))
    profile = {"sm_count": sm.value, "l2_bytes": l2.value, "cc": f"{ma.value}.{mi.value}",
               "description": torch.cuda.get_device_name()}
    entries, skipped, plans, seen = [], [], {}, []
    dev = a.row_ptr.device
    for k in ks:
        if k in seen:
            continue
        seen.append(k)
        if k not in specialization_sweep:
            skipped.append(k)
            continue
        g = torch.Generator(device=dev).manual_seed(seed ^ ((0x9E3779B97F4A7C15 * k) & 0x7FFFFFFFFFFFFFFF))
        b = torch.rand((a.n_cols, k), generator=g, device=dev, dtype=torch.float32)
        best, _ = tune_spmm(a, k, "sum", reps, x=b)
        default = Plan(a, k)
        out = torch.empty((a.n_rows, k), device=dev)

        def med(plan):
            ts = []
            for _ in range(reps):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                spmm_plan(a, b, "sum", plan, out)
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e))
            ts.sort()
            n = len(ts)
            return ts[n // 2] if n % 2 else 0.5 * (ts[n // 2 - 1] + ts[n // 2])

        spmm_plan(a, b, "sum", default, out)
        t_t, t_s = med(default), med(best)
        entries.append(TuningEntry(k, t_t, t_s, t_t / t_s))
        plans[k] = best
    if not entries:
        raise ConfigError("run_tuning: no requested K has a specialized kernel")
    top = entries[0]
    for e in entries:
        if e.speedup > top.speedup or (e.speedup == top.speedup and e.k < top.k):
            top = e
    return TuningReport(entries, top.k, profile, graph_id, skipped, plans)


def release_scratch(keep_bytes: int = 0) -> None:
    """Return the library's unused workspace to the driver (sgnn_release_scratch)."""
    check(lib().sgnn_release_scratch(int(keep_bytes)), "release_scratch")


def resolve_kernel(k: int, reduce) -> KernelKind:
    """resolve_kernel (kernels.hpp:38, dispatch.cpp:21-28)."""
    sk = C.c_uint32()
    tag = lib().sgnn_resolve_kernel(int(k), _reduce(reduce), C.byref(sk))
    return KernelKind.specialized(sk.value) if tag == _lib.SPECIALIZED else KernelKind.trusted()


def set_dispatch(enabled: bool) -> None:
    """set_dispatch (autotune.hpp:36, dispatch.cpp:12)."""
    lib().sgnn_set_dispatch(int(bool(enabled)))


def get_dispatch() -> bool:
    return bool(lib().sgnn_get_dispatch())


class DispatchGuard:
    """DispatchGuard (autotune.hpp:40-51)."""

    def __init__(self, enabled: bool):
        self.enabled = enabled

    def __enter__(self):
        self.prev = get_dispatch()
        set_dispatch(self.enabled)
        return self

    def __exit__(self, *exc):
        set_dispatch(self.prev)


def transpose(a: CsrMatrix) -> CsrMatrix:
    """transpose (sparse.hpp:72-89), bit-exact, on the device."""
    dev = a.row_ptr.device
    trp = torch.empty(a.n_cols + 1, dtype=torch.int64, device=dev)
    tci = torch.empty(a.nnz, dtype=torch.int32, device=dev)
    tv = torch.empty(a.nnz, dtype=torch.float32, device=dev)
    check(lib().sgnn_csr_transpose(C.byref(a.c()), trp.data_ptr(), tci.data_ptr() if a.nnz else None,
                                   tv.data_ptr() if a.nnz else None, None, 0, _stream()), "transpose")
    return CsrMatrix(a.n_cols, a.n_rows, trp, tci, tv)


def row_degrees(a: CsrMatrix) -> torch.Tensor:
    """row_degrees (sparse.hpp:105-109) as int32 (u32 bits)."""
    deg = torch.empty(a.n_rows, dtype=torch.int32, device=a.row_ptr.device)
    check(lib().sgnn_row_degrees(C.byref(a.c()), deg.data_ptr(), _stream()), "row_degrees")
    return deg


def is_symmetric(a: CsrMatrix) -> bool:
    """is_symmetric (sparse.hpp:179-192)."""
    out = C.c_int()
    check(lib().sgnn_is_symmetric(C.byref(a.c()), C.byref(out), _stream()), "is_symmetric")
    return bool(out.value)


class TrainingCache:
    """TrainingCache<float> + build_cache (gnn.hpp:113-196) over a device a_hat."""

    MODEL_KINDS = {"gcn": 0, "sage-sum": 1, "sage-mean": 2, "gin": 3}  # gnn.hpp:17-35

    def __init__(self, a: CsrMatrix, use_cache: bool = True, model_kind: str | None = None,
                 add_self_loops: bool = True):
        """model_kind None: `a` is already the propagation operand a_hat.
        Otherwise build_cache(kind, a, ...) (gnn.hpp:180-196): "gcn"
        normalizes A on the device (normalize_builds = 1)."""
        if a.n_rows != a.n_cols:
            raise ShapeError(f"build_cache: adjacency is {a.n_rows}x{a.n_cols}, expected square")
        self._a = a
        h = C.c_void_p()
        if model_kind is None:
            check(lib().sgnn_cache_create(C.byref(a.c()), int(bool(use_cache)), C.byref(h), _stream()),
                  "build_cache")
        else:
            if model_kind not in self.MODEL_KINDS:
                raise ConfigError(f"unknown model '{model_kind}' (expected gcn|sage-sum|sage-mean|gin)")
            check(lib().sgnn_cache_create_model(C.byref(a.c()), self.MODEL_KINDS[model_kind], int(bool(use_cache)),
                                                int(bool(add_self_loops)), C.byref(h), _stream()), "build_cache")
        self.handle = h
        if model_kind == "gcn":
            cs = _lib.Csr()
            check(lib().sgnn_cache_a_hat(self.handle, C.byref(cs)))
            self.a_hat = _View(cs, self)
        else:
            self.a_hat = a

    def _operand(self, fn) -> CsrMatrix:
        out = _lib.Csr()
        check(fn(self.handle, C.byref(out), _stream()), "cache operand")
        # one view per device operand, so its cached plans survive across epochs
        key = (out.row_ptr, out.col_idx, out.values, out.n_rows, out.nnz)
        views = self.__dict__.setdefault("_views", {})
        if key not in views:
            if out.row_ptr == self.a_hat.c().row_ptr and out.values == self.a_hat.c().values:
                views[key] = self.a_hat  # symmetric short-circuit: the operand is a_hat itself
            else:
                views[key] = _View(out, self)
        return views[key]

    def sum_operand(self) -> CsrMatrix:
        return self._operand(lib().sgnn_cache_sum_operand)

    def mean_operand(self) -> CsrMatrix:
        return self._operand(lib().sgnn_cache_mean_operand)

    @property
    def counters(self) -> dict:
        t, n, h, s = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        check(lib().sgnn_cache_counters(self.handle, C.byref(t), C.byref(n), C.byref(h), C.byref(s)))
        return {"transpose_builds": t.value, "normalize_builds": n.value, "cache_hits": h.value,
                "symmetric": bool(s.value)}

    def spmm_backward(self, dc: torch.Tensor, reduce="sum", out: torch.Tensor | None = None):
        """dX = spmm(sum_operand | mean_operand, dC, Sum) (gnn.hpp:275,290)."""
        _dense(dc, "spmm_backward")
        if out is None:
            out = torch.empty((self.a_hat.n_cols, dc.shape[1]), dtype=torch.float32, device=dc.device)
        check(lib().sgnn_spmm_backward_f32(self.handle, dc.data_ptr(), dc.shape[0], dc.shape[1],
                                           out.data_ptr(), _reduce(reduce), _stream()), "spmm_backward")
        return out

    def close(self):
        if getattr(self, "handle", None):
            lib().sgnn_cache_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _View(CsrMatrix):
    """A CSR view onto device arrays owned by a TrainingCache."""

    def __init__(self, cs: _lib.Csr, owner):
        self.n_rows, self.n_cols = cs.n_rows, cs.n_cols
        self._nnz = cs.nnz
        self._cstruct = cs
        self._owner = owner
        self._plans = {}

    @property
    def nnz(self) -> int:
        return int(self._nnz)

    def to_numpy(self):
        cs = self._cstruct
        rp = np.empty(cs.n_rows + 1, np.uint64)
        ci = np.empty(cs.nnz, np.uint32)
        v = np.empty(cs.nnz, np.float32)
        torch.cuda.synchronize()
        for host, ptr in ((rp, cs.row_ptr), (ci, cs.col_idx), (v, cs.values)):
            if host.nbytes:
                _lib.memcpy_d2h(host.ctypes.data, ptr, host.nbytes)
        return rp, ci, v


def normalize_adjacency(a: CsrMatrix, add_self_loops: bool = True) -> CsrMatrix:
    """normalize_adjacency (sparse.hpp:116-174) on the device, bit-exact."""
    nnz = C.c_uint64()
    check(lib().sgnn_normalize_adjacency(C.byref(a.c()), int(bool(add_self_loops)), C.byref(nnz),
                                         None, None, None, _stream()), "normalize_adjacency")
    dev = a.row_ptr.device
    trp = torch.empty(a.n_rows + 1, dtype=torch.int64, device=dev)
    tci = torch.empty(nnz.value, dtype=torch.int32, device=dev)
    tv = torch.empty(nnz.value, dtype=torch.float32, device=dev)
    check(lib().sgnn_normalize_adjacency(C.byref(a.c()), int(bool(add_self_loops)), C.byref(nnz),
                                         trp.data_ptr(), tci.data_ptr() if nnz.value else None,
                                         tv.data_ptr() if nnz.value else None, _stream()), "normalize_adjacency")
    return CsrMatrix(a.n_rows, a.n_cols, trp, tci, tv)


def sddmm(p: CsrMatrix, x: torch.Tensor, y: torch.Tensor) -> CsrMatrix:
    """sddmm (kernels.hpp:187-210): P's pattern with values p_e * <X_i, Y_j>."""
    _dense(x, "sddmm X")
    _dense(y, "sddmm Y")
    _on(p, "sddmm", x, y)
    if p.n_rows != x.shape[0] or p.n_cols != y.shape[0] or x.shape[1] != y.shape[1]:
        raise ShapeError(f"sddmm: pattern {p.n_rows}x{p.n_cols} needs X with {p.n_rows} rows and Y with "
                         f"{p.n_cols} rows of equal width; got X {x.shape[0]}x{x.shape[1]}, "
                         f"Y {y.shape[0]}x{y.shape[1]}")
    out = torch.empty(p.nnz, dtype=torch.float32, device=x.device)
    k = x.shape[1]
    if p.nnz and p.n_rows and k and k <= 1024 and (k % 4 == 0 or k <= 256):
        plan = p.plan(k, "fused")  # cached nnz-balanced split shared with fusedmm
        check(lib().sgnn_sddmm_plan_f32(C.byref(p.c()), x.data_ptr(), x.shape[0], y.data_ptr(), y.shape[0],
                                        k, out.data_ptr(), plan.handle, _stream()), "sddmm")
    else:
        check(lib().sgnn_sddmm_f32(C.byref(p.c()), x.data_ptr(), x.shape[0], y.data_ptr(), y.shape[0],
                                   k, out.data_ptr() if p.nnz else None, _stream()), "sddmm")
    return p.with_values(out)


EDGE_OPS = {"mul": _lib.EDGE_MUL, None: _lib.EDGE_MUL, "sigmoid_mul": _lib.EDGE_SIGMOID_MUL}


def fusedmm(p: CsrMatrix, x: torch.Tensor, y: torch.Tensor, edge_op="mul", reduce="sum",
            out: torch.Tensor | None = None, plan: Plan | None = None) -> torch.Tensor:
    """fusedmm (kernels.hpp:216-270) with a GPU-expressible combine
    (Semiring::combine, types.hpp:139-145): "mul" = p*dot (plus_times), or
    "sigmoid_mul" = p*sigmoid(dot).  An arbitrary Python callable is a
    DispatchError: there is no CPU fallback."""
    if callable(edge_op):
        raise DispatchError("fusedmm: arbitrary combine callables cannot run on the GPU; "
                            "use edge_op='mul' or 'sigmoid_mul'")
    if edge_op not in EDGE_OPS:
        raise ConfigError(f"fusedmm: unknown edge op {edge_op!r}")
    _dense(x, "fusedmm X")
    _dense(y, "fusedmm Y")
    if p.n_rows != x.shape[0] or p.n_cols != y.shape[0] or x.shape[1] != y.shape[1]:
        raise ShapeError(f"fusedmm: operand shapes do not compose (P {p.n_rows}x{p.n_cols}, X "
                         f"{x.shape[0]}x{x.shape[1]}, Y {y.shape[0]}x{y.shape[1]})")
    if out is None:
        out = torch.empty((p.n_rows, y.shape[1]), dtype=torch.float32, device=x.device)
    _out(out, (p.n_rows, y.shape[1]), "fusedmm")
    _on(p, "fusedmm", x, y, out)
    if plan is None and p.n_rows and x.shape[1] and x.shape[1] <= 1024 and (x.shape[1] % 4 == 0 or x.shape[1] <= 256):
        plan = p.plan(x.shape[1], "fused")  # cached split (built once per matrix and K)
    if plan is not None:
        check(lib().sgnn_fusedmm_plan_f32(C.byref(p.c()), x.data_ptr(), x.shape[0], y.data_ptr(), y.shape[0],
                                          x.shape[1], EDGE_OPS[edge_op], _reduce(reduce), out.data_ptr(),
                                          plan.handle, _stream()), "fusedmm")
        return out
    check(lib().sgnn_fusedmm_f32(C.byref(p.c()), x.data_ptr(), x.shape[0], y.data_ptr(), y.shape[0],
                                 x.shape[1], EDGE_OPS[edge_op], _reduce(reduce), out.data_ptr(),
                                 _stream()), "fusedmm")
    return out
