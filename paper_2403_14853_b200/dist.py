"""Multi-GPU face of the library: the communicator and the row-partitioned
GraphSAGE trainer of the C ABI (sgnn_comm_*, sgnn_dist_*; csrc/dist.cu).

The partition is the reference's thread fan-out (parallel.hpp:28-65,
balanced_row_partition) at GPU granularity: contiguous row blocks, rank r
owning rows [bounds[r], bounds[r+1]) of A (global column ids), of X and of
every activation; one training epoch is train()'s loop body
(gnn.hpp:427-435) with the feature blocks all-gathered in place (no padding:
the gathered buffer is the operand in its own row order) and the weight
gradients all-reduced.

    comm = Comm.from_torch()                 # one process per GPU (NCCL)
    eng = DistSage.from_graph(comm, row_ptr, col_idx, values, x, labels, mask, 128, 16)
    eng.set_weights(model); eng.epochs(10, 0.05); losses = eng.stats()[0]

`Comm.loopback(P)` runs P virtual ranks in one process on one GPU (the test
and balance-measurement mode; `DistSage.epochs_group`).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib, graphs, ops
from ._lib import check, lib

KIND_IDS = {"sage-sum": 1, "sage-mean": 2}
TIME_FIELDS = ("epoch_ms", "spmm_ms", "compute_ms", "exchange_ms", "spmm1_ms", "spmm2_ms", "spmm_bwd_ms", "dense_ms")
ROW_WEIGHT = 30  # GPU partition cost: nnz + ROW_WEIGHT * rows (DESIGN 6)


def row_partition(row_ptr, n_parts: int, row_weight: int = ROW_WEIGHT) -> np.ndarray:
    """Contiguous row bounds (u32[P+1]) of equal nnz + row_weight*rows cost
    (row_weight=1: balanced_row_partition, parallel.hpp:28-41)."""
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    out = np.empty(n_parts + 1, np.uint32)
    _lib.host().sgnn_host_weighted_row_partition(rp.ctypes.data, len(rp) - 1, n_parts, int(row_weight),
                                                 out.ctypes.data)
    return out


def row_block(row_ptr, col_idx, values, r0: int, r1: int):
    """Rows [r0, r1) of a CSR with global column ids (row_ptr rebased)."""
    rp = np.asarray(row_ptr, np.uint64)
    e0, e1 = int(rp[r0]), int(rp[r1])
    return (rp[r0:r1 + 1] - rp[r0]).astype(np.uint64), np.asarray(col_idx)[e0:e1], \
        (np.asarray(values, np.float32)[e0:e1] if values is not None else None)


class Comm:
    """sgnn_comm: NCCL (one process per GPU) or loopback (P virtual ranks)."""

    def __init__(self, handle, nranks, rank, kind):
        self.h, self.nranks, self.rank, self.kind = handle, nranks, rank, kind

    @classmethod
    def nccl(cls, unique_id: bytes, nranks: int, rank: int) -> "Comm":
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(lib().sgnn_comm_init_rank(buf, nranks, rank, C.byref(h)), "comm_init_rank")
        return cls(h, nranks, rank, "nccl")

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().sgnn_comm_get_unique_id(buf), "comm_get_unique_id")
        return buf.raw

    @classmethod
    def from_torch(cls, group=None) -> "Comm":
        """NCCL communicator over the ranks of a torch.distributed group (the
        id travels over the group's own backend)."""
        import torch.distributed as dist
        ws, rank = dist.get_world_size(group), dist.get_rank(group)
        obj = [cls.unique_id() if rank == 0 and ws > 1 else None]
        if ws > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        return cls.nccl(obj[0] or bytes(128), ws, rank)

    @classmethod
    def loopback(cls, nranks: int) -> "Comm":
        h = C.c_void_p()
        check(lib().sgnn_comm_init_loopback(nranks, C.byref(h)), "comm_init_loopback")
        return cls(h, nranks, 0, "loopback")

    def close(self):
        if self.h:
            lib().sgnn_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class DistSage:
    """One rank (engine) of the row-partitioned SAGE trainer (sgnn_dist)."""

    def __init__(self, comm: Comm | None, rank: int, bounds, block: ops.CsrMatrix, x_local, labels_local,
                 mask_local, hidden: int, classes: int, kind: str = "sage-mean", bwd_block: ops.CsrMatrix | None = None,
                 max_epochs: int = 128, device="cuda"):
        if kind not in KIND_IDS:
            raise _lib.UnsupportedError(f"dist: the row-partitioned trainer runs sage-sum / sage-mean, not {kind}")
        self.comm, self.kind = comm, kind
        self.bounds = np.ascontiguousarray(bounds, np.uint32)
        self.block, self.bwd_block = block, bwd_block  # borrowed by the engine: keep alive
        x = x_local.contiguous() if isinstance(x_local, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(x_local, np.float32)).to(device)
        lab = (labels_local if isinstance(labels_local, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(labels_local).astype(np.int64))).to(device).to(torch.int32).contiguous()
        msk = (mask_local if isinstance(mask_local, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(mask_local, np.uint8))).to(device).to(torch.uint8).contiguous()
        if lab.numel() and int(lab.min()) < 0:
            raise ops.ConfigError("softmax_xent: negative label")
        self.in_features, self.hidden, self.classes = int(x.shape[1]), int(hidden), int(classes)
        self.max_epochs = int(max_epochs)
        h = C.c_void_p()
        check(lib().sgnn_dist_create(comm.h if comm else None, int(rank), self.bounds.ctypes.data,
                                     C.byref(block.c()), C.byref(bwd_block.c()) if bwd_block is not None else None,
                                     KIND_IDS[kind], self.in_features, self.hidden, self.classes, x.data_ptr(),
                                     lab.data_ptr(), msk.data_ptr(), self.max_epochs, C.byref(h), ops._stream()),
              "dist_create")
        self.h = h
        r0, rows, nnz = C.c_uint32(), C.c_uint32(), C.c_uint64()
        check(lib().sgnn_dist_info(h, C.byref(r0), C.byref(rows), C.byref(nnz), None, None), "dist_info")
        self.r0, self.rows, self.nnz = r0.value, rows.value, nnz.value
        self.epochs_run = 0

    @classmethod
    def from_graph(cls, comm: Comm | None, row_ptr, col_idx, values, x, labels, mask, hidden, classes,
                   kind="sage-mean", rank: int | None = None, bounds=None, symmetric: bool | None = None,
                   row_weight: int = ROW_WEIGHT, max_epochs: int = 128, device="cuda"):
        """Engine of `rank` (default: the communicator's) from a host graph:
        partitions it (nnz + row_weight*rows), uploads the rank's row block
        (and, for a non-symmetric A, the same rows of A^T) and its slices of
        x / labels / mask (full-height host arrays)."""
        P = comm.nranks if comm else 1
        rank = (comm.rank if comm else 0) if rank is None else rank
        b = row_partition(row_ptr, P, row_weight) if bounds is None else np.ascontiguousarray(bounds, np.uint32)
        r0, r1 = int(b[rank]), int(b[rank + 1])
        n = len(row_ptr) - 1
        rp, ci, v = row_block(row_ptr, col_idx, values, r0, r1)
        block = ops.CsrMatrix.from_numpy(rp, ci, v, n, device=device)
        bwd = None
        full = None
        if symmetric is None:  # cache.symmetric = is_symmetric(a_hat) (gnn.hpp:194), on the device
            full = ops.CsrMatrix.from_numpy(row_ptr, col_idx, values, n, device=device)
            symmetric = ops.is_symmetric(full)
        if not symmetric:  # rows of A^T (gnn.hpp:127-144); mean scaling happens on the device
            full = full or ops.CsrMatrix.from_numpy(row_ptr, col_idx, values, n, device=device)
            trp, tci, tv = ops.transpose(full).to_numpy()
            brp, bci, bv = row_block(trp, tci, tv, r0, r1)
            bwd = ops.CsrMatrix.from_numpy(brp, bci, bv, n, device=device)
        del full
        xs = np.asarray(x)[r0:r1] if not isinstance(x, torch.Tensor) else x[r0:r1]
        return cls(comm, rank, b, block, xs, np.asarray(labels)[r0:r1], np.asarray(mask)[r0:r1], hidden, classes,
                   kind, bwd, max_epochs, device)

    # ---- parameters
    def set_weights(self, w1, w2, w1_self, w2_self):
        ts = [w.detach().float().contiguous() if isinstance(w, torch.Tensor) else
              torch.from_numpy(np.ascontiguousarray(w, np.float32)) for w in (w1, w2, w1_self, w2_self)]
        ts = [t.cuda() for t in ts]
        check(lib().sgnn_dist_set_weights(self.h, *(t.data_ptr() for t in ts), ops._stream()), "dist_set_weights")

    def get_weights(self):
        a, b = (self.in_features, self.hidden), (self.hidden, self.classes)
        out = [torch.empty(s, device="cuda") for s in (a, b, a, b)]
        check(lib().sgnn_dist_get_weights(self.h, *(t.data_ptr() for t in out), ops._stream()), "dist_get_weights")
        return out

    def set_features(self, x_local: torch.Tensor, borrow: bool = False):
        """New features for this rank's rows (device or pinned host tensor),
        copied into the engine (`borrow` is accepted and ignored)."""
        if x_local.shape != (self.rows, self.in_features) or x_local.dtype != torch.float32:
            raise ops.ShapeError(f"dist_set_features: expected float32 [{self.rows}, {self.in_features}]")
        x_local = x_local.contiguous()
        self._x_hold = x_local
        check(lib().sgnn_dist_set_features(self.h, x_local.data_ptr(), int(borrow), ops._stream()),
              "dist_set_features")

    # ---- training
    def epochs(self, n: int, lr: float):
        arr = (C.c_void_p * 1)(self.h)
        check(lib().sgnn_dist_epochs(arr, 1, int(n), float(lr), ops._stream()), "dist_epochs")
        self.epochs_run += n

    @staticmethod
    def epochs_group(engines, n: int, lr: float):
        """Loopback: all P engines of one comm, phase by phase on one stream."""
        arr = (C.c_void_p * len(engines))(*(e.h for e in engines))
        check(lib().sgnn_dist_epochs(arr, len(engines), int(n), float(lr), ops._stream()), "dist_epochs")
        for e in engines:
            e.epochs_run += n

    def stats(self, first: int = 0, count: int | None = None):
        """(loss[], accuracy[], times[count x 8]) of epochs [first, first+count)."""
        count = self.epochs_run - first if count is None else count
        loss = np.zeros(count)
        acc = np.zeros(count)
        times = np.zeros((count, len(TIME_FIELDS)))
        check(lib().sgnn_dist_stats(self.h, int(first), int(count), loss.ctypes.data, acc.ctypes.data,
                                    times.ctypes.data, ops._stream()), "dist_stats")
        return loss, acc, times

    def stats_copy(self, first: int, count: int, dst_ptr: int):
        """Async copy of (loss, accuracy) pairs to dst_ptr (host pinned or device)."""
        check(lib().sgnn_dist_stats_copy(self.h, int(first), int(count), dst_ptr, ops._stream()), "dist_stats_copy")

    def reset(self):
        check(lib().sgnn_dist_reset(self.h), "dist_reset")
        self.epochs_run = 0

    @property
    def n_masked(self) -> int:
        m = C.c_uint64()
        check(lib().sgnn_dist_info(self.h, None, None, None, C.byref(m), None), "dist_info")
        return m.value

    def close(self):
        if getattr(self, "h", None):
            lib().sgnn_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
