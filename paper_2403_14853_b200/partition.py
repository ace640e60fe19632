"""1D row partition of a square graph over GPUs.

Rank p owns the contiguous row block [b_p, b_{p+1}) chosen by the reference's
cost rule (nnz + rows, parallel.hpp:28-41, `balanced_row_partition`), the
matching feature rows X[b_p:b_{p+1}] and the output rows C[b_p:b_{p+1}].  The
only exchange is an all-gather of the feature blocks: every block is padded to
`stride` rows so the gathered buffer is [P*stride, K], and the block's column
ids are remapped once (host, `sgnn_host_partition_block`) to that padded
layout -- col' = owner*stride + (col - b_owner) -- so the unchanged SpMM
kernel reads the gathered buffer directly.  The remap is monotone, so every
row is accumulated in the same order as on one GPU: the P-GPU result is
bitwise the 1-GPU result.

Exchanges:
  NcclExchange      torch.distributed all_gather_into_tensor (NCCL over NVLink
                    on the B200 box; gloo on CPU for tests)
  LoopbackExchange  P virtual partitions in one process (device copies) -- the
                    SURVEY 4.5 test mode for partition/reassembly logic on one GPU
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, graphs


@dataclass
class RowPartition:
    bounds: np.ndarray  # u32[P+1]
    stride: int         # padded rows per block (>= max block size)
    n: int

    @property
    def parts(self) -> int:
        return len(self.bounds) - 1

    def rows(self, p: int):
        return int(self.bounds[p]), int(self.bounds[p + 1])

    def block(self, row_ptr, col_idx, values, p: int, threads: int = 0):
        """Rank p's CSR block with columns remapped to the padded layout."""
        r0, r1 = self.rows(p)
        rp = np.ascontiguousarray(row_ptr, np.uint64)
        ci = np.ascontiguousarray(col_idx, np.uint32)
        v = np.ascontiguousarray(values, np.float32) if values is not None else None
        nnz = int(rp[r1] - rp[r0])
        out_rp = np.empty(r1 - r0 + 1, np.uint64)
        out_ci = np.empty(nnz, np.uint32)
        out_v = np.empty(nnz, np.float32) if v is not None else None
        b = np.ascontiguousarray(self.bounds, np.uint32)
        got = _lib.host().sgnn_host_partition_block(
            rp.ctypes.data, ci.ctypes.data, v.ctypes.data if v is not None else None, b.ctypes.data,
            self.parts, p, self.stride, out_rp.ctypes.data, out_ci.ctypes.data,
            out_v.ctypes.data if out_v is not None else None, threads)
        assert got == nnz
        return out_rp, out_ci, out_v


def make_partition(row_ptr, n_parts: int, align: int = 1) -> RowPartition:
    """balanced_row_partition (parallel.hpp:28-41) at GPU granularity."""
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    bounds = graphs.balanced_row_partition(rp, n_parts)
    sizes = np.diff(bounds.astype(np.int64))
    stride = int(max(1, sizes.max() if len(sizes) else 1))
    stride = (stride + align - 1) // align * align
    return RowPartition(bounds, stride, len(rp) - 1)


def pad_block(x_local, stride: int):
    """[rows_p, K] -> [stride, K] (zero padding; padded rows are never read)."""
    import torch
    out = torch.zeros((stride, x_local.shape[1]), dtype=x_local.dtype, device=x_local.device)
    out[: x_local.shape[0]].copy_(x_local)
    return out


class NcclExchange:
    """All-gather of the padded feature blocks through torch.distributed
    (NCCL on GPUs; gloo on CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group

    def all_gather(self, block):
        import torch
        ws = self.dist.get_world_size(self.group)
        out = torch.empty((ws * block.shape[0], block.shape[1]), dtype=block.dtype, device=block.device)
        self.dist.all_gather_into_tensor(out, block.contiguous(), group=self.group)
        return out


class LoopbackExchange:
    """P virtual ranks in one process: all_gather takes the list of blocks."""

    def all_gather(self, blocks):
        import torch
        return torch.cat([b.contiguous() for b in blocks], dim=0)


class PartitionedSpmm:
    """Rank-local forward of C[rows_p] = reduce_j A[rows_p, j] X[j] with the
    all-gather exchange.  `compute(local_csr_arrays, gathered, reduce)` is the
    local SpMM; by default the B200 kernel (ops.spmm_plan on a cached plan)."""

    def __init__(self, row_ptr, col_idx, values, part: RowPartition, rank: int, k: int,
                 device="cuda", compute=None):
        self.part, self.rank, self.k = part, rank, int(k)
        self.r0, self.r1 = part.rows(rank)
        self.local = part.block(row_ptr, col_idx, values, rank)
        self.n_gathered = part.parts * part.stride
        self.device = device
        self._compute = compute
        self._plan = None
        self._a = None
        if compute is None:
            from . import ops
            self._a = ops.CsrMatrix.from_numpy(*self.local, self.n_gathered, device=device)
            self._plan = ops.Plan(self._a, self.k)

    def compute(self, gathered, reduce="sum", out=None):
        if self._compute is not None:
            return self._compute(self.local, gathered, reduce)
        from . import ops
        return ops.spmm_plan(self._a, gathered, reduce, self._plan, out)

    def forward(self, x_local, exchange, reduce="sum", out=None):
        """x_local: this rank's feature rows [r1-r0, K]."""
        gathered = exchange.all_gather(pad_block(x_local, self.part.stride))
        return self.compute(gathered, reduce, out)
