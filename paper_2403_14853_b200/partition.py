"""1D row partition of a square graph over GPUs.

Rank p owns the contiguous row block [b_p, b_{p+1}) chosen by the reference's
cost rule (parallel.hpp:28-41, `balanced_row_partition`) with the rows
weighted (`row_weight`, dist.row_partition), the matching feature rows
X[b_p:b_{p+1}] and the output rows C[b_p:b_{p+1}].  The only exchange is an
all-gather-v of the feature blocks into a full-height [n, K] buffer -- rank
q's rows land at rows b_q.., so the gathered buffer IS X in its own row order,
the block keeps its global column ids and the unchanged SpMM kernel reads it
directly.  Every row is accumulated in the same order as on one GPU: the
P-GPU result is bitwise the 1-GPU result.  (The native trainer,
csrc/dist.cu / dist.py, does the same exchange with grouped ncclSend/Recv;
this module is the torch.distributed mirror used by the gloo tests.)

Exchanges:
  NcclExchange      torch.distributed point-to-point all-gather-v (NCCL over
                    NVLink on the B200 box; gloo on CPU for tests)
  LoopbackExchange  P virtual partitions in one process (device copies) -- the
                    SURVEY 4.5 test mode for partition/reassembly logic on one GPU
  PeerBlocks        no copy at all: every rank's block lives in its own
                    cudaMalloc allocation, mapped into every other rank with
                    CUDA IPC (NVLink/NVSwitch peer memory); the SpMM kernel
                    (sgnn_spmm_peer_f32) gathers X rows straight from the
                    owner's HBM.  This path needs the *padded* layout: blocks
                    of a pow2 stride, columns remapped once to
                    col' = owner*stride + local (sgnn_host_partition_block),
                    so the owner lookup is a shift and a mask.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, graphs


@dataclass
class RowPartition:
    bounds: np.ndarray  # u32[P+1]
    stride: int         # padded rows per block (>= max block size); 0 = unpadded
    n: int

    @property
    def padded(self) -> bool:
        return self.stride > 0

    @property
    def n_gathered(self) -> int:
        """Rows of the gathered operand: n (unpadded) or P * stride."""
        return self.parts * self.stride if self.padded else self.n

    @property
    def parts(self) -> int:
        return len(self.bounds) - 1

    @property
    def shift(self) -> int:
        """log2(stride) for a pow2 partition (the peer path's part_shift)."""
        if self.stride & (self.stride - 1):
            raise ValueError("peer SpMM needs a power-of-two stride: make_partition(..., pow2=True)")
        return self.stride.bit_length() - 1

    def rows(self, p: int):
        return int(self.bounds[p]), int(self.bounds[p + 1])

    def block(self, row_ptr, col_idx, values, p: int, threads: int = 0):
        """Rank p's CSR block: global column ids (unpadded), or columns
        remapped to the padded owner layout."""
        r0, r1 = self.rows(p)
        if not self.padded:
            rp = np.asarray(row_ptr, np.uint64)
            e0, e1 = int(rp[r0]), int(rp[r1])
            return ((rp[r0:r1 + 1] - rp[r0]).astype(np.uint64), np.ascontiguousarray(np.asarray(col_idx)[e0:e1], np.uint32),
                    np.ascontiguousarray(np.asarray(values)[e0:e1], np.float32) if values is not None else None)
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


def make_partition(row_ptr, n_parts: int, align: int = 1, pow2: bool = False, padded: bool | None = None,
                   row_weight: int = 1) -> RowPartition:
    """balanced_row_partition (parallel.hpp:28-41) at GPU granularity, with
    cost nnz + row_weight * rows (row_weight = 1: the reference's rule).
    Unpadded by default; padded=True (implied by pow2=True, the peer path)
    pads every block to `stride` rows, rounded up to a power of two with pow2
    (the peer SpMM splits a remapped column into (owner, row) with a shift)."""
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    padded = pow2 if padded is None else padded
    if row_weight == 1:
        bounds = graphs.balanced_row_partition(rp, n_parts)
    else:
        out = np.empty(n_parts + 1, np.uint32)
        _lib.host().sgnn_host_weighted_row_partition(rp.ctypes.data, len(rp) - 1, n_parts, int(row_weight),
                                                     out.ctypes.data)
        bounds = out
    if not padded:
        return RowPartition(bounds, 0, len(rp) - 1)
    sizes = np.diff(bounds.astype(np.int64))
    stride = int(max(1, sizes.max() if len(sizes) else 1))
    stride = (stride + align - 1) // align * align
    if pow2:
        stride = 1 << (stride - 1).bit_length()
    return RowPartition(bounds, stride, len(rp) - 1)


def pad_block(x_local, stride: int):
    """[rows_p, K] -> [stride, K] (zero padding; padded rows are never read).
    A block that already has `stride` rows is used as it is (no copy)."""
    import torch
    if stride == 0 or x_local.shape[0] == stride:  # unpadded layout: the block as it is
        return x_local.contiguous()
    out = torch.zeros((stride, x_local.shape[1]), dtype=x_local.dtype, device=x_local.device)
    out[: x_local.shape[0]].copy_(x_local)
    return out


class NcclExchange:
    """All-gather of the feature blocks through torch.distributed (NCCL on
    GPUs; gloo on CPU tensors): all_gather_v for the unpadded layout,
    all_gather for the padded one."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group

    def all_gather_v(self, block, bounds):
        """Rank q's rows [bounds[q], bounds[q+1]) to every rank: a full-height
        [n, K] buffer (point-to-point, each rank receives only the others'
        rows)."""
        import torch
        ws = self.dist.get_world_size(self.group)
        if ws == 1:
            return block.contiguous()
        me = self.dist.get_rank(self.group)
        b = [int(v) for v in bounds]
        out = torch.empty((b[-1], block.shape[1]), dtype=block.dtype, device=block.device)
        out[b[me]:b[me + 1]].copy_(block)
        src = out[b[me]:b[me + 1]]
        ops = []
        for q in range(ws):
            if q == me:
                continue
            if b[me + 1] > b[me]:
                ops.append(self.dist.P2POp(self.dist.isend, src, q, self.group))
            if b[q + 1] > b[q]:
                ops.append(self.dist.P2POp(self.dist.irecv, out[b[q]:b[q + 1]], q, self.group))
        if ops:
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()
        return out

    def all_gather(self, block):
        import torch
        ws = self.dist.get_world_size(self.group)
        if ws == 1:  # the gathered operand is the block itself: no copy
            return block.contiguous()
        out = torch.empty((ws * block.shape[0], block.shape[1]), dtype=block.dtype, device=block.device)
        self.dist.all_gather_into_tensor(out, block.contiguous(), group=self.group)
        return out


class LoopbackExchange:
    """P virtual ranks in one process: all_gather takes the list of blocks."""

    def all_gather(self, blocks):
        import torch
        return torch.cat([b.contiguous() for b in blocks], dim=0)

    def all_gather_v(self, blocks, bounds):
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
        self.n_gathered = part.n_gathered
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
        if isinstance(exchange, PeerExchange):
            return self.forward_peer(x_local, exchange.blocks_for(self.part.stride, x_local.shape[1]), reduce, out)
        return self.compute(self.gather(x_local, exchange), reduce, out)

    def gather(self, local, exchange):
        """The full operand from this rank's rows of it."""
        if self.part.padded:
            return exchange.all_gather(pad_block(local, self.part.stride))
        return exchange.all_gather_v(local, self.part.bounds)

    # SDDMM / FusedMM shard the same way: X is this rank's rows,
    # Y the all-gathered feature blocks in the padded owner layout.
    def fusedmm_gathered(self, x_local, y_gathered, edge_op="mul", reduce="sum", out=None):
        """fusedmm (kernels.hpp:216-270) of this rank's row block."""
        if self._compute is not None:
            return self._compute_fused(x_local, y_gathered, edge_op, reduce)
        from . import ops
        return ops.fusedmm(self._a, x_local, y_gathered, edge_op, reduce, out)

    def sddmm_gathered(self, x_local, y_gathered):
        """sddmm (kernels.hpp:187-210) of this rank's row block: values of the
        block's nonzeros in CSR order."""
        if self._compute is not None:
            return self._compute_fused(x_local, y_gathered, None, None)
        from . import ops
        return ops.sddmm(self._a, x_local, y_gathered).values

    def fusedmm(self, x_local, y_local, exchange, edge_op="mul", reduce="sum", out=None):
        """Row block of fusedmm(A, X, Y): all-gather Y's blocks, then local."""
        return self.fusedmm_gathered(x_local, self.gather(y_local, exchange), edge_op, reduce, out)

    def sddmm(self, x_local, y_local, exchange):
        return self.sddmm_gathered(x_local, self.gather(y_local, exchange))

    def _compute_fused(self, x_local, y_gathered, edge_op, reduce):
        if not hasattr(self._compute, "fused"):
            raise TypeError("the injected compute has no fused(local, x, y, edge_op, reduce) entry")
        return self._compute.fused(self.local, x_local, y_gathered, edge_op, reduce)

    def compute_peer(self, parts, reduce="sum", out=None):
        """The local SpMM reading the partition's blocks in place (pointer
        table or tensors, one per rank): bitwise the gathered-buffer result."""
        from . import ops
        return ops.spmm_peer(self._a, parts, self.part.shift, self.k, reduce, self._plan, out)

    def forward_peer(self, x_local, blocks: "PeerBlocks", reduce="sum", out=None):
        """Fused all-gather + SpMM over peer memory."""
        return self.compute_peer(blocks.publish(x_local), reduce, out)


class _DeviceArray:
    """__cuda_array_interface__ over a library-owned device allocation."""

    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class PeerBlocks:
    """Feature blocks shared through peer memory (fused all-gather).

    Each rank owns `buffers` blocks of [stride, K] f32 in its own cudaMalloc
    allocation (sgnn_peer_alloc) and maps every other rank's blocks through
    CUDA IPC (sgnn_ipc_get_handle / sgnn_ipc_open_handle; handles travel by
    torch.distributed.all_gather_object).  publish(x_local) writes this rank's
    rows into the next block and runs one fence; after it every rank's block is
    readable by the SpMM.  With two buffers the fence of step t also orders the
    reads of step t-1 before the overwrite at step t+1, so one fence per step
    suffices.

    fence="device": an all_reduce of one element on the current stream (NCCL)
    -- stream-ordered, no host sync.  fence="host": synchronize + barrier
    (gloo; used where NCCL cannot run, e.g. two processes sharing one GPU)."""

    def __init__(self, stride: int, k: int, group=None, fence: str = "device", buffers: int = 2):
        import torch
        import torch.distributed as dist
        if fence not in ("device", "host"):
            raise ValueError("fence must be 'device' or 'host'")
        self.dist, self.group, self.fence = dist, group, fence
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        if self.world > 8:
            raise ValueError("peer SpMM maps at most 8 partitions")
        self.stride, self.k, self.buffers = int(stride), int(k), int(buffers)
        self.step = 0
        lib = _lib.lib()
        nbytes = self.stride * self.k * 4
        dev = torch.device("cuda", torch.cuda.current_device())
        self._own, self.views, handles = [], [], []
        for _ in range(self.buffers):
            p = _lib.C.c_void_p()
            _lib.check(lib.sgnn_peer_alloc(nbytes, _lib.C.byref(p)), "peer_alloc")
            self._own.append(p.value)
            v = torch.as_tensor(_DeviceArray(p.value, (self.stride, self.k)), device=dev)
            v.zero_()
            self.views.append(v)
            h = (_lib.C.c_char * 64)()
            _lib.check(lib.sgnn_ipc_get_handle(p.value, h), "ipc_get_handle")
            handles.append(bytes(h))
        torch.cuda.synchronize()
        gathered = [None] * self.world
        dist.all_gather_object(gathered, handles, group=group)
        self._opened = []
        self.ptrs = [[0] * self.world for _ in range(self.buffers)]
        for b in range(self.buffers):
            for q in range(self.world):
                if q == self.rank:
                    self.ptrs[b][q] = self._own[b]
                    continue
                out = _lib.C.c_void_p()
                h = (_lib.C.c_char * 64).from_buffer_copy(gathered[q][b])
                _lib.check(lib.sgnn_ipc_open_handle(h, _lib.C.byref(out)), "ipc_open_handle")
                self._opened.append(out.value)
                self.ptrs[b][q] = out.value
        if fence == "device":
            self._token = torch.zeros(1, device=dev)
        self._fence()

    def _fence(self):
        import torch
        if self.fence == "device":
            self.dist.all_reduce(self._token, group=self.group)
        else:
            torch.cuda.synchronize()
            self.dist.barrier(group=self.group)

    def publish(self, x_local):
        """Write this rank's rows; returns the part pointer table to read."""
        b = self.step % self.buffers
        self.step += 1
        self.views[b][: x_local.shape[0]].copy_(x_local)
        self._fence()
        return self.ptrs[b]

    def close(self):
        import torch
        if self._own is None:
            return
        torch.cuda.synchronize()
        self.dist.barrier(group=self.group)
        lib = _lib.lib()
        for p in self._opened:
            lib.sgnn_ipc_close_handle(p)
        self.dist.barrier(group=self.group)
        self.views = []
        for p in self._own:
            lib.sgnn_peer_free(p)
        self._own = None


class PeerExchange:
    """Exchange object for PartitionedSpmm.forward that selects the fused
    peer-memory path: one PeerBlocks per (stride, K), created on first use
    (collectively: every rank runs the same forward sequence)."""

    def __init__(self, group=None, fence: str = "device"):
        self.group, self.fence = group, fence
        self._blocks = {}

    def blocks_for(self, stride: int, k: int) -> PeerBlocks:
        key = (int(stride), int(k))
        if key not in self._blocks:
            self._blocks[key] = PeerBlocks(stride, k, self.group, self.fence)
        return self._blocks[key]

    def close(self):
        for b in self._blocks.values():
            b.close()
        self._blocks = {}
