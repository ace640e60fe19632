"""Row-partitioned 2-layer GraphSAGE training step over P ranks (BASELINE cfg5,
SURVEY 8e): the hot path (SpMM fwd x2, SpMM bwd x1 through the mean operand)
on each rank's row block, the all-gather of feature blocks as the only
sparse-path exchange (NCCL all-gather, or partition.PeerExchange: the SpMM
reads the other ranks' blocks in place over NVLink), and an all-reduce of the
dense weight gradients and the loss.  Mirrors gnn.hpp:234-244 (forward), :283-296 (backward), :318-349
(softmax_xent), :374-386 (sgd_step); with one rank it is exactly gnn.train's
step.

Ranks are torch.distributed processes (NCCL on the B200 box, gloo on CPU for
the tests); the local SpMM is the B200 kernel (or an injected `compute` on
CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import gnn, partition


def mean_operand_values(row_ptr, col_idx, values, degrees=None):
    """Values of TrainingCache::mean_operand (gnn.hpp:152-159): v / deg[col],
    IEEE fp32 divide.  `degrees` are a_hat's row degrees (default: those of
    row_ptr, the symmetric short-circuit where the operand is a_hat itself)."""
    deg = np.diff(np.asarray(row_ptr, np.uint64).astype(np.int64)) if degrees is None else np.asarray(degrees)
    deg = deg.astype(np.float32)
    return (np.asarray(values, np.float32) / deg[np.asarray(col_idx, np.int64)]).astype(np.float32)


def transpose_host(row_ptr, col_idx, values, n_cols):
    """transpose (sparse.hpp:72-89) on the host: column histogram, prefix sum,
    placement in ascending original row (a stable sort by column)."""
    rp = np.asarray(row_ptr, np.uint64).astype(np.int64)
    ci = np.asarray(col_idx, np.int64)
    rows = np.repeat(np.arange(len(rp) - 1, dtype=np.int64), np.diff(rp))
    order = np.argsort(ci, kind="stable")
    t_rp = np.zeros(n_cols + 1, np.uint64)
    t_rp[1:] = np.cumsum(np.bincount(ci, minlength=n_cols)).astype(np.uint64)
    return t_rp, rows[order].astype(np.uint32), np.asarray(values, np.float32)[order]


def is_symmetric_host(row_ptr, col_idx, values):
    """is_symmetric (sparse.hpp:179-192): A equals its transpose, structure
    and values."""
    n = len(row_ptr) - 1
    t_rp, t_ci, t_v = transpose_host(row_ptr, col_idx, values, n)
    return (np.array_equal(t_rp, np.asarray(row_ptr, np.uint64)) and np.array_equal(t_ci, np.asarray(col_idx, np.uint32))
            and np.array_equal(t_v, np.asarray(values, np.float32)))


@dataclass
class SageParams:
    w1: torch.Tensor
    w2: torch.Tensor
    w1_self: torch.Tensor
    w2_self: torch.Tensor


class DistSage:
    """One rank of the partitioned SAGE (sum or mean) trainer."""

    def __init__(self, row_ptr, col_idx, values, n_parts, rank, k_in, hidden, classes, reduce="mean",
                 device="cuda", exchange=None, allreduce=None, compute=None, symmetric=None, row_weight=1):
        """`symmetric`: None probes the graph like build_cache (gnn.hpp:194);
        a non-symmetric A runs its backward over rows of A^T (gnn.hpp:127-144,
        :149-160), partitioned at the same row bounds as A."""
        if symmetric is None:
            symmetric = is_symmetric_host(row_ptr, col_idx, values)
        self.symmetric = bool(symmetric)
        self.reduce = reduce
        self.exchange = exchange or partition.NcclExchange()
        # unpadded all-gather-v layout (global column ids); the peer path
        # splits remapped columns with a shift: padded pow2 block stride
        peer = isinstance(self.exchange, partition.PeerExchange)
        self.part = partition.make_partition(row_ptr, n_parts, pow2=peer, row_weight=row_weight)
        self.rank = rank
        self.r0, self.r1 = self.part.rows(rank)
        self.device = device
        self.allreduce = allreduce or _nccl_allreduce
        if self.symmetric:  # the operand is a_hat itself (mean: columns scaled in place)
            b_rp, b_ci = row_ptr, col_idx
            bwd_vals = mean_operand_values(row_ptr, col_idx, values) if reduce == "mean" else values
        else:  # rows of A^T; mean: scaled by the degree of the original row, now the column
            b_rp, b_ci, bwd_vals = transpose_host(row_ptr, col_idx, values, len(row_ptr) - 1)
            if reduce == "mean":
                bwd_vals = mean_operand_values(b_rp, b_ci, bwd_vals, degrees=np.diff(
                    np.asarray(row_ptr, np.uint64).astype(np.int64)))
        self.fwd = partition.PartitionedSpmm(row_ptr, col_idx, values, self.part, rank, k_in, device, compute)
        self.fwd2 = self.fwd if hidden == k_in else partition.PartitionedSpmm(
            row_ptr, col_idx, values, self.part, rank, hidden, device, compute)
        self.bwd = partition.PartitionedSpmm(b_rp, b_ci, bwd_vals, self.part, rank, hidden, device, compute)
        self.hidden, self.classes = hidden, classes
        self.use_glue = True  # the library's SAGE glue passes on CUDA tensors (False: torch ops)

    def step(self, params: SageParams, x_local, labels_local, mask_local, lr, n_masked_total):
        """One training step; returns the global mean loss."""
        if self.use_glue and x_local.is_cuda and gnn.sage_glue_ok(self.hidden, self.classes):
            return self._step_glue(params, x_local, labels_local, mask_local, lr, n_masked_total)
        red = self.reduce
        ex = self.exchange
        # forward (gnn.hpp:236-244)
        a1 = self.fwd.forward(x_local, ex, red)
        z1 = a1 @ params.w1 + x_local @ params.w1_self
        h1 = torch.relu(z1)
        a2 = self.fwd2.forward(h1, ex, red)
        logits = a2 @ params.w2 + h1 @ params.w2_self
        # softmax_xent over the global mask (gnn.hpp:318-349)
        ld = logits.double()
        row_max = ld.max(dim=1, keepdim=True).values
        e = torch.exp(ld - row_max)
        denom = e.sum(dim=1, keepdim=True)
        lab = labels_local.long()
        m = mask_local.bool()
        loss_rows = (row_max.squeeze(1) + torch.log(denom.squeeze(1))) - ld.gather(1, lab[:, None]).squeeze(1)
        loss_sum = loss_rows[m].sum().reshape(1)
        onehot = torch.zeros_like(e)
        onehot.scatter_(1, lab[:, None], 1.0)
        grad = ((e / denom - onehot) * (1.0 / n_masked_total)).float()
        grad[~m] = 0
        # backward (gnn.hpp:283-296); dense weight gradients are all-reduced
        g_w2 = a2.T @ grad
        g_w2s = h1.T @ grad
        ds2 = grad @ params.w2.T
        dh1 = self.bwd.forward(ds2, ex, "sum") + grad @ params.w2_self.T
        dz1 = torch.where(h1 <= 0, torch.zeros_like(dh1), dh1)
        g_w1 = a1.T @ dz1
        g_w1s = x_local.T @ dz1
        flat = self.allreduce(torch.cat([g_w1.ravel(), g_w2.ravel(), g_w1s.ravel(), g_w2s.ravel()]))
        loss_sum = self.allreduce(loss_sum)  # double, like the reference's accumulation
        sizes = [g_w1.numel(), g_w2.numel(), g_w1s.numel(), g_w2s.numel()]
        o = 0
        for p, g, n in zip((params.w1, params.w2, params.w1_self, params.w2_self), (g_w1, g_w2, g_w1s, g_w2s), sizes):
            p -= lr * flat[o:o + n].reshape(g.shape)
            o += n
        return float(loss_sum[0]) / n_masked_total


    def _step_glue(self, params: SageParams, x_local, labels_local, mask_local, lr, n_masked_total):
        """The same step with the library's SAGE glue passes (csrc/gnn.cu:
        add+relu, [a2|h1] logits, device softmax_xent, classes-wide weight
        gradients, grad W2s^T fused into relu_backward) around the
        partitioned SpMMs and the two big GEMMs per direction."""
        red = self.reduce
        ex = self.exchange
        # converted on every call (one cheap cast each): a cache keyed on the
        # labels alone would reuse a stale mask (train vs validation masks)
        lab = labels_local.to(torch.int32).contiguous()
        msk = mask_local.to(torch.uint8).contiguous()
        if lab.numel() and (int(lab.min()) < 0 or int(lab.max()) >= self.classes):
            raise partition._lib.ConfigError(f"softmax_xent: label out of range for {self.classes} classes")
        a1 = self.fwd.forward(x_local, ex, red)
        h1 = gnn.add_relu(gnn.dense_mm(a1, params.w1), gnn.dense_mm(x_local, params.w1_self))
        a2 = self.fwd2.forward(h1, ex, red)
        logits = gnn.sage_logits(a2, h1, params.w2, params.w2_self)
        grad, loss_sum, _ = gnn.softmax_xent_device(logits, lab, msk, 1.0 / n_masked_total)
        g_w2, g_w2s = gnn.sage_wgrad(a2, h1, grad)
        ds2 = gnn.sage_grad_wt(grad, params.w2)
        dz1 = gnn.sage_grad_wt(grad, params.w2_self, u=self.bwd.forward(ds2, ex, "sum"), act=h1)
        g_w1 = gnn.dense_mm(a1, dz1, transpose_a=True)
        g_w1s = gnn.dense_mm(x_local, dz1, transpose_a=True)
        flat = self.allreduce(torch.cat([g_w1.ravel(), g_w2.ravel(), g_w1s.ravel(), g_w2s.ravel()]))
        loss_sum = self.allreduce(loss_sum)
        o = 0
        for p, g in zip((params.w1, params.w2, params.w1_self, params.w2_self), (g_w1, g_w2, g_w1s, g_w2s)):
            p -= lr * flat[o:o + g.numel()].reshape(g.shape)
            o += g.numel()
        return float(loss_sum[0]) / n_masked_total


def _nccl_allreduce(t):
    import torch.distributed as dist
    dist.all_reduce(t)
    return t
