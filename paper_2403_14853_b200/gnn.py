"""GNN layer glue on the device -- the callers of the hot path
(gnn.hpp:75-438: init_model, forward, backward, softmax_xent, masked_accuracy,
sgd_step, train).  Every propagation is the B200 SpMM; every backward
propagation goes through the device TrainingCache (cached CSC / symmetric
short-circuit / 1/deg-scaled mean operand).  Dense products use torch
(cuBLAS SGEMM, TF32 disabled) and are outside the sparse hot path (north_star:
"any dense X·W ... is timed separately").
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False

KINDS = ("gcn", "sage-sum", "sage-mean", "gin")


@dataclass
class GnnModel:
    """GnnModel (gnn.hpp:40-63)."""
    kind: str
    in_features: int
    hidden: int
    classes: int
    w1: torch.Tensor
    w2: torch.Tensor
    w1_self: torch.Tensor | None = None
    w2_self: torch.Tensor | None = None
    epsilon: float = 0.0

    @property
    def has_self_weights(self):
        return self.kind in ("sage-sum", "sage-mean")

    @property
    def reduce(self):
        return "mean" if self.kind == "sage-mean" else "sum"

    def params(self):
        out = [self.w1, self.w2]
        if self.has_self_weights:
            out += [self.w1_self, self.w2_self]
        return out


@dataclass
class Gradients:
    w1: torch.Tensor
    w2: torch.Tensor
    w1_self: torch.Tensor | None = None
    w2_self: torch.Tensor | None = None
    epsilon: float = 0.0


def init_model(kind, in_features, hidden, classes, seed=1, device="cuda") -> GnnModel:
    """Glorot-uniform init (gnn.hpp:75-99 fill order w1, w2, w1_self, w2_self)."""
    if kind not in KINDS:
        raise ops.ConfigError(f"unknown model '{kind}' (expected gcn|sage-sum|sage-mean|gin)")
    if not (in_features and hidden and classes):
        raise ops.ConfigError("init_model: in_features, hidden, and classes must be positive")
    g = torch.Generator(device="cpu").manual_seed(seed)

    def glorot(r, c):
        lim = float(np.sqrt(6.0 / (r + c)))
        return ((torch.rand((r, c), generator=g, dtype=torch.float64) * 2 - 1) * lim).float().to(device)

    m = GnnModel(kind, in_features, hidden, classes, glorot(in_features, hidden), glorot(hidden, classes))
    if m.has_self_weights:
        m.w1_self, m.w2_self = glorot(in_features, hidden), glorot(hidden, classes)
    return m


def model_from_flat(kind, in_features, hidden, classes, flat, device="cuda") -> GnnModel:
    """Weights packed w1|w2|(w1_self|w2_self) (the reference's init order)."""
    flat = np.asarray(flat, np.float32)
    o = 0

    def take(r, c):
        nonlocal o
        t = torch.from_numpy(flat[o:o + r * c].reshape(r, c).copy()).to(device)
        o += r * c
        return t

    m = GnnModel(kind, in_features, hidden, classes, take(in_features, hidden), take(hidden, classes))
    if m.has_self_weights:
        m.w1_self, m.w2_self = take(in_features, hidden), take(hidden, classes)
    return m


def flat_weights(m: GnnModel) -> np.ndarray:
    return np.concatenate([p.detach().cpu().numpy().ravel() for p in m.params()])


@dataclass
class Tape:
    """Tape (gnn.hpp:199-207)."""
    n_nodes: int
    x: torch.Tensor
    h1: torch.Tensor | None = None
    a1: torch.Tensor | None = None
    a2: torch.Tensor | None = None


def build_cache(kind, a: ops.CsrMatrix, use_cache=True, add_self_loops=True) -> ops.TrainingCache:
    """build_cache (gnn.hpp:180-196) on the device."""
    return ops.TrainingCache(a, use_cache, model_kind=kind, add_self_loops=add_self_loops)


def _relu_backward(grad, act):
    return torch.where(act <= 0, torch.zeros_like(grad), grad)


def forward(model: GnnModel, cache: ops.TrainingCache, x: torch.Tensor):
    """forward (gnn.hpp:212-256)."""
    a_hat = cache.a_hat
    if x.shape[0] != a_hat.n_rows:
        raise ops.ShapeError(f"forward: features have {x.shape[0]} rows but graph has {a_hat.n_rows} nodes")
    if x.shape[1] != model.in_features:
        raise ops.ShapeError(f"forward: features have {x.shape[1]} columns but model expects {model.in_features}")
    tape = Tape(x.shape[0], x)
    if model.kind == "gcn":
        z1 = x @ model.w1
        tape.h1 = torch.relu(ops.spmm(a_hat, z1, "sum"))
        logits = ops.spmm(a_hat, tape.h1 @ model.w2, "sum")
    elif model.kind in ("sage-sum", "sage-mean"):
        red = model.reduce
        tape.a1 = ops.spmm(a_hat, x, red)
        z1 = tape.a1 @ model.w1 + x @ model.w1_self
        tape.h1 = torch.relu(z1)
        tape.a2 = ops.spmm(a_hat, tape.h1, red)
        logits = tape.a2 @ model.w2 + tape.h1 @ model.w2_self
    else:  # gin
        scale = 1.0 + model.epsilon
        tape.a1 = scale * x + ops.spmm(a_hat, x, "sum")
        tape.h1 = torch.relu(tape.a1 @ model.w1)
        tape.a2 = scale * tape.h1 + ops.spmm(a_hat, tape.h1, "sum")
        logits = tape.a2 @ model.w2
    return logits, tape


def backward(model: GnnModel, cache: ops.TrainingCache, tape: Tape, grad: torch.Tensor) -> Gradients:
    """backward (gnn.hpp:261-313); propagation transposes come from the cache."""
    if tape.n_nodes != cache.a_hat.n_rows or grad.shape[0] != tape.n_nodes:
        raise ops.TapeError(f"backward: tape covers {tape.n_nodes} nodes but graph/gradient expects "
                            f"{cache.a_hat.n_rows}/{grad.shape[0]}")
    if grad.shape[1] != model.classes:
        raise ops.TapeError(f"backward: grad_logits has {grad.shape[1]} columns, model has {model.classes} classes")
    if model.kind == "gcn":
        at = cache.sum_operand()  # fetched once per backward, used twice (gnn.hpp:274-279)
        dz2 = ops.spmm(at, grad.contiguous(), "sum")
        g = Gradients(None, tape.h1.T @ dz2)
        dp1 = _relu_backward(dz2 @ model.w2.T, tape.h1)
        dz1 = ops.spmm(at, dp1.contiguous(), "sum")
        g.w1 = tape.x.T @ dz1
        return g
    if model.kind in ("sage-sum", "sage-mean"):
        g = Gradients(None, tape.a2.T @ grad, None, tape.h1.T @ grad)
        ds2 = (grad @ model.w2.T).contiguous()
        dh1 = cache.spmm_backward(ds2, model.reduce) + grad @ model.w2_self.T
        dz1 = _relu_backward(dh1, tape.h1)
        g.w1 = tape.a1.T @ dz1
        g.w1_self = tape.x.T @ dz1
        return g
    scale = 1.0 + model.epsilon
    g = Gradients(None, tape.a2.T @ grad)
    dm2 = (grad @ model.w2.T).contiguous()
    deps = float((dm2.double() * tape.h1.double()).sum())
    dh1 = scale * dm2 + cache.spmm_backward(dm2, "sum")
    dz1 = _relu_backward(dh1, tape.h1)
    g.w1 = tape.a1.T @ dz1
    dm1 = dz1 @ model.w1.T
    deps += float((dm1.double() * tape.x.double()).sum())
    g.epsilon = deps
    return g


def softmax_xent(logits: torch.Tensor, labels: torch.Tensor, mask: torch.Tensor):
    """softmax_xent (gnn.hpp:318-349): mean -log softmax over masked rows, in double."""
    m = mask.bool()
    n_masked = int(m.sum())
    if n_masked == 0:
        raise ops.ConfigError("softmax_xent: mask selects no rows")
    if int(labels[m].max()) >= logits.shape[1]:
        raise ops.ConfigError("softmax_xent: label out of range")
    ld = logits.double()
    row_max = ld.max(dim=1, keepdim=True).values
    ex = torch.exp(ld - row_max)
    denom = ex.sum(dim=1, keepdim=True)
    lab = labels.long()
    loss_rows = (row_max.squeeze(1) + torch.log(denom.squeeze(1))) - ld.gather(1, lab[:, None]).squeeze(1)
    loss = float(loss_rows[m].sum()) / n_masked
    p = ex / denom
    onehot = torch.zeros_like(p)
    onehot.scatter_(1, lab[:, None], 1.0)
    grad = ((p - onehot) * (1.0 / n_masked)).float()
    grad[~m] = 0
    return loss, grad


def masked_accuracy(logits, labels, mask) -> float:
    """masked_accuracy (gnn.hpp:353-370); ties take the smallest class."""
    m = mask.bool()
    if int(m.sum()) == 0:
        return 0.0
    pred = logits.argmax(dim=1)
    return float((pred[m] == labels.long()[m]).double().mean())


def sgd_step(model: GnnModel, g: Gradients, lr: float) -> None:
    """sgd_step (gnn.hpp:374-386)."""
    model.w1 -= lr * g.w1
    model.w2 -= lr * g.w2
    if model.has_self_weights:
        model.w1_self -= lr * g.w1_self
        model.w2_self -= lr * g.w2_self
    if model.kind == "gin":
        model.epsilon -= lr * g.epsilon


@dataclass
class EpochStats:
    epoch: int
    loss: float
    train_accuracy: float
    epoch_seconds: float


@dataclass
class TrainOutput:
    stats: list = field(default_factory=list)
    cache: ops.TrainingCache | None = None


def _epoch_device(model: GnnModel, cache: ops.TrainingCache, x, lab, m, n_masked, lr, stats_out):
    """One epoch with no host synchronisation (CUDA-graph capturable): loss
    and accuracy are written to the device scalars in stats_out[0:2]; the
    weights move exactly as in the eager epoch (same gradients, same update)."""
    logits, tape = forward(model, cache, x)
    ld = logits.double()
    row_max = ld.max(dim=1, keepdim=True).values
    ex = torch.exp(ld - row_max)
    denom = ex.sum(dim=1, keepdim=True)
    loss_rows = (row_max.squeeze(1) + torch.log(denom.squeeze(1))) - ld.gather(1, lab[:, None]).squeeze(1)
    stats_out[0].copy_(torch.where(m, loss_rows, torch.zeros_like(loss_rows)).sum() / n_masked)
    pred = logits.argmax(dim=1)
    stats_out[1].copy_(((pred == lab) & m).sum().double() / n_masked)
    onehot = torch.zeros_like(ex)
    onehot.scatter_(1, lab[:, None], 1.0)
    grad = ((ex / denom - onehot) * (1.0 / n_masked)).float()
    grad = torch.where(m[:, None], grad, torch.zeros_like(grad))
    sgd_step(model, backward(model, cache, tape, grad), lr)


def _train_graphed(model, out, x, labels, mask, epochs, lr):
    """Epochs 2.. replay a CUDA graph of epoch 1 (captured after epoch 1 ran
    eagerly, which also builds every plan and cached operand): per epoch one
    graph launch instead of ~40 kernel launches and their Python dispatch.
    Operand fetches are counted once, at capture (the replays do not call the
    host API)."""
    m = mask.bool()
    n_masked = int(m.sum())
    if n_masked == 0:
        raise ops.ConfigError("softmax_xent: mask selects no rows")
    lab = labels.long()
    if int(lab[m].max()) >= model.classes:
        raise ops.ConfigError("softmax_xent: label out of range")
    stats = torch.zeros((epochs, 2), dtype=torch.float64, device=x.device)
    cur = torch.zeros(2, dtype=torch.float64, device=x.device)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(epochs + 1)]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # epoch 1, eager (warm-up for the capture)
        ev[0].record(side)
        _epoch_device(model, out.cache, x, lab, m, n_masked, lr, cur)
        stats[0].copy_(cur)
        ev[1].record(side)
    torch.cuda.current_stream().wait_stream(side)
    if epochs > 1:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            _epoch_device(model, out.cache, x, lab, m, n_masked, lr, cur)
        for e in range(1, epochs):
            g.replay()
            stats[e].copy_(cur)
            ev[e + 1].record()
    torch.cuda.synchronize()
    host = stats.cpu().numpy()
    for e in range(epochs):
        out.stats.append(EpochStats(e + 1, float(host[e, 0]), float(host[e, 1]),
                                    ev[e].elapsed_time(ev[e + 1]) * 1e-3))
    return out


def train(model: GnnModel, a: ops.CsrMatrix, x: torch.Tensor, labels: torch.Tensor, mask: torch.Tensor,
          epochs=100, lr=0.05, use_tuned=True, use_cache=True, add_self_loops=True,
          cuda_graph=False) -> TrainOutput:
    """train (gnn.hpp:414-438): the adjacency is prepared once (build_cache).
    cuda_graph=True replays a captured epoch (GCN / SAGE; GIN's epsilon
    update is a host scalar, so GIN always runs eagerly)."""
    if epochs < 1:
        raise ops.ConfigError("train: epochs must be >= 1")
    out = TrainOutput(cache=build_cache(model.kind, a, use_cache, add_self_loops))
    if cuda_graph and model.kind != "gin":
        with ops.DispatchGuard(use_tuned):
            return _train_graphed(model, out, x, labels, mask, epochs, lr)
    with ops.DispatchGuard(use_tuned):
        for epoch in range(1, epochs + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            logits, tape = forward(model, out.cache, x)
            loss, grad = softmax_xent(logits, labels, mask)
            acc = masked_accuracy(logits, labels, mask)
            sgd_step(model, backward(model, out.cache, tape, grad), lr)
            torch.cuda.synchronize()
            out.stats.append(EpochStats(epoch, loss, acc, time.perf_counter() - t0))
    return out


_KIND_IDS = {"gcn": 0, "sage-sum": 1, "sage-mean": 2, "gin": 3}


class NativeTrainOutput:
    """TrainOutput of the native engine: per-epoch stats and the engine's
    TrainingCache counters (gnn.hpp:121-123)."""

    def __init__(self, stats, counters):
        self.stats = stats
        self.counters = counters


def train_native(model: GnnModel, a: ops.CsrMatrix, x: torch.Tensor, labels: torch.Tensor, mask: torch.Tensor,
                 epochs=100, lr=0.05, use_cache=True, add_self_loops=True, cuda_graph=False) -> NativeTrainOutput:
    """train (gnn.hpp:414-438) in the native engine (sgnn_gnn_*, csrc/gnn.cu):
    every epoch runs inside the library (SpMM + cuBLAS + element-wise
    kernels); model's weights are updated in place at the end."""
    import ctypes as C
    from ._lib import check, lib
    L = lib()
    xs = x.contiguous()
    lab = labels.to(torch.int32).contiguous()
    msk = mask.to(torch.uint8).contiguous()
    h = C.c_void_p()
    check(L.sgnn_gnn_create(C.byref(a.c()), _KIND_IDS[model.kind], model.in_features, model.hidden, model.classes,
                            xs.data_ptr(), lab.data_ptr(), msk.data_ptr(), int(use_cache), int(add_self_loops),
                            int(epochs), C.byref(h), ops._stream()), "gnn_create")
    try:
        self_w = model.has_self_weights
        w1, w2 = model.w1.contiguous(), model.w2.contiguous()
        w1s = model.w1_self.contiguous() if self_w else None
        w2s = model.w2_self.contiguous() if self_w else None
        check(L.sgnn_gnn_set_weights(h, w1.data_ptr(), w2.data_ptr(), w1s.data_ptr() if self_w else None,
                                     w2s.data_ptr() if self_w else None, float(model.epsilon), ops._stream()),
              "gnn_set_weights")
        loss = (C.c_double * epochs)()
        acc = (C.c_double * epochs)()
        sec = (C.c_double * epochs)()
        check(L.sgnn_gnn_train(h, int(epochs), float(lr), int(cuda_graph), loss, acc, sec, ops._stream()), "train")
        eps = C.c_float()
        check(L.sgnn_gnn_get_weights(h, model.w1.data_ptr(), model.w2.data_ptr(),
                                     model.w1_self.data_ptr() if self_w else None,
                                     model.w2_self.data_ptr() if self_w else None, C.byref(eps), ops._stream()),
              "gnn_get_weights")
        model.epsilon = float(eps.value)
        t, n, hits, sym = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        check(L.sgnn_gnn_counters(h, C.byref(t), C.byref(n), C.byref(hits), C.byref(sym)), "gnn_counters")
        stats = [EpochStats(e + 1, float(loss[e]), float(acc[e]), float(sec[e])) for e in range(epochs)]
        return NativeTrainOutput(stats, {"transpose_builds": t.value, "normalize_builds": n.value,
                                         "cache_hits": hits.value, "symmetric": bool(sym.value)})
    finally:
        L.sgnn_gnn_destroy(h)


# ---------------------------------------------------------------- SAGE glue
# The library's SAGE layer-glue passes (sgnn_add_relu_f32, sgnn_sage_*_f32,
# sgnn_softmax_xent_f32; csrc/gnn.cu) over torch CUDA tensors, for trainers
# that sequence the layers themselves (sage_dist.DistSage on each rank).

def sage_glue_ok(hidden: int, classes: int) -> bool:
    """Shapes the classes-wide glue kernels take (hidden % 4 == 0, <= 128;
    1 <= classes <= 16)."""
    return hidden > 0 and hidden % 4 == 0 and hidden <= 128 and 1 <= classes <= 16


def _ptr(t):
    return t.data_ptr() if t is not None else None


def dense_mm(a: torch.Tensor, b: torch.Tensor, transpose_a: bool = False) -> torch.Tensor:
    """a @ b (or a.T @ b) for the layers' tall products on the tensor cores in
    FP32 emulation (sgnn_dense_mm_f32); shapes the kernels do not take
    (unaligned rows, short matrices) use torch's matmul on the same GPU."""
    from ._lib import lib
    if a.dim() != 2 or b.dim() != 2:
        raise ops.ShapeError(f"dense_mm: expected 2-D operands, got {tuple(a.shape)} and {tuple(b.shape)}")
    inner = a.shape[0] if transpose_a else a.shape[1]
    if b.shape[0] != inner:
        raise ops.ShapeError(f"dense_mm: {'A^T' if transpose_a else 'A'} is {tuple(a.T.shape if transpose_a else a.shape)}"
                             f" but B is {tuple(b.shape)}")
    if a.device != b.device:
        raise ops.ConfigError(f"dense_mm: operands on {a.device} and {b.device}")
    if a.shape[0] >= 4096 and a.is_cuda and a.is_contiguous() and b.is_contiguous() \
            and a.dtype == torch.float32 and b.dtype == torch.float32:
        m, k = a.shape
        n = b.shape[1]
        out = torch.empty((k, n) if transpose_a else (m, n), device=a.device)
        st = lib().sgnn_dense_mm_f32(1 if transpose_a else 0, m, n, k, a.data_ptr(), b.data_ptr(), out.data_ptr(),
                                     ops._stream())
        if st == 0:
            return out
        if st != _lib_status_unsupported():
            from ._lib import check
            check(st, "dense_mm")
    return a.T @ b if transpose_a else a @ b


def _lib_status_unsupported() -> int:
    return 10  # SGNN_ERR_UNSUPPORTED: a shape the tensor-core kernels do not take


def add_relu(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """relu(a + b) in one pass (SAGE's z1 = a1 W1 + X W1s, then relu)."""
    from ._lib import check, lib
    ops._dense(a, "add_relu a")
    ops._dense(b, "add_relu b")
    if a.shape != b.shape:
        raise ops.ShapeError(f"add_relu: {tuple(a.shape)} vs {tuple(b.shape)}")
    out = torch.empty_like(a) if out is None else out
    check(lib().sgnn_add_relu_f32(a.data_ptr(), b.data_ptr(), a.numel(), out.data_ptr(), ops._stream()), "add_relu")
    return out


def sage_logits(a2, h1, w2, w2s, out=None) -> torch.Tensor:
    """[a2 | h1] . [w2; w2s] (gnn.hpp:241-244)."""
    from ._lib import check, lib
    for t, nm in ((a2, "a2"), (h1, "h1"), (w2, "w2"), (w2s, "w2_self")):
        ops._dense(t, f"sage_logits {nm}")
    n, h = a2.shape
    c = w2.shape[1]
    if h1.shape != a2.shape or w2.shape != (h, c) or w2s.shape != (h, c):
        raise ops.ShapeError("sage_logits: operand shapes disagree")
    out = torch.empty(n, c, device=a2.device) if out is None else out
    check(lib().sgnn_sage_logits_f32(a2.data_ptr(), h1.data_ptr(), w2.data_ptr(), w2s.data_ptr(), n, h, c,
                                     out.data_ptr(), ops._stream()), "sage_logits")
    return out


def softmax_xent_device(logits, labels_u32, mask_u8, inv_count: float):
    """softmax_xent + masked_accuracy on the device (gnn.hpp:318-370):
    (grad, loss_sum double[1], correct int32[1]) -- sums, not means, so
    ranks can all-reduce them."""
    from ._lib import check, lib
    ops._dense(logits, "softmax_xent logits")
    n, c = logits.shape
    if labels_u32.dtype not in (torch.int32, torch.uint32) or labels_u32.numel() != n or not labels_u32.is_contiguous():
        raise ops.ConfigError("softmax_xent: labels must be a contiguous 32-bit integer tensor of one entry per row")
    if mask_u8.dtype != torch.uint8 or mask_u8.numel() != n or not mask_u8.is_contiguous():
        raise ops.ConfigError("softmax_xent: mask must be a contiguous uint8 tensor of one entry per row")
    if n and (int(labels_u32.min()) < 0 or int(labels_u32.max()) >= c):  # gnn.hpp:327
        raise ops.ConfigError(f"softmax_xent: label out of range for {c} classes")
    grad = torch.empty_like(logits)
    loss = torch.empty(1, dtype=torch.float64, device=logits.device)
    correct = torch.empty(1, dtype=torch.int32, device=logits.device)
    check(lib().sgnn_softmax_xent_f32(logits.data_ptr(), n, c, labels_u32.data_ptr(), mask_u8.data_ptr(),
                                      float(inv_count), grad.data_ptr(), loss.data_ptr(), correct.data_ptr(),
                                      ops._stream()), "softmax_xent")
    return grad, loss, correct


def sage_wgrad(a2, h1, grad):
    """(a2^T grad, h1^T grad): the classes-wide layer's weight gradients."""
    from ._lib import check, lib
    for t, nm in ((a2, "a2"), (h1, "h1"), (grad, "grad")):
        ops._dense(t, f"sage_wgrad {nm}")
    n, h = a2.shape
    c = grad.shape[1]
    if h1.shape != a2.shape or grad.shape[0] != n:
        raise ops.ShapeError("sage_wgrad: operand shapes disagree")
    g2 = torch.empty(h, c, device=a2.device)
    g2s = torch.empty(h, c, device=a2.device)
    check(lib().sgnn_sage_wgrad_f32(a2.data_ptr(), h1.data_ptr(), grad.data_ptr(), n, h, c, g2.data_ptr(),
                                    g2s.data_ptr(), ops._stream()), "sage_wgrad")
    return g2, g2s


def sage_grad_wt(grad, w, u=None, act=None, out=None):
    """grad w^T, or relu_backward(u + grad w^T, act) (gnn.hpp:285-292)."""
    from ._lib import check, lib
    ops._dense(grad, "sage_grad_wt grad")
    ops._dense(w, "sage_grad_wt w")
    n, c = grad.shape
    h = w.shape[0]
    if w.shape[1] != c:
        raise ops.ShapeError(f"sage_grad_wt: w is {tuple(w.shape)}, grad has {c} columns")
    if (u is None) != (act is None):
        raise ops.ConfigError("sage_grad_wt: u and act go together")
    for t, nm in ((u, "u"), (act, "act")):
        if t is not None:
            ops._dense(t, f"sage_grad_wt {nm}")
            if t.shape != (n, h):
                raise ops.ShapeError(f"sage_grad_wt: {nm} is {tuple(t.shape)}, expected {(n, h)}")
    out = torch.empty(n, h, device=grad.device) if out is None else out
    check(lib().sgnn_sage_grad_wt_f32(grad.data_ptr(), w.data_ptr(), n, h, c, _ptr(u), _ptr(act), out.data_ptr(),
                                      ops._stream()), "sage_grad_wt")
    return out
