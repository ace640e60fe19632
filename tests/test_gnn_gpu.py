"""GNN layer glue on the device (gnn.hpp:180-438) vs the reference's own
training runs (tests/golden/gnn_planted.npz, make_golden_gnn.py): per-epoch
losses, cache counters, cache/dispatch transparency, device
normalize_adjacency bit-exactness."""
import numpy as np
import pytest

from conftest import load_golden, rand_csr
from oracle import port

pytestmark = pytest.mark.gpu

HIDDEN, CLASSES, LR, EPOCHS = 32, 4, 0.05, 30


def _setup(kind):
    import torch

    from paper_2403_14853_b200 import gnn, ops
    g = load_golden("gnn_planted")
    a = ops.CsrMatrix.from_numpy(g["row_ptr"], g["col_idx"], g["values"], len(g["row_ptr"]) - 1)
    x = torch.from_numpy(g["x"]).cuda()
    lab = torch.from_numpy(g["labels"].astype(np.int64)).cuda()
    mask = torch.from_numpy(g["mask"]).cuda()
    m = gnn.model_from_flat(kind, x.shape[1], HIDDEN, CLASSES, g[f"{kind}_w0"])
    return g, a, x, lab, mask, m


@pytest.mark.parametrize("kind", ["gcn", "sage-sum", "sage-mean", "gin"])
def test_training_matches_reference(cuda, kind):
    from paper_2403_14853_b200 import gnn
    g, a, x, lab, mask, m = _setup(kind)
    out = gnn.train(m, a, x, lab, mask, epochs=EPOCHS, lr=LR)
    losses = np.array([s.loss for s in out.stats])
    want = g[f"{kind}_losses"]
    np.testing.assert_allclose(losses, want, rtol=2e-3, atol=1e-4)
    c = out.cache.counters
    assert [c["transpose_builds"], c["normalize_builds"], c["cache_hits"]] == [int(v) for v in g[f"{kind}_counters"]]
    assert abs(out.stats[-1].train_accuracy - g[f"{kind}_accs"][-1]) <= 0.02


@pytest.mark.parametrize("kind", ["gcn", "sage-sum", "sage-mean"])
def test_cuda_graph_training_matches_eager(cuda, kind):
    """train(cuda_graph=True) replays a captured epoch: final weights bitwise
    the eager run's, losses / accuracies equal (loss sums may differ in the
    last bits: masked-select vs masked-zero reduction), and faster epochs."""
    from paper_2403_14853_b200 import gnn
    g, a, x, lab, mask, m = _setup(kind)
    eager = gnn.train(m, a, x, lab, mask, epochs=EPOCHS, lr=LR)
    w_eager = gnn.flat_weights(m)
    _, _, _, _, _, m2 = _setup(kind)
    graphed = gnn.train(m2, a, x, lab, mask, epochs=EPOCHS, lr=LR, cuda_graph=True)
    np.testing.assert_array_equal(gnn.flat_weights(m2).view(np.uint32), w_eager.view(np.uint32))
    np.testing.assert_allclose([s.loss for s in graphed.stats], [s.loss for s in eager.stats], rtol=1e-12)
    assert [s.train_accuracy for s in graphed.stats] == [s.train_accuracy for s in eager.stats]
    np.testing.assert_allclose([s.loss for s in graphed.stats], g[f"{kind}_losses"], rtol=2e-3, atol=1e-4)
    t_eager = np.median([s.epoch_seconds for s in eager.stats[2:]])
    t_graph = np.median([s.epoch_seconds for s in graphed.stats[2:]])
    print(f"{kind}: eager {t_eager * 1e6:.1f} us/epoch, graphed {t_graph * 1e6:.1f} us/epoch")
    assert t_graph < t_eager


@pytest.mark.parametrize("kind", ["gcn", "sage-mean"])
def test_cache_and_dispatch_transparency(cuda, kind):
    """use_cache / use_tuned on vs off give bitwise-identical losses."""
    from paper_2403_14853_b200 import gnn
    g, a, x, lab, mask, m0 = _setup(kind)
    runs = {}
    for use_cache, use_tuned in ((True, True), (False, True), (True, False)):
        m = gnn.model_from_flat(kind, x.shape[1], HIDDEN, CLASSES, g[f"{kind}_w0"])
        out = gnn.train(m, a, x, lab, mask, epochs=10, lr=LR, use_cache=use_cache, use_tuned=use_tuned)
        runs[(use_cache, use_tuned)] = ([s.loss for s in out.stats], out.cache.counters)
    base = runs[(True, True)][0]
    assert runs[(False, True)][0] == base and runs[(True, False)][0] == base
    assert runs[(False, True)][1]["transpose_builds"] == int(g[f"{kind}_counters_nocache"][0]) * 10 // EPOCHS


def test_device_normalize_adjacency_bitexact(cuda):
    from paper_2403_14853_b200 import graphs, ops
    g = load_golden("gnn_planted")
    for rp, ci, v in ((g["row_ptr"], g["col_idx"], g["values"]),):
        a = ops.CsrMatrix.from_numpy(rp, ci, v, len(rp) - 1)
        for loops in (True, False):
            got = ops.normalize_adjacency(a, loops).to_numpy()
            want = port.normalize_adjacency(rp, ci, v, loops)
            for p, q in zip(got, want):
                np.testing.assert_array_equal(np.asarray(p).view(np.uint8), np.asarray(q).view(np.uint8))
    # weighted, with existing diagonals and empty rows; R-MAT with hubs
    rng = np.random.default_rng(2)
    rp, ci, v = rand_csr(rng, 700, 700, 0.01, hub_rows=(3,), empty_frac=0.2, value="positive")
    a = ops.CsrMatrix.from_numpy(rp, ci, v, 700)
    got = ops.normalize_adjacency(a, True).to_numpy()
    for p, q in zip(got, port.normalize_adjacency(rp, ci, v, True)):
        np.testing.assert_array_equal(np.asarray(p).view(np.uint8), np.asarray(q).view(np.uint8))
    rp, ci = graphs.rmat(12, 4096 * 12, seed=9, symmetrize=True)
    v = np.ones(len(ci), np.float32)
    got = ops.normalize_adjacency(ops.CsrMatrix.from_numpy(rp, ci, v, 4096), True).to_numpy()
    for p, q in zip(got, port.normalize_adjacency(rp, ci, v, True)):
        np.testing.assert_array_equal(np.asarray(p).view(np.uint8), np.asarray(q).view(np.uint8))
    with pytest.raises(ops.ConfigError):
        ops.normalize_adjacency(ops.CsrMatrix.from_numpy(np.array([0, 1], np.uint64), np.array([0], np.uint32),
                                                         np.array([-1.0], np.float32), 1))


def test_tape_and_shape_errors(cuda):
    import torch

    from paper_2403_14853_b200 import gnn, ops
    g, a, x, lab, mask, m = _setup("gcn")
    cache = gnn.build_cache("gcn", a)
    with pytest.raises(ops.ShapeError):
        gnn.forward(m, cache, x[:10])
    logits, tape = gnn.forward(m, cache, x)
    with pytest.raises(ops.TapeError):
        gnn.backward(m, cache, tape, torch.zeros(10, CLASSES, device="cuda"))


@pytest.mark.parametrize("kind", ["gcn", "sage-sum", "sage-mean", "gin"])
def test_native_engine_matches_reference(cuda, kind):
    """The native engine (sgnn_gnn_*, csrc/gnn.cu: SpMM + cuBLAS + device
    softmax-xent / SGD) reproduces the reference's train(): losses, cache
    counters, final accuracy; weights close to the torch engine's."""
    from paper_2403_14853_b200 import gnn
    g, a, x, lab, mask, m = _setup(kind)
    out = gnn.train_native(m, a, x, lab, mask, epochs=EPOCHS, lr=LR)
    losses = np.array([s.loss for s in out.stats])
    np.testing.assert_allclose(losses, g[f"{kind}_losses"], rtol=2e-3, atol=1e-4)
    c = out.counters
    assert [c["transpose_builds"], c["normalize_builds"], c["cache_hits"]] == [int(v) for v in g[f"{kind}_counters"]]
    assert abs(out.stats[-1].train_accuracy - g[f"{kind}_accs"][-1]) <= 0.02
    _, _, _, _, _, m2 = _setup(kind)
    gnn.train(m2, a, x, lab, mask, epochs=EPOCHS, lr=LR)
    np.testing.assert_allclose(gnn.flat_weights(m), gnn.flat_weights(m2), rtol=1e-3, atol=1e-5)


@pytest.mark.parametrize("kind", ["gcn", "sage-mean", "gin"])
def test_native_engine_cuda_graph_bitwise(cuda, kind):
    """Replaying the captured epoch gives bitwise the eager native run."""
    from paper_2403_14853_b200 import gnn
    _, a, x, lab, mask, m = _setup(kind)
    eager = gnn.train_native(m, a, x, lab, mask, epochs=EPOCHS, lr=LR)
    _, _, _, _, _, m2 = _setup(kind)
    graphed = gnn.train_native(m2, a, x, lab, mask, epochs=EPOCHS, lr=LR, cuda_graph=True)
    np.testing.assert_array_equal(gnn.flat_weights(m2).view(np.uint32), gnn.flat_weights(m).view(np.uint32))
    assert [s.loss for s in graphed.stats] == [s.loss for s in eager.stats]
    t_e = np.median([s.epoch_seconds for s in eager.stats[2:]])
    t_g = np.median([s.epoch_seconds for s in graphed.stats[2:]])
    print(f"native {kind}: eager {t_e * 1e6:.1f} us/epoch, graphed {t_g * 1e6:.1f} us/epoch")


def test_native_engine_errors(cuda):
    """gnn.hpp's error classes through the native engine."""
    import torch

    from paper_2403_14853_b200 import _lib, gnn, ops
    g, a, x, lab, mask, m = _setup("gcn")
    with pytest.raises(_lib.ConfigError):  # label out of range (softmax_xent)
        gnn.train_native(m, a, x, torch.full_like(lab, CLASSES), mask, epochs=2)
    with pytest.raises(_lib.ConfigError):  # empty mask
        gnn.train_native(m, a, x, lab, torch.zeros_like(mask), epochs=2)
    rect = ops.CsrMatrix.from_numpy(np.array([0, 1], np.uint64), np.array([1], np.uint32),
                                    np.array([1.0], np.float32), 2)
    with pytest.raises(_lib.ShapeError):  # build_cache: adjacency must be square
        gnn.train_native(m, rect, x[:1], lab[:1], mask[:1], epochs=2)


@pytest.mark.parametrize("hidden,classes", [(128, 16), (64, 10), (32, 3)])
def test_native_sage_classes_wide_kernels(cuda, monkeypatch, hidden, classes):
    """SAGE's classes-wide products (logits, W2/W2s gradients, grad W2^T and
    the fused grad W2s^T + relu_backward: sage_*_kernel in csrc/gnn.cu) vs
    the same engine on cuBLAS (SGNN_GNN_CUBLAS_SKINNY): losses and weights
    agree to fp32 reassociation, on a symmetric graph with hub and empty rows."""
    import torch

    from paper_2403_14853_b200 import gnn, graphs, ops
    rp, ci = graphs.rmat(11, 2048 * 8, seed=5, symmetrize=True)
    n = len(rp) - 1
    a = ops.CsrMatrix.from_numpy(rp, ci, np.ones(len(ci), np.float32), n)
    rng = np.random.default_rng(3)
    x = torch.from_numpy(rng.standard_normal((n, 48)).astype(np.float32)).cuda()
    lab = torch.from_numpy(rng.integers(0, classes, n)).cuda()
    mask = torch.from_numpy((rng.random(n) < 0.7).astype(np.uint8)).cuda()
    runs = []
    for cublas in (False, True):
        if cublas:
            monkeypatch.setenv("SGNN_GNN_CUBLAS_SKINNY", "1")
        m = gnn.init_model("sage-mean", 48, hidden, classes, seed=2)
        out = gnn.train_native(m, a, x, lab, mask, epochs=8, lr=0.05)
        runs.append(([s.loss for s in out.stats], gnn.flat_weights(m)))
    np.testing.assert_allclose(runs[0][0], runs[1][0], rtol=1e-5)
    np.testing.assert_allclose(runs[0][1], runs[1][1], rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("hidden,classes", [(128, 16), (64, 10)])
def test_dist_sage_glue_step_matches_torch_step(cuda, hidden, classes):
    """The row-partitioned SAGE-mean step (sage_dist.DistSage, one rank) with
    the library's glue passes vs the same step in torch ops: losses and
    weights agree to fp32 reassociation."""
    import torch

    from paper_2403_14853_b200 import graphs, sage_dist

    class Local:  # one rank: the gathered operand is the local block
        def all_gather(self, block):
            return block.contiguous()

        def all_gather_v(self, block, bounds):
            return block.contiguous()

    rp, ci = graphs.rmat(11, 2048 * 8, seed=9, symmetrize=True, self_loops=True)
    n = len(rp) - 1
    v = np.ones(len(ci), np.float32)
    rng = np.random.default_rng(4)
    f = 32
    x = torch.from_numpy(rng.standard_normal((n, f)).astype(np.float32)).cuda()
    lab = torch.from_numpy(rng.integers(0, classes, n)).cuda()
    mask = torch.from_numpy((rng.random(n) < 0.8).astype(np.uint8)).cuda()
    w0 = [torch.from_numpy((0.1 * rng.standard_normal(s)).astype(np.float32)).cuda()
          for s in ((f, hidden), (hidden, classes), (f, hidden), (hidden, classes))]
    runs = []
    for glue in (True, False):
        ds = sage_dist.DistSage(rp, ci, v, 1, 0, f, hidden, classes, "mean", device="cuda", exchange=Local(),
                                allreduce=lambda t: t)
        ds.use_glue = glue
        params = sage_dist.SageParams(*[w.clone() for w in w0])
        losses = [ds.step(params, x, lab, mask, 0.05, int(mask.sum())) for _ in range(5)]
        runs.append((losses, torch.cat([p.ravel() for p in (params.w1, params.w2, params.w1_self, params.w2_self)])))
    np.testing.assert_allclose(runs[0][0], runs[1][0], rtol=1e-5)
    np.testing.assert_allclose(runs[0][1].cpu().numpy(), runs[1][1].cpu().numpy(), rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("kind", ["sage-mean", "gcn"])
def test_native_tensor_core_gemms_match_sgemm(cuda, monkeypatch, kind):
    """The engine's tall products (X W, A^T G over all rows) on the tensor
    cores in FP32 emulation (csrc/dense_*.cu) vs the same engine on cuBLAS
    SGEMM (SGNN_GNN_CUBLAS_DENSE): losses and weights agree to fp32
    reassociation; the emulated products are checked against fp64 too."""
    import torch

    from paper_2403_14853_b200 import gnn, graphs, ops
    rp, ci = graphs.rmat(13, 8192 * 8, seed=6, symmetrize=True)
    n = len(rp) - 1
    a = ops.CsrMatrix.from_numpy(rp, ci, np.ones(len(ci), np.float32), n)
    rng = np.random.default_rng(8)
    x = torch.from_numpy(rng.standard_normal((n, 64)).astype(np.float32)).cuda()
    lab = torch.from_numpy(rng.integers(0, 8, n)).cuda()
    mask = torch.from_numpy((rng.random(n) < 0.6).astype(np.uint8)).cuda()
    runs = []
    for cublas in (False, True):
        if cublas:
            monkeypatch.setenv("SGNN_GNN_CUBLAS_DENSE", "1")
        m = gnn.init_model(kind, 64, 128, 8, seed=3)
        out = gnn.train_native(m, a, x, lab, mask, epochs=6, lr=0.05)
        runs.append(([s.loss for s in out.stats], gnn.flat_weights(m)))
    assert not np.array_equal(runs[0][1], runs[1][1])  # two different GEMM paths ran
    np.testing.assert_allclose(runs[0][0], runs[1][0], rtol=1e-5)
    np.testing.assert_allclose(runs[0][1], runs[1][1], rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("m,k,n", [(5000, 128, 128), (70000, 64, 96), (4100, 256, 32)])
def test_dense_mm_tensor_core_fp32(cuda, m, k, n):
    """sgnn_dense_mm_f32 (tensor-core FP32 emulation) vs fp64: A B and A^T B
    within 1e-6 of sum|a*b| -- tighter than SGEMM needs -- and deterministic."""
    import torch

    from paper_2403_14853_b200 import gnn
    g = torch.Generator(device="cuda").manual_seed(m + k + n)
    a = torch.randn(m, k, device="cuda", generator=g)
    b = torch.randn(k, n, device="cuda", generator=g)
    b2 = torch.randn(m, n, device="cuda", generator=g)
    c = gnn.dense_mm(a, b)
    want = a.double() @ b.double()
    den = a.double().abs() @ b.double().abs()
    assert ((c.double() - want).abs() <= 1e-6 * den).all()
    t = gnn.dense_mm(a, b2, transpose_a=True)
    want = a.double().T @ b2.double()
    den = a.double().abs().T @ b2.double().abs()
    assert ((t.double() - want).abs() <= 1e-6 * den).all()
    assert torch.equal(gnn.dense_mm(a, b2, transpose_a=True).view(torch.int32), t.view(torch.int32))


def test_native_cuda_graph_with_tensor_core_gemms(cuda):
    """CUDA-graph epochs with the tensor-core FP32 products in the captured
    graph (graph of 8192 nodes: tall products on dense_*.cu) replay bitwise
    the eager epochs."""
    import torch

    from paper_2403_14853_b200 import gnn, graphs, ops
    rp, ci = graphs.rmat(13, 8192 * 8, seed=12, symmetrize=True)
    n = len(rp) - 1
    a = ops.CsrMatrix.from_numpy(rp, ci, np.ones(len(ci), np.float32), n)
    rng = np.random.default_rng(9)
    x = torch.from_numpy(rng.standard_normal((n, 64)).astype(np.float32)).cuda()
    lab = torch.from_numpy(rng.integers(0, 8, n)).cuda()
    mask = torch.from_numpy((rng.random(n) < 0.6).astype(np.uint8)).cuda()
    m1 = gnn.init_model("sage-mean", 64, 128, 8, seed=4)
    eager = gnn.train_native(m1, a, x, lab, mask, epochs=5, lr=0.05)
    m2 = gnn.init_model("sage-mean", 64, 128, 8, seed=4)
    graphed = gnn.train_native(m2, a, x, lab, mask, epochs=5, lr=0.05, cuda_graph=True)
    np.testing.assert_array_equal(gnn.flat_weights(m2).view(np.uint32), gnn.flat_weights(m1).view(np.uint32))
    assert [s.loss for s in graphed.stats] == [s.loss for s in eager.stats]
