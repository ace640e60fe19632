"""Multi-GPU row partition.  CPU: the partitioner, the column
remap and the all-gather/reassembly logic with world_size 2 over gloo, local
compute by the oracle.  GPU: P virtual partitions on one device (loopback
exchange) must reproduce the single-GPU SpMM bit for bit."""
import os
import socket

import numpy as np
import pytest

from conftest import rand_csr
from oracle import port


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_compute(local, gathered, reduce):
    import torch
    rp, ci, v = local
    red = {"sum": 0, "min": 1, "max": 2, "mean": 3}[reduce]
    out = port.spmm(rp, ci, v, gathered.numpy(), red, np.float32)
    return torch.from_numpy(out)


def test_partition_blocks_cover_and_remap():
    """Padded owner layout (the peer path): blocks cover the graph, the remap
    is invertible and keeps every row strictly increasing."""
    from paper_2403_14853_b200 import partition
    rng = np.random.default_rng(0)
    n = 500
    rp, ci, v = rand_csr(rng, n, n, 0.02, hub_rows=(0, 7), empty_frac=0.1)
    for parts in (1, 2, 3, 8):
        pt = partition.make_partition(rp, parts, padded=True)
        np.testing.assert_array_equal(pt.bounds, port.balanced_row_partition(rp, parts))
        assert pt.stride >= max(np.diff(pt.bounds.astype(np.int64)))
        total = 0
        for p in range(parts):
            lrp, lci, lv = pt.block(rp, ci, v, p)
            r0, r1 = pt.rows(p)
            total += len(lci)
            # inverse remap recovers the global columns in the same order
            owner = lci // pt.stride
            glob = pt.bounds[owner] + (lci % pt.stride)
            np.testing.assert_array_equal(glob, ci[rp[r0]:rp[r1]])
            np.testing.assert_array_equal(lv, v[rp[r0]:rp[r1]])
            for i in range(len(lrp) - 1):  # the remap keeps every row strictly increasing
                row = lci[lrp[i]:lrp[i + 1]].astype(np.int64)
                assert (np.diff(row) > 0).all()
        assert total == len(ci)


def test_unpadded_partition_keeps_global_columns():
    """Default (all-gather-v) layout: no padding, blocks are plain row slices
    with global column ids; the gathered operand has exactly n rows."""
    from paper_2403_14853_b200 import partition
    rng = np.random.default_rng(1)
    n = 700
    rp, ci, v = rand_csr(rng, n, n, 0.02, hub_rows=(0, 3), empty_frac=0.1)
    for parts in (1, 2, 5, 8):
        for w in (1, 30):
            pt = partition.make_partition(rp, parts, row_weight=w)
            assert not pt.padded and pt.n_gathered == n
            if w == 1:
                np.testing.assert_array_equal(pt.bounds, port.balanced_row_partition(rp, parts))
            cat = [pt.block(rp, ci, v, p) for p in range(parts)]
            np.testing.assert_array_equal(np.concatenate([c[1] for c in cat]), ci)
            np.testing.assert_array_equal(np.concatenate([c[2] for c in cat]), v)
            for p, (lrp, _, _) in enumerate(cat):
                r0, r1 = pt.rows(p)
                np.testing.assert_array_equal(lrp, rp[r0:r1 + 1] - rp[r0])


@pytest.mark.parametrize("parts", [2, 3, 4, 8])
def test_weighted_row_partition_balances_cost(parts):
    """sgnn_host_weighted_row_partition: w = 1 is balanced_row_partition
    exactly; any w gives contiguous blocks whose cost nnz + w*rows is within
    one row's cost of the even share."""
    from paper_2403_14853_b200 import dist, graphs
    rp, _ = graphs.rmat(13, (1 << 13) * 20, seed=2, symmetrize=True, self_loops=True)
    np.testing.assert_array_equal(dist.row_partition(rp, parts, 1), port.balanced_row_partition(rp, parts))
    for w in (1, 7, 30, 1000):
        b = dist.row_partition(rp, parts, w).astype(np.int64)
        assert b[0] == 0 and b[-1] == len(rp) - 1 and (np.diff(b) >= 0).all()
        cost = rp.astype(np.int64) + w * np.arange(len(rp))
        total = int(cost[-1])
        for c in range(1, parts):
            target = total * c // parts
            assert cost[b[c]] >= target and (b[c] == 0 or cost[b[c] - 1] < target)


def _worker(rank, world, port_, rp, ci, v, x, reduce, q, row_weight=1):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_14853_b200 import partition
        pt = partition.make_partition(rp, world, row_weight=row_weight)
        ps = partition.PartitionedSpmm(rp, ci, v, pt, rank, x.shape[1], device="cpu", compute=_oracle_compute)
        r0, r1 = pt.rows(rank)
        c_local = ps.forward(torch.from_numpy(x[r0:r1].copy()), partition.NcclExchange(), reduce)
        # reassemble on every rank through the same all-gather-v (uneven blocks)
        full = partition.NcclExchange().all_gather_v(c_local, pt.bounds)
        if rank == 0:
            q.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("reduce,world,row_weight", [("sum", 2, 1), ("mean", 2, 30), ("max", 2, 1), ("sum", 3, 30)])
def test_two_rank_gloo_matches_single_process(reduce, world, row_weight):
    import torch.multiprocessing as mp
    rng = np.random.default_rng(3)
    n = 400
    rp, ci, v = rand_csr(rng, n, n, 0.03, hub_rows=(1,), empty_frac=0.1)
    x = rng.uniform(-1, 1, (n, 16)).astype(np.float32)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_, rp, ci, v, x, reduce, q, row_weight))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = port.spmm(rp, ci, v, x, {"sum": 0, "max": 2, "mean": 3}[reduce], np.float32)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def _sage_worker(rank, world, port_, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from conftest import load_golden

        from paper_2403_14853_b200 import partition, sage_dist
        g = load_golden("gnn_planted")
        rp, ci, v, x = g["row_ptr"], g["col_idx"], g["values"], g["x"]
        n, f = x.shape
        hidden, classes = 32, 4
        ds = sage_dist.DistSage(rp, ci, v, world, rank, f, hidden, classes, "mean", device="cpu",
                                exchange=partition.NcclExchange(), compute=_oracle_compute)
        w0 = g["sage-mean_w0"]
        o = [0]

        def take(r, c):
            t = torch.from_numpy(w0[o[0]:o[0] + r * c].reshape(r, c).copy())
            o[0] += r * c
            return t
        params = sage_dist.SageParams(take(f, hidden), take(hidden, classes), take(f, hidden), take(hidden, classes))
        r0, r1 = ds.r0, ds.r1
        xl = torch.from_numpy(x[r0:r1].copy())
        lab = torch.from_numpy(g["labels"][r0:r1].astype(np.int64))
        mask = torch.from_numpy(g["mask"][r0:r1].copy())
        losses = [ds.step(params, xl, lab, mask, 0.05, int(g["mask"].sum())) for _ in range(6)]
        if rank == 0:
            q.put(losses)
    finally:
        dist.destroy_process_group()


def test_two_rank_sage_mean_step_matches_reference():
    """The partitioned SAGE-mean step (gloo, 2 ranks, oracle SpMM) reproduces
    the reference's own training losses (tests/golden/gnn_planted.npz)."""
    import torch.multiprocessing as mp

    from conftest import load_golden
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_sage_worker, args=(r, 2, port_, q)) for r in range(2)]
    for p in procs:
        p.start()
    losses = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = load_golden("gnn_planted")["sage-mean_losses"][:6]
    np.testing.assert_allclose(losses, want, rtol=2e-3, atol=1e-5)


def _nonsym_case():
    rng = np.random.default_rng(11)
    n, f = 300, 16
    rp, ci, v = rand_csr(rng, n, n, 0.03, hub_rows=(2,), value="positive")
    x = rng.normal(0, 1, (n, f)).astype(np.float32)
    lab = rng.integers(0, 4, n).astype(np.uint32)
    mask = (rng.random(n) < 0.7).astype(np.uint8)
    return rp, ci, v, x, lab, mask


def _nonsym_worker(rank, world, port_, q, kind, w0):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_14853_b200 import partition, sage_dist
        rp, ci, v, x, lab, mask = _nonsym_case()
        n, f = x.shape
        hidden, classes = 32, 4
        ds = sage_dist.DistSage(rp, ci, v, world, rank, f, hidden, classes, kind.split("-")[1], device="cpu",
                                exchange=partition.NcclExchange(), compute=_oracle_compute)
        assert not ds.symmetric  # probed like build_cache (gnn.hpp:194)
        o = [0]

        def take(r, c):
            t = torch.from_numpy(w0[o[0]:o[0] + r * c].reshape(r, c).copy())
            o[0] += r * c
            return t
        params = sage_dist.SageParams(take(f, hidden), take(hidden, classes), take(f, hidden), take(hidden, classes))
        r0, r1 = ds.r0, ds.r1
        losses = [ds.step(params, torch.from_numpy(x[r0:r1].copy()), torch.from_numpy(lab[r0:r1].astype(np.int64)),
                          torch.from_numpy(mask[r0:r1].copy()), 0.05, int(mask.sum())) for _ in range(8)]
        if rank == 0:
            q.put(losses)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["sage-mean", "sage-sum"])
def test_two_rank_non_symmetric_backward_matches_reference(kind):
    """A non-symmetric A (gloo, 2 ranks, oracle SpMM): the backward runs over
    rows of A^T (mean: scaled by the original row's degree), gnn.hpp:127-160;
    losses match the reference's own train() on the same graph (oracle/_ref)."""
    import torch.multiprocessing as mp

    from oracle import ref
    from paper_2403_14853_b200 import sage_dist
    rp, ci, v, x, lab, mask = _nonsym_case()
    # the host transpose is the reference's, bit for bit
    t = sage_dist.transpose_host(rp, ci, v, x.shape[0])
    for a, b in zip(t, port.transpose(rp, ci, v, x.shape[0])):
        np.testing.assert_array_equal(np.asarray(a), np.asarray(b))
    w0 = ref.init_model(kind, x.shape[1], 32, 4, 5)
    want, _, _, _ = ref.train(kind, rp, ci, v, x, lab, mask, 32, 4, w0, 8, 0.05)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_nonsym_worker, args=(r, 2, port_, q, kind, w0)) for r in range(2)]
    for p in procs:
        p.start()
    losses = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_allclose(losses, want, rtol=2e-3, atol=1e-5)


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_loopback_partition_bitwise_equals_single_gpu(cuda, parts):
    import torch

    from paper_2403_14853_b200 import graphs, ops, partition
    rp, ci = graphs.rmat(14, (1 << 14) * 24, seed=5, symmetrize=True, self_loops=True)
    n = 1 << 14
    v = np.ones(len(ci), np.float32)
    x = torch.from_numpy(graphs.normal(n * 64, 0, 1, 3).reshape(n, 64)).cuda()
    a = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    for reduce in ("sum", "mean"):
        want = ops.spmm(a, x, reduce).cpu().numpy()
        pt = partition.make_partition(rp, parts)
        ranks = [partition.PartitionedSpmm(rp, ci, v, pt, p, 64) for p in range(parts)]
        blocks = [partition.pad_block(x[pt.rows(p)[0]:pt.rows(p)[1]], pt.stride) for p in range(parts)]
        gathered = partition.LoopbackExchange().all_gather(blocks)
        got = np.concatenate([r.compute(gathered, reduce).cpu().numpy() for r in ranks])
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [1, 2, 3, 8])
@pytest.mark.parametrize("k", [64, 128, 30])
def test_peer_spmm_bitwise_equals_single_gpu(cuda, parts, k):
    """sgnn_spmm_peer_f32 reading P separately allocated blocks (stand-ins for
    the peers' HBM) reproduces the single-GPU SpMM bit for bit."""
    import torch

    from paper_2403_14853_b200 import graphs, ops, partition
    n = 1 << 13
    rp, ci = graphs.rmat(13, n * 24, seed=9, symmetrize=True, self_loops=True)
    v = graphs.uniform(len(ci), 0.1, 1.0, 4)
    x = torch.from_numpy(graphs.normal(n * k, 0, 1, 3).reshape(n, k)).cuda()
    a = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    pt = partition.make_partition(rp, parts, pow2=True)
    ranks = [partition.PartitionedSpmm(rp, ci, v, pt, p, k) for p in range(parts)]
    blocks = [partition.pad_block(x[pt.rows(p)[0]:pt.rows(p)[1]], pt.stride) for p in range(parts)]
    for reduce in ("sum", "mean"):
        want = ops.spmm(a, x, reduce).cpu().numpy()
        got = np.concatenate([r.compute_peer(blocks, reduce).cpu().numpy() for r in ranks])
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    # raw pointer table form
    got0 = ranks[0].compute_peer([b.data_ptr() for b in blocks], "sum").cpu().numpy()
    np.testing.assert_array_equal(got0.view(np.uint32), ops.spmm(a, x, "sum")[: pt.rows(0)[1]].cpu().numpy().view(np.uint32))


@pytest.mark.gpu
def test_peer_spmm_rejects_bad_arguments(cuda):
    import torch

    from paper_2403_14853_b200 import _lib, graphs, ops, partition
    n = 1000
    rp, ci = graphs.er(n, n, 8, seed=1)
    v = np.ones(len(ci), np.float32)
    pt = partition.make_partition(rp, 2, pow2=True)
    r = partition.PartitionedSpmm(rp, ci, v, pt, 0, 32)
    blocks = [torch.zeros((pt.stride, 32), device="cuda") for _ in range(2)]
    with pytest.raises(_lib.UnsupportedError):
        r.compute_peer(blocks, "max")
    with pytest.raises(_lib.ShapeError):  # 1 part cannot cover 2*stride columns
        ops.spmm_peer(r._a, blocks[:1], pt.shift, 32, "sum", r._plan)
    with pytest.raises(ValueError):  # the peer path needs a pow2 stride
        partition.RowPartition(pt.bounds, pt.stride - 1, n).shift


def _ipc_worker(rank, world, port_, rp, ci, v, x, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_14853_b200 import partition
        torch.cuda.set_device(0)
        k = x.shape[1]
        pt = partition.make_partition(rp, world, pow2=True)
        r = partition.PartitionedSpmm(rp, ci, v, pt, rank, k)
        r0, r1 = pt.rows(rank)
        blocks = partition.PeerBlocks(pt.stride, k, fence="host")
        outs = []
        for step in range(3):  # exercises both buffers and the reuse fence
            xl = torch.from_numpy(x[r0:r1] * (step + 1)).cuda()
            outs.append(r.forward_peer(xl, blocks, "sum").cpu().numpy())
        blocks.close()
        gathered = [None] * world
        dist.all_gather_object(gathered, outs)
        if rank == 0:
            q.put([np.concatenate([g[s] for g in gathered]) for s in range(3)])
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_peer_blocks_ipc_two_processes(cuda):
    """The IPC handshake of PeerBlocks: two processes share the one GPU (host
    fences over gloo, so no kernel waits on another), each SpMM reads the
    other's block through an IPC mapping; bitwise the single-process result."""
    import torch
    import torch.multiprocessing as mp

    from paper_2403_14853_b200 import graphs, ops
    n = 3000
    rp, ci = graphs.er(n, n, 12, seed=2)
    v = graphs.uniform(len(ci), -1.0, 1.0, 5)
    x = graphs.normal(n * 64, 0, 1, 6).reshape(n, 64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port_, rp, ci, v, x, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    for s in range(3):
        want = ops.spmm(a, torch.from_numpy(x * (s + 1)).cuda(), "sum").cpu().numpy()
        np.testing.assert_array_equal(got[s].view(np.uint32), want.view(np.uint32))


def _sage_peer_worker(rank, world, port_, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from conftest import load_golden

        from paper_2403_14853_b200 import partition, sage_dist
        torch.cuda.set_device(0)
        g = load_golden("gnn_planted")
        rp, ci, v, x = g["row_ptr"], g["col_idx"], g["values"], g["x"]
        n, f = x.shape
        hidden, classes = 32, 4

        def allreduce(t):  # gloo reduces host tensors
            h = t.cpu()
            dist.all_reduce(h)
            return h.to(t.device)
        ex = partition.PeerExchange(fence="host")
        ds = sage_dist.DistSage(rp, ci, v, world, rank, f, hidden, classes, "mean", device="cuda",
                                exchange=ex, allreduce=allreduce)
        assert ds.part.stride & (ds.part.stride - 1) == 0
        w0 = g["sage-mean_w0"]
        o = [0]

        def take(r, c):
            t = torch.from_numpy(w0[o[0]:o[0] + r * c].reshape(r, c).copy()).cuda()
            o[0] += r * c
            return t
        params = sage_dist.SageParams(take(f, hidden), take(hidden, classes), take(f, hidden), take(hidden, classes))
        r0, r1 = ds.r0, ds.r1
        xl = torch.from_numpy(x[r0:r1].copy()).cuda()
        lab = torch.from_numpy(g["labels"][r0:r1].astype(np.int64)).cuda()
        mask = torch.from_numpy(g["mask"][r0:r1].copy()).cuda()
        losses = [ds.step(params, xl, lab, mask, 0.05, int(g["mask"].sum())) for _ in range(6)]
        ex.close()
        if rank == 0:
            q.put(losses)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_sage_peer_exchange_matches_reference(cuda):
    """cfg5's step with the fused peer exchange (two processes on one GPU,
    IPC-mapped blocks, host fences): losses track the reference's train()."""
    import torch.multiprocessing as mp

    from conftest import load_golden
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_sage_peer_worker, args=(r, 2, port_, q)) for r in range(2)]
    for p in procs:
        p.start()
    losses = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = load_golden("gnn_planted")["sage-mean_losses"][:6]
    np.testing.assert_allclose(losses, want, rtol=2e-3, atol=1e-5)


class _OracleCompute:
    """Local compute by the oracle (CPU gloo tests): SpMM and FusedMM/SDDMM."""

    def __call__(self, local, gathered, reduce):
        return _oracle_compute(local, gathered, reduce)

    def fused(self, local, x_local, y_gathered, edge_op, reduce):
        import torch
        rp, ci, v = local
        if edge_op is None:  # sddmm values
            return torch.from_numpy(port.sddmm(rp, ci, v, x_local.numpy(), y_gathered.numpy(), np.float64))
        op = {"mul": port.EDGE_MUL, "sigmoid_mul": port.EDGE_SIGMOID_MUL}[edge_op]
        red = {"sum": 0, "min": 1, "max": 2, "mean": 3}[reduce]
        return torch.from_numpy(port.fusedmm(rp, ci, v, x_local.numpy(), y_gathered.numpy(), op, red, np.float64))


def _fused_worker(rank, world, port_, rp, ci, v, x, y, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_14853_b200 import partition
        pt = partition.make_partition(rp, world)
        me = partition.PartitionedSpmm(rp, ci, v, pt, rank, x.shape[1], device="cpu", compute=_OracleCompute())
        r0, r1 = pt.rows(rank)
        xl = torch.from_numpy(x[r0:r1].astype(np.float64))
        yl = torch.from_numpy(y[r0:r1].astype(np.float64))
        ex = partition.NcclExchange()
        f = me.fusedmm(xl, yl, ex, "sigmoid_mul", "sum").numpy()
        sd = me.sddmm(xl, yl, ex).numpy()
        out = [None] * world
        dist.all_gather_object(out, (f, sd))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_fusedmm_sddmm_match_single_process():
    """SDDMM / FusedMM shard like SpMM: X local, Y all-gathered."""
    import torch.multiprocessing as mp
    rng = np.random.default_rng(8)
    n, k = 300, 8
    rp, ci, v = rand_csr(rng, n, n, 0.04, hub_rows=(2,), empty_frac=0.1)
    x = rng.normal(0, 0.5, (n, k)).astype(np.float32)
    y = rng.normal(0, 0.5, (n, k)).astype(np.float32)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, 2, port_, rp, ci, v, x, y, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    f = np.concatenate([g[0] for g in got])
    sd = np.concatenate([g[1] for g in got])
    xd, yd = x.astype(np.float64), y.astype(np.float64)
    np.testing.assert_array_equal(f, port.fusedmm(rp, ci, v, xd, yd, port.EDGE_SIGMOID_MUL, 0, np.float64))
    np.testing.assert_array_equal(sd, port.sddmm(rp, ci, v, xd, yd, np.float64))


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [2, 3, 8])
def test_loopback_partitioned_fusedmm_sddmm_bitwise(cuda, parts):
    """Row-partitioned FusedMM / SDDMM (Y all-gathered in the padded owner
    layout) reproduce the single-GPU results bit for bit (the fused dot and
    segments are plan-independent)."""
    import torch

    from paper_2403_14853_b200 import graphs, ops, partition
    n, k = 1 << 13, 64
    rp, ci = graphs.rmat(13, n * 16, seed=4, symmetrize=True, self_loops=True)
    v = graphs.uniform(len(ci), 0.0, 1.0, 2)
    x = torch.from_numpy(graphs.normal(n * k, 0, 0.1, 3).reshape(n, k)).cuda()
    y = torch.from_numpy(graphs.normal(n * k, 0, 0.1, 5).reshape(n, k)).cuda()
    a = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    want_f = ops.fusedmm(a, x, y, "sigmoid_mul", "sum").cpu().numpy()
    want_max = ops.fusedmm(a, x, y, "mul", "max").cpu().numpy()
    want_s = ops.sddmm(a, x, y).values.cpu().numpy()
    pt = partition.make_partition(rp, parts)
    ranks = [partition.PartitionedSpmm(rp, ci, v, pt, p, k) for p in range(parts)]
    gathered = partition.LoopbackExchange().all_gather(
        [partition.pad_block(y[pt.rows(p)[0]:pt.rows(p)[1]], pt.stride) for p in range(parts)])
    xs = [x[r.r0:r.r1].contiguous() for r in ranks]
    got_f = np.concatenate([r.fusedmm_gathered(xl, gathered, "sigmoid_mul", "sum").cpu().numpy()
                            for r, xl in zip(ranks, xs)])
    got_max = np.concatenate([r.fusedmm_gathered(xl, gathered, "mul", "max").cpu().numpy()
                              for r, xl in zip(ranks, xs)])
    got_s = np.concatenate([r.sddmm_gathered(xl, gathered).cpu().numpy() for r, xl in zip(ranks, xs)])
    np.testing.assert_array_equal(got_f.view(np.uint32), want_f.view(np.uint32))
    np.testing.assert_array_equal(got_max.view(np.uint32), want_max.view(np.uint32))
    np.testing.assert_array_equal(got_s.view(np.uint32), want_s.view(np.uint32))
