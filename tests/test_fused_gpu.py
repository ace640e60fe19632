"""SDDMM (kernels.hpp:187-210) and FusedMM (kernels.hpp:216-270) on the B200
against the reference's golden vectors and the oracle.  Tolerances:
SDDMM |gpu - ref64| <= 1e-5 * |p_e| * sum_k |x_ik y_jk|; FusedMM
|gpu - ref64| <= 1e-5 * sum_j |s_ij y_jk| (+ the dot's own rounding)."""
import numpy as np
import pytest

from conftest import assert_spmm_close, golden_cases, load_golden, rand_csr
from oracle import port

pytestmark = pytest.mark.gpu
REDS = {"sum": 0, "min": 1, "max": 2, "mean": 3}
EDGES = {"mul": 0, "sigmoid_mul": 1}


def _ops():
    from paper_2403_14853_b200 import ops
    return ops


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def run_sddmm(rp, ci, v, n, x, y):
    ops = _ops()
    out = ops.sddmm(ops.CsrMatrix.from_numpy(rp, ci, v, n), _t(x), _t(y))
    return out.values.cpu().numpy(), out


def run_fused(rp, ci, v, n, x, y, edge, red):
    ops = _ops()
    return ops.fusedmm(ops.CsrMatrix.from_numpy(rp, ci, v, n), _t(x), _t(y), edge, red).cpu().numpy()


def check_sddmm(rp, ci, v, n, x, y):
    got, _ = run_sddmm(rp, ci, v, n, x, y)
    want = port.sddmm(rp, ci, v, x, y)
    den = port.sddmm_absdenom(rp, ci, v, x, y)
    err = np.abs(got.astype(np.float64) - want)
    assert (err <= 1e-5 * den + 1e-30).all(), f"sddmm: max err/den {np.max(err / np.maximum(den, 1e-30))}"
    return got


def check_fused(rp, ci, v, n, x, y, edge, red):
    got = run_fused(rp, ci, v, n, x, y, edge, red)
    want = port.fusedmm(rp, ci, v, x, y, EDGES[edge], REDS[red])
    den = port.fusedmm_absdenom(rp, ci, v, x, y, EDGES[edge], REDS[red])
    assert_spmm_close(got, want, den, what=f"fusedmm {edge} {red}")
    return got


def test_kat_sddmm_fusedmm(cuda):
    ident = (np.arange(3, dtype=np.uint64), np.arange(2, dtype=np.uint32), np.ones(2, np.float32))
    x = np.array([[1, 2], [3, 4]], np.float32)
    got, out = run_sddmm(*ident, 2, x, x)
    np.testing.assert_array_equal(got, [5, 25])
    np.testing.assert_array_equal(out.row_ptr.cpu().numpy(), [0, 1, 2])  # pattern is P's
    np.testing.assert_array_equal(run_fused(*ident, 2, x, x, "mul", "sum"), [[5, 10], [75, 100]])
    # full pattern, values 1 -> X Y^T
    rng = np.random.default_rng(0)
    xx, yy = rng.uniform(-1, 1, (5, 8)).astype(np.float32), rng.uniform(-1, 1, (4, 8)).astype(np.float32)
    rp = np.arange(0, 21, 4, dtype=np.uint64)
    ci = np.tile(np.arange(4, dtype=np.uint32), 5)
    got, _ = run_sddmm(rp, ci, np.ones(20, np.float32), 4, xx, yy)
    np.testing.assert_allclose(got.reshape(5, 4), xx.astype(np.float64) @ yy.T.astype(np.float64), rtol=1e-5, atol=1e-6)


def test_empty(cuda):
    rp = np.zeros(4, np.uint64)
    x = np.ones((3, 16), np.float32)
    got, _ = run_sddmm(rp, np.zeros(0, np.uint32), np.zeros(0, np.float32), 5, x, np.ones((5, 16), np.float32))
    assert got.size == 0
    for red in REDS:
        out = run_fused(rp, np.zeros(0, np.uint32), np.zeros(0, np.float32), 5, x, np.ones((5, 16), np.float32), "mul", red)
        assert (out == 0).all()


@pytest.mark.parametrize("name", golden_cases())
def test_golden(cuda, name):
    g = load_golden(name)
    rp, ci, v, n = g["row_ptr"], g["col_idx"], g["values"], int(g["n_cols"])
    for k in g["ks"]:
        x, xi = g[f"x_{k}"], g[f"xi_{k}"]
        if k <= 1024:
            got, _ = run_sddmm(rp, ci, v, n, xi, x)
            den = port.sddmm_absdenom(rp, ci, v, xi, x)
            assert (np.abs(got - g[f"sddmm64_{k}"]) <= 1e-5 * den + 1e-30).all(), (name, k)
        for edge, eo in EDGES.items():
            for red, r in REDS.items():
                got = run_fused(rp, ci, v, n, xi, x, edge, red)
                den = port.fusedmm_absdenom(rp, ci, v, xi, x, eo, r)
                assert_spmm_close(got, g[f"fused64_{k}_{eo}_{r}"], den, what=f"{name} K={k} {edge} {red}")


@pytest.mark.parametrize("k", [1, 4, 7, 16, 32, 64, 100, 128, 256, 512, 1024])
def test_random(cuda, k):
    rng = np.random.default_rng(k)
    rp, ci, v = rand_csr(rng, 400, 700, 0.01, hub_rows=(3, 300), empty_frac=0.2)
    x = rng.normal(0, 0.3, (400, k)).astype(np.float32)
    y = rng.normal(0, 0.3, (700, k)).astype(np.float32)
    if k <= 256 or k % 4 == 0:
        check_sddmm(rp, ci, v, 700, x, y)
        for edge in EDGES:
            for red in REDS:
                check_fused(rp, ci, v, 700, x, y, edge, red)


def test_fusedmm_equals_spmm_of_sddmm(cuda):
    """SPEC.md:176 / acceptance #8: fusedmm = spmm(sddmm(P,X,Y), Y) within tolerance."""
    ops = _ops()
    rng = np.random.default_rng(4)
    rp, ci, v = rand_csr(rng, 300, 300, 0.03, hub_rows=(1,))
    x = rng.normal(0, 0.5, (300, 32)).astype(np.float32)
    y = rng.normal(0, 0.5, (300, 32)).astype(np.float32)
    p = ops.CsrMatrix.from_numpy(rp, ci, v, 300)
    s = ops.sddmm(p, _t(x), _t(y))
    for red in REDS:
        fused = ops.fusedmm(p, _t(x), _t(y), "mul", red).cpu().numpy()
        comp = ops.spmm(s, _t(y), red).cpu().numpy()
        sv = s.values.cpu().numpy()
        den = port.spmm_absdenom(rp, ci, sv, y, REDS[red]) + 1e-30
        assert (np.abs(fused - comp) <= 2e-5 * den).all(), red


def test_hub_rows_fused(cuda):
    rng = np.random.default_rng(12)
    n = 20000
    rp, ci, v = rand_csr(rng, 40, n, 0.0005, hub_rows=(0, 39), hub_density=0.7, value="positive")
    x = rng.normal(0, 0.1, (40, 64)).astype(np.float32)
    y = rng.normal(0, 0.1, (n, 64)).astype(np.float32)
    for red in REDS:
        check_fused(rp, ci, v, n, x, y, "sigmoid_mul", red)
    check_sddmm(rp, ci, v, n, x, y)


def test_fused_plan_transparency(cuda):
    """FusedMM/SDDMM results are bitwise independent of the register layout
    and work split (canonical high-bit-first dot tree, canonical segments)."""
    ops = _ops()
    rng = np.random.default_rng(21)
    rp, ci, v = rand_csr(rng, 600, 3000, 0.01, hub_rows=(0, 5), hub_density=0.3, empty_frac=0.1)
    x = rng.normal(0, 0.3, (600, 64)).astype(np.float32)
    y = rng.normal(0, 0.3, (3000, 64)).astype(np.float32)
    p = ops.CsrMatrix.from_numpy(rp, ci, v, 3000)
    for edge in ("sigmoid_mul", "mul"):
        base = ops.fusedmm(p, _t(x), _t(y), edge, "sum").cpu().numpy()
        for lv in ((16, 1, 8), (8, 2, 4), (4, 4, 4), (16, 2, 4), (32, 1, 8)):
            for pi in (32, 300):
                plan = ops.Plan(p, 64, lanes=lv[0], vec=lv[1], unroll=lv[2], path_items=pi)
                got = ops.fusedmm(p, _t(x), _t(y), edge, "sum", plan=plan).cpu().numpy()
                np.testing.assert_array_equal(got.view(np.uint32), base.view(np.uint32), err_msg=f"{edge} {lv} {pi}")
    check_fused(rp, ci, v, 3000, x, y, "sigmoid_mul", "sum")


def test_errors(cuda):
    import torch
    ops = _ops()
    p = ops.CsrMatrix.from_numpy(np.array([0, 1], np.uint64), np.array([0], np.uint32), np.ones(1, np.float32), 2)
    with pytest.raises(ops.ShapeError):
        ops.sddmm(p, torch.ones(2, 4, device="cuda"), torch.ones(2, 4, device="cuda"))
    with pytest.raises(ops.ShapeError):
        ops.fusedmm(p, torch.ones(1, 4, device="cuda"), torch.ones(3, 4, device="cuda"))
    with pytest.raises(ops.DispatchError):
        ops.fusedmm(p, torch.ones(1, 4, device="cuda"), torch.ones(2, 4, device="cuda"), edge_op=lambda a, b: a)


@pytest.mark.parametrize("k", [64, 128])
def test_tma_pipeline_bitwise_register_kernels(cuda, k, monkeypatch):
    """The warp-specialised TMA-gather kernels (fused_tma.cu: tile::gather4
    into mbarrier-paced shared-memory rings, K = 64 / 128) give bit for bit
    the register-gather kernels' FusedMM (both edge ops, sum and mean) and
    SDDMM, for every ring depth and work split: split hub rows (segment
    slots + fixup), empty rows, workers of only empty rows."""
    from paper_2403_14853_b200 import graphs
    ops = _ops()
    rng = np.random.default_rng(5)
    n = 1 << 13
    rp, ci = graphs.rmat(13, n * 12, seed=3)
    deg = np.diff(rp.astype(np.int64))
    v = rng.uniform(0, 1, len(ci)).astype(np.float32)
    x = rng.normal(0, 0.1, (n, k)).astype(np.float32)
    y = rng.normal(0, 0.1, (n, k)).astype(np.float32)
    assert (deg == 0).any() and deg.max() > 1000
    p = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    xt, yt = _t(x), _t(y)
    cases = [("sigmoid_mul", "sum"), ("mul", "sum"), ("sigmoid_mul", "mean")]
    for pi in (64, 512):
        plan = ops.Plan(p, k, **{**_fused_layout_kw(k), "path_items": pi})
        monkeypatch.delenv("SGNN_TMA_FUSED", raising=False)
        want = {c: ops.fusedmm(p, xt, yt, *c, plan=plan).cpu().numpy() for c in cases}
        want_s = ops.sddmm(p, xt, yt).values.cpu().numpy()
        monkeypatch.setenv("SGNN_TMA_FUSED", "1")
        for depth in ("2", "3", "4"):
            monkeypatch.setenv("SGNN_TMA_DEPTH", depth)
            for c in cases:
                got = ops.fusedmm(p, xt, yt, *c, plan=plan).cpu().numpy()
                np.testing.assert_array_equal(got.view(np.uint32), want[c].view(np.uint32), err_msg=f"{c} {pi} {depth}")
            got_s = ops.sddmm(p, xt, yt).values.cpu().numpy()
            np.testing.assert_array_equal(got_s.view(np.uint32), want_s.view(np.uint32), err_msg=f"sddmm {depth}")
    check_fused(rp, ci, v, n, x, y, "sigmoid_mul", "sum")
    check_sddmm(rp, ci, v, n, x, y)
    monkeypatch.delenv("SGNN_TMA_FUSED")


def _fused_layout_kw(k):
    return {"lanes": 16 if k == 64 else 32, "vec": 1, "unroll": 8, "k_tile": k}


@pytest.mark.parametrize("k", [32, 64])
def test_sddmm_lockstep_kernel_bitwise_generic(cuda, k, monkeypatch):
    """The full-width lockstep SDDMM (sddmm_lock_kernel, K = 32 / 64) gives bit
    for bit the generic kernel's results (same split, batches and dot tree):
    hub rows over many (col, val) windows, runs of empty rows longer than the
    row-end window, single-nonzero rows."""
    from paper_2403_14853_b200 import graphs
    ops = _ops()
    rng = np.random.default_rng(11)
    n = 1 << 13
    rp, ci = graphs.rmat(13, n * 10, seed=4)
    deg = np.diff(rp.astype(np.int64))
    assert (deg == 0).sum() > 100 and (deg == 1).any() and deg.max() > 1000
    v = rng.uniform(-1, 1, len(ci)).astype(np.float32)
    x = rng.normal(0, 0.1, (n, k)).astype(np.float32)
    y = rng.normal(0, 0.1, (n, k)).astype(np.float32)
    p = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    xt, yt = _t(x), _t(y)
    got = ops.sddmm(p, xt, yt).values.cpu().numpy()
    monkeypatch.setenv("SGNN_SDDMM_GENERIC", "1")
    want = ops.sddmm(p, xt, yt).values.cpu().numpy()
    monkeypatch.delenv("SGNN_SDDMM_GENERIC")
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    check_sddmm(rp, ci, v, n, x, y)


@pytest.mark.parametrize("parts", [2, 5])
def test_row_partitioned_fusedmm_sddmm_bitwise(cuda, parts):
    """SDDMM / FusedMM shard like the SpMM -- each rank holds a
    contiguous row block of P (global column ids, dist.row_partition's cost)
    and its rows of X, with Y all-gathered; the concatenated block results are
    bitwise the single-GPU ones (every row's chain, segments and dot tree
    depend only on the row), for both edge ops and all four reductions."""
    from paper_2403_14853_b200 import dist, graphs
    ops = _ops()
    rng = np.random.default_rng(parts)
    n, k = 1 << 12, 64
    rp, ci = graphs.rmat(12, n * 16, seed=6)
    v = rng.uniform(0, 1, len(ci)).astype(np.float32)
    x = rng.normal(0, 0.1, (n, k)).astype(np.float32)
    y = rng.normal(0, 0.1, (n, k)).astype(np.float32)
    p = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    xt, yt = _t(x), _t(y)
    bounds = dist.row_partition(rp, parts)
    blocks = [dist.row_block(rp, ci, v, int(bounds[r]), int(bounds[r + 1])) for r in range(parts)]
    for edge in ("sigmoid_mul", "mul"):
        for red in ("sum", "mean", "min", "max"):
            full = ops.fusedmm(p, xt, yt, edge, red).cpu().numpy()
            got = np.concatenate([ops.fusedmm(ops.CsrMatrix.from_numpy(b[0], b[1], b[2], n),
                                              xt[int(bounds[r]):int(bounds[r + 1])].contiguous(), yt, edge, red)
                                  .cpu().numpy() for r, b in enumerate(blocks)])
            np.testing.assert_array_equal(got.view(np.uint32), full.view(np.uint32), err_msg=f"{edge} {red}")
    full = ops.sddmm(p, xt, yt).values.cpu().numpy()
    got = np.concatenate([ops.sddmm(ops.CsrMatrix.from_numpy(b[0], b[1], b[2], n),
                                    xt[int(bounds[r]):int(bounds[r + 1])].contiguous(), yt).values.cpu().numpy()
                          for r, b in enumerate(blocks)])
    np.testing.assert_array_equal(got.view(np.uint32), full.view(np.uint32))


def test_output_operand_checks(cuda):
    """Caller-supplied outputs are validated before any launch (shape, dtype,
    layout): ShapeError / ConfigError, as the reference's shape checks."""
    import torch
    ops = _ops()
    p = ops.CsrMatrix.from_numpy(np.array([0, 1, 2], np.uint64), np.array([0, 1], np.uint32),
                                 np.ones(2, np.float32), 2)
    x = torch.ones(2, 4, device="cuda")
    with pytest.raises(ops.ShapeError):
        ops.fusedmm(p, x, x, out=torch.empty(3, 4, device="cuda"))
    with pytest.raises(ops.ConfigError):
        ops.fusedmm(p, x, x, out=torch.empty(2, 4, device="cuda", dtype=torch.float64))
    with pytest.raises(ops.ShapeError):
        ops.spmm(p, x, "sum", out=torch.empty(2, 5, device="cuda"))
    with pytest.raises(ops.ConfigError):
        ops.spmm_plan(p, x, "sum", out=torch.empty(4, 2, device="cuda").t())
    np.testing.assert_array_equal(ops.fusedmm(p, x, x, out=torch.empty(2, 4, device="cuda")).cpu().numpy(),
                                  ops.fusedmm(p, x, x).cpu().numpy())


@pytest.mark.parametrize("path_items", [0, 64, 512])
def test_fused_lockstep_kernel_bitwise_generic(cuda, path_items, monkeypatch):
    """The full-width lockstep FusedMM (fused_lock_kernel, K = 64, sum and
    mean, both edge ops) gives bit for bit the worker kernel's results
    (SGNN_FUSED_GENERIC): hub rows split over workers (segment slots +
    fixup), rows of several segments inside one worker (running totals in
    the output row), runs of empty rows, single-nonzero rows."""
    from paper_2403_14853_b200 import graphs
    ops = _ops()
    rng = np.random.default_rng(path_items + 1)
    n, k = 1 << 13, 64
    rp, ci = graphs.rmat(13, n * 12, seed=8)
    deg = np.diff(rp.astype(np.int64))
    assert (deg == 0).sum() > 100 and (deg == 1).any() and deg.max() > 1000
    v = rng.uniform(0, 1, len(ci)).astype(np.float32)
    x = rng.normal(0, 0.1, (n, k)).astype(np.float32)
    y = rng.normal(0, 0.1, (n, k)).astype(np.float32)
    p = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    xt, yt = _t(x), _t(y)
    plan = ops.Plan(p, k, **{**_fused_layout_kw(k), "path_items": path_items}) if path_items else None
    for edge in ("sigmoid_mul", "mul"):
        for red in ("sum", "mean"):
            got = ops.fusedmm(p, xt, yt, edge, red, plan=plan).cpu().numpy()
            monkeypatch.setenv("SGNN_FUSED_GENERIC", "1")
            want = ops.fusedmm(p, xt, yt, edge, red, plan=plan).cpu().numpy()
            monkeypatch.delenv("SGNN_FUSED_GENERIC")
            np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32), err_msg=f"{edge} {red}")
    check_fused(rp, ci, v, n, x, y, "sigmoid_mul", "sum")


@pytest.mark.parametrize("ring", [2, 3, 4])
@pytest.mark.parametrize("path_items", [0, 64, 512])
def test_fused_ring_kernel_bitwise_lockstep(cuda, ring, path_items, monkeypatch):
    """The lockstep FusedMM with its gathered rows in a shared-memory ring
    (cp.async, SGNN_FUSED_RING = ring chunks; K = 64, sum and mean, both edge
    ops) gives bit for bit the register kernel's results on the same graphs
    as above: split hub rows, multi-segment rows, runs of empty rows,
    workers shorter than the ring's lookahead (path_items = 64)."""
    from paper_2403_14853_b200 import graphs
    ops = _ops()
    rng = np.random.default_rng(path_items + 11)
    n, k = 1 << 13, 64
    rp, ci = graphs.rmat(13, n * 12, seed=8)
    v = rng.uniform(0, 1, len(ci)).astype(np.float32)
    x = rng.normal(0, 0.1, (n, k)).astype(np.float32)
    y = rng.normal(0, 0.1, (n, k)).astype(np.float32)
    p = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    xt, yt = _t(x), _t(y)
    plan = ops.Plan(p, k, **{**_fused_layout_kw(k), "path_items": path_items}) if path_items else None
    for edge in ("sigmoid_mul", "mul"):
        for red in ("sum", "mean"):
            monkeypatch.delenv("SGNN_FUSED_RING", raising=False)
            monkeypatch.setenv("SGNN_FUSED_RING", "0")
            want = ops.fusedmm(p, xt, yt, edge, red, plan=plan).cpu().numpy()
            monkeypatch.setenv("SGNN_FUSED_RING", str(ring))
            got = ops.fusedmm(p, xt, yt, edge, red, plan=plan).cpu().numpy()
            monkeypatch.delenv("SGNN_FUSED_RING")
            np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32), err_msg=f"{edge} {red}")
