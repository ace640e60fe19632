"""SpMM parity on the B200 against the CPU oracle (oracle/port.py, pinned to the
reference by tests/test_oracle_golden.py) and the reference's own golden
vectors (tests/golden/).  Tolerance: |gpu - ref64| <= 1e-5 * sum_j |a_ij x_jk|
(BASELINE north_star); rows with <= SGNN_SEGMENT nonzeros must additionally be
bit-identical to the reference's fp32 trusted kernel (no-FMA build)."""
import numpy as np
import pytest

from conftest import assert_spmm_close, golden_cases, load_golden, rand_csr
from oracle import port

pytestmark = pytest.mark.gpu

REDS = {"sum": 0, "min": 1, "max": 2, "mean": 3}


def _ops():
    from paper_2403_14853_b200 import ops
    return ops


def _run(a_np, x, reduce, n_cols, **plan_params):
    import torch
    ops = _ops()
    a = ops.CsrMatrix.from_numpy(*a_np, n_cols)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    if plan_params:
        out = ops.spmm_plan(a, xt, reduce, ops.Plan(a, x.shape[1], **plan_params))
    else:
        out = ops.spmm(a, xt, reduce)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _short_rows(rp):
    deg = np.diff(rp.astype(np.int64))
    return deg <= 256


def check_spmm(rp, ci, v, x, n_cols, reduce, **plan_params):
    got = _run((rp, ci, v), x, reduce, n_cols, **plan_params)
    r = REDS[reduce]
    want64 = port.spmm(rp, ci, v.astype(np.float64), x.astype(np.float64), r)
    denom = port.spmm_absdenom(rp, ci, v, x, r)
    assert_spmm_close(got, want64, denom, what=f"spmm {reduce}")
    want32 = port.spmm(rp, ci, v, x, r, np.float32)
    if reduce in ("min", "max"):  # exact regardless of segmenting
        np.testing.assert_array_equal(got.view(np.uint32), want32.view(np.uint32))
    else:
        short = _short_rows(rp)
        np.testing.assert_array_equal(got[short].view(np.uint32), want32[short].view(np.uint32))
    return got


# ---- SPEC known answers --------------------------------------
def test_kat_spmm(cuda):
    # A = 2x2 {(0,1)=2,(1,0)=3}, B=[[1,1],[2,2]] -> [[4,4],[3,3]]
    got = _run((np.array([0, 1, 2], np.uint64), np.array([1, 0], np.uint32), np.array([2, 3], np.float32)),
               np.array([[1, 1], [2, 2]], np.float32), "sum", 2)
    np.testing.assert_array_equal(got, [[4, 4], [3, 3]])
    a = (np.array([0, 2], np.uint64), np.array([0, 1], np.uint32), np.array([1, 1], np.float32))
    b = np.array([[2, 8], [4, 2]], np.float32)
    np.testing.assert_array_equal(_run(a, b, "min", 2), [[2, 2]])
    np.testing.assert_array_equal(_run(a, b, "max", 2), [[4, 8]])
    np.testing.assert_array_equal(_run(a, b, "mean", 2), [[3, 5]])
    # identity law
    ident = (np.arange(3, dtype=np.uint64), np.arange(2, dtype=np.uint32), np.ones(2, np.float32))
    bb = np.array([[1, 2], [3, 4]], np.float32)
    np.testing.assert_array_equal(_run(ident, bb, "sum", 2), bb)


def test_empty_rows_all_reductions(cuda):
    rp = np.array([0, 0, 2, 2, 3, 3], np.uint64)
    ci = np.array([0, 3, 1], np.uint32)
    v = np.array([1.5, -2.0, 0.5], np.float32)
    x = np.random.default_rng(0).uniform(-1, 1, (4, 8)).astype(np.float32)
    for red in REDS:
        got = check_spmm(rp, ci, v, x, 4, red)
        assert (got[[0, 2, 4]] == 0).all()


def test_empty_matrix(cuda):
    rp = np.zeros(6, np.uint64)
    x = np.ones((3, 16), np.float32)
    for red in REDS:
        got = _run((rp, np.zeros(0, np.uint32), np.zeros(0, np.float32)), x, red, 3)
        assert got.shape == (5, 16) and (got == 0).all()


@pytest.mark.parametrize("name", golden_cases())
def test_golden_fixtures(cuda, name):
    g = load_golden(name)
    rp, ci, v, n = g["row_ptr"], g["col_idx"], g["values"], int(g["n_cols"])
    for k in g["ks"]:
        x = g[f"x_{k}"]
        for red, r in REDS.items():
            got = _run((rp, ci, v), x, red, n)
            want64 = g[f"spmm64_{k}_{r}"]
            assert_spmm_close(got, want64, port.spmm_absdenom(rp, ci, v, x, r), what=f"{name} K={k} {red}")
            ref32 = g[f"spmm32_{k}_{r}"]
            short = _short_rows(rp) if red in ("sum", "mean") else np.ones(len(rp) - 1, bool)
            np.testing.assert_array_equal(got[short].view(np.uint32), ref32[short].view(np.uint32))


@pytest.mark.parametrize("k", [1, 3, 4, 16, 20, 32, 33, 64, 128, 200, 256, 512, 1024])
def test_random_widths(cuda, k):
    rng = np.random.default_rng(100 + k)
    rp, ci, v = rand_csr(rng, 300, 500, 0.02, hub_rows=(5, 100), empty_frac=0.1)
    x = rng.uniform(-1, 1, (500, k)).astype(np.float32)
    for red in REDS:
        check_spmm(rp, ci, v, x, 500, red)


def test_hub_rows_split_segments(cuda):
    """Rows far longer than SGNN_SEGMENT are split over workers; result within
    tolerance and identical for every plan."""
    rng = np.random.default_rng(7)
    n = 40000
    rp, ci, v = rand_csr(rng, 64, n, 0.001, hub_rows=(0, 1, 33, 63), hub_density=0.8)
    x = rng.standard_normal((n, 64)).astype(np.float32)
    base = check_spmm(rp, ci, v, x, n, "sum")
    for params in ({"path_items": 64}, {"path_items": 300, "lanes": 8, "vec": 2},
                   {"path_items": 4096, "split_rows_over": 100000}, {"scalar": 1, "path_items": 128},
                   {"k_tile": 16, "lanes": 4}):
        got = _run((rp, ci, v), x, "sum", n, **params)
        np.testing.assert_array_equal(got.view(np.uint32), base.view(np.uint32), err_msg=str(params))


@pytest.mark.parametrize("k", [16, 30, 128])
def test_single_row_150k_nonzeros(cuda, k):
    """SURVEY 4 test plan: one row of 150k nonzeros (split over hundreds of
    workers, 586 canonical segments) among short and empty rows; sum, mean
    and max within tolerance, sum/max bitwise plan-independent."""
    rng = np.random.default_rng(11)
    n_cols = 200_000
    hub = np.sort(rng.choice(n_cols, 150_000, replace=False)).astype(np.uint32)
    rows = [hub] + [np.sort(rng.choice(n_cols, int(rng.integers(0, 40)), replace=False)).astype(np.uint32)
                    for _ in range(300)]
    rp = np.zeros(len(rows) + 1, np.uint64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.concatenate(rows)
    v = rng.uniform(-1, 1, len(ci)).astype(np.float32)
    x = rng.standard_normal((n_cols, k)).astype(np.float32)
    for red in ("sum", "mean", "max"):
        base = check_spmm(rp, ci, v, x, n_cols, red)
        if red != "mean":
            got = _run((rp, ci, v), x, red, n_cols, path_items=512)
            np.testing.assert_array_equal(got.view(np.uint32), base.view(np.uint32))


def test_plans_bitwise_transparent(cuda):
    """Dispatch transparency: every plan gives bitwise the same C."""
    rng = np.random.default_rng(3)
    rp, ci, v = rand_csr(rng, 2000, 3000, 0.01, hub_rows=(1, 2, 1000), empty_frac=0.2)
    x = rng.uniform(-1, 1, (3000, 128)).astype(np.float32)
    ref = None
    for params in ({}, {"path_items": 16}, {"path_items": 1024}, {"lanes": 16, "vec": 2},
                   {"lanes": 8, "vec": 4, "unroll": 4}, {"unroll": 4}, {"k_tile": 64},
                   {"scalar": 1}, {"block": 64}, {"split_rows_over": 4096}):
        got = _run((rp, ci, v), x, "sum", 3000, **params) if params else _run((rp, ci, v), x, "sum", 3000)
        if ref is None:
            ref = got
            check_spmm(rp, ci, v, x, 3000, "sum")
        np.testing.assert_array_equal(got.view(np.uint32), ref.view(np.uint32), err_msg=str(params))


def test_shape_and_dispatch_errors(cuda):
    import torch
    ops = _ops()
    a = ops.CsrMatrix.from_numpy(np.array([0, 1], np.uint64), np.array([0], np.uint32),
                                 np.array([1], np.float32), 2)
    x = torch.ones((3, 32), device="cuda")
    with pytest.raises(ops.ShapeError):
        ops.spmm(a, x)
    x = torch.ones((2, 48), device="cuda")
    with pytest.raises(ops.DispatchError):
        ops.spmm_with(a, x, "sum", ops.KernelKind.specialized(32))
    with pytest.raises(ops.DispatchError):
        ops.spmm_with(a, x, "sum", ops.KernelKind.specialized(48))
    with pytest.raises(ops.DispatchError):
        ops.spmm_with(a, torch.ones((2, 32), device="cuda"), "mean", ops.KernelKind.specialized(32))
    with pytest.raises(ops.ConfigError):
        ops.spmm(a, torch.ones((2, 32), device="cuda"), "median")


def test_dispatch_toggle(cuda):
    ops = _ops()
    with ops.DispatchGuard(False):
        assert ops.resolve_kernel(32, "sum") == ops.KernelKind.trusted()
    assert ops.resolve_kernel(32, "sum") == ops.KernelKind.specialized(32)
    assert ops.resolve_kernel(48, "sum") == ops.KernelKind.trusted()
    assert ops.resolve_kernel(32, "mean") == ops.KernelKind.trusted()


def test_misaligned_operands_use_scalar_path(cuda):
    import torch
    rng = np.random.default_rng(11)
    rp, ci, v = rand_csr(rng, 100, 100, 0.05)
    x = rng.uniform(-1, 1, (100, 32)).astype(np.float32)
    ops = _ops()
    a = ops.CsrMatrix.from_numpy(rp, ci, v, 100)
    buf = torch.zeros(100 * 32 + 1, device="cuda")
    buf[1:] = torch.from_numpy(x.ravel()).cuda()
    xt = buf[1:].view(100, 32)  # 4-byte offset: not 16-byte aligned
    out = ops.spmm(a, xt, "sum")
    want = port.spmm(rp, ci, v, x, 0, np.float32)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))


# ---- dynamic worker schedule (common.cuh WarpSched, plan.cu plan_counter) ----
@pytest.mark.parametrize("k", [64, 256])
def test_dynamic_schedule_counter_reset_streams_graphs(cuda, k):
    """Many more workers than resident warps, so warps take workers from the
    plan's counter.  The counter resets itself at the end of each launch:
    repeated launches, a launch on a second stream (static schedule), and CUDA
    graph replays (static) are bitwise the first launch, which matches the
    oracle.  FusedMM and SDDMM share the counter of the fused plan."""
    import torch
    from paper_2403_14853_b200 import graphs
    ops = _ops()
    rp, ci = graphs.rmat(15, 16 << 15, seed=5)
    v = graphs.normal(len(ci), 0, 1, 9)
    n = len(rp) - 1
    x = graphs.normal(n * k, 0, 1, 10).reshape(n, k)
    a = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    xt = torch.from_numpy(x).cuda()
    plan = ops.Plan(a, k, path_items=32)
    assert plan.stats["workers"] > 2 * 148 * 20 * 2  # > 2 rounds of resident worker sets (occupancy 5)
    first = ops.spmm_plan(a, xt, "sum", plan)
    want32 = port.spmm(rp, ci, v, x, 0, np.float32)
    short = _short_rows(rp)
    np.testing.assert_array_equal(first.cpu().numpy()[short].view(np.uint32), want32[short].view(np.uint32))
    ref = first.cpu().numpy()
    out = torch.empty_like(first)

    def again():  # into a NaN-filled output: a skipped worker would show
        out.fill_(float("nan"))
        ops.spmm_plan(a, xt, "sum", plan, out)
        return out.cpu().numpy()

    for _ in range(5):
        np.testing.assert_array_equal(again(), ref)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        out.fill_(float("nan"))
        ops.spmm_plan(a, xt, "sum", plan, out)
    torch.cuda.current_stream().wait_stream(side)
    np.testing.assert_array_equal(out.cpu().numpy(), ref)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ops.spmm_plan(a, xt, "sum", plan, out)
    for _ in range(3):
        out.fill_(float("nan"))
        g.replay()
        np.testing.assert_array_equal(out.cpu().numpy(), ref)
    # after the capture, the owning stream still gets the dynamic schedule
    np.testing.assert_array_equal(again(), ref)
    # FusedMM / SDDMM over the fused plan's counter
    if k == 64:
        y = torch.from_numpy(graphs.normal(n * k, 0, 0.1, 11).reshape(n, k)).cuda()
        xs = xt * 0.1
        f0 = ops.fusedmm(a, xs, y, "mul", "sum").cpu().numpy()
        s0 = ops.sddmm(a, xs, y).values.cpu().numpy()
        for _ in range(3):
            out.fill_(float("nan"))
            ops.fusedmm(a, xs, y, "mul", "sum", out=out)
            np.testing.assert_array_equal(out.cpu().numpy(), f0)
            nan = torch.full((len(ci),), float("nan"), device="cuda")
            del nan  # the caching allocator hands this block to sddmm's output
            np.testing.assert_array_equal(ops.sddmm(a, xs, y).values.cpu().numpy(), s0)
        want_s = port.sddmm(rp, ci, v, xs.cpu().numpy().astype(np.float64), y.cpu().numpy().astype(np.float64))
        np.testing.assert_allclose(s0, want_s, rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("d0,d1,samples", [(1, 1 << 18, 512), ((1 << 24) - 4096, (1 << 24) + 4096, 4096),
                                           ((1 << 31) - 2048, (1 << 31), 4096)])
def test_mean_division_selftest(cuda, d0, d1, samples):
    """The mean epilogue's division (reciprocal in double + one rounding,
    common.cuh div_by_count) is bitwise IEEE __fdiv_rn for every degree in
    the range and every value class (specials, subnormals, all exponents)."""
    import ctypes as C

    from paper_2403_14853_b200 import _lib
    bad, fd, fs = C.c_uint64(), C.c_uint64(), C.c_uint32()
    _lib.check(_lib.lib().sgnn_selftest_count_division(d0, d1, samples, 1234, C.byref(bad), C.byref(fd),
                                                       C.byref(fs)), "selftest")
    assert bad.value == 0, f"{bad.value} mismatches, first at degree {fd.value} sample {fs.value}"


@pytest.mark.parametrize("k", [128, 64, 30])
def test_mean_epilogue_bitwise_sum_over_degree(cuda, k):
    """spmm(A, X, mean) == spmm(A, X, sum) / deg with IEEE division, bit for
    bit: rows split across workers, hub rows through the fixup kernels, tiny
    and signed-zero values (the divide moved into the kernels' row epilogue)."""
    import torch
    ops = _ops()
    rng = np.random.default_rng(17)
    n = 3000
    rp, ci, v = rand_csr(rng, n, n, 0.01, hub_rows=(0, 5, 77), hub_density=0.7, empty_frac=0.05)
    x = rng.normal(0, 1, (n, k)).astype(np.float32)
    x[::7] *= np.float32(1e-38)  # subnormal-range sums
    x[3] = -0.0
    a = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    xt = torch.from_numpy(x).cuda()
    layouts = ({}, {"lanes": 16, "split_rows_over": 256}, {"lanes": 32, "vec": 2, "unroll": 4}) if k % 4 == 0 else \
        ({}, {"split_rows_over": 256})
    for params in layouts:
        plan = ops.Plan(a, k, **params) if params else None
        s = ops.spmm_plan(a, xt, "sum", plan) if plan else ops.spmm(a, xt, "sum")
        m = ops.spmm_plan(a, xt, "mean", plan) if plan else ops.spmm(a, xt, "mean")
        deg = torch.from_numpy(np.diff(rp.astype(np.int64)).astype(np.float32)).cuda()[:, None]
        want = torch.where(deg > 0, s / torch.clamp(deg, min=1.0), torch.zeros_like(s))
        np.testing.assert_array_equal(m.cpu().numpy().view(np.uint32), want.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("k", [16, 20, 32, 64, 128])
def test_short_row_kernel_bitwise_worker(cuda, k, monkeypatch):
    """Small matrices whose rows all fit 2 G nonzeros take the short-row
    kernel (one group per row, no plan metadata); its results are bitwise the
    worker kernel's (SGNN_NO_SHORT_ROWS) and the reference's fp32 kernel, for
    every reduction, empty rows, a partial width (K = 20) and rows of exactly
    2 G nonzeros."""
    import torch
    ops = _ops()
    rng = np.random.default_rng(k)
    m, n = 3000, 5000
    lanes = 4 if k <= 16 else 8 if k <= 32 else 16 if k <= 64 else 32
    cnt = rng.integers(0, 2 * lanes + 1, m)
    cnt[rng.random(m) < 0.2] = 0
    cnt[:5] = 2 * lanes
    rows = [np.sort(rng.choice(n, size=int(c), replace=False)) for c in cnt]
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(cnt)
    ci = np.concatenate(rows).astype(np.uint32)
    v = rng.uniform(-1, 1, len(ci)).astype(np.float32)
    x = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    a = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    xt = torch.from_numpy(x).cuda()
    for red, r in REDS.items():
        got = ops.spmm(a, xt, red).cpu().numpy()
        monkeypatch.setenv("SGNN_NO_SHORT_ROWS", "1")
        want = ops.spmm(a, xt, red).cpu().numpy()
        monkeypatch.delenv("SGNN_NO_SHORT_ROWS")
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32), err_msg=red)
        w32 = port.spmm(rp, ci, v, x, r, np.float32)
        np.testing.assert_array_equal(got.view(np.uint32), w32.view(np.uint32), err_msg=f"{red} vs fp32 reference")


@pytest.mark.parametrize("k", [20, 32, 64])
@pytest.mark.parametrize("path_items", [0, 64])
def test_lockstep_worker_bitwise_generic(cuda, k, path_items, monkeypatch):
    """8- / 16-lane groups at one float4 per lane run the lockstep worker
    (lock_worker_kernel); it gives bit for bit the generic worker's results
    (SGNN_LOCK_GENERIC) for every reduction: hub rows split over workers
    (slots + fixup), multi-segment rows inside a worker, empty-row runs, a
    partial width (K = 20), and the reference's fp32 kernel on short rows."""
    import torch

    from paper_2403_14853_b200 import graphs
    ops = _ops()
    rng = np.random.default_rng(k + path_items)
    n = 1 << 13
    rp, ci = graphs.rmat(13, n * 12, seed=9)
    deg = np.diff(rp.astype(np.int64))
    assert (deg == 0).sum() > 100 and deg.max() > 1000
    v = rng.uniform(-1, 1, len(ci)).astype(np.float32)
    x = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    a = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    xt = torch.from_numpy(x).cuda()
    plan = ops.Plan(a, k, path_items=path_items) if path_items else None
    for red, r in REDS.items():
        got = (ops.spmm_plan(a, xt, red, plan) if plan else ops.spmm(a, xt, red)).cpu().numpy()
        monkeypatch.setenv("SGNN_LOCK_GENERIC", "1")
        want = (ops.spmm_plan(a, xt, red, plan) if plan else ops.spmm(a, xt, red)).cpu().numpy()
        monkeypatch.delenv("SGNN_LOCK_GENERIC")
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32), err_msg=red)
        short = deg <= 256
        w32 = port.spmm(rp, ci, v, x, r, np.float32)
        np.testing.assert_array_equal(got[short].view(np.uint32), w32[short].view(np.uint32),
                                      err_msg=f"{red} vs fp32 reference")
