"""On-device CSR->CSC transpose (bit-exact with sparse.hpp:72-89), row
degrees, is_symmetric, and the TrainingCache backward operands/counters
(gnn.hpp:113-196) against the reference's golden vectors and the oracle."""
import numpy as np
import pytest

from conftest import assert_spmm_close, golden_cases, load_golden, rand_csr
from oracle import port

pytestmark = pytest.mark.gpu


def _ops():
    from paper_2403_14853_b200 import ops
    return ops


def _dev(rp, ci, v, n):
    return _ops().CsrMatrix.from_numpy(rp, ci, v, n)


def _assert_csr_equal(got, want):
    for g, w, name in zip(got, want, ("row_ptr", "col_idx", "values")):
        g = np.asarray(g)
        w = np.asarray(w)
        assert g.shape == w.shape, name
        np.testing.assert_array_equal(g.view(np.uint8), w.view(np.uint8), err_msg=name)


@pytest.mark.parametrize("name", golden_cases())
def test_transpose_golden(cuda, name):
    g = load_golden(name)
    t = _ops().transpose(_dev(g["row_ptr"], g["col_idx"], g["values"], int(g["n_cols"])))
    _assert_csr_equal(t.to_numpy(), (g["t_row_ptr"], g["t_col_idx"], g["t_values"]))


@pytest.mark.parametrize("shape", [(1, 1), (3, 1), (1, 5000), (700, 300), (2000, 70000), (5000, 2049)])
def test_transpose_random(cuda, shape):
    m, n = shape
    rng = np.random.default_rng(m * 7 + n)
    rp, ci, v = rand_csr(rng, m, n, min(1.0, 20.0 / n), hub_rows=(0,) if m > 1 else (), empty_frac=0.2)
    t = _ops().transpose(_dev(rp, ci, v, n))
    _assert_csr_equal(t.to_numpy(), port.transpose(rp, ci, v, n))


def test_transpose_involution_and_empty(cuda):
    ops = _ops()
    rng = np.random.default_rng(5)
    rp, ci, v = rand_csr(rng, 1500, 900, 0.01, hub_rows=(3,), empty_frac=0.3)
    a = _dev(rp, ci, v, 900)
    _assert_csr_equal(ops.transpose(ops.transpose(a)).to_numpy(), (rp, ci, v))
    e = _dev(np.zeros(4, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32), 6)
    t = ops.transpose(e).to_numpy()
    assert t[0].shape == (7,) and (t[0] == 0).all() and t[1].size == 0
    # identity fixed point, single entry
    ident = _dev(np.arange(4, dtype=np.uint64), np.arange(3, dtype=np.uint32), np.ones(3, np.float32), 3)
    _assert_csr_equal(ops.transpose(ident).to_numpy(), ident.to_numpy())
    one = ops.transpose(_dev(np.array([0, 1, 1], np.uint64), np.array([1], np.uint32), np.array([2.0], np.float32), 2))
    _assert_csr_equal(one.to_numpy(), (np.array([0, 0, 1], np.uint64), np.array([0], np.uint32), np.array([2.0], np.float32)))


def test_row_degrees_and_symmetry(cuda):
    ops = _ops()
    for name in golden_cases():
        g = load_golden(name)
        a = _dev(g["row_ptr"], g["col_idx"], g["values"], int(g["n_cols"]))
        np.testing.assert_array_equal(ops.row_degrees(a).cpu().numpy().view(np.uint32), port.row_degrees(g["row_ptr"]))
        assert ops.is_symmetric(a) == bool(g["is_symmetric"]), name


def test_symmetry_value_mismatch(cuda):
    ops = _ops()
    rp = np.array([0, 1, 2], np.uint64)
    ci = np.array([1, 0], np.uint32)
    assert ops.is_symmetric(_dev(rp, ci, np.array([1.0, 1.0], np.float32), 2))
    assert not ops.is_symmetric(_dev(rp, ci, np.array([1.0, 2.0], np.float32), 2))
    assert not ops.is_symmetric(_dev(np.array([0, 1, 1], np.uint64), np.array([1], np.uint32), np.ones(1, np.float32), 2))


@pytest.mark.parametrize("name", [c for c in golden_cases() if c in ("empty_rows", "sym", "sym_ones")])
def test_cache_operands_and_counters_golden(cuda, name):
    """sum_operand / mean_operand and the build counters match the reference
    TrainingCache fetched 3 times (make_golden.py), with caching on and off."""
    ops = _ops()
    g = load_golden(name)
    for tag, which in (("sum", 0), ("mean", 1)):
        for use_cache in (0, 1):
            a = _dev(g["row_ptr"], g["col_idx"], g["values"], int(g["n_cols"]))
            cache = ops.TrainingCache(a, bool(use_cache))
            for _ in range(3):
                op = cache.sum_operand() if which == 0 else cache.mean_operand()
            _assert_csr_equal(op.to_numpy(), (g[f"cache_{tag}_{use_cache}_rp"], g[f"cache_{tag}_{use_cache}_ci"],
                                              g[f"cache_{tag}_{use_cache}_v"]))
            c = cache.counters
            want = g[f"cache_{tag}_{use_cache}_cnt"]
            assert [c["transpose_builds"], c["normalize_builds"], c["cache_hits"], int(c["symmetric"])] == \
                [int(x) for x in want], (name, tag, use_cache, c)


def test_spmm_backward_through_cache(cuda):
    """dX = A^T dC (sum) and (A D^-1)^T-style mean operand, vs the oracle."""
    import torch
    ops = _ops()
    rng = np.random.default_rng(9)
    n = 3000
    rp, ci, v = rand_csr(rng, n, n, 0.003, hub_rows=(0, 17), empty_frac=0.1, value="ones")
    a = _dev(rp, ci, v, n)
    cache = ops.TrainingCache(a, True)
    assert not cache.counters["symmetric"]
    g = rng.standard_normal((n, 64)).astype(np.float32)
    gt = torch.from_numpy(g).cuda()
    for red in ("sum", "mean"):
        dx = cache.spmm_backward(gt, red).cpu().numpy()
        if red == "sum":
            trp, tci, tv = port.transpose(rp, ci, v, n)
        else:
            trp, tci, tv = port.mean_operand(rp, ci, v, n, False)
        want = port.spmm(trp, tci, tv.astype(np.float64), g.astype(np.float64), 0)
        assert_spmm_close(dx, want, port.spmm_absdenom(trp, tci, tv, g, 0), what=f"backward {red}")
        short = np.diff(trp.astype(np.int64)) <= 256
        w32 = port.spmm(trp, tci, tv, g, 0, np.float32)
        np.testing.assert_array_equal(dx[short].view(np.uint32), w32[short].view(np.uint32))
    c = cache.counters
    assert c["transpose_builds"] == 2  # one for sum_operand, one for mean_operand (gnn.hpp:155)
    for _ in range(3):
        cache.spmm_backward(gt, "sum")
    assert cache.counters["transpose_builds"] == 2


def test_cache_symmetric_short_circuit(cuda):
    import torch
    ops = _ops()
    g = load_golden("sym")
    a = _dev(g["row_ptr"], g["col_idx"], g["values"], int(g["n_cols"]))
    cache = ops.TrainingCache(a, True)
    dc = torch.randn(a.n_rows, 32, device="cuda")
    for _ in range(4):
        cache.spmm_backward(dc, "sum")
    c = cache.counters
    assert c["symmetric"] and c["transpose_builds"] == 0 and c["cache_hits"] == 4


def test_backward_tape_error(cuda):
    import torch
    ops = _ops()
    g = load_golden("sym")
    cache = ops.TrainingCache(_dev(g["row_ptr"], g["col_idx"], g["values"], int(g["n_cols"])), True)
    with pytest.raises(ops.TapeError):
        cache.spmm_backward(torch.ones(5, 8, device="cuda"))
    with pytest.raises(ops.ShapeError):
        ops.TrainingCache(_dev(np.array([0, 0], np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32), 3))


def test_release_scratch_after_builds(cuda):
    """Workspace stays pooled for reuse; sgnn_release_scratch trims it and
    later builds still work."""
    import torch

    from paper_2403_14853_b200 import ops
    rng = np.random.default_rng(2)
    rp, ci, v = rand_csr(rng, 3000, 2000, 0.01)
    a = ops.CsrMatrix.from_numpy(rp, ci, v, 2000)
    t1 = ops.transpose(a)
    ops.release_scratch(0)
    t2 = ops.transpose(a)
    torch.cuda.synchronize()
    for x, y in zip(t1.to_numpy(), t2.to_numpy()):
        np.testing.assert_array_equal(x, y)


def test_is_symmetric_upper_lower_counting(cuda):
    """is_symmetric searches only the upper entries and compares the upper and
    lower counts: an extra lower entry, a value mismatch, a diagonal-only
    matrix and symmetric hub matrices all agree with the oracle."""
    import numpy as np

    from paper_2403_14853_b200 import graphs, ops

    def sym(rp, ci, v, n):
        got = ops.is_symmetric(ops.CsrMatrix.from_numpy(np.asarray(rp, np.uint64), np.asarray(ci, np.uint32),
                                                        np.asarray(v, np.float32), n))
        assert got == port.is_symmetric(np.asarray(rp, np.uint64), np.asarray(ci, np.uint32),
                                        np.asarray(v, np.float32), n)
        return got
    # (0,1),(1,0) mirrored; extra lower (2,0) without (0,2)
    assert not sym([0, 1, 2, 3], [1, 0, 0], [1, 1, 1], 3)
    # extra upper (0,2) without (2,0)
    assert not sym([0, 2, 3, 3], [1, 2, 0], [1, 1, 1], 3)
    # mirror present, value differs
    assert not sym([0, 1, 2], [1, 0], [1.0, 2.0], 2)
    assert sym([0, 1, 2], [1, 0], [2.0, 2.0], 2)
    assert sym([0, 1, 2, 3], [0, 1, 2], [5, 6, 7], 3)  # diagonal only
    rp, ci = graphs.rmat(12, 4096 * 16, seed=11, symmetrize=True, self_loops=True)
    v = np.ones(len(ci), np.float32)
    assert sym(rp, ci, v, 4096)
    v2 = v.copy()
    v2[len(v2) // 2] = 2.0  # one mirror pair now differs
    assert not sym(rp, ci, v2, 4096)
    rp2, ci2 = graphs.rmat(12, 4096 * 16, seed=11)
    assert not sym(rp2, ci2, np.ones(len(ci2), np.float32), 4096)


@pytest.mark.parametrize("shape,hub,empty", [((3000, (1 << 23) + 3), 0, 0.1),   # 24-bit columns: 3 passes of 8 bits
                                             ((20000, 1 << 18), 50000, 0.6),    # hub row over ~12 tiles, long empty runs
                                             ((9000, 2047), 0, 0.0),            # 11 bits: two 6-bit passes
                                             ((9000, 500), 0, 0.0)])            # 9 bits: one pass, 512 bins
def test_transpose_pass_counts_hubs_and_no_values(cuda, shape, hub, empty):
    """The radix plan's pass counts / digit widths (1 and 3 passes), a hub row
    spanning many 4096-nonzero tiles next to runs of empty rows longer than a
    tile (the tile-row precomputation), and the structure-only call (null
    values) -- all bit-exact with the reference's counting sort."""
    import ctypes as C

    import torch
    from paper_2403_14853_b200._lib import check, lib
    ops = _ops()
    m, n = shape
    rng = np.random.default_rng(m + n)
    cnt = rng.binomial(min(n, 40), 0.5, size=m)
    cnt[rng.random(m) < empty] = 0
    rows = [np.unique(rng.integers(0, n, size=int(c))) for c in cnt]  # sorted, distinct
    cnt = np.array([len(r) for r in rows], np.int64)
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(cnt)
    ci = np.concatenate(rows).astype(np.uint32)
    v = rng.uniform(-1, 1, len(ci)).astype(np.float32)
    if hub:
        cnt = np.diff(rp.astype(np.int64))
        cnt[0] = hub
        rows = [np.sort(rng.choice(n, size=int(c), replace=False)) if c else np.zeros(0, np.int64) for c in cnt]
        rp = np.zeros(m + 1, np.uint64)
        rp[1:] = np.cumsum(cnt)
        ci = np.concatenate(rows).astype(np.uint32)
        v = rng.uniform(-1, 1, len(ci)).astype(np.float32)
    a = _dev(rp, ci, v, n)
    want = port.transpose(rp, ci, v, n)
    _assert_csr_equal(ops.transpose(a).to_numpy(), want)
    trp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    tci = torch.empty(len(ci), dtype=torch.int32, device="cuda")
    check(lib().sgnn_csr_transpose(C.byref(a.c()), trp.data_ptr(), tci.data_ptr(), None, None, 0, ops._stream()),
          "transpose")
    np.testing.assert_array_equal(trp.cpu().numpy().view(np.uint64), want[0])
    np.testing.assert_array_equal(tci.cpu().numpy().view(np.uint32), want[1])
