import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: large BASELINE-size cases")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import torch
    return torch.device("cuda")


def golden_cases():
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and not f.startswith("gnn_"))


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def rand_csr(rng, m, n, density, hub_rows=(), hub_density=0.9, empty_frac=0.0, value="uniform"):
    """Random CSR built row by row (no dense m x n mask, so it scales)."""
    counts = rng.binomial(n, density, size=m)
    for h in hub_rows:
        counts[h] = int(n * hub_density)
    if empty_frac:
        counts[rng.random(m) < empty_frac] = 0
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(counts)
    ci = np.empty(int(rp[-1]), np.uint32)
    for i in range(m):
        c = int(counts[i])
        if c:
            ci[int(rp[i]):int(rp[i + 1])] = np.sort(rng.choice(n, size=c, replace=False))
    if value == "ones":
        v = np.ones(len(ci), np.float32)
    elif value == "positive":
        v = rng.uniform(0, 1, len(ci)).astype(np.float32)
    else:
        v = rng.uniform(-1, 1, len(ci)).astype(np.float32)
    return rp, ci, v


def assert_spmm_close(got, want64, denom, rtol=1e-5, what=""):
    """|gpu - ref64| <= rtol * sum_j |a_ij x_jk| (SURVEY 8c / north_star tolerance)."""
    err = np.abs(got.astype(np.float64) - want64)
    bound = rtol * denom
    bad = err > bound
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(f"{what}: {bad.sum()} elements exceed tolerance; first {idx.tolist()} "
                             f"err={err[bad][:5]} bound={bound[bad][:5]}")
