"""Small end-to-end exercise of every kernel family, for
`compute-sanitizer --tool memcheck|racecheck python scripts/sanitize_smoke.py`
(one tool per call, per B200_PROFILING.md)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402


def main():
    rp, ci = graphs.rmat(10, 1024 * 40, seed=3)  # hubs > SGNN_SEGMENT -> split rows + fixup
    n = 1024
    v = graphs.uniform(len(ci), -1, 1, seed=3)
    a = ops.CsrMatrix.from_numpy(rp, ci, v, n)
    for k in (16, 32, 33, 64, 128):
        x = torch.randn(n, k, device="cuda")
        for red in ("sum", "mean", "min", "max"):
            ops.spmm(a, x, red)
            ops.spmm_plan(a, x, red, ops.Plan(a, k, path_items=64))
        if k % 4 == 0:
            ops.fusedmm(a, x, x, "sigmoid_mul", "sum")
            ops.sddmm(a, x, x)
    t = ops.transpose(a)
    # transpose plans of 1 and 3 radix passes (2^11 and 2^23 + 3 columns)
    rng = np.random.default_rng(7)
    for m, nc in ((3000, 2047), (500, (1 << 23) + 3)):
        cnt = rng.integers(0, 40, m)
        rows = [np.unique(rng.integers(0, nc, size=int(c))) for c in cnt]
        rpw = np.zeros(m + 1, np.uint64)
        rpw[1:] = np.cumsum([len(r) for r in rows])
        ops.transpose(ops.CsrMatrix.from_numpy(rpw, np.concatenate(rows).astype(np.uint32),
                                               np.ones(int(rpw[-1]), np.float32), nc))
    cache = ops.TrainingCache(a, True)
    cache.spmm_backward(torch.randn(n, 32, device="cuda"), "mean")
    rps, cis = graphs.rmat(10, 1024 * 8, seed=4, symmetrize=True)
    s = ops.CsrMatrix.from_numpy(rps, cis, np.ones(len(cis), np.float32), n)
    ops.normalize_adjacency(s, True)
    ops.TrainingCache(s, True, model_kind="gcn")
    ops.tune_spmm(a, 32, "sum", reps=3)
    torch.cuda.synchronize()
    print("sanitize smoke ok", t.nnz)


if __name__ == "__main__":
    main()
