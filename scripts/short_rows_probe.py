"""Dev probe: cfg1 SpMM (and a K=128 short-row graph) with the short-row kernel
(SGNN_SHORT_ROWS=1) vs the worker kernel: event-timed, L2 flushed, results
compared bitwise in one process (the switch is read per call)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402
from scripts.fused_probe import t  # noqa: E402


def main():
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    w = graphs.cfg1(1)
    cases = [("cfg1", w.row_ptr, w.col_idx, w.values, w.n_cols, w.k)]
    rng = np.random.default_rng(3)
    n = 1 << 20
    cnt = rng.integers(0, 33, n)
    rows = [np.unique(rng.integers(0, n, size=int(c))) for c in cnt[:1]]
    for K in (64, 128):
        rp = np.zeros(n + 1, np.uint64)
        deg = rng.integers(0, 17, n)
        rp[1:] = np.cumsum(deg)
        ci = rng.integers(0, n, int(rp[-1])).astype(np.uint32)
        # sorted distinct columns within each row are not needed for timing; keep the CSR valid
        r = np.repeat(np.arange(n), deg)
        o = np.lexsort((ci, r))
        ci = ci[o]
        cases.append((f"uniform_deg<=16_K{K}", rp, ci, np.ones(len(ci), np.float32), n, K))
    for name, rp, ci, v, nc, k in cases:
        a = ops.CsrMatrix.from_numpy(rp, ci, v, nc)
        x = torch.rand(nc, k, device="cuda")
        plan = ops.Plan(a, k)
        c1 = torch.empty(len(rp) - 1, k, device="cuda")
        c2 = torch.empty_like(c1)
        out = {"case": name, "K": k}
        for red in ("sum", "mean"):
            os.environ.pop("SGNN_SHORT_ROWS", None)
            tw = t(lambda: ops.spmm_plan(a, x, red, plan, c1), flush, reps=30)
            os.environ["SGNN_SHORT_ROWS"] = "1"
            ts = t(lambda: ops.spmm_plan(a, x, red, plan, c2), flush, reps=30)
            os.environ.pop("SGNN_SHORT_ROWS", None)
            out[red] = {"worker_us": round(tw * 1e3, 2), "short_us": round(ts * 1e3, 2),
                        "bitwise": bool(torch.equal(c1.view(torch.int32), c2.view(torch.int32)))}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
