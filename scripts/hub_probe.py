"""Is the cfg2 SpMM limited by L2-slice hot spots on hub rows?  Times the
SpMM on the original graph and on copies where every occurrence of a hub
column (in-degree > T) is spread over R replicas of its X row (extra rows
appended to X; values and per-row order unchanged, so results stay equal).
Prints one JSON line per (T, R)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402


def timed(fn, reps=20, flush=None):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    w = graphs.cfg2(1)
    n, k = w.n_rows, w.k
    rp, ci, v = w.row_ptr, w.col_idx.astype(np.int64), w.values
    x = torch.from_numpy(graphs.normal(n * k, 0, 1, 7).reshape(n, k)).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    a = ops.CsrMatrix.from_numpy(rp, w.col_idx, v, n)
    base = ops.spmm(a, x, "sum")
    t0 = timed(lambda: ops.spmm(a, x, "sum"), flush=flush)
    deg = np.bincount(ci, minlength=n)
    order = np.argsort(-deg)
    print(json.dumps({"baseline_ms": round(t0, 4), "top_in_degrees": deg[order[:8]].tolist(),
                      "nnz": int(len(ci))}), flush=True)
    pos = np.arange(len(ci))
    for thr, reps in ((65536, 8), (16384, 8), (4096, 8), (4096, 32), (1024, 8)):
        hubs = np.nonzero(deg > thr)[0]
        if len(hubs) == 0:
            continue
        slot = np.full(n, -1, np.int64)
        slot[hubs] = np.arange(len(hubs))
        s = slot[ci]
        is_hub = s >= 0
        new_ci = ci.copy()
        # replica r of hub h lives at row n + h*reps + r - (r==0 ? keep original)
        r = pos % reps
        rep_id = n + s * reps + r
        new_ci[is_hub & (r > 0)] = rep_id[is_hub & (r > 0)]
        n2 = n + len(hubs) * reps
        a2 = ops.CsrMatrix.from_numpy(rp, new_ci.astype(np.uint32), v, n2)
        x2 = torch.empty(n2, k, device="cuda")
        x2[:n] = x
        hub_t = torch.from_numpy(hubs).cuda()
        x2[n:] = x[hub_t].repeat_interleave(reps, dim=0)
        same = torch.equal(ops.spmm(a2, x2, "sum"), base)
        t = timed(lambda: ops.spmm(a2, x2, "sum"), flush=flush)
        print(json.dumps({"threshold": thr, "replicas": reps, "hubs": int(len(hubs)),
                          "hub_nnz_frac": round(float(is_hub.mean()), 4), "ms": round(t, 4),
                          "speedup": round(t0 / t, 3), "bitwise_equal": bool(same)}), flush=True)


if __name__ == "__main__":
    main()
