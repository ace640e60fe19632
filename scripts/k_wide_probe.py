"""Wide-K SpMM (K = 768, 1024) on the cfg2 graph under a few layouts (dev probe)."""
import sys, json, torch, numpy as np
sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops
from scripts.ab_probe import timed
w = graphs.cfg2(1)
a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for k in (768, 1024):
    x = torch.rand(w.n_cols, k, device="cuda")
    out = torch.empty(w.n_rows, k, device="cuda")
    base = None
    for params in ({}, {"lanes": 32, "vec": 2, "unroll": 8}, {"lanes": 32, "vec": 2, "unroll": 4, "occupancy": 5},
                   {"lanes": 32, "vec": 1, "unroll": 8, "occupancy": 5}, {"lanes": 32, "vec": 4, "unroll": 2, "occupancy": 4}):
        p = ops.Plan(a, k, **params)
        t = timed(lambda: ops.spmm_plan(a, x, "sum", p, out), flush, reps=10)
        r = out.clone()
        if base is None: base = r
        print(json.dumps({"k": k, "params": params, "ms": t, "gflops": round(2*w.nnz*k/t/1e6,1), "same": bool(torch.equal(r, base))}))
