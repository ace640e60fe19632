"""A/B probe: time the cfg2 SpMM (fwd on A, bwd on the cached CSC) and the
cfg4 FusedMM with whichever libsgnn_b200.so SGNN_B200_LIB selects (L2
flushed between reps).  One JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402


def timed(fn, flush, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(float(np.median(ts)), 4)


def main():
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {"lib": os.path.basename(os.environ.get("SGNN_B200_LIB", "libsgnn_b200.so"))}
    w = graphs.cfg2(1)
    a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    x = torch.from_numpy(graphs.normal(w.n_cols * w.k, 0, 1, 7).reshape(w.n_cols, w.k)).cuda()
    c = torch.empty(w.n_rows, w.k, device="cuda")
    at = ops.TrainingCache(a).sum_operand()
    for occ in (5, 6):
        pf = ops.Plan(a, w.k, occupancy=occ)
        pb = ops.Plan(at, w.k, occupancy=occ)
        out[f"cfg2_fwd_occ{occ}"] = timed(lambda: ops.spmm_plan(a, x, "sum", pf, c), flush)
        out[f"cfg2_bwd_occ{occ}"] = timed(lambda: ops.spmm_plan(at, x, "sum", pb, c), flush)
    del a, at
    w4 = graphs.cfg4(1)
    p = ops.CsrMatrix.from_numpy(w4.row_ptr, w4.col_idx, w4.values, w4.n_cols)
    xs = torch.from_numpy(graphs.normal(w4.n_rows * w4.k, 0, 0.1, 3).reshape(w4.n_rows, w4.k)).cuda()
    ys = torch.from_numpy(graphs.normal(w4.n_cols * w4.k, 0, 0.1, 4).reshape(w4.n_cols, w4.k)).cuda()
    ops.fusedmm(p, xs, ys, "sigmoid_mul", "sum")
    out["cfg4_fusedmm"] = timed(lambda: ops.fusedmm(p, xs, ys, "sigmoid_mul", "sum"), flush)
    out["cfg4_sddmm"] = timed(lambda: ops.sddmm(p, xs, ys), flush)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
