"""Dev probe: SDDMM and FusedMM on cfg4 (R-MAT 2^20, N*32 samples, K=64),
CUDA events, L2 flushed between reps."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402

PEAK = 6558.7


def t(fn, flush, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def main():
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    w = graphs.cfg4()
    m, nnz, k = w.n_rows, w.nnz, w.k
    p = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    x = torch.from_numpy(graphs.normal(m * k, 0, 0.1, 5).reshape(m, k)).cuda()
    y = torch.from_numpy(graphs.normal(w.n_cols * k, 0, 0.1, 6).reshape(w.n_cols, k)).cuda()
    out = torch.empty(m, k, device="cuda")
    sd_bytes = 8 * (m + 1) + 8 * nnz + 4 * m * k + 4 * nnz * k + 4 * nnz
    fu_bytes = 8 * (m + 1) + 8 * nnz + 8 * m * k + 4 * nnz * k
    ms = t(lambda: ops.sddmm(p, x, y), flush)
    print(json.dumps({"op": "sddmm", "nnz": nnz, "ms": round(ms, 4), "GFLOPs": round(2 * nnz * k / ms / 1e6, 1),
                      "frac": round(sd_bytes / ms / 1e6 / PEAK, 3)}))
    for edge in ("sigmoid_mul", "mul"):
        for red in ("sum", "mean"):
            ms = t(lambda: ops.fusedmm(p, x, y, edge, red, out), flush)
            print(json.dumps({"op": f"fusedmm {edge} {red}", "ms": round(ms, 4),
                              "GFLOPs(2nnzK)": round(2 * nnz * k / ms / 1e6, 1),
                              "frac": round(fu_bytes / ms / 1e6 / PEAK, 3)}))
    for lv in ((16, 1, 8), (8, 2, 4), (16, 2, 4)):
        for pi in (64, 128, 256):
            try:
                plan = ops.Plan(p, k, lanes=lv[0], vec=lv[1], unroll=lv[2], path_items=pi)
            except Exception as ex:  # noqa: BLE001
                print("plan", lv, ex)
                continue
            ms = t(lambda: ops.fusedmm(p, x, y, "sigmoid_mul", "sum", out, plan=plan), flush)
            print(json.dumps({"op": "fusedmm sigmoid sum (plan)", "layout": lv, "path": pi, "ms": round(ms, 4),
                              "frac": round(fu_bytes / ms / 1e6 / PEAK, 3)}))
    # SpMM on the same graph (K=64)
    plan = ops.Plan(p, k)
    ms = t(lambda: ops.spmm_plan(p, y, "sum", plan, out), flush)
    sp_bytes = 8 * (m + 1) + 8 * nnz + 4 * nnz * k + 4 * m * k
    print(json.dumps({"op": "spmm K=64", "params": plan.params, "ms": round(ms, 4),
                      "frac": round(sp_bytes / ms / 1e6 / PEAK, 3)}))


if __name__ == "__main__":
    main()
