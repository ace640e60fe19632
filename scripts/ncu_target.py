"""One call of a hot-path op between cudaProfilerStart/Stop, for
`ncu --profile-from-start off --set full` captures (profiles/):
  python scripts/ncu_target.py cfg2_spmm | cfg2_spmm_bwd | cfg4_fused | cfg4_sddmm | cfg3_spmm | cfg5_spmm"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402


def main(which):
    if which.startswith("cfg2") or which.startswith("cfg3") or which.startswith("cfg5"):
        w = {"cfg2": graphs.cfg2, "cfg3": graphs.cfg3, "cfg5": graphs.cfg5}[which[:4]](1)
        a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
        if which.endswith("bwd"):
            a = ops.TrainingCache(a).sum_operand()
        x = torch.from_numpy(graphs.normal(a.n_cols * w.k, 0, 1, 7).reshape(a.n_cols, w.k)).cuda()
        c = torch.empty(a.n_rows, w.k, device="cuda")
        plan = ops.Plan(a, w.k)
        fn = lambda: ops.spmm_plan(a, x, "sum", plan, c)  # noqa: E731
    else:
        w = graphs.cfg4(1)
        p = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
        xs = torch.from_numpy(graphs.normal(w.n_rows * w.k, 0, 0.1, 3).reshape(w.n_rows, w.k)).cuda()
        ys = torch.from_numpy(graphs.normal(w.n_cols * w.k, 0, 0.1, 4).reshape(w.n_cols, w.k)).cuda()
        if which == "cfg4_fused":
            fn = lambda: ops.fusedmm(p, xs, ys, "sigmoid_mul", "sum")  # noqa: E731
        else:
            fn = lambda: ops.sddmm(p, xs, ys)  # noqa: E731
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    fn()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ok", which)


if __name__ == "__main__":
    main(sys.argv[1])
