"""cfg5 SAGE-mean step on one GPU, split into its phases with CUDA events
(dev probe): the three SpMMs vs the dense GEMMs / elementwise work."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops, sage_dist  # noqa: E402


def main():
    w = graphs.cfg5(1)
    n, k, hidden, classes = w.n_rows, w.k, 128, 16
    a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    mv = sage_dist.mean_operand_values(w.row_ptr, w.col_idx, w.values)
    am = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, mv, w.n_cols)
    x = torch.from_numpy(graphs.normal(n * k, 0, 1, 1, 51).reshape(n, k)).cuda()
    w1 = torch.randn(k, hidden, device="cuda") * 0.1
    w1s = torch.randn(k, hidden, device="cuda") * 0.1
    pf = ops.Plan(a, k)
    pb = ops.Plan(am, hidden)
    a1 = torch.empty(n, k, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    for it in range(3):
        ev[0].record()
        ops.spmm_plan(a, x, "mean", pf, a1)
        ev[1].record()
        z1 = a1 @ w1 + x @ w1s
        ev[2].record()
        h1 = torch.relu(z1)
        ev[3].record()
        ops.spmm_plan(am, h1, "sum", pb, a1)
        ev[4].record()
        g = a1.T @ h1
        ev[5].record()
        ld = h1[:, :classes].double()
        e = torch.exp(ld - ld.max(dim=1, keepdim=True).values)
        ev[6].record()
        torch.cuda.synchronize()
    names = ["spmm_mean_fwd", "gemm_2x_4Mx128x128", "relu", "spmm_bwd", "gemm_T_128x4Mx128", "softmax_double_4Mx16"]
    print(json.dumps({nm: round(ev[i].elapsed_time(ev[i + 1]), 3) for i, nm in enumerate(names)}))


if __name__ == "__main__":
    main()
