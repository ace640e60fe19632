"""cfg4 FusedMM / SDDMM: the TMA-gather kernels (fused_tma.cu) at ring depths
2/3/4 against the register-gather kernels (default; SGNN_TMA_FUSED=1 selects TMA), CUDA events,
L2 flushed between calls, median of 20; bitwise comparison of the outputs."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_14853_b200 import graphs, ops  # noqa: E402


def main():
    torch.cuda.set_device(0)
    w = graphs.cfg4(1)
    m, k = w.n_rows, w.k
    p = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    x = torch.from_numpy(graphs.normal(m * k, 0, 0.1, 1, 41).reshape(m, k)).cuda()
    y = torch.from_numpy(graphs.normal(w.n_cols * k, 0, 0.1, 1, 42).reshape(w.n_cols, k)).cuda()
    plan = p.plan(k, "fused")
    flush = bench.L2Flush("cuda")
    res = {}
    outs = {}
    for mode in ("reg", "tma2", "tma3", "tma4"):
        if mode == "reg":
            os.environ.pop("SGNN_TMA_FUSED", None)
        else:
            os.environ["SGNN_TMA_FUSED"] = "1"
            os.environ["SGNN_TMA_DEPTH"] = mode[-1]
        out = torch.empty(m, k, device="cuda")
        tf = bench._events_time(lambda: ops.fusedmm(p, x, y, "sigmoid_mul", "sum", out, plan=plan), 20, 3, flush)
        ts = bench._events_time(lambda: ops.sddmm(p, x, y), 20, 3, flush)
        outs[mode] = (out.cpu().numpy().copy(), ops.sddmm(p, x, y).values.cpu().numpy())
        res[mode] = {"fused_ms": round(float(np.median(tf)), 4), "sddmm_ms": round(float(np.median(ts)), 4)}
    for mode in ("tma2", "tma3", "tma4"):
        res[mode]["bitwise_fused"] = bool(np.array_equal(outs[mode][0].view(np.uint32), outs["reg"][0].view(np.uint32)))
        res[mode]["bitwise_sddmm"] = bool(np.array_equal(outs[mode][1].view(np.uint32), outs["reg"][1].view(np.uint32)))
    print(json.dumps({"cfg4": {"nnz": w.nnz, "K": k}, **res}), flush=True)


if __name__ == "__main__":
    main()
