"""Dev probe: is the cfg4 SDDMM bound by L2 misses?  The same row structure
with the columns folded into the first 2^s rows of Y (s = 20: the real
graph; 17: Y = 32 MiB, L2-resident), CUDA events, L2 flushed between reps."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402
from scripts.fused_probe import t  # noqa: E402


def main():
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    w = graphs.cfg4()
    m, k = w.n_rows, w.k
    x = torch.from_numpy(graphs.normal(m * k, 0, 0.1, 5).reshape(m, k)).cuda()
    y = torch.from_numpy(graphs.normal(w.n_cols * k, 0, 0.1, 6).reshape(w.n_cols, k)).cuda()
    out = torch.empty(m, k, device="cuda")
    for s in (20, 19, 18, 17, 15, 12):
        ci = (w.col_idx & np.uint32((1 << s) - 1)).astype(np.uint32)
        # keep each row's columns sorted (the CSR contract); duplicates are fine here
        rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(w.row_ptr.astype(np.int64)))
        ci = ci[np.lexsort((ci, rows))]
        p = ops.CsrMatrix.from_numpy(w.row_ptr, ci, w.values, w.n_cols)
        ms = t(lambda: ops.sddmm(p, x, y), flush)
        mf = t(lambda: ops.fusedmm(p, x, y, "sigmoid_mul", "sum", out), flush)
        ms2 = t(lambda: ops.spmm(p, y, "sum"), flush)
        print(json.dumps({"y_rows_bits": s, "y_MiB": (1 << s) * k * 4 >> 20, "sddmm_ms": round(ms, 4),
                          "fusedmm_ms": round(mf, 4), "spmm_ms": round(ms2, 4)}), flush=True)


if __name__ == "__main__":
    main()
