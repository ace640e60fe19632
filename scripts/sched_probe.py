"""Dev probe: worker size (path_items) sweep under the dynamic worker
schedule -- cfg2 / cfg3 SpMM (sum), cfg4 FusedMM and SDDMM; CUDA events, L2
flushed between reps.  One JSON line per graph."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402
from paper_2403_14853_b200.ops import _fused_layout  # noqa: E402
from scripts.ab_probe import timed  # noqa: E402

ITEMS = (128, 256, 512, 1024, 2048, 4096)


def spmm_sweep(name, w, flush):
    a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    x = torch.from_numpy(graphs.normal(w.n_cols * w.k, 0, 1, 7).reshape(w.n_cols, w.k)).cuda()
    c = torch.empty(w.n_rows, w.k, device="cuda")
    out = {"graph": name, "default": ops.Plan(a, w.k).params["path_items"]}
    for it in ITEMS:
        p = ops.Plan(a, w.k, path_items=it)
        out[it] = timed(lambda: ops.spmm_plan(a, x, "sum", p, c), flush)
        del p
    print(json.dumps(out), flush=True)


def fused_sweep(w, flush):
    p = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    xs = torch.from_numpy(graphs.normal(w.n_rows * w.k, 0, 0.1, 3).reshape(w.n_rows, w.k)).cuda()
    ys = torch.from_numpy(graphs.normal(w.n_cols * w.k, 0, 0.1, 4).reshape(w.n_cols, w.k)).cuda()
    out = {"graph": "cfg4", "default": p.plan(w.k, "fused").params["path_items"]}
    for it in ITEMS:
        pl = ops.Plan(p, w.k, path_items=it, **_fused_layout(w.k))
        p._plans[("fused", w.k)] = pl
        out[f"fused_{it}"] = timed(lambda: ops.fusedmm(p, xs, ys, "sigmoid_mul", "sum", plan=pl), flush)
        out[f"sddmm_{it}"] = timed(lambda: ops.sddmm(p, xs, ys), flush)
    print(json.dumps(out), flush=True)


def main():
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    spmm_sweep("cfg2", graphs.cfg2(1), flush)
    fused_sweep(graphs.cfg4(1), flush)
    w = graphs.cfg3(1)
    spmm_sweep("cfg3", w, flush)


if __name__ == "__main__":
    main()
