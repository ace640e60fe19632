"""Dev probe: cfg4 SDDMM (SGNN_SDDMM_VARIANT env, one process per variant)
and FusedMM sigmoid/sum with explicit plans (16 lanes, 8 or 16 gathers in
flight per group, register caps), CUDA events, L2 flushed between reps;
checks every variant against the default bitwise."""
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
    p = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    x = torch.from_numpy(graphs.normal(m * k, 0, 0.1, 5).reshape(m, k)).cuda()
    y = torch.from_numpy(graphs.normal(w.n_cols * k, 0, 0.1, 6).reshape(w.n_cols, k)).cuda()
    out = torch.empty(m, k, device="cuda")
    if sys.argv[1:] == ["sddmm"]:
        ms = t(lambda: ops.sddmm(p, x, y), flush)
        r = ops.sddmm(p, x, y)
        print(json.dumps({"op": "sddmm", "ms": round(ms, 4), "sum": float(r.values.double().sum())}))
        return
    if sys.argv[1:] == ["fused"]:
        ms = t(lambda: ops.fusedmm(p, x, y, "sigmoid_mul", "sum", out), flush)
        print(json.dumps({"op": "fusedmm sigmoid sum", "ms": round(ms, 4), "sum": float(out.double().sum())}))
        return
    ref = ops.fusedmm(p, x, y, "sigmoid_mul", "sum", out.clone())
    layouts = ((16, 1, 8, 5),) if sys.argv[1:] == ["paths"] else \
        ((16, 1, 8, 5), (16, 1, 8, 6), (16, 1, 16, 1), (16, 1, 16, 4), (16, 1, 16, 5))
    paths = (256, 512, 1024, 2048) if sys.argv[1:] == ["paths"] else (128, 256)
    for lv in layouts:
        for pi in paths:
            plan = ops.Plan(p, k, lanes=lv[0], vec=lv[1], unroll=lv[2], occupancy=lv[3], path_items=pi)
            ms = t(lambda: ops.fusedmm(p, x, y, "sigmoid_mul", "sum", out, plan=plan), flush)
            same = bool(torch.equal(out.view(torch.int32), ref.view(torch.int32)))
            print(json.dumps({"op": "fusedmm", "layout": lv, "path": pi, "ms": round(ms, 4), "bitwise": same}))


if __name__ == "__main__":
    main()
