"""cfg4 FusedMM / SDDMM under a few launch geometries (dev probe)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402
from scripts.ab_probe import timed  # noqa: E402


def main():
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    w4 = graphs.cfg4(1)
    p = ops.CsrMatrix.from_numpy(w4.row_ptr, w4.col_idx, w4.values, w4.n_cols)
    xs = torch.from_numpy(graphs.normal(w4.n_rows * w4.k, 0, 0.1, 3).reshape(w4.n_rows, w4.k)).cuda()
    ys = torch.from_numpy(graphs.normal(w4.n_cols * w4.k, 0, 0.1, 4).reshape(w4.n_cols, w4.k)).cuda()
    ref = ops.fusedmm(p, xs, ys, "sigmoid_mul", "sum")
    for params in ({}, {"lanes": 16, "vec": 1, "unroll": 8, "occupancy": 6},
                   {"lanes": 16, "vec": 1, "unroll": 4, "occupancy": 1},
                   {"lanes": 16, "vec": 1, "unroll": 4, "occupancy": 6},
                   {"lanes": 16, "vec": 1, "unroll": 4, "occupancy": 8},
                   {"lanes": 16, "vec": 1, "unroll": 8, "occupancy": 1},
                   {"lanes": 32, "vec": 1, "unroll": 8, "occupancy": 5}):
        try:
            plan = ops.Plan(p, w4.k, **params) if params else None
            got = ops.fusedmm(p, xs, ys, "sigmoid_mul", "sum", plan=plan)
            same = bool(torch.equal(got, ref))
            t = timed(lambda: ops.fusedmm(p, xs, ys, "sigmoid_mul", "sum", plan=plan), flush)
            print(json.dumps({"op": "fusedmm", "params": params, "ms": t, "bitwise_equal_default": same}), flush=True)
        except Exception as ex:  # noqa: BLE001
            print(json.dumps({"op": "fusedmm", "params": params, "error": str(ex)[:200]}), flush=True)


if __name__ == "__main__":
    main()
