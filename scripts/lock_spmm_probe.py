"""Dev probe: SpMM K=32 / 64 on the cfg4 graph, lockstep worker vs the generic
worker (SGNN_LOCK_GENERIC), event-timed with the L2 flushed, bitwise check."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402
from scripts.fused_probe import t  # noqa: E402


def main():
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    w = graphs.cfg4()
    a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    for k in (32, 64):
        x = torch.rand(w.n_cols, k, device="cuda")
        c1 = torch.empty(w.n_rows, k, device="cuda")
        c2 = torch.empty_like(c1)
        out = {"K": k}
        for red in ("sum", "mean"):
            os.environ["SGNN_LOCK_GENERIC"] = "1"
            tg = t(lambda: ops.spmm(a, x, red, out=c1), flush)
            os.environ.pop("SGNN_LOCK_GENERIC")
            tl = t(lambda: ops.spmm(a, x, red, out=c2), flush)
            out[red] = {"generic_ms": round(tg, 4), "lock_ms": round(tl, 4),
                        "bitwise": bool(torch.equal(c1.view(torch.int32), c2.view(torch.int32)))}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
