"""Dev probe: is_symmetric on cfg2 (non-symmetric: early exit) and cfg5
(symmetric: full check), event-timed (median of 5 warm calls)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402


def main():
    out = {}
    for name, w in (("cfg2", graphs.cfg2()), ("cfg5", graphs.cfg5(1))):
        a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
        ans = ops.is_symmetric(a)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ops.is_symmetric(a)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[name] = {"symmetric": ans, "ms": round(float(np.median(ts)), 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
