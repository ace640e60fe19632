"""Device transpose (CSR -> CSC, sparse.hpp:72-89) on cfg2: median of N
event-timed calls, plus a checksum of the result so A/B variants can be
compared for bit-identity in one process."""
import hashlib
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    which = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
    w = {"cfg2": graphs.cfg2, "cfg4": graphs.cfg4, "cfg5": graphs.cfg5}[which](1)
    a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    t = ops.transpose(a)  # warm the workspace pool
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t = ops.transpose(a)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    hs = hashlib.sha1()
    for v in (t.row_ptr, t.col_idx, t.values):
        hs.update(v.cpu().numpy().tobytes())
    h = hs.hexdigest()[:16]
    print(json.dumps({"nnz": int(a.nnz), "median_ms": round(float(np.median(times)), 4),
                      "min_ms": round(float(np.min(times)), 4), "hash": h}))


if __name__ == "__main__":
    main()
