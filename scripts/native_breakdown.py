"""Per-kernel breakdown of one cfg5 SAGE-mean epoch of the native engine:
run under `ncu --metrics gpu__time_duration.sum --csv` (dev probe); the
epoch is bracketed by cudaProfilerStart/Stop so only it is captured."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import gnn, graphs, ops  # noqa: E402


def main():
    w = graphs.cfg5(1)
    n, k, hidden, classes = w.n_rows, w.k, 128, 16
    a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    x = torch.from_numpy(graphs.normal(n * k, 0, 1, 1, 51).reshape(n, k)).cuda()
    lab = torch.from_numpy((np.arange(n) * 2654435761 % classes).astype(np.int64)).cuda()
    mask = torch.ones(n, dtype=torch.uint8, device="cuda")
    m = gnn.init_model("sage-mean", k, hidden, classes, seed=1)
    gnn.train_native(m, a, x, lab, mask, epochs=2, lr=0.05)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()  # create (cache build, plans) + one epoch
    gnn.train_native(m, a, x, lab, mask, epochs=1, lr=0.05)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
