"""cfg5 SAGE-mean training epochs in the native engine (one GPU) vs the
torch-based row-partitioned step at P=1 (dev probe)."""
import json
import sys
import time

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
    t0 = time.time()
    out = gnn.train_native(m, a, x, lab, mask, epochs=6, lr=0.05)
    wall = time.time() - t0
    m2 = gnn.init_model("sage-mean", k, hidden, classes, seed=1)
    outg = gnn.train_native(m2, a, x, lab, mask, epochs=6, lr=0.05, cuda_graph=True)
    print(json.dumps({"native_epoch_ms": [round(s.epoch_seconds * 1e3, 2) for s in out.stats],
                      "native_graph_epoch_ms": [round(s.epoch_seconds * 1e3, 2) for s in outg.stats],
                      "loss": [round(s.loss, 5) for s in out.stats], "wall_s": round(wall, 2)}))


if __name__ == "__main__":
    main()
