"""Does a locality-improving node order cut the cfg5 SpMM's DRAM traffic?
Relabels the cfg5 graph with reverse Cuthill-McKee (scipy) and with a
degree-descending order, keeps each row's neighbours in their ORIGINAL order
(so every row's accumulation chain -- and result -- is unchanged), and times
the K=128 mean SpMM (the epoch's layer-1 / layer-2 call) on each order."""
import json
import sys
import time

import numpy as np
import scipy.sparse as sp
import torch
from scipy.sparse.csgraph import reverse_cuthill_mckee

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2403_14853_b200 import graphs, ops  # noqa: E402


def relabel(rp, ci, perm):
    """new id of old node u = inv[u]; row new_i = old row perm[new_i], its
    columns mapped through inv in their original order."""
    n = len(rp) - 1
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    deg = np.diff(rp.astype(np.int64))[perm]
    nrp = np.zeros(n + 1, np.uint64)
    nrp[1:] = np.cumsum(deg)
    starts = rp[perm].astype(np.int64)
    idx = np.repeat(starts - np.concatenate([[0], np.cumsum(deg)[:-1]]), deg) + np.arange(int(nrp[-1]))
    nci = inv[ci.astype(np.int64)[idx]].astype(np.uint32)
    return nrp, nci


def time_spmm(rp, ci, k, x, flush):
    a = ops.CsrMatrix.from_numpy(rp, ci, np.ones(len(ci), np.float32), len(rp) - 1)
    plan = ops.Plan(a, k)
    out = torch.empty(len(rp) - 1, k, device="cuda")
    t = bench._events_time(lambda: ops.spmm_plan(a, x, "mean", plan, out), 10, 3, flush)
    return float(np.median(t))


def main():
    torch.cuda.set_device(0)
    w = graphs.cfg5(1)
    n, k = w.n_rows, 128
    x = torch.from_numpy(graphs.normal(n * k, 0, 1, 1, 51).reshape(n, k)).cuda()
    flush = bench.L2Flush("cuda")
    res = {"original_ms": time_spmm(w.row_ptr, w.col_idx, k, x, flush)}
    deg = np.diff(w.row_ptr.astype(np.int64))
    perm = np.argsort(-deg, kind="stable")
    rp2, ci2 = relabel(w.row_ptr, w.col_idx, perm)
    res["degree_desc_ms"] = time_spmm(rp2, ci2, k, x, flush)
    t0 = time.time()
    m = sp.csr_matrix((np.ones(len(w.col_idx), np.float32), w.col_idx.astype(np.int64), w.row_ptr.astype(np.int64)),
                      shape=(n, n))
    perm = reverse_cuthill_mckee(m, symmetric_mode=True)
    res["rcm_s"] = round(time.time() - t0, 1)
    rp3, ci3 = relabel(w.row_ptr, w.col_idx, perm.astype(np.int64))
    res["rcm_ms"] = time_spmm(rp3, ci3, k, x, flush)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
