"""Cost of the peer-table gather (sgnn_spmm_peer_f32) against the plain
gathered-buffer SpMM, on one GPU: the P blocks are separate local allocations
(stand-ins for the peers' HBM).  Prints one JSON line per P."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops, partition  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    w = graphs.cfg2(1)
    n, k = w.n_rows, w.k
    x = torch.from_numpy(graphs.normal(n * k, 0, 1, 7).reshape(n, k)).cuda()
    for parts in (1, 2, 4, 8):
        pt_g = partition.make_partition(w.row_ptr, parts)
        pt_p = partition.make_partition(w.row_ptr, parts, pow2=True)
        ranks_g = [partition.PartitionedSpmm(w.row_ptr, w.col_idx, w.values, pt_g, p, k) for p in range(parts)]
        ranks_p = [partition.PartitionedSpmm(w.row_ptr, w.col_idx, w.values, pt_p, p, k) for p in range(parts)]
        gathered = partition.LoopbackExchange().all_gather(
            [partition.pad_block(x[pt_g.rows(p)[0]:pt_g.rows(p)[1]], pt_g.stride) for p in range(parts)])
        blocks = [partition.pad_block(x[pt_p.rows(p)[0]:pt_p.rows(p)[1]], pt_p.stride) for p in range(parts)]
        outs = [torch.empty(r.r1 - r.r0, k, device="cuda") for r in ranks_g]
        tg = [timed(lambda r=r, o=o: r.compute(gathered, "sum", o)) for r, o in zip(ranks_g, outs)]
        tp = [timed(lambda r=r, o=o: r.compute_peer(blocks, "sum", o)) for r, o in zip(ranks_p, outs)]
        same = all(torch.equal(ranks_g[i].compute(gathered, "sum"), ranks_p[i].compute_peer(blocks, "sum"))
                   for i in range(parts))
        print(json.dumps({"parts": parts, "gathered_ms_per_rank": [round(t, 4) for t in tg],
                          "peer_ms_per_rank": [round(t, 4) for t in tp],
                          "max_gathered": round(max(tg), 4), "max_peer": round(max(tp), 4),
                          "stride_gathered": pt_g.stride, "stride_pow2": pt_p.stride, "bitwise_equal": same}),
              flush=True)


if __name__ == "__main__":
    main()
