"""Dev probe: time the SpMM kernel on cfg1/cfg2 for a few plans (CUDA events,
L2 flushed between reps).  Not the bench contract -- see bench.py."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402

PEAK = 6558.7


def alg_bytes(m, nnz, k):
    return 8 * (m + 1) + 8 * nnz + 4 * nnz * k + 4 * m * k


def time_it(fn, reps=10, flush=None):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def main():
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    which = sys.argv[1:2] or ["cfg1", "cfg2"]
    for name in which:
        t0 = time.time()
        w = getattr(graphs, name)()
        gen = time.time() - t0
        a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
        x = torch.from_numpy(graphs.normal(w.n_cols * w.k, 0, 1, 7).reshape(w.n_cols, w.k)).cuda()
        out = torch.empty(w.n_rows, w.k, device="cuda")
        by = alg_bytes(w.n_rows, w.nnz, w.k)
        if w.k == 128:
            variants = [{}, {"occupancy": 6}, {"lanes": 16, "vec": 2, "unroll": 4},
                        {"lanes": 16, "vec": 2, "unroll": 4, "occupancy": 4},
                        {"lanes": 16, "vec": 2, "unroll": 4, "occupancy": 6},
                        {"lanes": 16, "vec": 2, "unroll": 8, "occupancy": 4},
                        {"lanes": 8, "vec": 4, "unroll": 4, "occupancy": 4}]
            if len(sys.argv) > 2:
                variants = [json.loads(v) for v in sys.argv[2:]]
        elif w.k == 64:
            variants = [{}, {"occupancy": 5}, {"occupancy": 6}, {"unroll": 4, "occupancy": 6},
                        {"lanes": 32, "vec": 1, "unroll": 8}, {"path_items": 512}]
        elif w.k == 256:
            variants = [{}, {"lanes": 32, "vec": 2, "unroll": 4, "occupancy": 5},
                        {"lanes": 32, "vec": 1, "unroll": 8}, {"lanes": 32, "vec": 1, "unroll": 8, "occupancy": 5}]
        else:
            variants = [{}, {"occupancy": 5}, {"occupancy": 6}, {"unroll": 16}, {"lanes": 4, "vec": 2},
                        {"path_items": 64}, {"path_items": 16}, {"path_items": 8}, {"path_items": 8, "unroll": 4}]
        for red in ("sum", "mean"):
            for v in variants:
                try:
                    plan = ops.Plan(a, w.k, **v)
                except Exception as ex:  # noqa: BLE001
                    print(name, red, v, "ERR", ex)
                    continue
                fn = lambda: ops.spmm_plan(a, x, red, plan, out)  # noqa: E731
                ms = time_it(fn, flush=flush)
                ms_warm = time_it(fn)
                print(json.dumps({"cfg": name, "reduce": red, "params": plan.params, "stats": plan.stats,
                                  "ms": round(ms, 4), "ms_warm": round(ms_warm, 4),
                                  "GBps": round(by / ms / 1e6, 1), "frac": round(by / ms / 1e6 / PEAK, 3),
                                  "GFLOPs": round(2 * w.nnz * w.k / ms / 1e6, 1), "gen_s": round(gen, 2)}))
                sys.stdout.flush()


if __name__ == "__main__":
    main()
