"""Runs the on-device autotuner (sgnn_tune_spmm) on BASELINE configs and
prints the best entries against the default plan (dev probe)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402


def main():
    for name in sys.argv[1:] or ["cfg2", "cfg3"]:
        w = getattr(graphs, name)(1)
        a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
        torch.cuda.synchronize()
        t0 = time.time()
        plan, table = ops.tune_spmm(a, w.k, "sum", reps=5)
        torch.cuda.synchronize()
        dt = time.time() - t0
        table.sort(key=lambda e: e["ms"])
        default = ops.Plan(a, w.k).params
        dms = [e["ms"] for e in table if all(e["params"][k] == default[k] for k in ("lanes", "vec", "unroll", "occupancy", "path_items", "k_tile"))]
        print(json.dumps({"cfg": name, "tune_s": round(dt, 2), "candidates": len(table), "default": default,
                          "default_ms": dms[0] if dms else None,
                          "best": table[:5]}), flush=True)
        del a, plan


if __name__ == "__main__":
    main()
