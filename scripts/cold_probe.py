"""Dev probe: where the cold (first-in-process) cfg2 cache build goes --
first vs second TrainingCache build, CUDA events and wall clock; run with and
without CUDA_MODULE_LOADING=EAGER to separate lazy kernel loading."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402


def main():
    w = graphs.cfg2(1)
    a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    torch.cuda.synchronize()
    out = {"module_loading": os.environ.get("CUDA_MODULE_LOADING", "default(lazy)")}
    for tag in ("first", "second"):
        t0 = time.perf_counter()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        c = ops.TrainingCache(a, True)
        e1.record()
        c.sum_operand()
        e2.record()
        torch.cuda.synchronize()
        out[tag] = {"wall_ms": round((time.perf_counter() - t0) * 1e3, 2), "create_ms": round(e0.elapsed_time(e1), 3),
                    "transpose_ms": round(e1.elapsed_time(e2), 3)}
        del c
    print(json.dumps(out))


if __name__ == "__main__":
    main()
