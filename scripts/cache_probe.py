"""TrainingCache build cost on cfg2 (is_symmetric probe + device transpose),
cold (first use in the process) and warm, CUDA events + wall clock."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops  # noqa: E402


def main():
    w = graphs.cfg2(1)
    a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    out = {}
    for tag in ("cold", "warm", "warm2"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        cache = ops.TrainingCache(a, True)
        e1.record()
        at = cache.sum_operand()
        e2.record()
        torch.cuda.synchronize()
        out[tag] = {"wall_ms": round((time.perf_counter() - t0) * 1e3, 3), "create_ms": round(e0.elapsed_time(e1), 3),
                    "transpose_ms": round(e1.elapsed_time(e2), 3)}
        del at, cache
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t = ops.transpose(a)
    e1.record()
    torch.cuda.synchronize()
    out["ops.transpose_ms"] = round(e0.elapsed_time(e1), 3)
    e0.record()
    s = ops.is_symmetric(a)
    e1.record()
    torch.cuda.synchronize()
    out["is_symmetric_ms"] = round(e0.elapsed_time(e1), 3)
    out["symmetric"] = s
    print(json.dumps(out))


if __name__ == "__main__":
    main()
