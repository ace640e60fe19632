"""run_tuning (autotune.hpp:99-164) on the cfg2 graph over the reference's
specialization sweep K = 16..1024, saved in report.cpp's dialect (plus the
plans sidecar) under profiles/: per K the default-plan vs tuned-plan time."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops, report  # noqa: E402


def main(out):
    w = graphs.cfg2(1)
    a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
    rep = ops.run_tuning(a, ops.specialization_sweep, reps=5, graph_id="cfg2_rmat18_k256")
    report.save_report(rep, out)
    for e in rep.entries:
        gf = 2 * w.nnz * e.k / (e.t_specialized_ms * 1e-3) / 1e9
        print(f"K={e.k:5d} trusted {e.t_trusted_ms:8.3f} ms  tuned {e.t_specialized_ms:8.3f} ms  "
              f"speedup {e.speedup:.3f}  {gf:8.1f} GFLOP/s")
    print("best_k", rep.best_k)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/tuning_cfg2.csv")
