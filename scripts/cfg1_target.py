"""cfg1 SpMM: a few calls between cudaProfilerStart/Stop for ncu launch timing (dev probe)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs, ops
w = graphs.cfg1(1)
a = ops.CsrMatrix.from_numpy(w.row_ptr, w.col_idx, w.values, w.n_cols)
x = torch.rand(w.n_cols, w.k, device="cuda")
c = torch.empty(w.n_rows, w.k, device="cuda")
p = ops.Plan(a, w.k)
for _ in range(5): ops.spmm_plan(a, x, "sum", p, c)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(3): ops.spmm_plan(a, x, "sum", p, c)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
