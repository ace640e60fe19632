"""Writes the col_idx of a BASELINE config (CSR order) as raw u32 for gather_probe."""
import sys

sys.path.insert(0, ".")
from paper_2403_14853_b200 import graphs  # noqa: E402

w = getattr(graphs, sys.argv[1])(1)
w.col_idx.astype("uint32").tofile(sys.argv[2])
print(w.n_cols)
