"""Generate tests/golden/gnn_*.npz: the reference's own training runs
(gnn.hpp:414-438 train, io.hpp synth_planted, gnn.hpp init_model) compiled
from /root/reference/proj (oracle/_ref).  Run in the build container:

    make -C oracle && python tests/golden/make_golden_gnn.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402

# planted partition of SPEC acceptance #7 (n=400, 4 classes, p_intra 0.1,
# p_inter 0.01, feat_dim 16, noise 0.1), data seed 7, init seed 1
N, C_, PI, PO, F, NOISE, DSEED, WSEED = 400, 4, 0.1, 0.01, 16, 0.1, 7, 1
HIDDEN, LR, EPOCHS = 32, 0.05, 30


def main():
    rp, ci, v, x, lab, mask = ref.synth_planted(N, C_, PI, PO, F, NOISE, DSEED)
    out = dict(row_ptr=rp, col_idx=ci, values=v, x=x, labels=lab, mask=mask)
    for kind in ("gcn", "sage-sum", "sage-mean", "gin"):
        w0 = ref.init_model(kind, F, HIDDEN, C_, WSEED)
        losses, accs, w1, cnt = ref.train(kind, rp, ci, v, x, lab, mask, HIDDEN, C_, w0, EPOCHS, LR, True)
        out[f"{kind}_w0"] = w0
        out[f"{kind}_losses"] = losses
        out[f"{kind}_accs"] = accs
        out[f"{kind}_w_final"] = w1
        out[f"{kind}_counters"] = np.array([cnt["transpose_builds"], cnt["normalize_builds"], cnt["cache_hits"]], np.uint64)
        l2, _, _, cnt2 = ref.train(kind, rp, ci, v, x, lab, mask, HIDDEN, C_, w0, EPOCHS, LR, False)
        assert np.array_equal(l2, losses)  # cache transparency in the reference itself
        out[f"{kind}_counters_nocache"] = np.array([cnt2["transpose_builds"], cnt2["normalize_builds"], cnt2["cache_hits"]], np.uint64)
        print(kind, losses[0], losses[-1], accs[-1], cnt, cnt2)
    np.savez_compressed(os.path.join(HERE, "gnn_planted.npz"), **out)


if __name__ == "__main__":
    main()
