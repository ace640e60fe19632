"""Generate tests/golden/*.npz from the reference itself (oracle/_ref, compiled
from /root/reference/proj by oracle/Makefile).  Run in the build container:

    make -C oracle && python tests/golden/make_golden.py

Each fixture holds seeded inputs plus the reference's outputs for every hot
path function (spmm fp32 trusted/specialized and fp64 for all four reduces,
transpose, sddmm, fusedmm for both edge ops and all reduces, the TrainingCache
operands and counters, is_symmetric, normalize_adjacency, balanced_row_partition).
The tests pin oracle/port.py against these and the GPU path against both.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402


def rand_csr(rng, m, n, density, hub_rows=(), empty_frac=0.0, symmetric=False, value="uniform"):
    mask = rng.random((m, n)) < density
    for h in hub_rows:
        mask[h, :] = rng.random(n) < 0.9
    if empty_frac:
        mask[rng.random(m) < empty_frac, :] = False
    if symmetric:
        assert m == n
        mask = mask | mask.T
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(mask.sum(1))
    ci = np.nonzero(mask)[1].astype(np.uint32)
    if value == "ones":
        v = np.ones(len(ci), np.float32)
    else:
        v = rng.uniform(-1, 1, len(ci)).astype(np.float32)
        if symmetric:  # mirror values so the matrix is value-symmetric too
            dense = np.zeros((m, n), np.float32)
            r = np.repeat(np.arange(m), np.diff(rp).astype(np.int64))
            dense[r, ci] = v
            dense = np.triu(dense) + np.triu(dense, 1).T
            v = dense[r, ci].astype(np.float32)
    return rp, ci, v


CASES = [
    # name, m, n, density, hubs, empty_frac, symmetric, K list
    ("er_small", 64, 48, 0.10, (), 0.0, False, (1, 3, 16, 32)),
    ("hub", 64, 300, 0.03, (3, 50), 0.2, False, (16, 33, 64)),
    ("empty_rows", 80, 80, 0.05, (), 0.6, False, (4, 32, 128)),
    ("sym", 120, 120, 0.04, (7,), 0.0, True, (8, 32)),
    ("sym_ones", 100, 100, 0.05, (), 0.1, True, (16,)),
    ("wide", 24, 400, 0.02, (0,), 0.0, False, (256,)),
]


def main():
    if not ref.available("O2"):
        raise SystemExit("oracle/_ref not built (make -C oracle) -- needs /root/reference")
    for ci_, (name, m, n, dens, hubs, ef, sym, ks) in enumerate(CASES):
        rng = np.random.default_rng(1000 + ci_)
        value = "ones" if name.endswith("ones") else "uniform"
        rp, col, v = rand_csr(rng, m, n, dens, hubs, ef, sym, value)
        out = dict(row_ptr=rp, col_idx=col, values=v, n_cols=np.uint32(n), ks=np.array(ks, np.uint32))
        out["transpose"] = np.array(0)
        trp, tci, tv = ref.transpose_f32(rp, col, v, n)
        out.update(t_row_ptr=trp, t_col_idx=tci, t_values=tv)
        out["is_symmetric"] = np.uint8(ref.is_symmetric(rp, col, v, n))
        out["partition7"] = ref.balanced_row_partition(rp, 7)
        for k in ks:
            x = rng.uniform(-1, 1, (n, k)).astype(np.float32)
            xi = rng.uniform(-1, 1, (m, k)).astype(np.float32)
            out[f"x_{k}"] = x
            out[f"xi_{k}"] = xi
            for red in range(4):
                out[f"spmm32_{k}_{red}"] = ref.spmm_f32(rp, col, v, x, n, red)
                out[f"spmm64_{k}_{red}"] = ref.spmm_f64(rp, col, v, x.astype(np.float64), n, red)
                for eo in (0, 1):
                    out[f"fused32_{k}_{eo}_{red}"] = ref.fusedmm(rp, col, v, xi, x, n, eo, red, np.float32)
                    out[f"fused64_{k}_{eo}_{red}"] = ref.fusedmm(rp, col, v, xi.astype(np.float64),
                                                                 x.astype(np.float64), n, eo, red)
            if k in (16, 32, 64, 128, 256):
                out[f"spmm32spec_{k}"] = ref.spmm_f32(rp, col, v, x, n, 0, specialized=True)
            out[f"sddmm32_{k}"] = ref.sddmm(rp, col, v, xi, x, n, np.float32)
            out[f"sddmm64_{k}"] = ref.sddmm(rp, col, v, xi.astype(np.float64), x.astype(np.float64), n)
        if m == n:
            for kind, which, tag in ((1, 0, "sum"), (2, 1, "mean")):
                for use_cache in (0, 1):
                    a, b, c, cnt = ref.cache_operand(rp, col, v, kind, use_cache, which, 3)
                    out[f"cache_{tag}_{use_cache}_rp"] = a
                    out[f"cache_{tag}_{use_cache}_ci"] = b
                    out[f"cache_{tag}_{use_cache}_v"] = c
                    out[f"cache_{tag}_{use_cache}_cnt"] = np.array(
                        [cnt["transpose_builds"], cnt["normalize_builds"], cnt["cache_hits"], cnt["symmetric"]],
                        np.uint64)
            if (v >= 0).all():
                nrp, nci, nv = ref.normalize_adjacency(rp, col, v, True)
                out.update(norm_row_ptr=nrp, norm_col_idx=nci, norm_values=nv)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
