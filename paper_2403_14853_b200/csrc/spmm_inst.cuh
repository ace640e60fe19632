// spmm_inst.cuh -- instantiates the worker kernels (SpMM, and FusedMM for each
// edge op) for one reduction and exposes them through lookup functions.
// Included once per (reduction, mode) file so the variants compile in parallel.
#pragma once

#include <algorithm>

#include "spmm_kernel.cuh"

namespace sgnn {

template <int G, int V, int U, int RED, bool VEC, int OP, int MINB>
sgnn_status launch_spmm_worker(const SpmmArgs& a, uint32_t block, uint32_t max_blocks,
                               cudaStream_t s) {
    static int per_sm[2] = {-1, -1};  // for block = 64, 128
    const int bi = block <= 64 ? 0 : 1;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    if (per_sm[bi] < 0) {
        int n = 0;
        SGNN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &n, dev::spmm_worker_kernel<G, V, U, RED, VEC, OP, MINB>, int(block), 0));
        per_sm[bi] = std::max(n, 1);
    }
    const uint64_t want = ceil_div_u64(uint64_t(a.n_workers) * G, block);
    uint64_t blocks = std::min<uint64_t>(want, uint64_t(dp.sm_count) * per_sm[bi]);
    if (max_blocks) blocks = std::min<uint64_t>(blocks, max_blocks);
    if (blocks == 0) return SGNN_OK;
    dev::spmm_worker_kernel<G, V, U, RED, VEC, OP, MINB><<<unsigned(blocks), block, 0, s>>>(a);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

// (lanes, vec, unroll, reduce, float4?, mode, occupancy) combinations for SpMM.
#define SGNN_SPMM_CONFIGS(X, RED, OP) \
    X(4, 1, 4, RED, true, OP, 1)      \
    X(4, 1, 8, RED, true, OP, 1)      \
    X(4, 2, 8, RED, true, OP, 1)      \
    X(4, 4, 4, RED, true, OP, 1)      \
    X(8, 4, 4, RED, true, OP, 1)      \
    X(8, 1, 4, RED, true, OP, 1)      \
    X(8, 1, 8, RED, true, OP, 1)      \
    X(16, 1, 4, RED, true, OP, 1)     \
    X(16, 1, 8, RED, true, OP, 1)     \
    X(32, 1, 4, RED, true, OP, 1)     \
    X(32, 1, 8, RED, true, OP, 1)     \
    X(32, 1, 16, RED, true, OP, 1)    \
    X(16, 1, 16, RED, true, OP, 1)    \
    X(8, 1, 16, RED, true, OP, 1)     \
    X(8, 2, 4, RED, true, OP, 1)      \
    X(8, 2, 8, RED, true, OP, 1)      \
    X(16, 2, 4, RED, true, OP, 1)     \
    X(16, 2, 8, RED, true, OP, 1)     \
    X(32, 2, 4, RED, true, OP, 1)     \
    X(32, 2, 8, RED, true, OP, 1)     \
    X(16, 4, 2, RED, true, OP, 1)     \
    X(16, 4, 4, RED, true, OP, 1)     \
    X(32, 4, 2, RED, true, OP, 1)     \
    X(32, 4, 4, RED, true, OP, 1)     \
    X(32, 8, 2, RED, true, OP, 1)     \
    X(32, 1, 4, RED, false, OP, 1)    \
    X(32, 1, 8, RED, false, OP, 1)    \
    X(32, 2, 4, RED, false, OP, 1)    \
    X(32, 2, 8, RED, false, OP, 1)    \
    X(32, 4, 2, RED, false, OP, 1)    \
    X(32, 4, 4, RED, false, OP, 1)    \
    X(32, 8, 2, RED, false, OP, 1)    \
    X(32, 8, 4, RED, false, OP, 1)

// Register-capped (occupancy) variants of the main float4 layouts, for the
// reductions GNN training uses (sum, mean).
#define SGNN_SPMM_OCC_CONFIGS(X, RED, OP) \
    X(4, 2, 8, RED, true, OP, 4)          \
    X(4, 2, 8, RED, true, OP, 6)          \
    X(8, 2, 4, RED, true, OP, 6)          \
    X(8, 2, 4, RED, true, OP, 8)          \
    X(8, 2, 8, RED, true, OP, 4)          \
    X(16, 2, 4, RED, true, OP, 4)         \
    X(16, 2, 4, RED, true, OP, 6)         \
    X(16, 2, 4, RED, true, OP, 8)         \
    X(16, 2, 8, RED, true, OP, 4)         \
    X(16, 2, 8, RED, true, OP, 6)         \
    X(32, 1, 4, RED, true, OP, 6)         \
    X(32, 1, 4, RED, true, OP, 8)         \
    X(32, 1, 8, RED, true, OP, 4)         \
    X(32, 1, 8, RED, true, OP, 5)         \
    X(32, 1, 8, RED, true, OP, 6)         \
    X(16, 1, 8, RED, true, OP, 5)         \
    X(16, 1, 8, RED, true, OP, 6)         \
    X(16, 1, 4, RED, true, OP, 6)         \
    X(8, 1, 8, RED, true, OP, 5)          \
    X(8, 1, 8, RED, true, OP, 6)          \
    X(32, 2, 4, RED, true, OP, 5)         \
    X(32, 2, 4, RED, true, OP, 4)         \
    X(32, 2, 4, RED, true, OP, 6)         \
    X(16, 4, 2, RED, true, OP, 6)         \
    X(16, 4, 4, RED, true, OP, 4)         \
    X(32, 4, 2, RED, true, OP, 4)         \
    X(32, 4, 4, RED, true, OP, 4)

#define SGNN_NO_OCC_CONFIGS(X, RED, OP)

// FusedMM needs all of K in registers (the dot); a smaller set suffices.
#define SGNN_FUSED_CONFIGS(X, RED, OP) \
    X(16, 1, 8, RED, true, OP, 5)      \
    X(8, 1, 8, RED, true, OP, 5)       \
    X(32, 1, 8, RED, true, OP, 5)      \
    X(4, 1, 8, RED, true, OP, 1)       \
    X(4, 2, 8, RED, true, OP, 1)       \
    X(4, 4, 4, RED, true, OP, 1)       \
    X(8, 2, 4, RED, true, OP, 1)       \
    X(8, 4, 4, RED, true, OP, 1)       \
    X(16, 2, 4, RED, true, OP, 1)      \
    X(8, 1, 8, RED, true, OP, 1)       \
    X(16, 1, 8, RED, true, OP, 1)      \
    X(32, 1, 4, RED, true, OP, 1)      \
    X(32, 1, 8, RED, true, OP, 1)      \
    X(8, 2, 8, RED, true, OP, 1)       \
    X(16, 2, 8, RED, true, OP, 1)      \
    X(32, 2, 4, RED, true, OP, 1)      \
    X(32, 4, 4, RED, true, OP, 1)      \
    X(32, 8, 2, RED, true, OP, 1)      \
    X(32, 1, 4, RED, false, OP, 1)     \
    X(32, 2, 4, RED, false, OP, 1)     \
    X(32, 4, 2, RED, false, OP, 1)     \
    X(32, 8, 2, RED, false, OP, 1)

#define SGNN_WORKER_CASE(G, V, U, RED, VEC, OP, MINB)                                      \
    if (vec == VEC && lanes == G && vregs == V && unroll == U && occ == MINB)              \
        return &launch_spmm_worker<G, V, U, RED, VEC, OP, MINB>;

#define SGNN_DEFINE_SPMM_LOOKUP(NAME, RED, OCCS)                                      \
    SpmmLauncher NAME(bool vec, int lanes, int vregs, int unroll, int occ) {         \
        if (occ == 0) occ = 1;                                                        \
        SGNN_SPMM_CONFIGS(SGNN_WORKER_CASE, RED, dev::OP_SPMM)                        \
        OCCS(SGNN_WORKER_CASE, RED, dev::OP_SPMM)                                     \
        return nullptr;                                                               \
    }                                                                                 \
    sgnn_status NAME##_fixup(const FixupArgs& f, cudaStream_t s) {                    \
        if (f.n_fix == 0 || f.width == 0) return SGNN_OK;                             \
        DeviceProps dp;                                                               \
        SGNN_TRY(device_props(&dp));                                                  \
        const bool v4 = f.width % 4 == 0 && f.ldc % 4 == 0 && f.ld_slot % 4 == 0 &&    \
                        reinterpret_cast<uintptr_t>(f.c) % 16 == 0 &&                 \
                        reinterpret_cast<uintptr_t>(f.slots) % 16 == 0;               \
        if (v4) {                                                                     \
            const uint64_t items = uint64_t(f.n_fix) * ((f.width + 127) / 128);        \
            const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(items * 32, 256), \
                                                       uint64_t(dp.sm_count) * 8);    \
            dev::spmm_fixup_vec_kernel<RED><<<unsigned(blocks), 256, 0, s>>>(f);      \
            SGNN_LAUNCH_CHECK();                                                      \
            if (f.fix_long && f.n_long) {                                             \
                dev::spmm_fixup_long_kernel<RED><<<f.n_long, dev::kFixupLongThreads, 0, s>>>(f); \
                SGNN_LAUNCH_CHECK();                                                  \
            }                                                                         \
            return SGNN_OK;                                                           \
        }                                                                             \
        const uint64_t total = uint64_t(f.n_fix) * f.width;                           \
        const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(total, 256),          \
                                                   uint64_t(dp.sm_count) * 8);        \
        dev::spmm_fixup_kernel<RED><<<unsigned(blocks), 256, 0, s>>>(f);              \
        SGNN_LAUNCH_CHECK();                                                          \
        return SGNN_OK;                                                               \
    }

// Peer-partitioned SpMM (OP_SPMM_PEER): the default layouts per K, sum (and mean).
#define SGNN_PEER_CONFIGS(X, RED, OP) \
    X(4, 1, 8, RED, true, OP, 1)      \
    X(8, 1, 8, RED, true, OP, 4)      \
    X(16, 1, 8, RED, true, OP, 4)     \
    X(32, 1, 8, RED, true, OP, 4)     \
    X(32, 2, 4, RED, true, OP, 4)     \
    X(32, 4, 4, RED, true, OP, 1)     \
    X(32, 1, 4, RED, false, OP, 1)    \
    X(32, 2, 4, RED, false, OP, 1)    \
    X(32, 4, 2, RED, false, OP, 1)    \
    X(32, 8, 2, RED, false, OP, 1)

#define SGNN_DEFINE_PEER_LOOKUP(NAME, RED)                                            \
    SpmmLauncher NAME(bool vec, int lanes, int vregs, int unroll, int occ) {         \
        if (occ == 0) occ = 1;                                                        \
        SGNN_PEER_CONFIGS(SGNN_WORKER_CASE, RED, dev::OP_SPMM_PEER)                   \
        return nullptr;                                                               \
    }

#define SGNN_DEFINE_FUSED_LOOKUP(NAME, RED, OP)                                       \
    SpmmLauncher NAME(bool vec, int lanes, int vregs, int unroll, int occ) {         \
        if (occ == 0) occ = 1;                                                        \
        SGNN_FUSED_CONFIGS(SGNN_WORKER_CASE, RED, OP)                                 \
        return nullptr;                                                               \
    }

// Mean has kernels of its own (the divide in the row epilogue); layouts
// without one run the Sum kernels plus run_mean_divide (spmm.cu).
SpmmLauncher spmm_lookup_sum(bool, int, int, int, int);
SpmmLauncher spmm_lookup_mean(bool, int, int, int, int);
sgnn_status spmm_lookup_mean_fixup(const FixupArgs&, cudaStream_t);
SpmmLauncher spmm_peer_lookup_sum(bool, int, int, int, int);
SpmmLauncher spmm_lookup_min(bool, int, int, int, int);
SpmmLauncher spmm_lookup_max(bool, int, int, int, int);
sgnn_status spmm_lookup_sum_fixup(const FixupArgs&, cudaStream_t);
sgnn_status spmm_lookup_min_fixup(const FixupArgs&, cudaStream_t);
sgnn_status spmm_lookup_max_fixup(const FixupArgs&, cudaStream_t);
SpmmLauncher fused_lookup_mul_sum(bool, int, int, int, int);
SpmmLauncher fused_lookup_mul_min(bool, int, int, int, int);
SpmmLauncher fused_lookup_mul_max(bool, int, int, int, int);
SpmmLauncher fused_lookup_sig_sum(bool, int, int, int, int);
SpmmLauncher fused_lookup_sig_min(bool, int, int, int, int);
SpmmLauncher fused_lookup_sig_max(bool, int, int, int, int);

}  // namespace sgnn
