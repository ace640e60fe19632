// spmm_inst.cuh -- instantiates the worker kernels (SpMM, and FusedMM for each
// edge op) for one reduction and exposes them through lookup functions.
// Included once per (reduction, mode) file so the variants compile in parallel.
#pragma once

#include <algorithm>

#include "spmm_kernel.cuh"

namespace sgnn {

template <int G, int V, int U, int RED, bool VEC, int OP>
sgnn_status launch_spmm_worker(const SpmmArgs& a, uint32_t block, uint32_t max_blocks,
                               cudaStream_t s) {
    static int per_sm[3] = {-1, -1, -1};  // for block = 64, 128, 256
    const int bi = block <= 64 ? 0 : block <= 128 ? 1 : 2;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    if (per_sm[bi] < 0) {
        int n = 0;
        SGNN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &n, dev::spmm_worker_kernel<G, V, U, RED, VEC, OP>, int(block), 0));
        per_sm[bi] = std::max(n, 1);
    }
    const uint64_t want = ceil_div_u64(uint64_t(a.n_workers) * G, block);
    uint64_t blocks = std::min<uint64_t>(want, uint64_t(dp.sm_count) * per_sm[bi]);
    if (max_blocks) blocks = std::min<uint64_t>(blocks, max_blocks);
    if (blocks == 0) return SGNN_OK;
    dev::spmm_worker_kernel<G, V, U, RED, VEC, OP><<<unsigned(blocks), block, 0, s>>>(a);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

// (lanes, vec, unroll, float4?) combinations compiled for SpMM.
#define SGNN_SPMM_CONFIGS(X, RED, OP) \
    X(4, 1, 4, RED, true, OP)         \
    X(4, 1, 8, RED, true, OP)         \
    X(4, 2, 8, RED, true, OP)         \
    X(8, 4, 4, RED, true, OP)         \
    X(8, 1, 4, RED, true, OP)         \
    X(8, 1, 8, RED, true, OP)         \
    X(16, 1, 4, RED, true, OP)        \
    X(16, 1, 8, RED, true, OP)        \
    X(32, 1, 4, RED, true, OP)        \
    X(32, 1, 8, RED, true, OP)        \
    X(8, 2, 4, RED, true, OP)         \
    X(8, 2, 8, RED, true, OP)         \
    X(16, 2, 4, RED, true, OP)        \
    X(16, 2, 8, RED, true, OP)        \
    X(32, 2, 4, RED, true, OP)        \
    X(32, 2, 8, RED, true, OP)        \
    X(16, 4, 2, RED, true, OP)        \
    X(16, 4, 4, RED, true, OP)        \
    X(32, 4, 2, RED, true, OP)        \
    X(32, 4, 4, RED, true, OP)        \
    X(32, 8, 2, RED, true, OP)        \
    X(32, 1, 4, RED, false, OP)       \
    X(32, 1, 8, RED, false, OP)       \
    X(32, 2, 4, RED, false, OP)       \
    X(32, 2, 8, RED, false, OP)       \
    X(32, 4, 2, RED, false, OP)       \
    X(32, 4, 4, RED, false, OP)       \
    X(32, 8, 2, RED, false, OP)       \
    X(32, 8, 4, RED, false, OP)

// FusedMM needs all of K in registers (the dot); a smaller set suffices.
#define SGNN_FUSED_CONFIGS(X, RED, OP) \
    X(4, 1, 8, RED, true, OP)          \
    X(8, 1, 8, RED, true, OP)          \
    X(16, 1, 8, RED, true, OP)         \
    X(32, 1, 4, RED, true, OP)         \
    X(32, 1, 8, RED, true, OP)         \
    X(8, 2, 8, RED, true, OP)          \
    X(16, 2, 8, RED, true, OP)         \
    X(32, 2, 4, RED, true, OP)         \
    X(32, 4, 4, RED, true, OP)         \
    X(32, 8, 2, RED, true, OP)         \
    X(32, 1, 4, RED, false, OP)        \
    X(32, 2, 4, RED, false, OP)        \
    X(32, 4, 2, RED, false, OP)        \
    X(32, 8, 2, RED, false, OP)

#define SGNN_WORKER_CASE(G, V, U, RED, VEC, OP) \
    if (vec == VEC && lanes == G && vregs == V && unroll == U) return &launch_spmm_worker<G, V, U, RED, VEC, OP>;

#define SGNN_DEFINE_SPMM_LOOKUP(NAME, RED)                                            \
    SpmmLauncher NAME(bool vec, int lanes, int vregs, int unroll) {                  \
        SGNN_SPMM_CONFIGS(SGNN_WORKER_CASE, RED, dev::OP_SPMM)                        \
        return nullptr;                                                               \
    }                                                                                 \
    sgnn_status NAME##_fixup(const FixupArgs& f, cudaStream_t s) {                    \
        if (f.n_fix == 0 || f.width == 0) return SGNN_OK;                             \
        DeviceProps dp;                                                               \
        SGNN_TRY(device_props(&dp));                                                  \
        const uint64_t total = uint64_t(f.n_fix) * f.width;                           \
        const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(total, 256),          \
                                                   uint64_t(dp.sm_count) * 8);        \
        dev::spmm_fixup_kernel<RED><<<unsigned(blocks), 256, 0, s>>>(f);              \
        SGNN_LAUNCH_CHECK();                                                          \
        return SGNN_OK;                                                               \
    }

#define SGNN_DEFINE_FUSED_LOOKUP(NAME, RED, OP)                                       \
    SpmmLauncher NAME(bool vec, int lanes, int vregs, int unroll) {                  \
        SGNN_FUSED_CONFIGS(SGNN_WORKER_CASE, RED, OP)                                 \
        return nullptr;                                                               \
    }

SpmmLauncher spmm_lookup_sum(bool, int, int, int);
SpmmLauncher spmm_lookup_mean(bool, int, int, int);
SpmmLauncher spmm_lookup_min(bool, int, int, int);
SpmmLauncher spmm_lookup_max(bool, int, int, int);
sgnn_status spmm_lookup_sum_fixup(const FixupArgs&, cudaStream_t);
sgnn_status spmm_lookup_mean_fixup(const FixupArgs&, cudaStream_t);
sgnn_status spmm_lookup_min_fixup(const FixupArgs&, cudaStream_t);
sgnn_status spmm_lookup_max_fixup(const FixupArgs&, cudaStream_t);
SpmmLauncher fused_lookup_mul_sum(bool, int, int, int);
SpmmLauncher fused_lookup_mul_mean(bool, int, int, int);
SpmmLauncher fused_lookup_mul_min(bool, int, int, int);
SpmmLauncher fused_lookup_mul_max(bool, int, int, int);
SpmmLauncher fused_lookup_sig_sum(bool, int, int, int);
SpmmLauncher fused_lookup_sig_mean(bool, int, int, int);
SpmmLauncher fused_lookup_sig_min(bool, int, int, int);
SpmmLauncher fused_lookup_sig_max(bool, int, int, int);

}  // namespace sgnn
