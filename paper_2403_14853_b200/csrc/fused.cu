// fused.cu -- SDDMM (kernels.hpp:187-210) and FusedMM (kernels.hpp:216-270).
//
// SDDMM: each output is independent, so workers take equal nnz ranges
// (no row snapping, no fixup).  A group holds X_i (re-loaded on row change)
// and, per nonzero, gathers Y_j, forms the canonical group dot product
// (group_dot) and writes p_e * dot.  Results are collected in the lane that
// loaded the nonzero so the stores are coalesced.
//
// FusedMM: the SpMM worker kernel in fused mode (spmm_kernel.cuh): per edge
// Y_j is gathered once and used for both the dot and the accumulation
// (the reference reads it twice, kernels.hpp:238,244), with the plan's
// nnz-balanced split, canonical segments and fixup for hub rows.
#include <algorithm>
#include <cstdlib>

#include "ops.cuh"
#include "plan.cuh"
#include "spmm_inst.cuh"

#ifndef SGNN_SDDMM_U16
#define SGNN_SDDMM_U16 8  // gathers in flight per group of the K=64 SDDMM
#endif
#ifndef SGNN_SDDMM_MINB
#define SGNN_SDDMM_MINB 7  // register cap for the K=64 SDDMM (cfg4 probe: 7 best of {1, 6, 7, 8})
#endif

namespace sgnn {

// fused_tma.cu: the TMA-gather (warp-specialised) kernels for K = 64 / 128
sgnn_status run_fused_tma(const sgnn_csr* p, const float* x, const float* y, uint32_t k, int op, int reduce,
                          float* out, const sgnn_plan_s* plan, cudaStream_t s, bool* ran);
int tma_op_sddmm();

namespace {

struct SddmmArgs {
    const uint64_t* __restrict__ rp;
    const uint32_t* __restrict__ ci;
    const float* __restrict__ val;
    const float* __restrict__ x;
    const float* __restrict__ y;
    float* __restrict__ out;
    uint64_t nnz;
    uint64_t per_worker;
    const uint32_t* __restrict__ wrow;  // optional plan split (row of each worker start)
    const uint64_t* __restrict__ wnz;
    uint32_t n_rows;
    uint32_t n_workers;
    uint32_t k;
    uint64_t ld;
    uint32_t* wctr;  // dynamic worker schedule (plan_counter), null: static
};

__device__ __forceinline__ uint32_t row_of(const uint64_t* __restrict__ rp, uint32_t m, uint64_t e) {
    uint32_t lo = 0, hi = m;  // largest r with rp[r] <= e
    while (hi - lo > 1) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (__ldg(rp + mid) <= e) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Same hot-loop shape as the SpMM worker: 32-bit worker-local positions,
// (col, val) of the next batch prefetched, one IMAD per gather address, and
// the U dot products of a batch formed together when the batch stays in one
// row (independent shuffle trees interleave).
template <int G, int V, int U, bool VEC, int MINB = 1>
__global__ void __launch_bounds__(128, MINB) sddmm_kernel(const SddmmArgs a) {
    using F = dev::Frag<G, V, VEC>;
    constexpr int CH = (U + G - 1) / G;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const int gl_eff = min(gl, int(a.k / F::W) - 1);
    const char* ylane = reinterpret_cast<const char*>(a.y + F::W * gl_eff);
    const uint32_t ldb = uint32_t(a.ld) * 4u;
    const int nq = F::blocks_in(gl, a.k);
    const bool full = a.k == uint32_t(F::W * G * V);
    // LOCK (groups narrower than a warp): the groups of a warp step through
    // their batches together so the batch-body shuffles use the full warp mask
    // (see spmm_worker_kernel); batches are cut at row ends, so every batch's
    // U dots share one X_i.
    constexpr bool LOCK = G < 32;
    constexpr unsigned FULL = 0xffffffffu;
    dev::WarpSched<32 / G> ws(a.wctr);
    for (uint32_t w = ws.base + uint32_t(lane / G); LOCK ? __any_sync(FULL, w < a.n_workers) : (w < a.n_workers);
         ws.next(), w = ws.base + uint32_t(lane / G)) {
        const bool wact = w < a.n_workers;
        const uint32_t wq = wact ? w : a.n_workers - 1;
        // a plan's split (no search) or an even nnz split (binary search)
        const uint64_t j0 = a.wnz ? __ldg(a.wnz + wq) : uint64_t(wq) * a.per_worker;
        const uint32_t E = !wact ? 0u
                           : a.wnz ? uint32_t(__ldg(a.wnz + wq + 1) - j0)
                                   : uint32_t(min(a.per_worker, a.nnz - j0));
        uint32_t r = a.wrow ? __ldg(a.wrow + wq) : row_of(a.rp, a.n_rows, j0);
        uint32_t rb = r;
        uint64_t rwin = __ldg(a.rp + min(rb + 1 + uint32_t(gl), a.n_rows));
        uint32_t rend_l = uint32_t(min(dev::shfl_u64(gmask, rwin, 0, G), j0 + E) - j0);
        F xrow;
        xrow.load(a.x + uint64_t(r) * a.ld, gl, a.k);  // zero-filled past K
        uint32_t cc[CH];
        float vv[CH];
        auto load_cv = [&](uint32_t base) {
#pragma unroll
            for (int h = 0; h < CH; ++h) {
                const uint32_t lq = base + uint32_t(gl + G * h);
                const bool ok = (gl + G * h) < U && lq < E;
                cc[h] = ok ? dev::ld_stream(a.ci + j0 + lq) : 0u;
                vv[h] = ok ? dev::ld_stream(a.val + j0 + lq) : 0.0f;
            }
        };
        auto next_row = [&](uint32_t l) {  // advance to the row holding local position l
            do {
                ++r;
                if (r - rb >= uint32_t(G)) {
                    rb = r;
                    rwin = __ldg(a.rp + min(rb + 1 + uint32_t(gl), a.n_rows));
                }
                rend_l = uint32_t(min(dev::shfl_u64(gmask, rwin, int(r - rb), G), j0 + E) - j0);
            } while (l >= rend_l);
            xrow.load(a.x + uint64_t(r) * a.ld, gl, a.k);
        };
        if (E) load_cv(0);
        const uint64_t l2pol = dev::gather_policy();
        if constexpr (LOCK) {
            uint32_t base = 0;
            while (__any_sync(FULL, base < E)) {
                const bool act = base < E;
                int n = 0;
                if (act) {
                    if (base >= rend_l) next_row(base);
                    const uint32_t room = rend_l - base;
                    n = room < uint32_t(U) ? int(room) : U;
                }
                F yf[U];
                float pv[U];
                uint32_t colu[U];
                // with the transpose-reduce a lane needs only the value of the
                // nonzero it owns (taken before load_cv overwrites vv)
                constexpr bool ALL_VALS = U > G;
                float pv_own = 0.0f;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    colu[u] = __shfl_sync(FULL, cc[u / G], u % G, G);
                    if constexpr (ALL_VALS) pv[u] = __shfl_sync(FULL, vv[u / G], u % G, G);
                }
                if constexpr (!ALL_VALS) pv_own = __shfl_sync(FULL, vv[0], gl / (G / U), G);
                if (act) {
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        yf[u].template gather<false>(
                            reinterpret_cast<const float*>(ylane + uint64_t(colu[u]) * ldb), nq, l2pol);
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) yf[u].zero();
                }
                const uint32_t nb = base + uint32_t(n);
                if (act && nb < E) load_cv(nb);
                float res[CH];
#pragma unroll
                for (int h = 0; h < CH; ++h) res[h] = 0.0f;
                if constexpr (U <= G) {
                    constexpr int PER = G / U;
                    const float r_own = __fmul_rn(pv_own, dev::batch_dots(xrow, yf, FULL, gl, nq));  // kernels.hpp:206
                    res[0] = __shfl_sync(FULL, r_own, (gl * PER) & (G - 1), G);
                } else {
                    float d[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) d[u] = dev::group_dot(xrow, yf[u], FULL, nq);
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (gl == u % G) res[u / G] = __fmul_rn(pv[u], d[u]);  // kernels.hpp:206
                }
#pragma unroll
                for (int h = 0; h < CH; ++h) {
                    const int q = gl + G * h;
                    if (q < n) __stcs(a.out + j0 + base + uint32_t(q), res[h]);
                }
                base = nb;
            }
        } else {
            for (uint32_t base = 0; base < E; base += U) {
                const int n = (E - base) < uint32_t(U) ? int(E - base) : U;
                F yf[U];
                float pv[U];
    #pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t col = __shfl_sync(gmask, cc[u / G], u % G, G);
                    pv[u] = __shfl_sync(gmask, vv[u / G], u % G, G);
                    const float* lrow = reinterpret_cast<const float*>(ylane + uint64_t(col) * ldb);
                    if (full) yf[u].template gather<false>(lrow, nq, l2pol);
                    else yf[u].template gather<true>(lrow, nq, l2pol);
                }
                if (base + U < E) load_cv(base + U);
                float res[CH];
    #pragma unroll
                for (int h = 0; h < CH; ++h) res[h] = 0.0f;
                if (base >= rend_l) next_row(base);
                if (base + uint32_t(n) <= rend_l) {
                    if constexpr (U <= G) {
                        // transpose-reduce: lane gl owns nonzero gl/(G/U); lane u stores nonzero u
                        constexpr int PER = G / U;
                        const int u_own = gl / PER;
                        float pv_own = pv[0];
    #pragma unroll
                        for (int u = 1; u < U; ++u)
                            if (u == u_own) pv_own = pv[u];
                        const float r_own = __fmul_rn(pv_own, dev::batch_dots(xrow, yf, gmask, gl));  // kernels.hpp:206
                        res[0] = __shfl_sync(gmask, r_own, (gl * PER) & (G - 1), G);
                    } else {
                        float d[U];
    #pragma unroll
                        for (int u = 0; u < U; ++u) d[u] = dev::group_dot(xrow, yf[u], gmask);
    #pragma unroll
                        for (int u = 0; u < U; ++u)
                            if (gl == u % G) res[u / G] = __fmul_rn(pv[u], d[u]);  // kernels.hpp:206
                    }
                } else {
    #pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (u >= n) break;
                        if (base + uint32_t(u) >= rend_l) next_row(base + uint32_t(u));
                        const float d = dev::group_dot(xrow, yf[u], gmask);
                        if (gl == u % G) res[u / G] = __fmul_rn(pv[u], d);
                    }
                }
    #pragma unroll
                for (int h = 0; h < CH; ++h) {
                    const uint32_t lq = base + uint32_t(gl + G * h);
                    if ((gl + G * h) < U && lq < E) __stcs(a.out + j0 + lq, res[h]);
                }
            }
        }
    }
    ws.finish();
}

// Full-width float4 SDDMM for K = 4 G (one float4 of every row per lane,
// G < 32 lanes per nonzero, 32 / G groups per warp in lockstep): the same
// work split, batches and dot tree as sddmm_kernel's LOCK path -- so bitwise
// the same results -- with the per-batch overhead cut, since these shapes are
// bound by instruction issue, not by memory (profiles/r02_cfg4_k64_probes):
// (col, val) arrive in G-wide windows (one load per lane per G nonzeros, the
// next window prefetched when the next batch would leave this one), a gather
// address is one mad.wide, no lane masking of the dot (every lane's float4 is
// inside K), idle groups gather nothing, and the row advance is warp-uniform
// and skips up to G rows per step with one ballot over the row-end window.
template <int G, int U, int MINB>
__global__ void __launch_bounds__(128, MINB) sddmm_lock_kernel(const SddmmArgs a) {
    static_assert(G < 32 && U <= G, "lockstep groups, one owned dot per lane");
    using F = dev::Frag<G, 1, true>;
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int PER = G / U;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1), gbase = lane & ~(G - 1);
    const unsigned gbits = (G == 32) ? FULL : ((1u << G) - 1u);
    const char* ylane = reinterpret_cast<const char*>(a.y + 4 * gl);
    const uint32_t ldb = uint32_t(a.ld) * 4u;
    const uint64_t l2pol = dev::gather_policy();
    dev::WarpSched<32 / G> ws(a.wctr);
    for (uint32_t w = ws.base + uint32_t(lane / G); __any_sync(FULL, w < a.n_workers);
         ws.next(), w = ws.base + uint32_t(lane / G)) {
        const bool wact = w < a.n_workers;
        const uint32_t wq = wact ? w : a.n_workers - 1;
        const uint64_t j0 = a.wnz ? __ldg(a.wnz + wq) : uint64_t(wq) * a.per_worker;
        const uint32_t E = !wact ? 0u
                           : a.wnz ? uint32_t(__ldg(a.wnz + wq + 1) - j0)
                                   : uint32_t(min(a.per_worker, a.nnz - j0));
        uint32_t r = a.wrow ? __ldg(a.wrow + wq) : row_of(a.rp, a.n_rows, j0);
        // lane gl of the window: worker-local end of row rb + gl (clamped to E)
        auto window = [&](uint32_t rb_) -> uint32_t {
            const uint64_t e = __ldg(a.rp + min(rb_ + 1 + uint32_t(gl), a.n_rows));
            return uint32_t(min(e - j0, uint64_t(E)));
        };
        uint32_t rb = r;
        uint32_t rwin = window(rb);
        // X rows are read once each (a DRAM miss at every row start): the
        // window's later non-empty rows go to L2 when the window is loaded
        auto prefetch_x = [&](bool mine) {  // every lane calls it; the groups in `mine` prefetch
            const uint32_t prev = __shfl_up_sync(FULL, rwin, 1, G);
            if (mine && gl >= 1 && rwin > prev && rb + uint32_t(gl) < a.n_rows) {
                const char* xp = reinterpret_cast<const char*>(a.x + uint64_t(rb + uint32_t(gl)) * a.ld);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(xp));
                if (a.k > 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(xp + 128));
            }
        };
        prefetch_x(wact);
        uint32_t rend_l = __shfl_sync(FULL, rwin, gbase);
        F xrow;
        xrow.load(a.x + uint64_t(r) * a.ld, gl, a.k);
        // (col, val) window: lane gl holds nonzero wb + gl
        uint32_t wb = 0, cw = 0;
        float vw = 0.0f;
        auto load_window = [&](uint32_t at) {
            wb = at;
            const bool ok = at + uint32_t(gl) < E;
            cw = ok ? dev::ld_stream(a.ci + j0 + at + gl) : 0u;  // 0: a safe dummy row
            vw = ok ? dev::ld_stream(a.val + j0 + at + gl) : 0.0f;
        };
        if (E) load_window(0);
        uint32_t base = 0;
        while (__any_sync(FULL, base < E)) {
            const bool act = base < E;
            // row advance: the first row of the window ending after `base`
            // (rows before it end at or before base), else the next window
            while (true) {
                const bool need = act && base >= rend_l;
                if (!__any_sync(FULL, need)) break;
                const unsigned later = (__ballot_sync(FULL, rwin > base) >> gbase) & gbits;
                const bool found = need && later != 0u;
                if (found) r = rb + uint32_t(__ffs(later) - 1);
                if (need && !found) {
                    rb += G;
                    rwin = window(rb);
                }
                if (__any_sync(FULL, need && !found)) prefetch_x(need && !found);
                const uint32_t t = __shfl_sync(FULL, rwin, gbase + int(r - rb) * int(found));
                if (found) {
                    rend_l = t;
                    xrow.load(a.x + uint64_t(r) * a.ld, gl, a.k);
                }
            }
            int n = 0;
            if (act) {
                const uint32_t room = rend_l - base;
                n = room < uint32_t(U) ? int(room) : U;
            }
            // an active group's batch lies inside the window (base - wb <= G - U);
            // an idle group's shuffles read anything and gather nothing
            const int s0 = gbase + int(base - wb);
            uint32_t colu[U];
#pragma unroll
            for (int u = 0; u < U; ++u) colu[u] = __shfl_sync(FULL, cw, s0 + u);
            const float pv_own = __shfl_sync(FULL, vw, s0 + gl / PER);
            F yf[U];
            if (act) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const char* p;
                    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(colu[u]), "r"(ldb), "l"(ylane));
                    const float4 t = dev::ld_gather(reinterpret_cast<const float4*>(p), l2pol);
                    yf[u].v[0] = t.x; yf[u].v[1] = t.y; yf[u].v[2] = t.z; yf[u].v[3] = t.w;
                }
            }
            const uint32_t nb = base + uint32_t(n);
            if (act && nb < E && nb + uint32_t(U) > wb + uint32_t(G)) load_window(nb);
            const float r_own = __fmul_rn(pv_own, dev::batch_dots(xrow, yf, FULL, gl));  // kernels.hpp:206
            const float res = __shfl_sync(FULL, r_own, gbase + ((gl * PER) & (G - 1)));
            if (gl < n) __stcs(a.out + j0 + base + uint32_t(gl), res);
            base = nb;
        }
    }
    ws.finish();
}

template <int G, int U, int MINB>
sgnn_status launch_sddmm_lock(const SddmmArgs& a, cudaStream_t s) {
    static int per_sm = -1;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    if (per_sm < 0) {
        int n = 0;
        SGNN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sddmm_lock_kernel<G, U, MINB>, 128, 0));
        per_sm = std::max(n, 1);
    }
    const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(uint64_t(a.n_workers) * G, 128),
                                               uint64_t(dp.sm_count) * per_sm);
    if (blocks == 0) return SGNN_OK;
    sddmm_lock_kernel<G, U, MINB><<<unsigned(blocks), 128, 0, s>>>(a);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

using SddmmLaunch = sgnn_status (*)(const SddmmArgs&, cudaStream_t);

template <int G, int V, int U, bool VEC, int MINB = 1>
sgnn_status launch_sddmm(const SddmmArgs& a, cudaStream_t s) {
    static int per_sm = -1;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    if (per_sm < 0) {
        int n = 0;
        SGNN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sddmm_kernel<G, V, U, VEC, MINB>, 128, 0));
        per_sm = std::max(n, 1);
    }
    const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(uint64_t(a.n_workers) * G, 128),
                                               uint64_t(dp.sm_count) * per_sm);
    if (blocks == 0) return SGNN_OK;
    sddmm_kernel<G, V, U, VEC, MINB><<<unsigned(blocks), 128, 0, s>>>(a);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

// (lanes, float4-or-float registers) covering K in one pass.
bool full_k_layout(uint32_t k, bool vec, int* lanes, int* vregs) {
    if (vec) {
        if (k <= 16) { *lanes = 4; *vregs = 1; }
        else if (k <= 32) { *lanes = 8; *vregs = 1; }
        else if (k <= 64) { *lanes = 16; *vregs = 1; }
        else if (k <= 128) { *lanes = 32; *vregs = 1; }
        else if (k <= 256) { *lanes = 32; *vregs = 2; }
        else if (k <= 512) { *lanes = 32; *vregs = 4; }
        else if (k <= 1024) { *lanes = 32; *vregs = 8; }
        else return false;
    } else {
        *lanes = 32;
        if (k <= 32) *vregs = 1;
        else if (k <= 64) *vregs = 2;
        else if (k <= 128) *vregs = 4;
        else if (k <= 256) *vregs = 8;
        else return false;
    }
    return true;
}

// Unroll of the compiled FusedMM configuration for a full-K layout
// (SGNN_FUSED_CONFIGS in spmm_inst.cuh).
int fused_unroll(bool vec, int lanes, int vregs) {
    if (vec) return (lanes < 32 || vregs == 1) ? 8 : (vregs == 8 ? 2 : 4);
    return vregs >= 4 ? 2 : 4;
}

SpmmLauncher find_fused_launcher_occ(bool vec, int lanes, int vregs, int unroll, int edge, int reduce,
                                     int occ) {
    const bool sig = edge == SGNN_EDGE_SIGMOID_MUL;
    switch (reduce) {
        case SGNN_REDUCE_SUM:
        case SGNN_REDUCE_MEAN:  // sum kernels + the divide pass (run_mean_divide)
            return sig ? fused_lookup_sig_sum(vec, lanes, vregs, unroll, occ) : fused_lookup_mul_sum(vec, lanes, vregs, unroll, occ);
        case SGNN_REDUCE_MIN:
            return sig ? fused_lookup_sig_min(vec, lanes, vregs, unroll, occ) : fused_lookup_mul_min(vec, lanes, vregs, unroll, occ);
        case SGNN_REDUCE_MAX:
            return sig ? fused_lookup_sig_max(vec, lanes, vregs, unroll, occ) : fused_lookup_mul_max(vec, lanes, vregs, unroll, occ);
    }
    return nullptr;
}

// Prefers the register-capped (5 CTAs/SM) variant when one is compiled.
// the full-width lockstep FusedMM (dev::fused_lock_kernel), K = 64, Sum / Mean
template <int OP, int MINB>
sgnn_status launch_fused_lock(const SpmmArgs& a, cudaStream_t s) {
    static int per_sm = -1;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    if (per_sm < 0) {
        int n = 0;
        SGNN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, dev::lock_worker_kernel<16, 8, OP, SGNN_REDUCE_SUM, MINB>, 128, 0));
        per_sm = std::max(n, 1);
    }
    const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(uint64_t(a.n_workers) * 16, 128), uint64_t(dp.sm_count) * per_sm);
    if (blocks == 0) return SGNN_OK;
    dev::lock_worker_kernel<16, 8, OP, SGNN_REDUCE_SUM, MINB><<<unsigned(blocks), 128, 0, s>>>(a);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

// the lockstep FusedMM with its gathered rows in a shared-memory ring of NCH
// chunks (cp.async, spmm_kernel.cuh): the ring sets the CTAs per SM
template <int OP, int NCH, int MINB = (NCH >= 4 ? 3 : NCH == 3 ? 4 : 5)>
sgnn_status launch_fused_ring(const SpmmArgs& a, cudaStream_t s) {
    auto kern = dev::lock_worker_kernel<16, 8, OP, SGNN_REDUCE_SUM, MINB, NCH>;
    constexpr uint32_t smem = dev::ring_smem_bytes<NCH>();
    static int per_sm = -1;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    if (per_sm < 0) {
        SGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        int n = 0;
        SGNN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, 128, smem));
        per_sm = std::max(n, 1);
    }
    const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(uint64_t(a.n_workers) * 16, 128), uint64_t(dp.sm_count) * per_sm);
    if (blocks == 0) return SGNN_OK;
    kern<<<unsigned(blocks), 128, smem, s>>>(a);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

SpmmLauncher find_fused_launcher(bool vec, int lanes, int vregs, int unroll, int edge, int reduce) {
    SpmmLauncher l = find_fused_launcher_occ(vec, lanes, vregs, unroll, edge, reduce, 5);
    return l ? l : find_fused_launcher_occ(vec, lanes, vregs, unroll, edge, reduce, 1);
}

}  // namespace

sgnn_status run_sddmm(const sgnn_csr* p, const float* x, const float* y, uint32_t k, float* out,
                      const sgnn_plan_s* plan, cudaStream_t s) {
    if (p->nnz == 0) return SGNN_OK;
    if (plan && !plan_matches(plan, p, plan->k))
        return fail(SGNN_ERR_DISPATCH, "sddmm: plan was built for another matrix");
    const bool vec = (k % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(y) % 16 == 0);
    int lanes, vregs;
    if (!full_k_layout(k, vec, &lanes, &vregs))
        return fail(SGNN_ERR_UNSUPPORTED, "sddmm: K=" + std::to_string(k) +
                                              " exceeds the register-resident width of this build");
    SddmmArgs a;
    a.rp = p->row_ptr;
    a.ci = p->col_idx;
    a.val = p->values;
    a.x = x;
    a.y = y;
    a.out = out;
    a.nnz = p->nnz;
    a.n_rows = p->n_rows;
    a.k = k;
    a.ld = k;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    // ~4 workers per resident group, at least 64 nonzeros each
    const uint64_t groups = uint64_t(dp.sm_count) * 2048 / lanes;
    a.per_worker = std::max<uint64_t>(64, ceil_div_u64(p->nnz, 4 * groups));
    a.n_workers = uint32_t(ceil_div_u64(p->nnz, a.per_worker));
    a.wrow = nullptr;
    a.wnz = nullptr;
    a.wctr = nullptr;
    if (plan) {  // reuse the plan's nnz-balanced split: worker starts need no row search
        if (vec && p->n_cols) {
            bool ran = false;
            SGNN_TRY(run_fused_tma(p, x, y, k, tma_op_sddmm(), SGNN_REDUCE_SUM, out, plan, s, &ran));
            if (ran) return SGNN_OK;
        }
        a.wrow = plan->wrow;
        a.wnz = plan->wnz;
        a.n_workers = plan->n_workers;
        a.wctr = plan_counter(plan, s);
    }
    SddmmLaunch fn = nullptr;
    const bool generic = std::getenv("SGNN_SDDMM_GENERIC") != nullptr;  // A/B switch (tests)
    // full-width lockstep kernels (cfg4: 0.79 -> 0.70 ms; register caps 6 / 7 / 8: 0.78 / 0.70 / 0.70,
    // a two-batch software pipeline at 4-5 CTAs/SM: 0.89-0.93)
    if (vec && !generic && k == 64 && lanes == 16 && vregs == 1) return launch_sddmm_lock<16, 8, 7>(a, s);
    if (vec && !generic && k == 32 && lanes == 8 && vregs == 1) return launch_sddmm_lock<8, 8, 1>(a, s);
    if (vec) {
        if (lanes == 4) fn = &launch_sddmm<4, 1, 8, true>;
        else if (lanes == 8) fn = &launch_sddmm<8, 1, 8, true>;
        else if (lanes == 16) fn = &launch_sddmm<16, 1, SGNN_SDDMM_U16, true, SGNN_SDDMM_MINB>;
        else if (vregs == 1) fn = &launch_sddmm<32, 1, 8, true>;
        else if (vregs == 2) fn = &launch_sddmm<32, 2, 4, true>;
        else if (vregs == 4) fn = &launch_sddmm<32, 4, 4, true>;
        else fn = &launch_sddmm<32, 8, 2, true>;
    } else {
        if (vregs == 1) fn = &launch_sddmm<32, 1, 4, false>;
        else if (vregs == 2) fn = &launch_sddmm<32, 2, 4, false>;
        else if (vregs == 4) fn = &launch_sddmm<32, 4, 2, false>;
        else fn = &launch_sddmm<32, 8, 2, false>;
    }
    return fn(a, s);
}

sgnn_status run_fusedmm(const sgnn_csr* p, const float* x, const float* y, uint32_t k, int edge_op,
                        int reduce, float* out, const sgnn_plan_s* plan, cudaStream_t s) {
    if (reduce < 0 || reduce > 3) return fail(SGNN_ERR_CONFIG, "fusedmm: unknown reduce op");
    if (edge_op != SGNN_EDGE_MUL && edge_op != SGNN_EDGE_SIGMOID_MUL)
        return fail(SGNN_ERR_CONFIG, "fusedmm: unknown edge op");
    if (k == 0 || p->n_rows == 0) return SGNN_OK;
    const bool vec = (k % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(y) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    int lanes, vregs;
    if (!full_k_layout(k, vec, &lanes, &vregs))
        return fail(SGNN_ERR_UNSUPPORTED, "fusedmm: K=" + std::to_string(k) +
                                              " exceeds the register-resident width of this build");
    sgnn_plan_s* own = nullptr;
    if (!plan) {
        sgnn_plan_params pp{};
        pp.lanes = uint32_t(lanes);
        pp.vec = uint32_t(vregs);
        pp.k_tile = k;
        pp.unroll = uint32_t(fused_unroll(vec, lanes, vregs));
        if (!vec) pp.scalar = 1;
        SGNN_TRY(build_plan(p, k, &pp, vec, &own, s));
        plan = own;
    } else if (!plan_matches(plan, p, k)) {
        return fail(SGNN_ERR_DISPATCH, "fusedmm: plan was built for another matrix or K");
    }
    sgnn_status st = SGNN_OK;
    int unroll = fused_unroll(vec, lanes, vregs);
    // A caller's plan may choose the register layout if it holds all of K and
    // a fused kernel is compiled for it (the split is reusable either way).
    if (!own && plan->vec == vec) {
        const int pl = int(plan->p.lanes), pv = int(plan->p.vec), pu = int(plan->p.unroll);
        if (uint32_t((vec ? 4 : 1) * pl * pv) >= k && find_fused_launcher(vec, pl, pv, pu, edge_op, reduce)) {
            lanes = pl;
            vregs = pv;
            unroll = pu;
        }
    }
    if (plan->n_slots && plan->kt < k)  // the dot needs all of K: slots must be K wide
        st = fail(SGNN_ERR_DISPATCH, "fusedmm: plan workspace is narrower than K; build the plan with k_tile=K");
    bool tma_ran = false;
    if (st == SGNN_OK && vec && p->n_cols) {
        const int op = edge_op == SGNN_EDGE_SIGMOID_MUL ? dev::OP_FUSED_SIGMOID : dev::OP_FUSED_MUL;
        st = run_fused_tma(p, x, y, k, op, reduce, out, plan, s, &tma_ran);
    }
    SpmmLauncher launch = st == SGNN_OK && !tma_ran ? find_fused_launcher(vec, lanes, vregs, unroll, edge_op, reduce)
                                                    : nullptr;
    if (st == SGNN_OK && !tma_ran && !launch)
        st = fail(SGNN_ERR_UNSUPPORTED, "fusedmm: no kernel for lanes=" + std::to_string(lanes) +
                                            " vec=" + std::to_string(vregs) + " unroll=" + std::to_string(unroll));
    if (st == SGNN_OK && !tma_ran) {
        SpmmArgs args{};
        args.rp = p->row_ptr;
        args.ci = p->col_idx;
        args.val = p->values;
        args.x = y;
        args.xi = x;
        args.ldxi = k;
        args.c = out;
        args.slots = plan->slots;
        args.wrow = plan->wrow;
        args.wnz = plan->wnz;
        args.wslot = plan->wslot;
        args.n_rows = p->n_rows;
        args.n_workers = plan->n_workers;
        args.ldx = k;
        args.ldc = k;
        args.ld_slot = plan->kt;
        args.width = k;
        args.wctr = plan_counter(plan, s);
        const bool generic = std::getenv("SGNN_FUSED_GENERIC") != nullptr;  // A/B switch (tests)
        const char* ring_env = std::getenv("SGNN_FUSED_RING");  // A/B switch: ring chunks (2 / 3 / 4), else registers
        const int ring = ring_env ? std::atoi(ring_env) : 0;
        const bool sig = edge_op == SGNN_EDGE_SIGMOID_MUL;
        if (!generic && vec && k == 64 && (reduce == SGNN_REDUCE_SUM || reduce == SGNN_REDUCE_MEAN) && ring == 4)
            st = sig ? launch_fused_ring<dev::OP_FUSED_SIGMOID, 4>(args, s) : launch_fused_ring<dev::OP_FUSED_MUL, 4>(args, s);
        else if (!generic && vec && k == 64 && (reduce == SGNN_REDUCE_SUM || reduce == SGNN_REDUCE_MEAN) && ring == 2)
            st = sig ? launch_fused_ring<dev::OP_FUSED_SIGMOID, 2>(args, s) : launch_fused_ring<dev::OP_FUSED_MUL, 2>(args, s);
        else if (!generic && vec && k == 64 && (reduce == SGNN_REDUCE_SUM || reduce == SGNN_REDUCE_MEAN) && ring == 3)
            st = sig ? launch_fused_ring<dev::OP_FUSED_SIGMOID, 3>(args, s) : launch_fused_ring<dev::OP_FUSED_MUL, 3>(args, s);
        else if (!generic && vec && k == 64 && (reduce == SGNN_REDUCE_SUM || reduce == SGNN_REDUCE_MEAN))
            // 5 CTAs/SM (96 registers): 1.175 -> 1.086 ms on cfg4; capped at
            // 6 / 7 it spills (44 / 136 bytes) and runs 1.098 / 1.211 ms
            st = sig ? launch_fused_lock<dev::OP_FUSED_SIGMOID, 5>(args, s)
                     : launch_fused_lock<dev::OP_FUSED_MUL, 5>(args, s);
        else
            st = launch(args, plan->p.block, 0, s);
    }
    if (st == SGNN_OK && plan->n_fix) {
        FixupArgs f;
        f.rp = p->row_ptr;
        f.fix_row = plan->fix_row;
        f.fix_slot = plan->fix_slot;
        f.fix_long = plan->fix_long;
        f.n_long = plan->n_long;
        f.slots = plan->slots;
        f.c = out;
        f.ldc = k;
        f.ld_slot = plan->kt;
        f.n_fix = plan->n_fix;
        f.width = k;
        // the fused kernels of mean are the sum kernels; the divide is the pass below
        st = launch_spmm_fixup(f, reduce == SGNN_REDUCE_MEAN ? SGNN_REDUCE_SUM : reduce, s);
    }
    if (st == SGNN_OK && reduce == SGNN_REDUCE_MEAN)  // kernels.hpp:263-266
        st = run_mean_divide(p->row_ptr, p->n_rows, out, k, k, s);
    if (own) destroy_plan(own);
    return st;
}

}  // namespace sgnn
