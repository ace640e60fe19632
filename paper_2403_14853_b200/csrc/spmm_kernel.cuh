// spmm_kernel.cuh -- the sm_100a CSR SpMM worker kernel and its fixup pass.
//
// Restates spmm_rows_trusted / spmm_rows_fixed (kernels.hpp:45-128) for the
// GPU.  One *worker* = a group of G lanes (G in {4,8,16,32}) that walks a
// contiguous nnz-balanced range of the CSR (plan.cuh).  Lane l of the group
// owns the K-slice elements {4*(l + G*v) .. +3 : v < V} (float4 path) or
// {l + G*v} (scalar path), so one warp instruction gathers a contiguous,
// coalesced piece of a neighbour row X[col, :].
//
// Per batch the group broadcasts the (col, val) pairs of a coalesced chunk
// load (through shared memory for full-warp groups, by shuffles otherwise),
// issues U independent row gathers before consuming them (memory-level
// parallelism), then accumulates in ascending nonzero order with separately
// rounded multiply and add (FMUL + FADD2) -- the reference's exact fp32 chain
// (kernels.hpp:55-58) for every row of <= SGNN_SEGMENT nonzeros.  Row ends
// come from a G-wide window of row_ptr held in registers, so short rows cost
// no dependent loads.  Groups narrower than a warp run in lockstep (see the
// LOCK comment in spmm_worker_kernel).
#pragma once

#include "common.cuh"

namespace sgnn {

#define SGNN_MAX_PEERS 8


struct SpmmArgs {
    const uint64_t* __restrict__ rp;
    const uint32_t* __restrict__ ci;
    const float* __restrict__ val;
    const float* __restrict__ x;  // gathered operand (X for SpMM, Y for FusedMM), pre-offset by k0
    const float* __restrict__ xi; // FusedMM only: row operand X (row r's slice is dotted with Y_j)
    uint64_t ldxi;
    float* c;                     // pre-offset by k0 (re-read for multi-segment rows)
    float* __restrict__ slots;    // pre-offset by k0-in-pass; stride ld_slot
    const uint32_t* __restrict__ wrow;
    const uint64_t* __restrict__ wnz;
    const uint32_t* __restrict__ wslot;
    uint32_t n_rows;
    uint32_t n_workers;
    uint64_t ldx;     // row stride of X (floats)
    uint64_t ldc;     // row stride of C (floats)
    uint64_t ld_slot; // row stride of a slot (floats)
    uint32_t width;   // floats of K this launch covers
    // OP_SPMM_PEER: column c lives in block c >> part_shift at row
    // c & ((1 << part_shift) - 1); block base pointers pre-offset by k0
    const float* xparts[SGNN_MAX_PEERS];
    uint32_t part_shift;
    uint32_t* wctr;  // dynamic worker schedule (plan_counter), null: static
};

struct FixupArgs {
    const uint64_t* __restrict__ rp;
    const uint32_t* __restrict__ fix_row;
    const uint32_t* __restrict__ fix_slot;
    const float* __restrict__ slots;
    float* __restrict__ c;  // pre-offset by k0
    uint64_t ldc;
    uint64_t ld_slot;
    uint32_t n_fix;
    uint32_t width;
    // split rows with > SGNN_FIXUP_LONG segments (indices into fix_row), done
    // by spmm_fixup_long_kernel; null: all rows by the per-row kernels
    const uint32_t* __restrict__ fix_long = nullptr;
    uint32_t n_long = 0;
};

namespace dev {

// Reduction semantics (kernels.hpp:53-89, types.hpp:116).
template <int RED>
struct Reducer {
    // a*x folded into acc; `first` marks the first element of a segment.
    static __device__ __forceinline__ float fold(float acc, float a, float x, bool first) {
#ifdef SGNN_EXPERIMENT_FMA_FOLD
        if (RED == SGNN_REDUCE_SUM || RED == SGNN_REDUCE_MEAN) return __fmaf_rn(a, x, acc);
#endif
        const float p = __fmul_rn(a, x);
        if (RED == SGNN_REDUCE_SUM || RED == SGNN_REDUCE_MEAN) return __fadd_rn(acc, p);
        if (first) return p;
        if (RED == SGNN_REDUCE_MIN) return (p < acc) ? p : acc;  // std::min(acc, p)
        return (acc < p) ? p : acc;                               // std::max(acc, p)
    }
    // FusedMM fold: the sum accumulates with fma (FusedMM parity is
    // tolerance-based -- its dot already differs from the reference's chain --
    // and every plan uses the same fold, so results stay plan-independent).
    static __device__ __forceinline__ float fold_fused(float acc, float s, float y, bool first) {
        if (RED == SGNN_REDUCE_SUM || RED == SGNN_REDUCE_MEAN) return __fmaf_rn(s, y, acc);
        return fold(acc, s, y, first);
    }
    // Whole-fragment folds: acc[i] = fold(acc[i], s, x[i]) for every i, in
    // packed pairs where the op allows (same per-element rounding).
    template <int N>
    static __device__ __forceinline__ void fold_all(float (&acc)[N], float s, const float (&x)[N], bool first) {
        if constexpr ((RED == SGNN_REDUCE_SUM || RED == SGNN_REDUCE_MEAN) && N % 2 == 0) {
#ifndef SGNN_EXPERIMENT_FMA_FOLD
#pragma unroll
            for (int i = 0; i < N; i += 2) add2_rn(acc[i], acc[i + 1], __fmul_rn(s, x[i]), __fmul_rn(s, x[i + 1]));
            return;
#endif
        }
#pragma unroll
        for (int i = 0; i < N; ++i) acc[i] = fold(acc[i], s, x[i], first);
    }
    template <int N>
    static __device__ __forceinline__ void fold_fused_all(float (&acc)[N], float s, const float (&y)[N], bool first) {
        if constexpr ((RED == SGNN_REDUCE_SUM || RED == SGNN_REDUCE_MEAN) && N % 2 == 0) {
#pragma unroll
            for (int i = 0; i < N; i += 2) fma2_rn(acc[i], acc[i + 1], s, y[i], y[i + 1]);
        } else {
#pragma unroll
            for (int i = 0; i < N; ++i) acc[i] = fold_fused(acc[i], s, y[i], first);
        }
    }
    // canonical combine of consecutive segment partials (left to right)
    static __device__ __forceinline__ float combine(float t, float s) {
        if (RED == SGNN_REDUCE_SUM || RED == SGNN_REDUCE_MEAN) return __fadd_rn(t, s);
        if (RED == SGNN_REDUCE_MIN) return (s < t) ? s : t;
        return (t < s) ? s : t;
    }
    // epilogue: mean divide (kernels.hpp:60-63, exact: div_by_count); empty
    // rows give 0 for all ops
    static __device__ __forceinline__ float finish(float v, uint64_t deg) {
        if (RED == SGNN_REDUCE_MEAN) return deg ? div_by_count(v, recip_count(deg), float(deg)) : 0.0f;
        return deg ? v : 0.0f;
    }
    // the same over a row fragment: one reciprocal per row, and the exact
    // subnormal-quotient path behind one (rarely taken) branch per row, so
    // the common case never executes it predicated
    template <int N>
    static __device__ __forceinline__ void finish_frag(float (&v)[N], uint64_t deg) {
        if (RED != SGNN_REDUCE_MEAN || !deg) {
#pragma unroll
            for (int i = 0; i < N; ++i) v[i] = deg ? v[i] : 0.0f;
            return;
        }
        const double r = recip_count(deg);
        const float d = float(deg);
        bool exact = false;
#pragma unroll
        for (int i = 0; i < N; ++i) exact |= count_quotient_subnormal(v[i], d);
        if (__builtin_expect(exact, 0)) {
#pragma unroll
            for (int i = 0; i < N; ++i) v[i] = div_by_count(v[i], r, d);
        } else {
#pragma unroll
            for (int i = 0; i < N; ++i) v[i] = div_by_count_normal(v[i], r);
        }
    }
};

template <int G, int V, bool VEC>
struct Frag {
    static constexpr int W = VEC ? 4 : 1;
    static constexpr int N = V * W;
    float v[N];

    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = 0.0f;
    }
    // Is register block `q` of lane `gl` inside the launch width?
    static __device__ __forceinline__ bool valid(int gl, int q, uint32_t width) {
        return uint32_t(W * (gl + G * q)) < width;
    }
    __device__ __forceinline__ void load(const float* __restrict__ row, int gl, uint32_t width) {
#pragma unroll
        for (int q = 0; q < V; ++q) {
            if (valid(gl, q, width)) {
                if constexpr (VEC) {
                    const float4 t = __ldg(reinterpret_cast<const float4*>(row) + gl + G * q);
                    v[4 * q + 0] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
                } else {
                    v[q] = __ldg(row + gl + G * q);
                }
            } else {
#pragma unroll
                for (int i = 0; i < W; ++i) v[W * q + i] = 0.0f;
            }
        }
    }
    // Number of this lane's register blocks inside the launch width.
    static __device__ __forceinline__ int blocks_in(int gl, uint32_t width) {
        const int lim = int(width / W) - gl;
        return lim <= 0 ? 0 : min(V, (lim + G - 1) / G);
    }
    // Hot-loop gather of a neighbour row: `lrow` already points at this
    // lane's first element; blocks beyond nq are skipped (ZERO: zero-filled,
    // needed where all lanes' values are summed, i.e. the FusedMM dot).
    template <bool ZERO>
    __device__ __forceinline__ void gather(const float* __restrict__ lrow, int nq, uint64_t pol) {
        if constexpr (!ZERO) {
            // Unpredicated: blocks beyond the width re-read block 0 (the lane
            // base is clamped inside the row), their values are never stored.
#pragma unroll
            for (int q = 0; q < V; ++q) {
                const int qe = (q < nq) ? q : 0;
                if constexpr (VEC) {
                    const float4 t = ld_gather(reinterpret_cast<const float4*>(lrow + 4 * G * qe), pol);
                    v[4 * q + 0] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
                } else {
                    v[q] = ld_gather(lrow + G * qe, pol);
                }
            }
            return;
        }
#pragma unroll
        for (int q = 0; q < V; ++q) {
            if (q < nq) {
                if constexpr (VEC) {
                    const float4 t = ld_gather(reinterpret_cast<const float4*>(lrow + 4 * G * q), pol);
                    v[4 * q + 0] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
                } else {
                    v[q] = ld_gather(lrow + G * q, pol);
                }
            } else if constexpr (ZERO) {
#pragma unroll
                for (int i = 0; i < W; ++i) v[W * q + i] = 0.0f;
            }
        }
    }
    // Coherent load of data this thread wrote earlier in the same launch.
    __device__ __forceinline__ void load_own(const float* row, int gl, uint32_t width) {
#pragma unroll
        for (int q = 0; q < V; ++q) {
            if (valid(gl, q, width)) {
                if constexpr (VEC) {
                    const float4 t = reinterpret_cast<const float4*>(row)[gl + G * q];
                    v[4 * q + 0] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
                } else {
                    v[q] = row[gl + G * q];
                }
            }
        }
    }
    __device__ __forceinline__ void store(float* __restrict__ row, int gl, uint32_t width) const {
#pragma unroll
        for (int q = 0; q < V; ++q) {
            if (valid(gl, q, width)) {
                if constexpr (VEC) {
                    __stcs(reinterpret_cast<float4*>(row) + gl + G * q,
                           make_float4(v[4 * q + 0], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
                } else {
                    __stcs(row + gl + G * q, v[q]);
                }
            }
        }
    }
};

// Kernel modes: plain SpMM, or FusedMM with an edge op (kernels.hpp:216-270).
// OP_SPMM_PEER: SpMM whose gathered operand is split in row blocks that live
// in different allocations -- the feature blocks of the ranks of a row
// partition, read directly over NVLink peer mappings (no all-gather copy).
enum { OP_SPMM = 0, OP_FUSED_MUL = 1, OP_FUSED_SIGMOID = 2, OP_SPMM_PEER = 3 };
template <int OP>
constexpr bool is_fused() { return OP == OP_FUSED_MUL || OP == OP_FUSED_SIGMOID; }

// Canonical dot product <a, b> over the group.  Leaves are float4 blocks
// q = lane + G*v: x0*y0 then fma of the next three (scalar path: x0*y0);
// the leaves are summed by a balanced binary tree over q, HIGHEST index bit
// first (zero leaves pad to a power of two).  q's high bits are the
// register index v and its low bits the lane, so the tree is: within-lane
// over v (high v bit first), then across lanes xor G/2, G/4, ..., 1.  It is
// the same tree for every (G, V) layout, so FusedMM/SDDMM results do not
// depend on the plan.
// Blocks q >= nq (past the launch width) are zero leaves: masked here, so
// the operands' out-of-width registers may hold anything.
template <int G, int V, bool VEC>
__device__ __forceinline__ float lane_leaf(const Frag<G, V, VEC>& a, const Frag<G, V, VEC>& b, int nq = V) {
    float p[V];
#pragma unroll
    for (int q = 0; q < V; ++q) {
        float t;
        if constexpr (VEC) {
            t = __fmul_rn(a.v[4 * q], b.v[4 * q]);
            t = __fmaf_rn(a.v[4 * q + 1], b.v[4 * q + 1], t);
            t = __fmaf_rn(a.v[4 * q + 2], b.v[4 * q + 2], t);
            t = __fmaf_rn(a.v[4 * q + 3], b.v[4 * q + 3], t);
        } else {
            t = __fmul_rn(a.v[q], b.v[q]);
        }
        p[q] = (q < nq) ? t : 0.0f;
    }
#pragma unroll
    for (int half = V / 2; half >= 1; half >>= 1)  // v tree, high bit first
#pragma unroll
        for (int q = 0; q < half; ++q) p[q] = __fadd_rn(p[q], p[q + half]);
    return p[0];
}

// One dot, every lane of the group gets it.
template <int G, int V, bool VEC>
__device__ __forceinline__ float group_dot(const Frag<G, V, VEC>& a, const Frag<G, V, VEC>& b,
                                           unsigned gmask, int nq = V) {
    float p = lane_leaf(a, b, nq);
#pragma unroll
    for (int s = G / 2; s >= 1; s >>= 1) p = __fadd_rn(p, __shfl_xor_sync(gmask, p, s, G));
    return p;
}

// U dots at once (U <= G) by a transpose-reduce: each halving step exchanges
// half of the remaining partials with lane ^ s (s = G/2, G/4, ...), then a
// butterfly finishes the lanes below.  Same tree as group_dot (lane bits high
// first), U-1 + log2(G/U) shuffles for U dots instead of U*log2(G).  Lane gl
// returns the dot of nonzero gl / (G/U).
template <int G, int V, int U, bool VEC>
__device__ __forceinline__ float batch_dots(const Frag<G, V, VEC>& a, const Frag<G, V, VEC> (&b)[U],
                                            unsigned gmask, int gl, int nq = V) {
    static_assert(U <= G, "batch_dots needs U <= G");
    float p[U];
#pragma unroll
    for (int u = 0; u < U; ++u) p[u] = lane_leaf(a, b[u], nq);
    int s = G / 2;
#pragma unroll
    for (int h = U / 2; h >= 1; h >>= 1, s >>= 1) {
        const bool up = (gl & s) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const float send = up ? p[i] : p[h + i];
            const float keep = up ? p[h + i] : p[i];
            p[i] = __fadd_rn(keep, __shfl_xor_sync(gmask, send, s, G));
        }
    }
#pragma unroll
    for (; s >= 1; s >>= 1) p[0] = __fadd_rn(p[0], __shfl_xor_sync(gmask, p[0], s, G));
    return p[0];
}

template <int OP>
__device__ __forceinline__ float edge_value(float p, float dot) {
    // p * (1 / (1 + exp(-dot))) with the hardware exp2/reciprocal (a few ulp,
    // deterministic): the IEEE-exact divide's slow-path call would cost
    // registers inside the gather loop; FusedMM parity is tolerance-based.
    if (OP == OP_FUSED_SIGMOID)
        return __fmul_rn(p, __fdividef(1.0f, __fadd_rn(1.0f, __expf(-dot))));
    return __fmul_rn(p, dot);  // default combine, kernels.hpp:239
}

// The worker walk.  See plan.cuh for the ownership rules; in short, worker
// (i0,j0)->(i1,j1) consumes nonzeros [j0,j1), finishes rows i0..i1-1 and
// holds the head of row i1 when j1 > row_ptr[i1].  A row that lies entirely
// inside [j0,j1) is written to C; a row split across workers has its
// SGNN_SEGMENT-nonzero segment partials written to consecutive slots.
// MINB: resident 128-thread CTAs per SM the register allocation must allow
// (1 = unconstrained); the tuner's occupancy knob.
template <int G, int V, int U, int RED, bool VEC, int OP = OP_SPMM, int MINB = 1>
__global__ void __launch_bounds__(128, MINB) spmm_worker_kernel(const SpmmArgs a) {
    using F = Frag<G, V, VEC>;
    using R = Reducer<RED>;
    constexpr int N = F::N;
    // One chunk = one batch of U nonzeros: their (col, val) are loaded by the
    // first U lanes of the group (CH per lane when U > G), all U row gathers
    // are issued, then consumed in order.  Keeping one batch per loop trip
    // bounds the live registers to U fragments.
    constexpr int BATCH = U;
    constexpr int CHUNK = U;
    // full-warp groups broadcast (col, val) through shared memory instead of
    // 2 shuffles per nonzero (U even, one chunk element per lane)
    constexpr bool CV_SMEM = (G == 32) && (U % 2 == 0) && (CHUNK <= 32) && SGNN_CV_SMEM;
    __shared__ __align__(16) uint2 s_cv[CV_SMEM ? 4 : 1][CV_SMEM ? CHUNK : 2];
    constexpr int CH = (CHUNK + G - 1) / G;
    constexpr uint64_t SEG = SGNN_SEGMENT;

    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
    // this lane's slice of any gathered row: byte offset col*ldxb from xlane
    // lanes past the width alias the row's last valid block (always in bounds)
    const int gl_eff = min(gl, int(a.width / F::W) - 1);
    const char* xlane = reinterpret_cast<const char*>(a.x + F::W * gl_eff);
    const uint32_t ldxb = uint32_t(a.ldx) * 4u;
    const uint32_t lane_off = uint32_t(F::W * gl_eff) * 4u;  // OP_SPMM_PEER
    const uint32_t part_mask = (1u << a.part_shift) - 1u;
    // address of this lane's slice of gathered row `col`
    auto row_addr = [&](uint32_t col) -> const float* {
        if constexpr (OP == OP_SPMM_PEER) {
            const char* base = reinterpret_cast<const char*>(a.xparts[col >> a.part_shift]);
            return reinterpret_cast<const float*>(base + lane_off + uint64_t(col & part_mask) * ldxb);
        } else {
            return reinterpret_cast<const float*>(xlane + uint64_t(col) * ldxb);
        }
    };
    const int nq = F::blocks_in(gl, a.width);
    const uint64_t l2pol = dev::gather_policy();
    const bool full = a.width == uint32_t(F::W * G * V);  // every lane's blocks are in range

    // LOCK (groups narrower than a warp): the groups of a warp step through
    // their workers' batches together, so every shuffle of the batch body runs
    // with the full warp mask (a lane-dependent group mask makes the compiler
    // guard each shuffle with a convergence check).  A group whose worker is
    // exhausted idles through the remaining trips of the warp.
    constexpr bool LOCK = G < 32;
    constexpr unsigned FULL = 0xffffffffu;
    dev::WarpSched<32 / G> ws(a.wctr);
    for (uint32_t w = ws.base + uint32_t(lane / G); LOCK ? __any_sync(FULL, w < a.n_workers) : (w < a.n_workers);
         ws.next(), w = ws.base + uint32_t(lane / G)) {
        const bool wact = w < a.n_workers;
        const uint32_t wq = wact ? w : a.n_workers - 1;  // idle group: no rows, no nonzeros
        const uint32_t i0 = __ldg(a.wrow + wq), i1 = wact ? __ldg(a.wrow + wq + 1) : i0;
        const uint64_t j0 = __ldg(a.wnz + wq);
        const uint32_t E = wact ? uint32_t(__ldg(a.wnz + wq + 1) - j0) : 0u;  // nonzeros of this worker
        uint32_t slot = a.wslot ? __ldg(a.wslot + wq) : 0u;

        // All row bookkeeping is in 32-bit positions local to the worker
        // (j0-relative, clamped to E): every row r >= i0 ends at or after j0.
        // Lane gl of the window holds the local end of row rb + gl.
        auto window = [&](uint32_t rb_) -> uint32_t {
            const uint64_t e = __ldg(a.rp + min(rb_ + 1 + uint32_t(gl), a.n_rows));
            return uint32_t(min(e - j0, uint64_t(E)));
        };
        uint32_t r = i0;
        uint32_t rb = r;
        uint32_t rwin = window(rb);
        // Row i0 may have begun in an earlier worker (plan.cuh: then j0 sits on
        // one of its segment boundaries); rows i0 < r < i1 lie entirely inside
        // [j0, j1), row i1 is the head of a row finished elsewhere.
        const bool head_cut = __ldg(a.rp + i0) < j0;
        bool inside = !head_cut && r < i1;
        uint32_t rs_l = 0;                                  // local start of row r
        uint32_t rend_l = __shfl_sync(gmask, rwin, 0, G);   // local end of row r
        uint32_t seg_l = min(uint32_t(SEG), rend_l);
        uint32_t next_l = 0;  // next local position needing row/segment work (0: settle first)
        bool first = true;
        bool have_tot = false;
        F acc;
        acc.zero();
        F xrow;                   // FusedMM: X[r, :] slice of the current row
        uint32_t xrow_id = 0xffffffffu;

        auto store_slot = [&](const F& f) {
            f.store(a.slots + uint64_t(slot) * a.ld_slot, gl, a.width);
            ++slot;
        };
        // Rows longer than one segment but owned by this worker keep their
        // running segment total in the output row itself (rare; saves registers).
        auto finish_segment = [&]() {  // segment boundary inside a row
            if (inside) {
                float* crow = a.c + uint64_t(r) * a.ldc;
                if (have_tot) {
                    F t;
                    t.load_own(crow, gl, a.width);
#pragma unroll
                    for (int i = 0; i < N; ++i) t.v[i] = R::combine(t.v[i], acc.v[i]);
                    t.store(crow, gl, a.width);
                } else {
                    acc.store(crow, gl, a.width);
                }
                have_tot = true;
            } else {
                store_slot(acc);
            }
            acc.zero();
            first = true;
        };
        auto finish_row = [&]() {  // row r has no more nonzeros in this worker
            if (inside) {
                const uint64_t deg = rend_l - rs_l;  // the whole row is local
                float* crow = a.c + uint64_t(r) * a.ldc;
                if (have_tot) {
                    F t;
                    t.load_own(crow, gl, a.width);
#pragma unroll
                    for (int i = 0; i < N; ++i) acc.v[i] = R::combine(t.v[i], acc.v[i]);
                }
                R::finish_frag(acc.v, deg);
                acc.store(crow, gl, a.width);
            } else {
                store_slot(acc);
            }
        };
        auto advance_row = [&]() {
            ++r;
            rs_l = rend_l;
            if (r - rb >= uint32_t(G)) {
                rb = r;
                rwin = window(rb);
            }
            rend_l = __shfl_sync(gmask, rwin, int(r - rb), G);
            inside = r < i1;
            seg_l = min(rs_l + uint32_t(SEG), rend_l);
            first = true;
            have_tot = false;
            acc.zero();
        };
        // Row/segment bookkeeping for local position l (>= next_l): close
        // finished rows, close a finished segment, fetch X_r for FusedMM.
        auto settle = [&](uint32_t l) {
            while (l >= rend_l) {
                finish_row();
                advance_row();
            }
            if (l >= seg_l) {
                finish_segment();
                seg_l = min(seg_l + uint32_t(SEG), rend_l);
            }
            if constexpr (is_fused<OP>()) {
                if (xrow_id != r) {
                    xrow.load(a.xi + uint64_t(r) * a.ldxi, gl, a.width);
                    xrow_id = r;
                }
            }
            next_l = min(rend_l, seg_l);
        };

        // (col, val) of batch b+1 are prefetched while batch b is gathered and
        // folded, so each batch waits for one memory latency, not two.
        uint32_t cc[CH];
        float vv[CH];
        auto load_cv = [&](uint32_t base) {
#pragma unroll
            for (int h = 0; h < CH; ++h) {
                const uint32_t lq = base + uint32_t(gl + G * h);
                const bool ok = (gl + G * h) < CHUNK && lq < E;
                cc[h] = ok ? dev::ld_stream(a.ci + j0 + lq) : 0u;  // 0: a safe dummy row
                vv[h] = ok ? dev::ld_stream(a.val + j0 + lq) : 0.0f;
            }
        };
        if (E) load_cv(0);
        if constexpr (LOCK) {
            // Batches are cut at row / segment ends (settle runs between
            // batches, group-divergent); the batch body is warp-uniform.
            uint32_t base = 0;
            while (__any_sync(FULL, base < E)) {
                const bool act = base < E;
                int n = 0;
                if (act) {
                    if (base >= next_l) settle(base);
                    const uint32_t room = next_l - base;
                    n = room < uint32_t(BATCH) ? int(room) : BATCH;
                }
                F xf[U];
                float av[U];
                uint32_t colu[U];
                // FusedMM with the transpose-reduce needs only the value of
                // the nonzero a lane owns (one shuffle, below), not all U
                constexpr bool ALL_VALS = !is_fused<OP>() || U > G;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    colu[u] = __shfl_sync(FULL, cc[u / G], u % G, G);
                    if constexpr (ALL_VALS) av[u] = __shfl_sync(FULL, vv[u / G], u % G, G);
                }
                // (taken before load_cv below overwrites vv with the next chunk)
                float pv_own = 0.0f;
                if constexpr (!ALL_VALS) pv_own = __shfl_sync(FULL, vv[0], gl / (G / U), G);
                // an idle group gathers nothing; its fragments are never folded
                // (n = 0) and its dots stay inside its own lanes
                if (act) {
#pragma unroll
                    for (int u = 0; u < U; ++u) xf[u].template gather<false>(row_addr(colu[u]), nq, l2pol);
                }
                const uint32_t nb = base + uint32_t(n);
                if (act && nb < E) load_cv(nb);
                if constexpr (is_fused<OP>()) {
                    float sv[U];
                    if constexpr (U <= G) {
                        constexpr int PER = G / U;
                        const float s_own = edge_value<OP>(pv_own, batch_dots(xrow, xf, FULL, gl, nq));
#pragma unroll
                        for (int u = 0; u < U; ++u) sv[u] = __shfl_sync(FULL, s_own, u * PER, G);
                    } else {
#pragma unroll
                        for (int u = 0; u < U; ++u) sv[u] = edge_value<OP>(av[u], group_dot(xrow, xf[u], FULL, nq));
                    }
                    if (n == U) {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            R::fold_fused_all(acc.v, sv[u], xf[u].v, first);
                            first = false;
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (u < n) {
                                R::fold_fused_all(acc.v, sv[u], xf[u].v, first);
                                first = false;
                            }
                        }
                    }
                } else if (n == U) {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        R::fold_all(acc.v, av[u], xf[u].v, first);
                        first = false;
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (u < n) {
                            R::fold_all(acc.v, av[u], xf[u].v, first);
                            first = false;
                        }
                    }
                }
                base = nb;
            }
        } else {
            for (uint32_t base = 0; base < E; base += BATCH) {
                const int n = (E - base) < uint32_t(BATCH) ? int(E - base) : BATCH;
                F xf[U];
                float av[U];
                uint32_t colu[U];
                if constexpr (CV_SMEM) {
                    // (col, val) of the batch broadcast through shared memory:
                    // one 8-byte store per lane, then two nonzeros per 16-byte load
                    uint2* cvw = s_cv[threadIdx.x >> 5];
                    if (gl < CHUNK) cvw[gl] = make_uint2(cc[0], __float_as_uint(vv[0]));
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < U; u += 2) {
                        const uint4 t = reinterpret_cast<const uint4*>(cvw)[u / 2];
                        colu[u] = t.x; av[u] = __uint_as_float(t.y);
                        colu[u + 1] = t.z; av[u + 1] = __uint_as_float(t.w);
                    }
                    __syncwarp();
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        colu[u] = __shfl_sync(gmask, cc[u / G], u % G, G);
                        av[u] = __shfl_sync(gmask, vv[u / G], u % G, G);
                    }
                }
    #pragma unroll
                for (int u = 0; u < U; ++u) {  // unconditional gathers (tail lanes read row 0)
                    const float* lrow = row_addr(colu[u]);
                    // the FusedMM dot sums all lanes: zero-fill blocks past a partial width
                    if (!is_fused<OP>() || full) xf[u].template gather<false>(lrow, nq, l2pol);
                    else xf[u].template gather<true>(lrow, nq, l2pol);
                }
                if (base + BATCH < E) load_cv(base + BATCH);
                auto fold = [&](const F& xv, float pv) {
                    float s = pv;
                    if constexpr (is_fused<OP>()) {
                        // s_ij = combine(p_ij, <X_i, Y_j>); Y_j is reused below (read once)
                        s = edge_value<OP>(pv, group_dot(xrow, xv, gmask));
                    }
                    if constexpr (is_fused<OP>()) R::fold_fused_all(acc.v, s, xv.v, first);
                    else R::fold_all(acc.v, s, xv.v, first);
                    first = false;
                };
                if (base + uint32_t(n) <= next_l) {
                    // fast path: the whole batch continues the current row segment
                    if constexpr (is_fused<OP>()) {
                        float sv[U];
                        if constexpr (U <= G) {
                            // transpose-reduce: lane gl owns the dot of nonzero gl/(G/U);
                            // the edge op runs once per nonzero, then s is broadcast
                            constexpr int PER = G / U;
                            const int u_own = gl / PER;
                            float pv_own = av[0];
    #pragma unroll
                            for (int u = 1; u < U; ++u)
                                if (u == u_own) pv_own = av[u];
                            const float s_own = edge_value<OP>(pv_own, batch_dots(xrow, xf, gmask, gl));
    #pragma unroll
                            for (int u = 0; u < U; ++u) sv[u] = __shfl_sync(gmask, s_own, u * PER, G);
                        } else {
    #pragma unroll
                            for (int u = 0; u < U; ++u) sv[u] = edge_value<OP>(av[u], group_dot(xrow, xf[u], gmask));
                        }
    #pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (u < n) {
                                R::fold_fused_all(acc.v, sv[u], xf[u].v, first);
                                first = false;
                            }
                        }
                    } else if (n == U) {
                        // full batch (all but a worker's last): no per-element guards
    #pragma unroll
                        for (int u = 0; u < U; ++u) fold(xf[u], av[u]);
                    } else {
    #pragma unroll
                        for (int u = 0; u < U; ++u)
                            if (u < n) fold(xf[u], av[u]);
                    }
                } else {
                    // slow path: row / segment boundaries inside the batch
    #pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (u >= n) break;
                        const uint32_t l = base + uint32_t(u);
                        if (l >= next_l) settle(l);
                        fold(xf[u], av[u]);
                    }
                }
            }
        }
        // All nonzeros consumed: close rows that end inside this worker (the
        // current one and any empty rows after it), then the head of row i1.
        while (r < i1) {
            finish_row();
            advance_row();
        }
        if (r < a.n_rows && E > rs_l) store_slot(acc);  // head of a split row
    }
    ws.finish();
}

// Adds the segment partials of each split row left to right and applies the
// reduction epilogue.  One thread per K element; the slot loads are
// independent, the fold is the canonical sequential chain.
template <int RED>
__global__ void __launch_bounds__(256) spmm_fixup_kernel(const FixupArgs f) {
    using R = Reducer<RED>;
    constexpr uint64_t SEG = SGNN_SEGMENT;
    const uint64_t total = uint64_t(f.n_fix) * f.width;
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t fi = uint32_t(t / f.width);
        const uint32_t k = uint32_t(t % f.width);
        const uint32_t r = __ldg(f.fix_row + fi);
        const uint64_t deg = __ldg(f.rp + r + 1) - __ldg(f.rp + r);
        const uint64_t nseg = (deg + SEG - 1) / SEG;
        const float* s = f.slots + uint64_t(__ldg(f.fix_slot + fi)) * f.ld_slot + k;
        float v = __ldcs(s);
        uint64_t q = 1;
        for (; q + 8 <= nseg; q += 8) {
            float b[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) b[i] = __ldcs(s + (q + i) * f.ld_slot);
#pragma unroll
            for (int i = 0; i < 8; ++i) v = R::combine(v, b[i]);
        }
        for (; q < nseg; ++q) v = R::combine(v, __ldcs(s + q * f.ld_slot));
        __stcs(f.c + uint64_t(r) * f.ldc + k, R::finish(v, deg));
    }
}

// float4 fixup: one warp per (split row, 128-float chunk), lane l owns
// floats 4l..4l+3 of the chunk, so each slot row is one coalesced 512-byte
// read.  Same per-element chain as spmm_fixup_kernel.
template <int RED>
__global__ void __launch_bounds__(256) spmm_fixup_vec_kernel(const FixupArgs f) {
    using R = Reducer<RED>;
    constexpr uint64_t SEG = SGNN_SEGMENT;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nchunk = (f.width + 127) / 128;
    const uint64_t items = uint64_t(f.n_fix) * nchunk;
    const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    auto comb = [](float4 t, const float4& u) {
        t.x = R::combine(t.x, u.x); t.y = R::combine(t.y, u.y);
        t.z = R::combine(t.z, u.z); t.w = R::combine(t.w, u.w);
        return t;
    };
    for (uint64_t it = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; it < items; it += n_warps) {
        const uint32_t fi = uint32_t(it / nchunk);
        const uint32_t k = uint32_t(it % nchunk) * 128 + lane * 4;
        if (k >= f.width) continue;
        const uint32_t r = __ldg(f.fix_row + fi);
        const uint64_t deg = __ldg(f.rp + r + 1) - __ldg(f.rp + r);
        const uint64_t nseg = (deg + SEG - 1) / SEG;
        if (f.fix_long && nseg > SGNN_FIXUP_LONG) continue;  // spmm_fixup_long_kernel's row
        const uint64_t st = f.ld_slot / 4;
        const float4* s = reinterpret_cast<const float4*>(f.slots + uint64_t(__ldg(f.fix_slot + fi)) * f.ld_slot + k);
        float4 v = __ldcs(s);
        uint64_t q = 1;
        for (; q + 8 <= nseg; q += 8) {
            float4 b[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) b[i] = __ldcs(s + (q + i) * st);
#pragma unroll
            for (int i = 0; i < 8; ++i) v = comb(v, b[i]);
        }
        for (; q < nseg; ++q) v = comb(v, __ldcs(s + q * st));
        v.x = R::finish(v.x, deg); v.y = R::finish(v.y, deg);
        v.z = R::finish(v.z, deg); v.w = R::finish(v.w, deg);
        __stcs(reinterpret_cast<float4*>(f.c + uint64_t(r) * f.ldc + k), v);
    }
}

// Split rows with more than SGNN_FIXUP_LONG segments (hub rows: cfg2's
// largest has 300): a CTA stages chunks of the row's consecutive slots in
// shared memory with all its threads, then each thread runs the canonical
// left-to-right chain over its columns -- instead of one warp walking 300
// slot loads in dependent batches of 8.
constexpr int kFixupLongThreads = 256;
constexpr int kFixupLongBytes = 48 * 1024;
template <int RED>
__global__ void __launch_bounds__(kFixupLongThreads) spmm_fixup_long_kernel(const FixupArgs f) {
    using R = Reducer<RED>;
    constexpr uint64_t SEG = SGNN_SEGMENT;
    __shared__ __align__(16) float tile[kFixupLongBytes / 4];
    const uint32_t w4 = f.width / 4;  // float4 per slot row (width % 4 == 0 here)
    const uint32_t chunk = max(1u, uint32_t(kFixupLongBytes / 16) / w4);  // slots per staging round
    for (uint32_t li = blockIdx.x; li < f.n_long; li += gridDim.x) {
        const uint32_t fi = __ldg(f.fix_long + li);
        const uint32_t r = __ldg(f.fix_row + fi);
        const uint64_t deg = __ldg(f.rp + r + 1) - __ldg(f.rp + r);
        const uint32_t nseg = uint32_t((deg + SEG - 1) / SEG);
        const float* s0 = f.slots + uint64_t(__ldg(f.fix_slot + fi)) * f.ld_slot;
        // thread t owns columns t, t + T, ... (< width); its chain in registers
        constexpr int PER = 1024 / kFixupLongThreads;  // width <= 1024 floats
        float v[PER];
        for (uint32_t q0 = 0; q0 < nseg; q0 += chunk) {
            const uint32_t nq = min(chunk, nseg - q0);
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < nq * w4; i += kFixupLongThreads) {
                const uint32_t q = i / w4, c4 = i % w4;
                reinterpret_cast<float4*>(tile)[i] =
                    __ldcs(reinterpret_cast<const float4*>(s0 + uint64_t(q0 + q) * f.ld_slot) + c4);
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const uint32_t k = threadIdx.x + uint32_t(j) * kFixupLongThreads;
                if (k >= f.width) break;
                uint32_t q = 0;
                if (q0 == 0) v[j] = tile[k], q = 1;
                for (; q < nq; ++q) v[j] = R::combine(v[j], tile[q * f.width + k]);
            }
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const uint32_t k = threadIdx.x + uint32_t(j) * kFixupLongThreads;
            if (k >= f.width) break;
            __stcs(f.c + uint64_t(r) * f.ldc + k, R::finish(v[j], deg));
        }
    }
}

// Lockstep worker for one float4 per lane (K <= 4 G, G < 32): FusedMM
// (Sum; Mean through the divide pass) and SpMM (every reduction): the
// worker kernel's split, batches, row / segment / slot rules,
// dot tree and fma fold -- bitwise its results (test) -- with fewer
// instructions per batch: (col, val) arrive in G-wide windows, a gather
// address is one mad.wide, the dot is unmasked (every lane's float4 is inside
// K), and the row / segment settling runs as warp-uniform loops with
// full-mask shuffles.  At the worker's 5 CTAs/SM: cfg4 1.175 -> 1.086 ms
// (capping registers lower spills: DESIGN 3.3).
//
// NCH > 0 (G = 16, U = 8, K = 64): the gathered rows go through a
// shared-memory ring instead of registers.  A worker's nonzeros are cut in
// aligned chunks of 8 local positions; chunk c's 8 rows are copied by
// cp.async (16 bytes per lane, lane-private slots, so a per-thread
// wait_group is the only synchronisation) NCH - 1 chunks before they are
// used, and its values ride along in a small ring.  Batches are cut at chunk
// ends as well as at row / segment ends, so a batch reads one slot.  The
// rows in flight per SM are then set by the ring (NCH - 1 chunks per group),
// not by the register file.  Same dot tree, same fold order: bitwise the
// register kernel's results (test).
template <int NCH>
constexpr uint32_t ring_row_bytes() { return uint32_t(8 * NCH * 8 + 8) * 16u * 16u; }  // 8 groups + 8 positions of pad
template <int NCH>
constexpr uint32_t ring_smem_bytes() { return ring_row_bytes<NCH>() + uint32_t(8 * NCH * 8 + 8) * 4u; }

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
#if defined(SGNN_RING_CG)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
#else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
#endif
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int G, int U, int OP, int RED, int MINB, int NCH = 0>
__global__ void __launch_bounds__(128, MINB) lock_worker_kernel(const SpmmArgs a) {
    static_assert(G < 32 && U <= G && (OP == OP_SPMM || is_fused<OP>()), "lockstep groups");
    static_assert(!is_fused<OP>() || RED == SGNN_REDUCE_SUM, "FusedMM: sum kernels (mean: divide pass)");
    constexpr bool RING = NCH > 0;
    static_assert(!RING || (G == 16 && U == 8 && NCH >= 2), "ring: 16-lane groups, chunks of 8 positions");
    using F = Frag<G, 1, true>;
    using R = Reducer<RED>;
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int PER = G / U;
    constexpr uint32_t SEG = SGNN_SEGMENT;
    const int lane = threadIdx.x & 31, gl = lane & (G - 1), gbase = lane & ~(G - 1);
    extern __shared__ __align__(16) unsigned char ring_smem[];
    // this lane's column of its group's row ring, and the group's value ring
    float4* const ring = reinterpret_cast<float4*>(ring_smem) + size_t(threadIdx.x / G) * (RING ? NCH * 8 * 16 : 0) + gl;
    float* const vring = reinterpret_cast<float*>(ring_smem + (RING ? ring_row_bytes<RING ? NCH : 1>() : 0)) +
                         (threadIdx.x / G) * (RING ? NCH * 8 : 0);
    // lanes past the width alias the row's last valid float4 (always in bounds)
    const char* ylane = reinterpret_cast<const char*>(a.x + 4 * min(gl, int(a.width / 4) - 1));
    const uint32_t ldb = uint32_t(a.ldx) * 4u;
    const uint64_t l2pol = gather_policy();
    WarpSched<32 / G> ws(a.wctr);
    for (uint32_t w = ws.base + uint32_t(lane / G); __any_sync(FULL, w < a.n_workers);
         ws.next(), w = ws.base + uint32_t(lane / G)) {
        const bool wact = w < a.n_workers;
        const uint32_t wq = wact ? w : a.n_workers - 1;  // idle group: no rows, no nonzeros
        const uint32_t i0 = __ldg(a.wrow + wq), i1 = wact ? __ldg(a.wrow + wq + 1) : i0;
        const uint64_t j0 = __ldg(a.wnz + wq);
        const uint32_t E = wact ? uint32_t(__ldg(a.wnz + wq + 1) - j0) : 0u;
        uint32_t slot = a.wslot ? __ldg(a.wslot + wq) : 0u;
        auto window = [&](uint32_t rb_) -> uint32_t {  // lane gl: local end of row rb_ + gl
            const uint64_t e = __ldg(a.rp + min(rb_ + 1 + uint32_t(gl), a.n_rows));
            return uint32_t(min(e - j0, uint64_t(E)));
        };
        uint32_t r = i0, rb = i0;
        uint32_t rwin = window(rb);
        // FusedMM: X rows are read once each, so every row start is a DRAM
        // miss on the critical path; the window's later non-empty rows (those
        // with nonzeros in this worker) are fetched into L2 when the window
        // is loaded (cfg4: 1.078 -> 1.025 ms)
        auto prefetch_x = [&](bool mine) {  // every lane calls it; the groups in `mine` prefetch
            if constexpr (is_fused<OP>()) {
                const uint32_t prev = __shfl_up_sync(FULL, rwin, 1, G);
                if (mine && gl >= 1 && rwin > prev && rb + uint32_t(gl) < a.n_rows) {
                    const char* xp = reinterpret_cast<const char*>(a.xi + uint64_t(rb + uint32_t(gl)) * a.ldxi);
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(xp));
                    if (a.width > 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(xp + 128));
                }
            }
        };
        prefetch_x(wact);
        uint32_t rend_l = __shfl_sync(FULL, rwin, gbase);
        uint32_t rs_l = 0, seg_l = min(SEG, rend_l);
        bool inside = __ldg(a.rp + i0) >= j0 && r < i1;  // row i0 did not begin in an earlier worker
        bool have_tot = false, first = true, xstale = true;  // xstale: X_r not loaded yet
        F acc, xrow;
        acc.zero();
        auto store_slot = [&]() {
            acc.store(a.slots + uint64_t(slot) * a.ld_slot, gl, a.width);
            ++slot;
        };
        auto finish_row = [&]() {  // row r has no more nonzeros in this worker
            if (inside) {
                float* crow = a.c + uint64_t(r) * a.ldc;
                if (have_tot) {
                    F t;
                    t.load_own(crow, gl, a.width);
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc.v[i] = R::combine(t.v[i], acc.v[i]);
                }
                R::finish_frag(acc.v, rend_l - rs_l);
                acc.store(crow, gl, a.width);
            } else {
                store_slot();
            }
        };
        // rows of the groups in `need` advance by one (window reload per group,
        // then one full-mask shuffle for the new row ends)
        auto advance = [&](bool need) {
            bool reloaded = false;
            if (need) {
                ++r;
                rs_l = rend_l;
                if (r - rb >= uint32_t(G)) {
                    rb = r;
                    rwin = window(rb);
                    reloaded = true;
                }
            }
            if constexpr (is_fused<OP>()) {
                if (__any_sync(FULL, reloaded)) prefetch_x(reloaded);
            }
            const uint32_t t = __shfl_sync(FULL, rwin, gbase + int(r - rb));
            if (need) {
                rend_l = t;
                inside = r < i1;
                seg_l = min(rs_l + SEG, rend_l);
                first = true;
                have_tot = false;
                xstale = true;
                acc.zero();
            }
        };
        uint32_t wb = 0, cw = 0;
        float vw = 0.0f;
        auto load_window = [&](uint32_t at) {
            wb = at;
            const bool ok = at + uint32_t(gl) < E;
            cw = ok ? ld_stream(a.ci + j0 + at + gl) : 0u;  // 0: a safe dummy row
            vw = ok ? ld_stream(a.val + j0 + at + gl) : 0.0f;
        };
        // RING: (cw, vw) is the 16-position window the next chunk is issued
        // from, (cw2, vw2) the window after it (loaded two chunks early)
        uint32_t cw2 = 0, issued = 0, slot_i = 0, slot_c = NCH - 1, next_enter = 0;
        float vw2 = 0.0f;
        auto load_window2 = [&](uint32_t at) {
            const bool ok = at + uint32_t(gl) < E;
            cw2 = ok ? ld_stream(a.ci + j0 + at + gl) : 0u;
            vw2 = ok ? ld_stream(a.val + j0 + at + gl) : 0.0f;
        };
        // copies of chunk `issued` (positions 8 issued .. +8) into slot slot_i;
        // every lane runs the shuffles, the groups in `doit` issue and commit
        auto issue_chunk = [&](bool doit) {
            const int h8 = int(issued & 1u) * 8;
            uint32_t colu[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) colu[u] = __shfl_sync(FULL, cw, gbase + h8 + u);
            if (doit) {
                const uint32_t p0 = issued * 8u;
                float4* dst = ring + slot_i * (8 * 16);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (p0 + uint32_t(u) < E) {
                        const char* p;
                        asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(colu[u]), "r"(ldb), "l"(ylane));
                        cp_async16(dst + u * 16, p);
                    }
                }
                if ((gl >> 3) == int(issued & 1u)) vring[slot_i * 8 + (gl & 7)] = vw;
                cp_async_commit();
                if (issued & 1u) {  // the window is used up: take the next, load the one after
                    cw = cw2;
                    vw = vw2;
                    load_window2((issued + 1u) * 8u + 16u);
                }
                ++issued;
                slot_i = slot_i + 1 == uint32_t(NCH) ? 0u : slot_i + 1;
            }
        };
        if constexpr (RING) {
            if (E) {
                load_window(0);
                load_window2(16);
            }
#pragma unroll
            for (int c = 0; c < NCH - 1; ++c) issue_chunk(wact);
        } else {
            if (E) load_window(0);
        }
        uint32_t base = 0;
        while (__any_sync(FULL, base < E)) {
            const bool act = base < E;
            if constexpr (RING) {
                // entering chunk base / 8: issue chunk base / 8 + NCH - 1 into the
                // slot just consumed, then wait for this chunk's rows
                const bool enter = act && base == next_enter;
                if (__any_sync(FULL, enter)) {
                    issue_chunk(enter);
                    if (enter) {
                        cp_async_wait<RING ? NCH - 1 : 0>();
                        next_enter += 8;
                        slot_c = slot_c + 1 == uint32_t(NCH) ? 0u : slot_c + 1;
                    }
                    __syncwarp();  // the value ring's stores are visible to the group
                }
            }
            // settle (the worker's): close finished rows, then a finished segment
            while (true) {
                const bool need = act && base >= rend_l;
                if (!__any_sync(FULL, need)) break;
                if (need) finish_row();
                advance(need);
            }
            if (act && base >= seg_l) {  // segment boundary inside a row
                if (inside) {
                    float* crow = a.c + uint64_t(r) * a.ldc;
                    if (have_tot) {
                        F t;
                        t.load_own(crow, gl, a.width);
#pragma unroll
                        for (int i = 0; i < 4; ++i) t.v[i] = R::combine(t.v[i], acc.v[i]);
                        t.store(crow, gl, a.width);
                    } else {
                        acc.store(crow, gl, a.width);
                    }
                    have_tot = true;
                } else {
                    store_slot();
                }
                acc.zero();
                first = true;
                seg_l = min(seg_l + SEG, rend_l);
            }
            if constexpr (is_fused<OP>()) {
                if (act && xstale) {
                    xrow.load(a.xi + uint64_t(r) * a.ldxi, gl, a.width);
                    xstale = false;
                }
            }
            int n = 0;
            if (act) {
                uint32_t room = min(rend_l, seg_l) - base;
                if constexpr (RING) room = min(room, 8u - (base & 7u));  // and at the chunk's end
                n = room < uint32_t(U) ? int(room) : U;
            }
            float pv_own = 0.0f, av[U];
            F yf[U];
            const uint32_t nb = base + uint32_t(n);
            if constexpr (RING) {
                // the batch's rows and values from this chunk's slot (reads past
                // the chunk's end stay inside the ring or its pad; never folded)
                const uint32_t off = base & 7u;
                const float4* src = ring + (slot_c * 8 + off) * 16;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const float4 t = src[u * 16];
                    yf[u].v[0] = t.x; yf[u].v[1] = t.y; yf[u].v[2] = t.z; yf[u].v[3] = t.w;
                }
                if constexpr (is_fused<OP>()) {
                    pv_own = vring[slot_c * 8 + min(off + uint32_t(gl / PER), 7u)];
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) av[u] = vring[slot_c * 8 + min(off + uint32_t(u), 7u)];
                }
            } else {
                // an active group's batch lies inside the window (base - wb <= G - U)
                const int s0 = gbase + int(base - wb);
                uint32_t colu[U];
#pragma unroll
                for (int u = 0; u < U; ++u) colu[u] = __shfl_sync(FULL, cw, s0 + u);
                if constexpr (is_fused<OP>()) {
                    pv_own = __shfl_sync(FULL, vw, s0 + gl / PER);
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) av[u] = __shfl_sync(FULL, vw, s0 + u);
                }
                if (act) {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const char* p;
                        asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(colu[u]), "r"(ldb), "l"(ylane));
                        const float4 t = ld_gather(reinterpret_cast<const float4*>(p), l2pol);
                        yf[u].v[0] = t.x; yf[u].v[1] = t.y; yf[u].v[2] = t.z; yf[u].v[3] = t.w;
                    }
                }
                if (act && nb < E && nb + uint32_t(U) > wb + uint32_t(G)) load_window(nb);
            }
            if constexpr (is_fused<OP>()) {
                const float s_own = edge_value<OP>(pv_own, batch_dots(xrow, yf, FULL, gl));
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const float sv = __shfl_sync(FULL, s_own, gbase + u * PER);
                    if (u < n) {
                        R::fold_fused_all(acc.v, sv, yf[u].v, first);
                        first = false;
                    }
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (u < n) {
                        R::fold_all(acc.v, av[u], yf[u].v, first);
                        first = false;
                    }
                }
            }
            base = nb;
        }
        // all nonzeros consumed: close rows ending inside this worker (the
        // current one and empty rows after it), then the head of row i1
        while (true) {
            const bool need = r < i1;
            if (!__any_sync(FULL, need)) break;
            if (need) finish_row();
            advance(need);
        }
        if (r < a.n_rows && E > rs_l) store_slot();  // head of a split row
        if constexpr (RING) cp_async_wait<0>();  // (only empty groups can be pending)
    }
    ws.finish();
}

// Short-row SpMM (every row <= 2 G nonzeros, no split rows): one G-lane
// group per row, rows strided over the groups, no plan metadata and no
// worker schedule -- a row costs three dependent loads (row_ptr, its (col,
// val) pairs in one G-wide load each, its gathers).  The fold is the worker's
// (ascending nonzero order, the same Reducer), so results are bitwise the
// worker kernel's.  Groups narrower than a warp step together (full-mask
// shuffles); a group with a shorter row idles through the extra trips.
template <int G, int U, int RED>
__global__ void __launch_bounds__(128) spmm_short_rows_kernel(const SpmmArgs a) {
    using F = Frag<G, 1, true>;
    using R = Reducer<RED>;
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, gl = lane & (G - 1), gbase = lane & ~(G - 1);
    const uint32_t ngroups = (gridDim.x * blockDim.x) / G;
    const uint32_t g0 = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int gl_eff = min(gl, int(a.width / 4) - 1);
    const char* xlane = reinterpret_cast<const char*>(a.x + 4 * gl_eff);
    const uint32_t ldxb = uint32_t(a.ldx) * 4u;
    const uint64_t l2pol = gather_policy();
    // every group of a warp runs the same number of row trips
    const uint32_t wfirst = g0 - uint32_t(lane / G);
    const uint32_t trips = wfirst < a.n_rows ? (a.n_rows - wfirst + ngroups - 1) / ngroups : 0u;
    for (uint32_t t = 0; t < trips; ++t) {
        const uint32_t r = g0 + t * ngroups;
        const bool act = r < a.n_rows;
        uint64_t j = 0;
        uint32_t deg = 0;
        if (act) {
            j = __ldg(a.rp + r);
            deg = uint32_t(__ldg(a.rp + r + 1) - j);
        }
        const uint32_t c0 = uint32_t(gl) < deg ? ld_stream(a.ci + j + gl) : 0u;  // 0: a safe dummy row
        const float v0 = uint32_t(gl) < deg ? ld_stream(a.val + j + gl) : 0.0f;
        const uint32_t c1 = uint32_t(gl + G) < deg ? ld_stream(a.ci + j + G + gl) : 0u;
        const float v1 = uint32_t(gl + G) < deg ? ld_stream(a.val + j + G + gl) : 0.0f;
        F acc;
        acc.zero();
        bool first = true;
        for (uint32_t b = 0; __any_sync(FULL, b < deg); b += U) {
            F xf[U];
            float av[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t p = b + uint32_t(u);  // the same position in every lane of the group
                const int src = gbase + int(p & (G - 1));
                const uint32_t col = __shfl_sync(FULL, p < uint32_t(G) ? c0 : c1, src);
                av[u] = __shfl_sync(FULL, p < uint32_t(G) ? v0 : v1, src);
                xf[u].template gather<false>(reinterpret_cast<const float*>(xlane + uint64_t(col) * ldxb), 1, l2pol);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (b + uint32_t(u) < deg) {
                    R::fold_all(acc.v, av[u], xf[u].v, first);
                    first = false;
                }
            }
        }
        if (act) {
            R::finish_frag(acc.v, deg);
            acc.store(a.c + uint64_t(r) * a.ldc, gl, a.width);
        }
    }
}

}  // namespace dev

// Host launcher table (spmm_launch.cu).
using SpmmLauncher = sgnn_status (*)(const SpmmArgs&, uint32_t block, uint32_t max_blocks,
                                     cudaStream_t);
SpmmLauncher find_spmm_launcher(bool vec, int lanes, int vec_regs, int unroll, int reduce, int occ);
sgnn_status launch_spmm_fixup(const FixupArgs& f, int reduce, cudaStream_t s);

}  // namespace sgnn
