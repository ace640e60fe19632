// fused_tma.cu -- warp-specialised SDDMM / FusedMM (kernels.hpp:187-270) for
// K = 64 and 128: Y rows are gathered by the Tensor Memory Accelerator into
// shared-memory rings instead of into registers.
//
// STATUS: opt-in (SGNN_TMA_FUSED=1), slower than the register kernels on
// cfg4 -- see tma_fused_enabled() below and DESIGN.md 3.3.
//
// Why: at K = 64 the register-gather worker (spmm_kernel.cuh, fused mode) is
// latency-bound -- per batch of 8 nonzeros it waits for the 8 row gathers,
// then runs the dependent dot -> transpose-reduce -> edge op -> fold chain,
// and the fragments in flight cap residency at ~19 warps/SM (ncu, cfg4).
// Here one producer warp per CTA keeps D stages of 8 rows in flight for each
// consumer worker with `cp.async.bulk.tensor.2d ... tile::gather4` (4 rows of
// Y per instruction, completion on an mbarrier), so rows in flight cost
// shared memory, not registers, and the consumers never issue a global load
// for Y.
//
// CTA = NCW consumer warps + 1 producer warp.  Each consumer warp runs two
// workers of G = 16 lanes (lane gl holds float4 block(s) gl + 16 v of a row,
// V = K / 64) in lockstep, exactly like the LOCK path of the register kernel:
// same worker split (the plan's wrow / wnz / wslot), same row / canonical
// 256-nonzero segment bookkeeping, same dot tree (dev::batch_dots), edge op
// and fold order -- results are bitwise those of the register kernel
// (tests/test_fused_gpu.py).  Ring slot c (c = 2 * consumer warp + half)
// belongs to one consumer worker; producer lane c fills it.
//
// Ring protocol per slot: stage s holds up to 8 consecutive nonzeros of one
// worker (its chunk ch = positions 8ch..8ch+7): the gathered Y rows, their
// values and a header (worker id, chunk).  full[s]: producer arrive +
// expect_tx, completed by the TMA bytes; empty[s]: the consumer half's lane 0
// after its lanes have read the stage.  Workers are taken from the plan's
// dynamic counter (first round static), like dev::WarpSched; a worker
// without nonzeros still gets one (data-less) stage so its empty rows are
// written; a sentinel header ends the slot.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "ops.cuh"
#include "plan.cuh"
#include "spmm_kernel.cuh"

namespace sgnn {

namespace {

constexpr int kStageRows = 8;           // nonzeros (Y rows) per ring stage: two gather4
constexpr uint32_t kSentinel = 0xffffffffu;
constexpr int OP_SDDMM = 100;           // SDDMM through the same pipeline (no fold)

struct TmaArgs {
    const uint64_t* __restrict__ rp;
    const uint32_t* __restrict__ ci;
    const float* __restrict__ val;
    const float* __restrict__ xi;  // row operand X [n_rows x K]
    float* c;                      // FusedMM output [n_rows x K]
    float* __restrict__ slots;     // segment partials of split rows (stride ld_slot)
    float* __restrict__ out;       // SDDMM values [nnz]
    const uint32_t* __restrict__ wrow;
    const uint64_t* __restrict__ wnz;
    const uint32_t* __restrict__ wslot;
    uint64_t ld_slot;
    uint32_t n_rows;
    uint32_t n_workers;
    uint32_t* wctr;  // dynamic worker schedule (plan_counter), null: static stride
};

// ---- PTX: shared-memory mbarriers and the TMA row gather
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// rows r0..r3 of the 2-D tensor map (box {K, 1}) -> 4 consecutive rows at dst
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint64_t* bar, uint32_t r0,
                                            uint32_t r1, uint32_t r2, uint32_t r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

template <int V, int NCW, int D>
struct TmaSmem {
    static constexpr int K = 64 * V;
    static constexpr int NSLOT = 2 * NCW;
    static constexpr size_t kStageBytes = size_t(kStageRows) * K * 4;
    static constexpr size_t kData = size_t(NSLOT) * D * kStageBytes;
    static constexpr size_t kBars = size_t(NSLOT) * D * 2 * 8;
    static constexpr size_t kHdr = size_t(NSLOT) * D * 2 * 4;
    static constexpr size_t kVals = size_t(NSLOT) * D * kStageRows * 4;
    static constexpr size_t kBytes = kData + kBars + kHdr + kVals + 1024;  // + alignment slack
};

template <int V, int OP, int RED, int NCW, int D>
__global__ void __launch_bounds__(32 * (NCW + 1)) fused_tma_kernel(const TmaArgs a,
                                                                   const __grid_constant__ CUtensorMap tmap) {
    constexpr int G = 16, U = kStageRows;
    constexpr int K = 64 * V;
    constexpr int NSLOT = 2 * NCW;
    using L = TmaSmem<V, NCW, D>;
    using F = dev::Frag<G, V, true>;
    using R = dev::Reducer<RED>;
    constexpr int N = F::N;
    constexpr uint64_t SEG = SGNN_SEGMENT;
    constexpr unsigned FULL = 0xffffffffu;
    constexpr bool SDDMM = OP == OP_SDDMM;
    constexpr int EDGE_OP = SDDMM ? dev::OP_FUSED_MUL : OP;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float* sdata = reinterpret_cast<float*>(base);                      // [NSLOT][D][8][K]
    uint64_t* full = reinterpret_cast<uint64_t*>(base + L::kData);     // [NSLOT][D]
    uint64_t* empty = full + NSLOT * D;                                 // [NSLOT][D]
    uint32_t* hdr = reinterpret_cast<uint32_t*>(empty + NSLOT * D);     // [NSLOT][D][2]
    float* svals = reinterpret_cast<float*>(hdr + NSLOT * D * 2);       // [NSLOT][D][8]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NSLOT * D; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NCW) {
        // ------------------------------------------------------- producer
        if (lane >= NSLOT) return;
        const int c = lane;
        const uint32_t first_round = gridDim.x * NSLOT;
        // The slot's stream of items (worker, chunk) is generated PF items
        // ahead of the one being emitted: each item's (col, val) loads are in
        // flight for PF emits before its TMA is issued.  The worker after the
        // current one is taken from the schedule when the current one starts.
        constexpr int PF = 3;
        uint32_t w = blockIdx.x * NSLOT + c, ch = 0;
        bool have = w < a.n_workers;
        uint64_t j0 = have ? __ldg(a.wnz + w) : 0;
        uint32_t E = have ? uint32_t(__ldg(a.wnz + w + 1) - j0) : 0u;
        uint32_t nw = have ? (a.wctr ? first_round + atomicAdd(a.wctr, 1u) : w + first_round) : kSentinel;
        bool nhave = nw < a.n_workers;
        uint64_t nj0 = nhave ? __ldg(a.wnz + nw) : 0;
        uint32_t nE = nhave ? uint32_t(__ldg(a.wnz + nw + 1) - nj0) : 0u;
        uint32_t cs[PF][U], hw[PF], hc[PF], hn[PF];
        float vs[PF][U];
        // the next item into slot q of the lookahead (cols/vals loads issued)
        auto gen = [&](int q) {
            hw[q] = have ? w : kSentinel;
            hc[q] = ch;
            hn[q] = have ? E : 0u;
#pragma unroll
            for (int t = 0; t < U; ++t) {
                const uint32_t p = ch * U + uint32_t(t);
                const uint32_t qq = p < E ? p : (E ? E - 1 : 0);  // clamp: duplicate rows are harmless
                cs[q][t] = have && E ? __ldcs(a.ci + j0 + qq) : 0u;
                vs[q][t] = have && p < E ? __ldcs(a.val + j0 + p) : 0.0f;
            }
            if (!have) return;  // the sentinel repeats
            if ((ch + 1) * U < E) {
                ++ch;
                return;
            }
            w = nw;  // next worker; take the one after it now
            have = nhave;
            j0 = nj0;
            E = nE;
            ch = 0;
            if (have) {
                nw = a.wctr ? first_round + atomicAdd(a.wctr, 1u) : w + first_round;
                nhave = nw < a.n_workers;
                nj0 = nhave ? __ldg(a.wnz + nw) : 0;
                nE = nhave ? uint32_t(__ldg(a.wnz + nw + 1) - nj0) : 0u;
            }
        };
#pragma unroll
        for (int q = 0; q < PF; ++q) gen(q);
        // emit item q (loaded PF emits ago), then refill lookahead slot q: the
        // slots rotate by unrolling (no register copies, which would stall on
        // the loads still in flight)
        uint32_t it = 0;
        bool fin = false;
        while (!fin) {
#pragma unroll
            for (int q = 0; q < PF; ++q) {
                if (fin) break;
                const uint32_t s = it % D;
                if (it >= uint32_t(D)) mbar_wait(empty + c * D + s, ((it / D) - 1) & 1);
                uint32_t* h = hdr + (c * D + s) * 2;
                h[0] = hw[q];
                h[1] = hc[q];
                float* sv = svals + (c * D + s) * U;
#pragma unroll
                for (int t = 0; t < U; ++t) sv[t] = vs[q][t];
                uint64_t* fb = full + c * D + s;
                if (hw[q] != kSentinel && hn[q]) {
                    float* dst = sdata + (size_t(c) * D + s) * (U * K);
                    mbar_arrive_tx(fb, uint32_t(L::kStageBytes));
                    tma_gather4(dst, &tmap, fb, cs[q][0], cs[q][1], cs[q][2], cs[q][3]);
                    tma_gather4(dst + 4 * K, &tmap, fb, cs[q][4], cs[q][5], cs[q][6], cs[q][7]);
                } else {
                    mbar_arrive(fb);
                }
                ++it;
                if (hw[q] == kSentinel) fin = true;
                else gen(q);
            }
        }
        if (a.wctr && atomicAdd(a.wctr + 1, 1u) == first_round - 1) {  // last slot out resets the schedule
            atomicExch(a.wctr, 0u);
            atomicExch(a.wctr + 1, 0u);
        }
        return;
    }

    // ----------------------------------------------------------- consumers
    const int half = lane >> 4, gl = lane & (G - 1);
    const int c = 2 * warp + half;
    const float* stage_base = sdata + size_t(c) * D * (U * K);
    const int nq = V;  // every lane's blocks are inside K (K = 64 V exactly)

    uint32_t it = 0;
    bool done = false, need = true, wact = false;
    uint32_t i0 = 0, i1 = 0, E = 0, slot = 0, r = 0, rb = 0, rwin = 0, rs_l = 0, rend_l = 0, seg_l = 0;
    uint32_t next_l = 0, pos = 0;
    uint64_t j0 = 0;
    bool inside = false, first = true, have_tot = false;
    F acc, xrow, xnext;
    acc.zero();
    uint32_t xrow_id = 0xffffffffu, xnext_id = 0xffffffffu;

    // (row bookkeeping of spmm_worker_kernel, per half-warp worker)
    auto window = [&](uint32_t rb_) -> uint32_t {
        const uint64_t e = __ldg(a.rp + min(rb_ + 1 + uint32_t(gl), a.n_rows));
        return uint32_t(min(e - j0, uint64_t(E)));
    };
    // row bookkeeping runs half-divergently: its shuffles name only this half
    const unsigned hmask = 0xffffu << (16 * half);
    auto hshfl = [&](uint32_t v, int src) { return __shfl_sync(hmask, v, src, G); };
    auto store_slot = [&](const F& f) {
        f.store(a.slots + uint64_t(slot) * a.ld_slot, gl, K);
        ++slot;
    };
    auto finish_segment = [&]() {
        if (inside) {
            float* crow = a.c + uint64_t(r) * K;
            if (have_tot) {
                F t;
                t.load_own(crow, gl, K);
#pragma unroll
                for (int i = 0; i < N; ++i) t.v[i] = R::combine(t.v[i], acc.v[i]);
                t.store(crow, gl, K);
            } else {
                acc.store(crow, gl, K);
            }
            have_tot = true;
        } else {
            store_slot(acc);
        }
        acc.zero();
        first = true;
    };
    auto finish_row = [&]() {
        if constexpr (SDDMM) return;
        if (inside) {
            const uint64_t deg = rend_l - rs_l;
            float* crow = a.c + uint64_t(r) * K;
            if (have_tot) {
                F t;
                t.load_own(crow, gl, K);
#pragma unroll
                for (int i = 0; i < N; ++i) acc.v[i] = R::combine(t.v[i], acc.v[i]);
            }
#pragma unroll
            for (int i = 0; i < N; ++i) acc.v[i] = R::finish(acc.v[i], deg);
            acc.store(crow, gl, K);
        } else {
            store_slot(acc);
        }
    };
    // rows are contiguous inside a worker: the next row's X is prefetched
    // one row ahead (its load overlaps the current row's batches)
    auto fetch_x = [&]() {
        if (xrow_id == r) return;
        if (xnext_id == r) {
            xrow = xnext;
        } else {
            xrow.load(a.xi + uint64_t(r) * K, gl, K);
        }
        xrow_id = r;
        if (r + 1 < a.n_rows) {
            xnext.load(a.xi + uint64_t(r + 1) * K, gl, K);
            xnext_id = r + 1;
        }
    };
    auto advance_row = [&]() {
        ++r;
        rs_l = rend_l;
        if (r - rb >= uint32_t(G)) {
            rb = r;
            rwin = window(rb);
        }
        rend_l = hshfl(rwin, int(r - rb));
        inside = r < i1;
        seg_l = min(rs_l + uint32_t(SEG), rend_l);
        first = true;
        have_tot = false;
        acc.zero();
    };
    auto settle = [&](uint32_t l) {
        while (l >= rend_l) {
            finish_row();
            advance_row();
        }
        if constexpr (!SDDMM) {
            if (l >= seg_l) {
                finish_segment();
                seg_l = min(seg_l + uint32_t(SEG), rend_l);
            }
            next_l = min(rend_l, seg_l);
        } else {
            next_l = rend_l;
        }
        fetch_x();
    };
    auto start_worker = [&](uint32_t w) {
        i0 = __ldg(a.wrow + w);
        i1 = __ldg(a.wrow + w + 1);
        j0 = __ldg(a.wnz + w);
        E = uint32_t(__ldg(a.wnz + w + 1) - j0);
        slot = a.wslot ? __ldg(a.wslot + w) : 0u;
        r = i0;
        rb = r;
        rwin = window(rb);
        inside = !(__ldg(a.rp + i0) < j0) && r < i1;
        rs_l = 0;
        rend_l = hshfl(rwin, 0);
        seg_l = min(uint32_t(SEG), rend_l);
        next_l = 0;
        first = true;
        have_tot = false;
        acc.zero();
        pos = 0;
        wact = true;
    };
    auto close_worker = [&]() {
        if constexpr (!SDDMM) {
            while (r < i1) {
                finish_row();
                advance_row();
            }
            if (r < a.n_rows && E > rs_l) store_slot(acc);  // head of a split row
        }
        wact = false;
    };

    // LOCK-style loop: the two half-warp workers step together so the batch
    // body's shuffles run with the full warp converged (shuffle offsets stay
    // inside a half); rows / stages are handled half-divergently between.
    while (__any_sync(FULL, !done)) {
        int n = 0;
        uint32_t s = 0, s0 = 0;
        bool release = false;
        if (!done) {
            if (need) {
                s = it % D;
                mbar_wait(full + c * D + s, (it / D) & 1);
                const uint32_t* h = hdr + (c * D + s) * 2;
                const uint32_t hw = h[0], hc = h[1];
                if (hw == kSentinel) {
                    if (wact) close_worker();
                    done = true;
                    release = true;
                } else {
                    if (hc == 0) {
                        if (wact) close_worker();
                        start_worker(hw);
                    }
                    need = false;
                    if (E == 0) {  // a worker without nonzeros: its rows are empty
                        close_worker();
                        release = true;
                    }
                }
            }
            if (!done && !release) {
                s = it % D;
                if (pos >= next_l) settle(pos);
                const uint32_t room = next_l - pos, sroom = uint32_t(U) - (pos % U);
                n = int(min(min(room, sroom), uint32_t(U)));
                s0 = pos % U;
            }
        }
        // ---- batch body: rows s0 .. s0+n-1 of stage s (smem), all lanes
        F yf[U];
        const float* rows = stage_base + size_t(s) * (U * K) + size_t(s0) * K;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (u < n) {
#pragma unroll
                for (int q = 0; q < V; ++q) {
                    const float4 t = reinterpret_cast<const float4*>(rows + size_t(u) * K)[gl + G * q];
                    yf[u].v[4 * q + 0] = t.x;
                    yf[u].v[4 * q + 1] = t.y;
                    yf[u].v[4 * q + 2] = t.z;
                    yf[u].v[4 * q + 3] = t.w;
                }
            } else {
                yf[u].zero();
            }
        }
        constexpr int PER = G / U;  // lanes per nonzero in the transpose-reduce
        const int u_own = gl / PER;
        const float pv_own = u_own < n ? svals[(c * D + s) * U + s0 + u_own] : 0.0f;
        const float d_own = dev::batch_dots(xrow, yf, FULL, gl, nq);
        if constexpr (SDDMM) {
            if (gl % PER == 0 && u_own < n) __stcs(a.out + j0 + pos + uint32_t(u_own), __fmul_rn(pv_own, d_own));
        } else {
            const float s_own = dev::edge_value<EDGE_OP>(pv_own, d_own);
            float sv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) sv[u] = __shfl_sync(FULL, s_own, u * PER, G);
            if (n == U) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    R::fold_fused_all(acc.v, sv[u], yf[u].v, first);
                    first = false;
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (u < n) {
                        R::fold_fused_all(acc.v, sv[u], yf[u].v, first);
                        first = false;
                    }
                }
            }
        }
        if (n > 0) {
            pos += uint32_t(n);
            if (pos % U == 0 || pos == E) release = true;
        }
        __syncwarp();
        if (release) {
            if (gl == 0) mbar_arrive(empty + c * D + (it % D));
            ++it;
            need = true;
        }
    }
}

// ---- host side
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiled>(p);
    }();
    return fn;
}

// Y [rows x K] fp32 row-major as a 2-D tensor with a {K, 1} box (gather4 rows).
bool make_row_map(CUtensorMap* m, const float* y, uint32_t rows, uint32_t k) {
    EncodeTiled enc = encode_fn();
    if (!enc || rows == 0) return false;
    const cuuint64_t dims[2] = {k, rows};
    const cuuint64_t strides[1] = {cuuint64_t(k) * 4};
    const cuuint32_t box[2] = {k, 1};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(y), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr int kNcw = 4;  // consumer warps per CTA (8 ring slots)

template <int V, int OP, int RED, int D>
sgnn_status launch_tma(const TmaArgs& a, const CUtensorMap& map, cudaStream_t s) {
    using L = TmaSmem<V, kNcw, D>;
    static int per_sm = -1;
    auto kern = fused_tma_kernel<V, OP, RED, kNcw, D>;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    if (per_sm < 0) {
        SGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L::kBytes)));
        int nb = 0;
        SGNN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32 * (kNcw + 1), L::kBytes));
        per_sm = std::max(nb, 1);
    }
    const uint64_t want = ceil_div_u64(a.n_workers, 2 * kNcw);
    const uint64_t blocks = std::min<uint64_t>(want, uint64_t(dp.sm_count) * per_sm);
    if (blocks == 0) return SGNN_OK;
    kern<<<unsigned(blocks), 32 * (kNcw + 1), L::kBytes, s>>>(a, map);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

// ring stages per slot (SGNN_TMA_DEPTH = 2, 3 or 4; read per call)
int tma_depth() {
    const char* e = std::getenv("SGNN_TMA_DEPTH");
    const int v = e ? std::atoi(e) : 3;
    return (v == 2 || v == 3 || v == 4) ? v : 3;
}

template <int V, int OP, int RED>
sgnn_status launch_depth(const TmaArgs& a, const CUtensorMap& map, cudaStream_t s) {
    switch (tma_depth()) {
        case 2: return launch_tma<V, OP, RED, 2>(a, map, s);
        case 4: return launch_tma<V, OP, RED, 4>(a, map, s);
        default: return launch_tma<V, OP, RED, 3>(a, map, s);
    }
}

}  // namespace

// Opt-in (SGNN_TMA_FUSED set, read per call): measured slower than the
// register-gather kernels on cfg4 -- 1.77-2.3 ms vs 1.17 ms FusedMM, 1.5-2.2
// vs 0.79 ms SDDMM (scripts/tma_probe.py, profiles/r02_tma_*): the consumers
// spend their issue slots spinning on the full barriers, i.e. the gather4
// rows arrive at ~23 GB/s per SM with 96 stages (192 KB) in flight per SM.
bool tma_fused_enabled() { return std::getenv("SGNN_TMA_FUSED") != nullptr; }

// 1 = ran; 0 = not applicable here (the caller takes the register kernels).
sgnn_status run_fused_tma(const sgnn_csr* p, const float* x, const float* y, uint32_t k, int op, int reduce,
                          float* out, const sgnn_plan_s* plan, cudaStream_t s, bool* ran) {
    *ran = false;
    if (!tma_fused_enabled() || !plan || (k != 64 && k != 128)) return SGNN_OK;
    if (reinterpret_cast<uintptr_t>(x) % 16 || reinterpret_cast<uintptr_t>(y) % 16 ||
        reinterpret_cast<uintptr_t>(out) % 16)
        return SGNN_OK;
    if (op != OP_SDDMM && plan->n_slots && plan->kt < k) return SGNN_OK;
    if (reduce == SGNN_REDUCE_MEAN) reduce = SGNN_REDUCE_SUM;  // the caller runs the divide pass
    CUtensorMap map;
    if (!make_row_map(&map, y, p->n_cols, k)) return SGNN_OK;
    TmaArgs a{};
    a.rp = p->row_ptr;
    a.ci = p->col_idx;
    a.val = p->values;
    a.xi = x;
    a.c = out;
    a.out = out;
    a.slots = plan->slots;
    a.ld_slot = plan->kt;
    a.wrow = plan->wrow;
    a.wnz = plan->wnz;
    a.wslot = plan->wslot;
    a.n_rows = p->n_rows;
    a.n_workers = plan->n_workers;
    a.wctr = plan_counter(plan, s);
    sgnn_status st = SGNN_ERR_UNSUPPORTED;
#define SGNN_TMA_CASE(OPV, OPC, REDV)                                                     \
    if (op == OPC && reduce == REDV) {                                                    \
        st = k == 64 ? launch_depth<1, OPV, REDV>(a, map, s) : launch_depth<2, OPV, REDV>(a, map, s); \
    }
    SGNN_TMA_CASE(OP_SDDMM, OP_SDDMM, SGNN_REDUCE_SUM)
    SGNN_TMA_CASE(dev::OP_FUSED_SIGMOID, dev::OP_FUSED_SIGMOID, SGNN_REDUCE_SUM)
    SGNN_TMA_CASE(dev::OP_FUSED_MUL, dev::OP_FUSED_MUL, SGNN_REDUCE_SUM)
#undef SGNN_TMA_CASE
    if (st == SGNN_ERR_UNSUPPORTED) return SGNN_OK;  // min / max: register kernels
    if (st == SGNN_OK) *ran = true;
    return st;
}

int tma_op_sddmm() { return OP_SDDMM; }

}  // namespace sgnn
