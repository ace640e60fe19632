// plan.cu -- builds the nnz-balanced worker split (see plan.cuh).
#include <algorithm>
#include <cstdlib>

#include "plan.cuh"

namespace sgnn {

namespace {

constexpr uint64_t kSeg = SGNN_SEGMENT;

// Boundary w of the cost-balanced split (parallel.hpp:28-41 cost model,
// at worker granularity, with snapping -- see plan.cuh).
__global__ void plan_coords_kernel(const uint64_t* __restrict__ rp, uint32_t m, uint64_t nnz,
                                   uint64_t d, uint64_t split_t, uint32_t n_workers,
                                   uint32_t* __restrict__ wrow, uint64_t* __restrict__ wnz) {
    const uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w > n_workers) return;
    const uint64_t total = nnz + m;
    const uint64_t b = min(w * d, total);
    if (w == n_workers || b >= total) {
        wrow[w] = m;
        wnz[w] = nnz;
        return;
    }
    // largest r in [0, m) with rp[r] + r <= b
    uint32_t lo = 0, hi = m;
    while (hi - lo > 1) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (__ldg(rp + mid) + mid <= b) lo = mid;
        else hi = mid;
    }
    const uint32_t r = lo;
    const uint64_t rs = __ldg(rp + r), re = __ldg(rp + r + 1);
    const uint64_t deg = re - rs;
    const uint64_t o = b - (rs + r);  // in [0, deg]
    uint32_t outr;
    uint64_t outj;
    if (o == 0) {
        outr = r; outj = rs;
    } else if (deg <= split_t) {
        // short row: never split; snap to the nearer row boundary
        if (2 * o > deg + 1) { outr = r + 1; outj = re; }
        else { outr = r; outj = rs; }
    } else {
        const uint64_t mm = (o / kSeg) * kSeg;  // segment boundary at or below
        if (mm == 0) { outr = r; outj = rs; }
        else if (mm >= deg) { outr = r + 1; outj = re; }
        else { outr = r; outj = rs + mm; }
    }
    wrow[w] = outr;
    wnz[w] = outj;
}

// Per worker: number of segment partials it emits and whether a split row starts in it.
// longest row of the matrix (clamped to u32), for the short-row kernel
__global__ void row_max_degree_kernel(const uint64_t* __restrict__ rp, uint32_t m, uint32_t* __restrict__ out) {
    uint32_t best = 0;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x)
        best = max(best, uint32_t(min(rp[r + 1] - rp[r], uint64_t(0xffffffffu))));
    for (int o = 16; o >= 1; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

__global__ void plan_count_kernel(const uint64_t* __restrict__ rp, uint32_t m, uint32_t n_workers,
                                  const uint32_t* __restrict__ wrow,
                                  const uint64_t* __restrict__ wnz, uint32_t* __restrict__ nslot,
                                  uint32_t* __restrict__ nfix) {
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= n_workers) return;
    const uint32_t i0 = wrow[w], i1 = wrow[w + 1];
    const uint64_t j0 = wnz[w], j1 = wnz[w + 1];
    uint32_t n = 0, f = 0;
    if (i0 < m) {
        const uint64_t rs0 = rp[i0];
        if (j0 > rs0) {  // continuation of a row split before this worker
            const uint64_t end = min(j1, rp[i0 + 1]);
            n += uint32_t((end - j0 + kSeg - 1) / kSeg);
        }
    }
    if (i1 < m) {
        const uint64_t rs1 = rp[i1];
        if (j1 > rs1 && rs1 >= j0) {  // a split row starts here and continues
            n += uint32_t((j1 - rs1) / kSeg);
            f = 1;
        }
    }
    nslot[w] = n;
    nfix[w] = f;
}

__global__ void plan_fix_kernel(const uint64_t* __restrict__ rp, uint32_t m, uint32_t n_workers,
                                const uint32_t* __restrict__ wrow, const uint64_t* __restrict__ wnz,
                                const uint32_t* __restrict__ wslot,
                                const uint32_t* __restrict__ fixscan,
                                uint32_t* __restrict__ fix_row, uint32_t* __restrict__ fix_slot) {
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= n_workers) return;
    if (fixscan[w + 1] == fixscan[w]) return;
    const uint32_t i0 = wrow[w], i1 = wrow[w + 1];
    const uint64_t j0 = wnz[w];
    uint32_t first = 0;
    if (i0 < m && j0 > rp[i0]) {
        const uint64_t end = min(wnz[w + 1], rp[i0 + 1]);
        first = uint32_t((end - j0 + kSeg - 1) / kSeg);
    }
    fix_row[fixscan[w]] = i1;
    fix_slot[fixscan[w]] = wslot[w] + first;
}

// 1 for split rows with more than SGNN_FIXUP_LONG segments (long fixup list)
__global__ void plan_long_flag_kernel(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ fix_row,
                                      uint32_t n_fix, uint32_t* __restrict__ flag) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_fix) return;
    const uint32_t r = fix_row[i];
    flag[i] = (rp[r + 1] - rp[r] + kSeg - 1) / kSeg > SGNN_FIXUP_LONG ? 1u : 0u;
}

__global__ void plan_long_scatter_kernel(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                                         uint32_t n_fix, uint32_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_fix && flag[i]) out[pos[i]] = i;
}

uint32_t pow2_floor(uint64_t v) {
    uint32_t p = 1;
    while (uint64_t(p) * 2 <= v && p < (1u << 30)) p *= 2;
    return p;
}

}  // namespace

void default_params(const sgnn_csr* a, uint32_t k, bool vec_ok, const DeviceProps& dp,
                    sgnn_plan_params* p) {
    sgnn_plan_params d{};
    if (vec_ok && !p->scalar) {
        // one float4 per lane, 8 gathers in flight measured best on B200 (cfg1/cfg2 probes)
        if (k <= 16) { d.lanes = 4; d.vec = 1; }
        else if (k <= 32) { d.lanes = 8; d.vec = 1; }
        else if (k <= 64) { d.lanes = 16; d.vec = 1; }
        else if (k <= 128) { d.lanes = 32; d.vec = 1; }
        else if (k <= 256) { d.lanes = 32; d.vec = 2; }
        else { d.lanes = 32; d.vec = 2; }  // 256-wide passes: cfg2 1.28x (K=512), 1.26x (K=1024) over vec 4
        // 8 gathers in flight except with 4 float4 per lane; two float4 per
        // lane (128 < K <= 256) at the compiler's register allocation: the
        // tuner's choice on cfg2 K=256 (1.04x) and cfg3 (1.08x over U=4 at
        // the 5-CTA cap; profiles/r01_tuning_cfg2.csv, r01_tune_cfg35.log)
        d.unroll = d.vec >= 4 ? 4 : 8;
        // register cap for 5 resident 128-thread CTAs: best or equal on cfg1-cfg4 probes
        if (d.vec == 1 && k > 16) d.occupancy = 5;
    } else {
        d.lanes = 32;
        d.vec = k <= 32 ? 1 : k <= 64 ? 2 : k <= 128 ? 4 : 8;
        d.unroll = d.vec >= 8 ? 2 : 4;
    }
    d.block = 128;
    // Workers per resident lane group (warps take workers dynamically, so
    // shorter workers even out the tail but cost row/segment cuts).  Probes
    // (scripts/sched_probe.py): 16-lane groups 4 (cfg4 FusedMM: 8 is 1.28x
    // slower), 4-lane groups (K <= 16, little work per nonzero) 2 (cfg2
    // tuner: 1.29x over 4); full-warp groups 8, capped below.
    const uint64_t total = a->nnz + a->n_rows;
    const uint64_t groups = uint64_t(dp.sm_count > 0 ? dp.sm_count : 148) *
                            uint64_t(dp.max_threads_per_sm > 0 ? dp.max_threads_per_sm : 2048) /
                            d.lanes;
    // full-warp groups: 8 workers per group at one float4 per lane, 4 at two
    // or more (twice the work per nonzero: cfg3 K=256 tuner, 1024 items
    // 1.08x over 512)
    const uint64_t per_group = d.lanes <= 4 ? 2 : d.lanes == 32 ? (d.vec >= 2 ? 4 : 8) : 4;
    uint64_t want = total / (per_group * groups);
    // full-warp groups: at most 1024 rows+nonzeros per worker (cfg5 tuner:
    // 1.035x over 2048; cfg2 1.55 ms, 8 per group)
    const uint32_t cap = d.lanes == 32 ? 1024 : 4096;
    d.path_items = std::max<uint32_t>(32, std::min<uint32_t>(cap, pow2_floor(std::max<uint64_t>(want, 1))));
    d.split_rows_over = std::max<uint32_t>(d.path_items, SGNN_SEGMENT);
    d.k_tile = 0;
    d.scalar = p->scalar;
    if (!p->lanes) p->lanes = d.lanes;
    if (!p->vec) p->vec = d.vec;
    if (!p->unroll) p->unroll = d.unroll;
    if (!p->path_items) p->path_items = d.path_items;
    if (!p->split_rows_over) p->split_rows_over = std::max<uint32_t>(p->path_items, SGNN_SEGMENT);
    if (!p->block) p->block = d.block;
    // the occupancy default belongs to the default layout only
    if (!p->occupancy && p->lanes == d.lanes && p->vec == d.vec && p->unroll == d.unroll)
        p->occupancy = d.occupancy;
}

sgnn_status resolve_params(const sgnn_csr* a, uint32_t k, bool vec_ok, const DeviceProps& dp,
                           const sgnn_plan_params* in, sgnn_plan_s* plan) {
    sgnn_plan_params p{};
    if (in) p = *in;
    default_params(a, k, vec_ok, dp, &p);
    const bool scalar = p.scalar || !vec_ok;
    if (p.lanes != 4 && p.lanes != 8 && p.lanes != 16 && p.lanes != 32)
        return fail(SGNN_ERR_CONFIG, "plan: lanes must be 4, 8, 16 or 32");
    if (p.vec != 1 && p.vec != 2 && p.vec != 4 && p.vec != 8)
        return fail(SGNN_ERR_CONFIG, "plan: vec must be 1, 2, 4 or 8");
    if (p.unroll != 2 && p.unroll != 4 && p.unroll != 8 && p.unroll != 16)
        return fail(SGNN_ERR_CONFIG, "plan: unroll must be 2, 4, 8 or 16");
    if (p.block != 64 && p.block != 128)
        return fail(SGNN_ERR_CONFIG, "plan: block must be 64 or 128");
    if (p.occupancy > 8 || p.occupancy == 2 || p.occupancy == 3 || p.occupancy == 7)
        return fail(SGNN_ERR_CONFIG, "plan: occupancy must be 0, 1, 4, 5, 6 or 8");
    if (p.path_items == 0) return fail(SGNN_ERR_CONFIG, "plan: path_items must be >= 1");
    const uint32_t width = (scalar ? 1u : 4u) * p.lanes * p.vec;  // floats one pass covers
    uint32_t kt = p.k_tile ? p.k_tile : k;
    kt = std::min(kt, k);
    kt = std::min(kt, width);
    if (!scalar && (kt % 4)) kt = (kt / 4) * 4;
    if (kt == 0) kt = std::min<uint32_t>(k, width);
    plan->p = p;
    plan->p.scalar = scalar ? 1 : 0;
    plan->p.k_tile = kt;
    plan->vec = !scalar;
    plan->kt = kt;
    uint64_t t = std::max<uint64_t>(p.split_rows_over, SGNN_SEGMENT);
    plan->split_T = ceil_div_u64(t, SGNN_SEGMENT) * SGNN_SEGMENT;
    plan->p.split_rows_over = uint32_t(plan->split_T);
    return SGNN_OK;
}

uint32_t* plan_counter(const sgnn_plan_s* p, cudaStream_t s) {
    static const bool off = std::getenv("SGNN_STATIC_SCHEDULE") != nullptr;  // A/B switch
    if (off || !p || !p->wctr || s == cudaStreamPerThread) return nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) {
        (void)cudaGetLastError();
        return nullptr;
    }
    if (cs != cudaStreamCaptureStatusNone) return nullptr;
    const uintptr_t key = reinterpret_cast<uintptr_t>(s) + 1;
    uintptr_t owner = p->ctr_owner.load(std::memory_order_acquire);
    if (owner == 0 && p->ctr_owner.compare_exchange_strong(owner, key, std::memory_order_acq_rel)) return p->wctr;
    return owner == key ? p->wctr : nullptr;
}

bool plan_matches(const sgnn_plan_s* p, const sgnn_csr* a, uint32_t k) {
    return p && p->row_ptr == a->row_ptr && p->n_rows == a->n_rows && p->nnz == a->nnz && p->k == k;
}

void destroy_plan(sgnn_plan_s* p) {
    if (!p) return;
    if (p->mem) cudaFree(p->mem);
    if (p->fmem) cudaFree(p->fmem);
    delete p;
}

sgnn_status build_plan(const sgnn_csr* a, uint32_t k, const sgnn_plan_params* params, bool vec_ok,
                       sgnn_plan_s** out, cudaStream_t s) {
    *out = nullptr;
    SGNN_TRY(check_csr(a, "plan"));
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    auto* plan = new sgnn_plan_s;
    plan->row_ptr = a->row_ptr;
    plan->n_rows = a->n_rows;
    plan->n_cols = a->n_cols;
    plan->nnz = a->nnz;
    plan->k = k;
    sgnn_status st = resolve_params(a, k, vec_ok, dp, params, plan);
    if (st != SGNN_OK) {
        delete plan;
        return st;
    }
    const uint64_t total = a->nnz + a->n_rows;
    const uint64_t nw = ceil_div_u64(total, plan->p.path_items);
    if (nw >= (1ull << 32) - 2) {
        delete plan;
        return fail(SGNN_ERR_CONFIG, "plan: too many workers; raise path_items");
    }
    const uint32_t W = uint32_t(nw);
    plan->n_workers = W;
    // layout: wrow u32[W+1] | wnz u64[W+1] | wslot u32[W+1] | nfix u32[W+1] | fix arrays later
    auto align = [](size_t v) { return (v + 255) & ~size_t(255); };
    const size_t o_wrow = 0;
    const size_t o_wnz = align(o_wrow + sizeof(uint32_t) * (size_t(W) + 1));
    const size_t o_wslot = align(o_wnz + sizeof(uint64_t) * (size_t(W) + 1));
    const size_t o_fscan = align(o_wslot + sizeof(uint32_t) * (size_t(W) + 1));
    const size_t o_ctr = align(o_fscan + sizeof(uint32_t) * (size_t(W) + 1));
    const size_t o_maxd = align(o_ctr + 2 * sizeof(uint32_t));
    const size_t o_end = align(o_maxd + sizeof(uint32_t));
    cudaError_t ce = cudaMalloc(&plan->mem, o_end);
    if (ce != cudaSuccess) {
        delete plan;
        return fail(SGNN_ERR_NOMEM, std::string("plan alloc: ") + cudaGetErrorString(ce));
    }
    char* base = static_cast<char*>(plan->mem);
    plan->wrow = reinterpret_cast<uint32_t*>(base + o_wrow);
    plan->wnz = reinterpret_cast<uint64_t*>(base + o_wnz);
    plan->wslot = reinterpret_cast<uint32_t*>(base + o_wslot);
    uint32_t* fscan = reinterpret_cast<uint32_t*>(base + o_fscan);
    plan->wctr = reinterpret_cast<uint32_t*>(base + o_ctr);
    uint32_t* maxd = reinterpret_cast<uint32_t*>(base + o_maxd);
    ce = cudaMemsetAsync(plan->wctr, 0, o_end - o_ctr, s);  // counters + max degree; ordered by the readback sync below
    if (ce != cudaSuccess) {
        destroy_plan(plan);
        return fail(SGNN_ERR_CUDA, std::string("plan counter: ") + cudaGetErrorString(ce));
    }

    const int tb = 256;
    if (a->n_rows)
        row_max_degree_kernel<<<unsigned(std::min<uint64_t>(ceil_div_u64(a->n_rows, tb), uint64_t(dp.sm_count) * 8)), tb,
                                0, s>>>(a->row_ptr, a->n_rows, maxd);
    plan_coords_kernel<<<unsigned(ceil_div_u64(uint64_t(W) + 1, tb)), tb, 0, s>>>(
        a->row_ptr, a->n_rows, a->nnz, plan->p.path_items, plan->split_T, W, plan->wrow, plan->wnz);
    ce = cudaGetLastError();
    if (ce == cudaSuccess && W > 0) {
        plan_count_kernel<<<unsigned(ceil_div_u64(W, tb)), tb, 0, s>>>(
            a->row_ptr, a->n_rows, W, plan->wrow, plan->wnz, plan->wslot, fscan);
        ce = cudaGetLastError();
    }
    if (ce != cudaSuccess) {
        destroy_plan(plan);
        return fail(SGNN_ERR_CUDA, std::string("plan kernels: ") + cudaGetErrorString(ce));
    }
    st = exclusive_scan_u32(plan->wslot, plan->wslot, W, s);
    if (st == SGNN_OK) st = exclusive_scan_u32(fscan, fscan, W, s);
    if (st != SGNN_OK) {
        destroy_plan(plan);
        return st;
    }
    uint32_t counts[3] = {0, 0, 0};
    ce = cudaMemcpyAsync(&counts[0], plan->wslot + W, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess)
        ce = cudaMemcpyAsync(&counts[1], fscan + W, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(&counts[2], maxd, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) {
        destroy_plan(plan);
        return fail(SGNN_ERR_CUDA, std::string("plan readback: ") + cudaGetErrorString(ce));
    }
    plan->n_slots = counts[0];
    plan->n_fix = counts[1];
    plan->max_deg = counts[2];
    if (plan->n_fix > 0) {
        // fix arrays + slot workspace
        void* fmem = nullptr;
        const size_t fbytes = align(sizeof(uint32_t) * plan->n_fix) * 4 +
                              sizeof(float) * size_t(plan->n_slots) * plan->kt;
        ce = cudaMalloc(&fmem, fbytes);
        if (ce != cudaSuccess) {
            destroy_plan(plan);
            return fail(SGNN_ERR_NOMEM, std::string("plan workspace: ") + cudaGetErrorString(ce));
        }
        plan->fmem = fmem;
        char* fb = static_cast<char*>(fmem);
        plan->fix_row = reinterpret_cast<uint32_t*>(fb);
        plan->fix_slot = reinterpret_cast<uint32_t*>(fb + align(sizeof(uint32_t) * plan->n_fix));
        plan->fix_long = reinterpret_cast<uint32_t*>(fb + 2 * align(sizeof(uint32_t) * plan->n_fix));
        uint32_t* long_pos = reinterpret_cast<uint32_t*>(fb + 3 * align(sizeof(uint32_t) * plan->n_fix));
        plan->slots = reinterpret_cast<float*>(fb + 4 * align(sizeof(uint32_t) * plan->n_fix));
        plan_fix_kernel<<<unsigned(ceil_div_u64(W, tb)), tb, 0, s>>>(
            a->row_ptr, a->n_rows, W, plan->wrow, plan->wnz, plan->wslot, fscan, plan->fix_row,
            plan->fix_slot);
        ce = cudaGetLastError();
        if (ce != cudaSuccess) {
            destroy_plan(plan);
            return fail(SGNN_ERR_CUDA, std::string("plan fix: ") + cudaGetErrorString(ce));
        }
        // compact the long split rows (their fixup gets a CTA each):
        // flags -> exclusive scan (scratch) -> scatter of the fix indices
        const unsigned fb_blocks = unsigned(ceil_div_u64(plan->n_fix, tb));
        uint32_t* pos = nullptr;
        st = scratch_alloc(reinterpret_cast<void**>(&pos), sizeof(uint32_t) * plan->n_fix, s);
        if (st == SGNN_OK) {
            plan_long_flag_kernel<<<fb_blocks, tb, 0, s>>>(a->row_ptr, plan->fix_row, plan->n_fix, long_pos);
            st = exclusive_scan_u32(long_pos, pos, plan->n_fix, s);
        }
        uint32_t last[2] = {0, 0};
        if (st == SGNN_OK &&
            (cudaMemcpyAsync(&last[0], pos + plan->n_fix - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s) !=
                 cudaSuccess ||
             cudaMemcpyAsync(&last[1], long_pos + plan->n_fix - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s) !=
                 cudaSuccess))
            st = fail(SGNN_ERR_CUDA, "plan long rows: readback");
        if (st == SGNN_OK)
            plan_long_scatter_kernel<<<fb_blocks, tb, 0, s>>>(long_pos, pos, plan->n_fix, plan->fix_long);
        if (st == SGNN_OK && cudaStreamSynchronize(s) != cudaSuccess)
            st = fail(SGNN_ERR_CUDA, "plan long rows: sync");
        scratch_free(pos, s);
        if (st != SGNN_OK) {
            destroy_plan(plan);
            return st;
        }
        plan->n_long = last[0] + last[1];
    }
    *out = plan;
    return SGNN_OK;
}

}  // namespace sgnn
