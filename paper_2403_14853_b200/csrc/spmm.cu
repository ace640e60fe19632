// spmm.cu -- host driver of the SpMM worker + fixup kernels (K-tile passes),
// and the Mean epilogue.
//
// Mean (kernels.hpp:60-63): the mean kernels divide by the row's nonzero
// count where the row is stored (dev::div_by_count, bit-identical to
// __fdiv_rn without its slow-path call); layouts without a mean kernel, the
// peer path and FusedMM run the Sum kernels and one divide pass over C.
#include <algorithm>
#include <cstdlib>

#include "ops.cuh"
#include "plan.cuh"
#include "spmm_inst.cuh"

namespace sgnn {

namespace {

// C[r, :] /= deg(r) for rows with deg > 0 (empty rows already hold 0).
// One warp per row; float4 when the row is 16-byte aligned.
__global__ void __launch_bounds__(256) mean_divide_kernel(const uint64_t* __restrict__ rp, uint32_t m,
                                                          float* __restrict__ c, uint64_t ldc,
                                                          uint32_t k, bool vec) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t n_warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m; r += n_warps) {
        const uint64_t deg = __ldg(rp + r + 1) - __ldg(rp + r);
        if (!deg) continue;
        const float d = float(deg);
        float* row = c + uint64_t(r) * ldc;
        if (vec) {
            float4* row4 = reinterpret_cast<float4*>(row);
            for (uint32_t q = lane; q < k / 4; q += 32) {
                float4 t = row4[q];
                t.x = __fdiv_rn(t.x, d); t.y = __fdiv_rn(t.y, d);
                t.z = __fdiv_rn(t.z, d); t.w = __fdiv_rn(t.w, d);
                row4[q] = t;
            }
        } else {
            for (uint32_t q = lane; q < k; q += 32) row[q] = __fdiv_rn(row[q], d);
        }
    }
}

// The lockstep worker (dev::lock_worker_kernel) for 8- and 16-lane groups
template <int G, int RED>
sgnn_status launch_spmm_lock(const SpmmArgs& a, uint32_t block, cudaStream_t s) {
    constexpr int MINB = 5;
    static int per_sm = -1;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    if (per_sm < 0) {
        int n = 0;
        SGNN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &n, dev::lock_worker_kernel<G, 8, dev::OP_SPMM, RED, MINB>, 128, 0));
        per_sm = std::max(n, 1);
    }
    (void)block;
    const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(uint64_t(a.n_workers) * G, 128), uint64_t(dp.sm_count) * per_sm);
    if (blocks == 0) return SGNN_OK;
    dev::lock_worker_kernel<G, 8, dev::OP_SPMM, RED, MINB><<<unsigned(blocks), 128, 0, s>>>(a);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

template <int RED>
sgnn_status spmm_lock_red(int lanes, const SpmmArgs& a, uint32_t block, cudaStream_t s) {
    return lanes == 8 ? launch_spmm_lock<8, RED>(a, block, s) : launch_spmm_lock<16, RED>(a, block, s);
}

sgnn_status run_spmm_lock(int lanes, int reduce, const SpmmArgs& a, uint32_t block, cudaStream_t s) {
    switch (reduce) {
        case SGNN_REDUCE_SUM: return spmm_lock_red<SGNN_REDUCE_SUM>(lanes, a, block, s);
        case SGNN_REDUCE_MEAN: return spmm_lock_red<SGNN_REDUCE_MEAN>(lanes, a, block, s);
        case SGNN_REDUCE_MIN: return spmm_lock_red<SGNN_REDUCE_MIN>(lanes, a, block, s);
        case SGNN_REDUCE_MAX: return spmm_lock_red<SGNN_REDUCE_MAX>(lanes, a, block, s);
    }
    return fail(SGNN_ERR_CONFIG, "unknown reduce op");
}

template <int G, int RED>
sgnn_status launch_short_rows(const SpmmArgs& a, cudaStream_t s) {
    static int per_sm = -1;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    if (per_sm < 0) {
        int n = 0;
        SGNN_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, dev::spmm_short_rows_kernel<G, 8, RED>, 128, 0));
        per_sm = std::max(n, 1);
    }
    const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(uint64_t(a.n_rows) * G, 128), uint64_t(dp.sm_count) * per_sm);
    if (blocks == 0) return SGNN_OK;
    dev::spmm_short_rows_kernel<G, 8, RED><<<unsigned(blocks), 128, 0, s>>>(a);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

template <int RED>
sgnn_status short_rows_red(int lanes, const SpmmArgs& a, cudaStream_t s) {
    switch (lanes) {
        case 4: return launch_short_rows<4, RED>(a, s);
        case 8: return launch_short_rows<8, RED>(a, s);
        case 16: return launch_short_rows<16, RED>(a, s);
        case 32: return launch_short_rows<32, RED>(a, s);
    }
    return fail(SGNN_ERR_UNSUPPORTED, "short rows: lanes");
}

sgnn_status run_short_rows(int lanes, int reduce, const SpmmArgs& a, cudaStream_t s) {
    switch (reduce) {
        case SGNN_REDUCE_SUM: return short_rows_red<SGNN_REDUCE_SUM>(lanes, a, s);
        case SGNN_REDUCE_MEAN: return short_rows_red<SGNN_REDUCE_MEAN>(lanes, a, s);
        case SGNN_REDUCE_MIN: return short_rows_red<SGNN_REDUCE_MIN>(lanes, a, s);
        case SGNN_REDUCE_MAX: return short_rows_red<SGNN_REDUCE_MAX>(lanes, a, s);
    }
    return fail(SGNN_ERR_CONFIG, "unknown reduce op");
}

}  // namespace

// Self-test of the mean epilogue's division (dev::div_by_count) against
// __fdiv_rn: degrees [d0, d1) x `samples` values per degree (a counter-hashed
// mix of random bit patterns -- every exponent, subnormals, signs -- and the
// specials 0, -0, +-inf, NaN, +-FLT_MAX, +-FLT_MIN, +-denorm_min).
__global__ void count_division_check_kernel(uint64_t d0, uint64_t d1, uint32_t samples, uint64_t seed,
                                            unsigned long long* bad, unsigned long long* first_bad) {
    const uint64_t n = (d1 - d0) * samples;
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t deg = d0 + t / samples;
        const uint32_t j = uint32_t(t % samples);
        uint32_t bits;
        constexpr uint32_t kSpecial[] = {0x00000000u, 0x80000000u, 0x7f800000u, 0xff800000u, 0x7fc00000u,
                                         0x7f7fffffu, 0xff7fffffu, 0x00800000u, 0x80800000u, 0x00000001u,
                                         0x80000001u, 0x3f800000u, 0x007fffffu};
        if (j < sizeof(kSpecial) / sizeof(kSpecial[0])) {
            bits = kSpecial[j];
        } else {
            uint64_t z = seed + t * 0x9E3779B97F4A7C15ull;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            z ^= z >> 31;
            bits = uint32_t(z);
            if (j & 1) bits = (bits & 0x807fffffu) | (uint32_t(96 + (z >> 40) % 64) << 23);  // |v| ~ 2^-31..2^32
        }
        const float v = __uint_as_float(bits);
        const float want = __fdiv_rn(v, float(deg));
        const float got = dev::div_by_count(v, dev::recip_count(deg), float(deg));
        const bool same = __float_as_uint(want) == __float_as_uint(got) || (want != want && got != got);
        if (!same) {
            atomicAdd(bad, 1ull);
            atomicMin(first_bad, (unsigned long long)t);
        }
    }
}

sgnn_status selftest_count_division(uint64_t d0, uint64_t d1, uint32_t samples, uint64_t seed, uint64_t* mismatches,
                                    uint64_t* first_deg, uint32_t* first_bits) {
    if (d0 == 0 || d1 <= d0 || samples == 0) return fail(SGNN_ERR_CONFIG, "selftest: need 0 < d0 < d1, samples > 0");
    unsigned long long* buf = nullptr;
    SGNN_CUDA_TRY(cudaMalloc(&buf, 2 * sizeof(unsigned long long)));
    unsigned long long h[2] = {0ull, ~0ull};
    cudaMemcpy(buf, h, sizeof(h), cudaMemcpyHostToDevice);
    count_division_check_kernel<<<148 * 16, 256>>>(d0, d1, samples, seed, buf, buf + 1);
    const cudaError_t e = cudaMemcpy(h, buf, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(buf);
    if (e != cudaSuccess) return fail(SGNN_ERR_CUDA, std::string("selftest: ") + cudaGetErrorString(e));
    *mismatches = h[0];
    if (first_deg) *first_deg = h[0] ? d0 + h[1] / samples : 0;
    if (first_bits) *first_bits = h[0] ? uint32_t(h[1] % samples) : 0;
    return SGNN_OK;
}

sgnn_status run_mean_divide(const uint64_t* rp, uint32_t m, float* c, uint64_t ldc, uint32_t k,
                            cudaStream_t s) {
    if (m == 0 || k == 0) return SGNN_OK;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(uint64_t(m) * 32, 256), uint64_t(dp.sm_count) * 16);
    const bool vec = (k % 4 == 0) && (ldc % 4 == 0) && (reinterpret_cast<uintptr_t>(c) % 16 == 0);
    mean_divide_kernel<<<unsigned(blocks), 256, 0, s>>>(rp, m, c, ldc, k, vec);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

SpmmLauncher find_spmm_launcher(bool vec, int lanes, int vregs, int unroll, int reduce, int occ) {
    switch (reduce) {
        case SGNN_REDUCE_SUM: return spmm_lookup_sum(vec, lanes, vregs, unroll, occ);
        case SGNN_REDUCE_MEAN: return spmm_lookup_mean(vec, lanes, vregs, unroll, occ);
        case SGNN_REDUCE_MIN: return spmm_lookup_min(vec, lanes, vregs, unroll, occ);
        case SGNN_REDUCE_MAX: return spmm_lookup_max(vec, lanes, vregs, unroll, occ);
    }
    return nullptr;
}

sgnn_status launch_spmm_fixup(const FixupArgs& f, int reduce, cudaStream_t s) {
    switch (reduce) {
        case SGNN_REDUCE_SUM: return spmm_lookup_sum_fixup(f, s);
        case SGNN_REDUCE_MEAN: return spmm_lookup_mean_fixup(f, s);
        case SGNN_REDUCE_MIN: return spmm_lookup_min_fixup(f, s);
        case SGNN_REDUCE_MAX: return spmm_lookup_max_fixup(f, s);
    }
    return fail(SGNN_ERR_CONFIG, "unknown reduce op");
}

sgnn_status run_spmm(const sgnn_csr* a, const float* x, uint32_t k, float* c, int reduce,
                     const sgnn_plan_s* plan, cudaStream_t s) {
    return run_spmm_ld(a, x, k, k, c, k, reduce, plan, s);
}

sgnn_status run_spmm_ld(const sgnn_csr* a, const float* x, uint64_t ldx, uint32_t k, float* c, uint64_t ldc,
                        int reduce, const sgnn_plan_s* plan, cudaStream_t s) {
    if (ldx < k || ldc < k) return fail(SGNN_ERR_CONFIG, "spmm: row strides must be >= K");
    if (reduce < 0 || reduce > 3) return fail(SGNN_ERR_CONFIG, "spmm: unknown reduce op");
    if (k == 0 || a->n_rows == 0) return SGNN_OK;
    if (!plan_matches(plan, a, k))
        return fail(SGNN_ERR_DISPATCH, "spmm: plan was built for another matrix or K");
    const bool aligned = (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(c) % 16 == 0) && (k % 4 == 0) && (ldx % 4 == 0) &&
                         (ldc % 4 == 0);
    const bool vec = plan->vec && aligned;
    int lanes = int(plan->p.lanes), vregs = int(plan->p.vec), unroll = int(plan->p.unroll);
    if (!vec) {
        lanes = 32;
        if (plan->vec) {  // float4 plan on misaligned operands: scalar kernel, same split
            vregs = std::min<int>(8, int(ceil_div_u64(plan->kt, 32)));
            vregs = vregs <= 1 ? 1 : vregs <= 2 ? 2 : vregs <= 4 ? 4 : 8;
            unroll = vregs >= 4 ? 2 : 4;
        }
    }
    // register-capped variants exist for sum (and hence mean); min/max use
    // the uncapped kernel of the same layout (occupancy is not numerics)
    const int occ = vec ? int(plan->p.occupancy) : 1;
    SpmmLauncher launch = find_spmm_launcher(vec, lanes, vregs, unroll, reduce, occ);
    if (!launch && occ > 1) launch = find_spmm_launcher(vec, lanes, vregs, unroll, reduce, 1);
    // mean: the divide happens in the row epilogue of the mean kernels; a
    // layout without one runs the sum kernels and the divide pass
    int kred = reduce;
    if (!launch && reduce == SGNN_REDUCE_MEAN) {
        kred = SGNN_REDUCE_SUM;
        launch = find_spmm_launcher(vec, lanes, vregs, unroll, kred, occ);
        if (!launch && occ > 1) launch = find_spmm_launcher(vec, lanes, vregs, unroll, kred, 1);
    }
    if (!launch)
        return fail(SGNN_ERR_UNSUPPORTED, "spmm: no kernel compiled for lanes=" +
                                              std::to_string(lanes) + " vec=" +
                                              std::to_string(vregs) + " unroll=" +
                                              std::to_string(unroll));
    const uint32_t kernel_width = uint32_t((vec ? 4 : 1) * lanes * vregs);
    // Small short-row matrices (every row <= 2 G nonzeros, every row's group
    // resident at once): the short-row kernel -- three dependent loads per row
    // instead of the worker's metadata / row window / (col, val) / gather
    // chain (cfg1: 14.4 -> 10.2 us, bitwise the same).  Larger ones keep the
    // worker (equal or faster once rows outnumber the resident groups).
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    const uint64_t resident = uint64_t(dp.sm_count) * uint64_t(dp.max_threads_per_sm > 0 ? dp.max_threads_per_sm : 2048);
    const bool no_short = std::getenv("SGNN_NO_SHORT_ROWS") != nullptr;  // A/B switch (tests)
    if (!no_short && vec && vregs == 1 && plan->kt == k && kernel_width >= k && plan->n_fix == 0 &&
        plan->max_deg <= uint32_t(2 * lanes) && uint64_t(a->n_rows) * lanes <= resident) {
        SpmmArgs args{};
        args.rp = a->row_ptr;
        args.ci = a->col_idx;
        args.val = a->values;
        args.x = x;
        args.c = c;
        args.n_rows = a->n_rows;
        args.ldx = ldx;
        args.ldc = ldc;
        args.width = k;
        return run_short_rows(lanes, reduce, args, s);
    }

    for (uint32_t k0 = 0; k0 < k; k0 += plan->kt) {
        const uint32_t kp = std::min(plan->kt, k - k0);
        for (uint32_t sk = 0; sk < kp; sk += kernel_width) {
            SpmmArgs args{};
            args.rp = a->row_ptr;
            args.ci = a->col_idx;
            args.val = a->values;
            args.x = x + k0 + sk;
            args.c = c + k0 + sk;
            args.slots = plan->slots ? plan->slots + sk : nullptr;
            args.wrow = plan->wrow;
            args.wnz = plan->wnz;
            args.wslot = plan->wslot;
            args.n_rows = a->n_rows;
            args.n_workers = plan->n_workers;
            args.wctr = plan_counter(plan, s);
            args.ldx = ldx;
            args.ldc = ldc;
            args.ld_slot = plan->kt;
            args.width = std::min(kernel_width, kp - sk);
            // 8- / 16-lane groups at one float4 per lane: the lockstep worker
            // (same results; fewer instructions per batch)
            const bool lock = vec && vregs == 1 && unroll == 8 && (lanes == 8 || lanes == 16) &&
                              !std::getenv("SGNN_LOCK_GENERIC");  // A/B switch (tests)
            if (lock) SGNN_TRY(run_spmm_lock(lanes, kred, args, plan->p.block, s));
            else SGNN_TRY(launch(args, plan->p.block, 0, s));
        }
        if (plan->n_fix) {
            FixupArgs f;
            f.rp = a->row_ptr;
            f.fix_row = plan->fix_row;
            f.fix_slot = plan->fix_slot;
            f.fix_long = plan->fix_long;
            f.n_long = plan->n_long;
            f.slots = plan->slots;
            f.c = c + k0;
            f.ldc = ldc;
            f.ld_slot = plan->kt;
            f.n_fix = plan->n_fix;
            f.width = kp;
            SGNN_TRY(launch_spmm_fixup(f, kred, s));
        }
    }
    if (reduce == SGNN_REDUCE_MEAN && kred != reduce) SGNN_TRY(run_mean_divide(a->row_ptr, a->n_rows, c, ldc, k, s));
    return SGNN_OK;
}

sgnn_status run_spmm_peer(const sgnn_csr* a, const float* const* parts, uint32_t n_parts,
                          uint32_t part_shift, uint32_t k, float* c, int reduce,
                          const sgnn_plan_s* plan, cudaStream_t s) {
    if (reduce != SGNN_REDUCE_SUM && reduce != SGNN_REDUCE_MEAN)
        return fail(SGNN_ERR_UNSUPPORTED, "spmm_peer: sum and mean only");
    if (n_parts == 0 || n_parts > SGNN_MAX_PEERS)
        return fail(SGNN_ERR_CONFIG, "spmm_peer: 1.." + std::to_string(SGNN_MAX_PEERS) + " parts");
    if (part_shift > 31 || (uint64_t(n_parts) << part_shift) < a->n_cols)
        return fail(SGNN_ERR_SHAPE, "spmm_peer: n_parts << part_shift must cover the remapped columns");
    if (k == 0 || a->n_rows == 0) return SGNN_OK;
    if (!plan_matches(plan, a, k))
        return fail(SGNN_ERR_DISPATCH, "spmm_peer: plan was built for another matrix or K");
    bool aligned = (reinterpret_cast<uintptr_t>(c) % 16 == 0) && (k % 4 == 0);
    for (uint32_t i = 0; i < n_parts; ++i) aligned &= reinterpret_cast<uintptr_t>(parts[i]) % 16 == 0;
    const bool vec = plan->vec && aligned;
    int lanes = int(plan->p.lanes), vregs = int(plan->p.vec), unroll = int(plan->p.unroll);
    if (!vec) {
        lanes = 32;
        vregs = std::min<int>(8, int(ceil_div_u64(plan->kt, 32)));
        vregs = vregs <= 1 ? 1 : vregs <= 2 ? 2 : vregs <= 4 ? 4 : 8;
        unroll = vregs >= 4 ? 2 : 4;
    }
    SpmmLauncher launch = spmm_peer_lookup_sum(vec, lanes, vregs, unroll, vec ? int(plan->p.occupancy) : 1);
    // peer kernels carry the part table: they are compiled at occupancy 4 / 1
    if (!launch && vec) launch = spmm_peer_lookup_sum(vec, lanes, vregs, unroll, 4);
    if (!launch && vec) launch = spmm_peer_lookup_sum(vec, lanes, vregs, unroll, 1);
    if (!launch)
        return fail(SGNN_ERR_UNSUPPORTED, "spmm_peer: no peer kernel for lanes=" + std::to_string(lanes) +
                                              " vec=" + std::to_string(vregs) + " unroll=" + std::to_string(unroll));
    const uint32_t kernel_width = uint32_t((vec ? 4 : 1) * lanes * vregs);
    for (uint32_t k0 = 0; k0 < k; k0 += plan->kt) {
        const uint32_t kp = std::min(plan->kt, k - k0);
        for (uint32_t sk = 0; sk < kp; sk += kernel_width) {
            SpmmArgs args{};
            args.rp = a->row_ptr;
            args.ci = a->col_idx;
            args.val = a->values;
            args.x = parts[0] + k0 + sk;  // (unused base for the lane clamp)
            for (uint32_t i = 0; i < n_parts; ++i) args.xparts[i] = parts[i] + k0 + sk;
            args.part_shift = part_shift;
            args.c = c + k0 + sk;
            args.slots = plan->slots ? plan->slots + sk : nullptr;
            args.wrow = plan->wrow;
            args.wnz = plan->wnz;
            args.wslot = plan->wslot;
            args.n_rows = a->n_rows;
            args.n_workers = plan->n_workers;
            args.wctr = plan_counter(plan, s);
            args.ldx = k;
            args.ldc = k;
            args.ld_slot = plan->kt;
            args.width = std::min(kernel_width, kp - sk);
            SGNN_TRY(launch(args, plan->p.block, 0, s));
        }
        if (plan->n_fix) {
            FixupArgs f;
            f.rp = a->row_ptr;
            f.fix_row = plan->fix_row;
            f.fix_slot = plan->fix_slot;
            f.fix_long = plan->fix_long;
            f.n_long = plan->n_long;
            f.slots = plan->slots;
            f.c = c + k0;
            f.ldc = k;
            f.ld_slot = plan->kt;
            f.n_fix = plan->n_fix;
            f.width = kp;
            SGNN_TRY(launch_spmm_fixup(f, SGNN_REDUCE_SUM, s));
        }
    }
    if (reduce == SGNN_REDUCE_MEAN) SGNN_TRY(run_mean_divide(a->row_ptr, a->n_rows, c, k, k, s));
    return SGNN_OK;
}

}  // namespace sgnn
