// normalize.cu -- normalize_adjacency (sparse.hpp:116-174) on the device:
// A_hat = D^-1/2 (A + I) D^-1/2, bit-exact with the reference.
//
//  1. per row: binary-search the diagonal, count (deg + missing diagonal)
//  2. exclusive scan -> row_ptr of A + I
//  3. one warp per row: copy the row, inserting the diagonal at its sorted
//     place (or adding 1 to an existing one), exactly like sparse.hpp:131-149
//  4. one thread per row: d_i = sum of the row's values in double, in row
//     order (sparse.hpp:157-161), s_i = 1/sqrt(d_i) (0 for d_i = 0)
//  5. one warp per row: v = float(double(v) * (s_i * s_j)) (sparse.hpp:165-171)
// All arithmetic uses the same IEEE operations in the same order as the
// reference, so the result is bitwise identical.
#include <algorithm>

#include "ops.cuh"

namespace sgnn {
namespace {

__device__ __forceinline__ uint64_t lower_bound_col(const uint32_t* __restrict__ ci, uint64_t lo,
                                                    uint64_t hi, uint32_t key) {
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (__ldg(ci + mid) < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void norm_count_kernel(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                                  const float* __restrict__ v, uint32_t n, int add_loops,
                                  uint32_t* __restrict__ cnt, int* __restrict__ bad) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t lo = rp[i], hi = rp[i + 1];
        uint32_t c = uint32_t(hi - lo);
        if (add_loops) {
            const uint64_t p = lower_bound_col(ci, lo, hi, i);
            if (p == hi || __ldg(ci + p) != i) ++c;
        }
        cnt[i] = c;
        for (uint64_t e = lo; e < hi; ++e)  // sparse.hpp:122-123
            if (__ldg(v + e) < 0.0f) { atomicExch(bad, 1); break; }
    }
}

__global__ void norm_copy_kernel(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                                 const float* __restrict__ v, uint32_t n, int add_loops,
                                 const uint64_t* __restrict__ trp, uint32_t* __restrict__ tci,
                                 float* __restrict__ tv) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t n_warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += n_warps) {
        const uint64_t lo = rp[i], hi = rp[i + 1], out = trp[i];
        uint64_t p = hi;
        bool has = false;
        if (add_loops) {
            p = lower_bound_col(ci, lo, hi, i);
            has = p < hi && __ldg(ci + p) == i;
        }
        const bool insert = add_loops && !has;
        for (uint64_t e = lo + lane; e < hi; e += 32) {
            const uint32_t j = __ldg(ci + e);
            float x = __ldg(v + e);
            if (add_loops && j == i) x = __fadd_rn(x, 1.0f);  // a_ii + 1 (sparse.hpp:136)
            const uint64_t o = out + (e - lo) + ((insert && e >= p) ? 1 : 0);
            tci[o] = j;
            tv[o] = x;
        }
        if (insert && lane == 0) {
            tci[out + (p - lo)] = i;
            tv[out + (p - lo)] = 1.0f;
        }
    }
}

__global__ void norm_scale_kernel(const uint64_t* __restrict__ trp, const float* __restrict__ tv,
                                  uint32_t n, double* __restrict__ inv) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double d = 0.0;
        for (uint64_t e = trp[i]; e < trp[i + 1]; ++e) d = __dadd_rn(d, double(tv[e]));
        inv[i] = d > 0 ? __ddiv_rn(1.0, __dsqrt_rn(d)) : 0.0;
    }
}

__global__ void norm_apply_kernel(const uint64_t* __restrict__ trp, const uint32_t* __restrict__ tci,
                                  float* __restrict__ tv, uint32_t n, const double* __restrict__ inv) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t n_warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += n_warps) {
        const double si = inv[i];
        for (uint64_t e = trp[i] + lane; e < trp[i + 1]; e += 32)
            tv[e] = __double2float_rn(__dmul_rn(double(tv[e]), __dmul_rn(si, __ldg(inv + tci[e]))));
    }
}

}  // namespace

sgnn_status run_normalize_count(const sgnn_csr* a, int add_loops, uint32_t* cnt, int* bad,
                                cudaStream_t s) {
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    const unsigned blocks = unsigned(std::min<uint64_t>(ceil_div_u64(a->n_rows, 256), uint64_t(dp.sm_count) * 8));
    if (a->n_rows) norm_count_kernel<<<blocks, 256, 0, s>>>(a->row_ptr, a->col_idx, a->values, a->n_rows, add_loops, cnt, bad);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

sgnn_status run_normalize(const sgnn_csr* a, int add_loops, uint64_t* out_nnz, uint64_t* trp,
                          uint32_t* tci, float* tv, cudaStream_t s) {
    if (a->n_rows != a->n_cols)
        return fail(SGNN_ERR_SHAPE, "normalize_adjacency: matrix is " + std::to_string(a->n_rows) + "x" +
                                        std::to_string(a->n_cols) + ", expected square");
    const uint32_t n = a->n_rows;
    uint32_t* cnt = nullptr;
    uint64_t* scan = nullptr;
    int* bad = nullptr;
    double* inv = nullptr;
    sgnn_status st = scratch_alloc(reinterpret_cast<void**>(&cnt), sizeof(uint32_t) * (size_t(n) + 1), s);
    if (st == SGNN_OK) st = scratch_alloc(reinterpret_cast<void**>(&scan), sizeof(uint64_t) * (size_t(n) + 1), s);
    if (st == SGNN_OK) st = scratch_alloc(reinterpret_cast<void**>(&bad), sizeof(int), s);
    if (st == SGNN_OK && cudaMemsetAsync(bad, 0, sizeof(int), s) != cudaSuccess) st = fail(SGNN_ERR_CUDA, "memset");
    if (st == SGNN_OK) st = run_normalize_count(a, add_loops, cnt, bad, s);
    if (st == SGNN_OK) st = exclusive_scan_u32_to_u64(cnt, trp ? trp : scan, n, s);
    int hbad = 0;
    uint64_t total = 0;
    if (st == SGNN_OK) {
        const uint64_t* tot = (trp ? trp : scan) + n;
        if (cudaMemcpyAsync(&total, tot, sizeof(uint64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            st = fail(SGNN_ERR_CUDA, "normalize_adjacency: readback failed");
    }
    if (st == SGNN_OK && hbad) st = fail(SGNN_ERR_CONFIG, "normalize_adjacency: negative edge value");
    if (st == SGNN_OK) *out_nnz = total;
    if (st == SGNN_OK && trp && n) {
        DeviceProps dp;
        st = device_props(&dp);
        if (st == SGNN_OK) st = scratch_alloc(reinterpret_cast<void**>(&inv), sizeof(double) * n, s);
        if (st == SGNN_OK) {
            const unsigned wb = unsigned(std::min<uint64_t>(ceil_div_u64(uint64_t(n) * 32, 256), uint64_t(dp.sm_count) * 16));
            const unsigned tb = unsigned(std::min<uint64_t>(ceil_div_u64(n, 256), uint64_t(dp.sm_count) * 8));
            norm_copy_kernel<<<wb, 256, 0, s>>>(a->row_ptr, a->col_idx, a->values, n, add_loops, trp, tci, tv);
            norm_scale_kernel<<<tb, 256, 0, s>>>(trp, tv, n, inv);
            norm_apply_kernel<<<wb, 256, 0, s>>>(trp, tci, tv, n, inv);
            if (cudaGetLastError() != cudaSuccess) st = fail(SGNN_ERR_CUDA, "normalize_adjacency: launch failed");
        }
    }
    scratch_free(cnt, s);
    scratch_free(scan, s);
    scratch_free(bad, s);
    scratch_free(inv, s);
    return st;
}

}  // namespace sgnn
