// runtime.cu -- error state, device properties, scratch memory and the
// device-wide exclusive scans used by the planner and the transpose.
#include <mutex>

#include "common.cuh"

namespace sgnn {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

sgnn_status device_props(DeviceProps* out) {
    static std::mutex mu;
    static DeviceProps cache[64];
    static bool have[64] = {};
    int dev = 0;
    SGNN_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 0 || dev >= 64) return fail(SGNN_ERR_CUDA, "device ordinal out of range");
    if (!have[dev]) {
        DeviceProps p;
        SGNN_CUDA_TRY(cudaDeviceGetAttribute(&p.sm_count, cudaDevAttrMultiProcessorCount, dev));
        SGNN_CUDA_TRY(cudaDeviceGetAttribute(&p.l2_bytes, cudaDevAttrL2CacheSize, dev));
        SGNN_CUDA_TRY(cudaDeviceGetAttribute(&p.cc_major, cudaDevAttrComputeCapabilityMajor, dev));
        SGNN_CUDA_TRY(cudaDeviceGetAttribute(&p.cc_minor, cudaDevAttrComputeCapabilityMinor, dev));
        SGNN_CUDA_TRY(cudaDeviceGetAttribute(&p.max_threads_per_sm,
                                             cudaDevAttrMaxThreadsPerMultiProcessor, dev));
        if (p.cc_major != 10)
            return fail(SGNN_ERR_CUDA, "this library is built for sm_100a (B200); device has cc " +
                                           std::to_string(p.cc_major) + "." +
                                           std::to_string(p.cc_minor));
        // Scratch comes from the device's default stream-ordered pool; keep
        // freed blocks in the pool (no release back to the driver at every
        // synchronisation), so repeated plan / transpose / cache builds reuse
        // their workspace instead of re-mapping it.
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cache[dev] = p;
        have[dev] = true;
    }
    *out = cache[dev];
    return SGNN_OK;
}

sgnn_status scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
    *p = nullptr;
    if (bytes == 0) return SGNN_OK;
    SGNN_CUDA_TRY(cudaMallocAsync(p, bytes, s));
    return SGNN_OK;
}

void scratch_free(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

sgnn_status check_csr(const sgnn_csr* a, const char* what) {
    if (!a) return fail(SGNN_ERR_CONFIG, std::string(what) + ": null csr");
    if (!a->row_ptr) return fail(SGNN_ERR_CONFIG, std::string(what) + ": null row_ptr");
    if (a->nnz > 0 && (!a->col_idx || !a->values))
        return fail(SGNN_ERR_CONFIG, std::string(what) + ": null col_idx/values with nnz > 0");
    return SGNN_OK;
}

// ------------------------------------------------------------------ scans
namespace {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr uint64_t kScanTile = uint64_t(kScanThreads) * kScanItems;

template <class T>
__device__ __forceinline__ T warp_inclusive(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread; returns the block total too.
template <class T>
__device__ __forceinline__ T block_exclusive(T v, T* total) {
    __shared__ T warp_sums[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const T inc = warp_inclusive(v);
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        T s = lane < nw ? warp_sums[lane] : T(0);
        s = warp_inclusive(s);
        if (lane < nw) warp_sums[lane] = s;
    }
    __syncthreads();
    const T prefix = (wid > 0 ? warp_sums[wid - 1] : T(0)) + inc - v;
    *total = warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
    return prefix;
}

template <class TIn, class TOut>
__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const TIn* __restrict__ in,
                                                                   uint64_t n,
                                                                   TOut* __restrict__ sums) {
    const uint64_t base = uint64_t(blockIdx.x) * kScanTile;
    TOut s = 0;
    for (int i = 0; i < kScanItems; ++i) {
        const uint64_t idx = base + uint64_t(i) * kScanThreads + threadIdx.x;
        if (idx < n) s += TOut(in[idx]);
    }
    TOut total;
    block_exclusive(s, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// Exclusive scan of each tile plus its block offset.  If offsets == nullptr,
// there is exactly one block with offset 0.  Thread t handles the blocked
// items [t*kScanItems, (t+1)*kScanItems) of the tile.
template <class TIn, class TOut>
__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(const TIn* in, TOut* out,
                                                                 uint64_t n,
                                                                 const TOut* __restrict__ offsets) {
    const uint64_t base = uint64_t(blockIdx.x) * kScanTile + uint64_t(threadIdx.x) * kScanItems;
    // a thread's 8 consecutive items move as 16-byte vectors when the whole
    // run is in range and aligned (a scalar blocked load touches 8 sectors
    // per warp instruction)
    const bool vin = sizeof(TIn) == 4 && base + kScanItems <= n &&
                     (reinterpret_cast<uintptr_t>(in + base) & 15) == 0;
    const bool vout = base + kScanItems <= n && (reinterpret_cast<uintptr_t>(out + base) & 15) == 0 &&
                      (sizeof(TOut) == 4 || sizeof(TOut) == 8);
    TOut vals[kScanItems];
    TOut s = 0;
    if (vin) {
        static_assert(kScanItems == 8, "two 16-byte vectors per thread");
        const uint4 a = *reinterpret_cast<const uint4*>(in + base);
        const uint4 b = *reinterpret_cast<const uint4*>(in + base + 4);
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            vals[i] = TOut(w[i]);
            s += vals[i];
        }
    } else {
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            const uint64_t idx = base + i;
            vals[i] = idx < n ? TOut(in[idx]) : TOut(0);
            s += vals[i];
        }
    }
    TOut total;
    TOut run = block_exclusive(s, &total) + (offsets ? offsets[blockIdx.x] : TOut(0));
    if (vout) {
        TOut o[kScanItems];
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            o[i] = run;
            run += vals[i];
        }
        uint4* dst = reinterpret_cast<uint4*>(out + base);
        constexpr int NV = int(kScanItems * sizeof(TOut) / 16);
#pragma unroll
        for (int q = 0; q < NV; ++q) dst[q] = reinterpret_cast<const uint4*>(o)[q];
    } else {
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            const uint64_t idx = base + i;
            if (idx < n) out[idx] = run;
            run += vals[i];
        }
    }
    // the thread owning the last element writes the grand total to out[n]
    if (n > 0 && base <= n - 1 && n - 1 < base + kScanItems) out[n] = run;
    if (n == 0 && blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
}

template <class TIn, class TOut>
sgnn_status scan_impl(const TIn* in, TOut* out, uint64_t n, cudaStream_t s) {
    const uint64_t nb = n == 0 ? 1 : ceil_div_u64(n, kScanTile);
    if (nb == 1) {
        scan_down_kernel<TIn, TOut><<<1, kScanThreads, 0, s>>>(in, out, n, nullptr);
        SGNN_LAUNCH_CHECK();
        return SGNN_OK;
    }
    TOut* sums = nullptr;
    SGNN_TRY(scratch_alloc(reinterpret_cast<void**>(&sums), sizeof(TOut) * (nb + 1), s));
    scan_reduce_kernel<TIn, TOut><<<unsigned(nb), kScanThreads, 0, s>>>(in, n, sums);
    SGNN_LAUNCH_CHECK();
    sgnn_status st = scan_impl<TOut, TOut>(sums, sums, nb, s);
    if (st == SGNN_OK) {
        scan_down_kernel<TIn, TOut><<<unsigned(nb), kScanThreads, 0, s>>>(in, out, n, sums);
        if (cudaGetLastError() != cudaSuccess) st = fail(SGNN_ERR_CUDA, "scan_down launch failed");
    }
    scratch_free(sums, s);
    return st;
}

}  // namespace

sgnn_status exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
    return scan_impl<uint32_t, uint32_t>(in, out, n, s);
}
sgnn_status exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t s) {
    return scan_impl<uint64_t, uint64_t>(in, out, n, s);
}
sgnn_status exclusive_scan_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n,
                                      cudaStream_t s) {
    return scan_impl<uint32_t, uint64_t>(in, out, n, s);
}

}  // namespace sgnn
