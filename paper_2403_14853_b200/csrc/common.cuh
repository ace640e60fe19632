// common.cuh -- shared device helpers and host-side error plumbing for the
// sm_100a sparse hot path.  See include/sgnn_b200.h for the ABI contract.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/sgnn_b200.h"

namespace sgnn {

// ---------------------------------------------------------------- host side
// Thread-local last-error message (sgnn_last_error).
void set_error(const std::string& msg);
const char* last_error();

struct Error {
    sgnn_status status;
};

inline sgnn_status fail(sgnn_status st, const std::string& msg) {
    set_error(msg);
    return st;
}

#define SGNN_CUDA_TRY(expr)                                                                 \
    do {                                                                                    \
        cudaError_t err_ = (expr);                                                          \
        if (err_ != cudaSuccess) {                                                          \
            return ::sgnn::fail(err_ == cudaErrorMemoryAllocation ? SGNN_ERR_NOMEM          \
                                                                  : SGNN_ERR_CUDA,          \
                                std::string(#expr) + ": " + cudaGetErrorString(err_));      \
        }                                                                                   \
    } while (0)

#define SGNN_TRY(expr)                              \
    do {                                            \
        sgnn_status st_ = (expr);                   \
        if (st_ != SGNN_OK) return st_;             \
    } while (0)

// Launch check: catches configuration errors synchronously (no device sync).
#define SGNN_LAUNCH_CHECK() SGNN_CUDA_TRY(cudaGetLastError())

inline uint64_t ceil_div_u64(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

struct DeviceProps {
    int sm_count = 0;
    int l2_bytes = 0;
    int cc_major = 0;
    int cc_minor = 0;
    int max_threads_per_sm = 0;
};
// Cached per current device; returns SGNN_ERR_CUDA when no usable device.
sgnn_status device_props(DeviceProps* out);

// Stream-ordered scratch allocation (cudaMallocAsync on the device's default pool).
sgnn_status scratch_alloc(void** p, size_t bytes, cudaStream_t s);
void scratch_free(void* p, cudaStream_t s);

// Exclusive prefix sums on the device (scan.cu).  `out` may alias `in`.
// Writes the grand total to out[n] (so out has n+1 entries).
sgnn_status exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s);
sgnn_status exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t s);
// Same, but input is u32 counts widened into u64 offsets.
sgnn_status exclusive_scan_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n,
                                      cudaStream_t s);

// Validation shared by the entry points (kernels.hpp:131-136 shape rules).
sgnn_status check_csr(const sgnn_csr* a, const char* what);

}  // namespace sgnn

// --------------------------------------------------------------- device side
namespace sgnn {
namespace dev {

__device__ __forceinline__ uint64_t shfl_u64(unsigned mask, uint64_t v, int src, int width) {
    const uint32_t lo = __shfl_sync(mask, static_cast<uint32_t>(v), src, width);
    const uint32_t hi = __shfl_sync(mask, static_cast<uint32_t>(v >> 32), src, width);
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

// Streaming (evict-first) loads for the CSR arrays, which are read once.
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) { return __ldcs(p); }
__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }

}  // namespace dev
}  // namespace sgnn
