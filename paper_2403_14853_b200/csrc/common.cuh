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
#ifndef SGNN_CV_SMEM
#define SGNN_CV_SMEM 1
#endif

#ifndef SGNN_FIXUP_LONG
#define SGNN_FIXUP_LONG 32  // split rows with more segments go to spmm_fixup_long_kernel
#endif

namespace sgnn {
namespace dev {

// Worker schedule of a warp running PER consecutive workers at a time (one
// per lane group).  The first round is static (warp i takes workers
// i*PER..); later rounds are taken from a counter (ctr[0]) so warps that drew
// short workers pick up more instead of idling through a static grid stride
// -- power-law rows make per-worker times uneven.  The last warp to leave
// zeroes the counters for the next launch on the stream.  ctr == null: the
// static grid-stride schedule.  Which warp runs a worker never changes its
// results.
template <int PER>
struct WarpSched {
    uint32_t* ctr;
    uint32_t first_round;  // workers of the static first round (all warps)
    uint32_t base;         // first worker of this warp's current set
    __device__ __forceinline__ explicit WarpSched(uint32_t* c) : ctr(c) {
        const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        first_round = ((gridDim.x * blockDim.x) >> 5) * PER;
        base = warp * PER;
    }
    __device__ __forceinline__ void next() {
        if (ctr) {
            uint32_t t = 0;
            if ((threadIdx.x & 31) == 0) t = atomicAdd(ctr, uint32_t(PER));
            base = first_round + __shfl_sync(0xffffffffu, t, 0);
        } else {
            base += first_round;
        }
    }
    __device__ __forceinline__ void finish() {
        if (ctr && (threadIdx.x & 31) == 0) {
            if (atomicAdd(ctr + 1, 1u) == first_round / PER - 1) {
                atomicExch(ctr, 0u);
                atomicExch(ctr + 1, 0u);
            }
        }
    }
};

__device__ __forceinline__ uint64_t shfl_u64(unsigned mask, uint64_t v, int src, int width) {
    const uint32_t lo = __shfl_sync(mask, static_cast<uint32_t>(v), src, width);
    const uint32_t hi = __shfl_sync(mask, static_cast<uint32_t>(v >> 32), src, width);
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

// Streaming (evict-first) loads for the CSR arrays, which are read once.
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) { return __ldcs(p); }
__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }

// Packed fp32 pair arithmetic (FADD2 / FFMA2 on sm_100): each lane of the
// pair is an ordinary IEEE round-to-nearest add / fma, so results are those
// of the scalar ops.  (A packed multiply is not used: ptxas contracts
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2, which would change the rounding.)
__device__ __forceinline__ void add2_rn(float& a0, float& a1, float b0, float b1) {
    uint64_t a, b;
    asm("mov.b64 %0, {%1,%2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1,%2};" : "=l"(b) : "f"(b0), "f"(b1));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(a) : "l"(a), "l"(b));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a0), "=f"(a1) : "l"(a));
}
// (a0, a1) = fma((s, s), (y0, y1), (a0, a1))
__device__ __forceinline__ void fma2_rn(float& a0, float& a1, float s, float y0, float y1) {
    uint64_t a, y, ss;
    asm("mov.b64 %0, {%1,%2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1,%2};" : "=l"(y) : "f"(y0), "f"(y1));
    asm("mov.b64 %0, {%1,%1};" : "=l"(ss) : "f"(s));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(a) : "l"(ss), "l"(y), "l"(a));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a0), "=f"(a1) : "l"(a));
}

// Mean epilogue (kernels.hpp:60-63): v / T(nnz(i)), IEEE round-to-nearest,
// bit-identical to __fdiv_rn(v, float(deg)) but without div.rn.f32's
// slow-path subroutine call (whose register cost would land in the gather
// loop).  d = float(deg) is a 24-bit float.  For a NORMAL quotient, the exact
// quotient of two 24-bit floats is either representable or at least 2^-49
// (relative) away from every rounding midpoint, so any approximation within
// 2^-50 of v/d rounds to the same float: recip_count gives 1/d within
// ~2^-52.5 (rcp.approx seed, two Newton steps in double), v * r in double
// adds 2^-53, and the final cvt.rn.f32.f64 performs the single rounding
// (inf and NaN included).  A SUBNORMAL quotient (|v| < d 2^-126) has fewer
// bits, so exact midpoints occur (e.g. v = 3077091 * 2^-143, d = 15744): it is
// computed exactly on the 2^-149 grid: |v| 2^149 is an integer < 2^48, the
// integer quotient and remainder come exactly out of double arithmetic, and
// ties go to even.  Checked bitwise against __fdiv_rn
// over every degree up to 2^18 and special values (tests/test_spmm_gpu.py).
__device__ __forceinline__ double recip_count(uint64_t deg) {
    const float d = float(deg);
    float r0;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(d));
    const double dd = double(d);
    double r = double(r0);
    r = __fma_rn(__fma_rn(-dd, r, 1.0), r, r);
    r = __fma_rn(__fma_rn(-dd, r, 1.0), r, r);
    return r;
}
__device__ __forceinline__ float div_by_count_subnormal(float v, double r, float d) {
    // all in double, all exact: num < 2^48, q * d < 2^49, the remainder fma
    const double num = double(fabsf(v)) * 0x1p149;
    const double dd = double(d);
    double q = trunc(num * r);  // within one of the integer quotient
    double rem = __fma_rn(-q, dd, num);
    if (rem < 0.0) {
        q -= 1.0;
        rem += dd;
    } else if (rem >= dd) {
        q += 1.0;
        rem -= dd;
    }
    const double rem2 = 2.0 * rem;
    if (rem2 > dd || (rem2 == dd && (static_cast<long long>(q) & 1))) q += 1.0;  // ties to even
    return copysignf(float(q) * 0x1p-149f, v);
}
// nonzero v whose quotient by d is subnormal (zero takes the normal path)
__device__ __forceinline__ bool count_quotient_subnormal(float v, float d) {
    return fabsf(v) < d * 0x1p-126f && v != 0.0f;
}
__device__ __forceinline__ float div_by_count_normal(float v, double r) {
    return __double2float_rn(__dmul_rn(double(v), r));
}
__device__ __forceinline__ float div_by_count(float v, double r, float d) {
    if (count_quotient_subnormal(v, d)) return div_by_count_subnormal(v, r, d);
    return div_by_count_normal(v, r);
}

// (a0, a1) = fma((s, s), (w0, w1), (a0, a1)): the same as fma2_rn, named for
// call sites where the pair runs over outputs (w0, w1 from two rows of W)
__device__ __forceinline__ void fma2s_rn(float& a0, float& a1, float s, float w0, float w1) {
    fma2_rn(a0, a1, s, w0, w1);
}

#ifndef SGNN_LD_MODE
#define SGNN_LD_MODE 0  // gathers through __ldg (ld.global.nc); 1-3: A/B variants, see ld_gather
#endif
// L2 policy for gathered operand rows (reused across the whole launch):
// evict-last, so the streamed CSR arrays and the output do not push them out.
__device__ __forceinline__ uint64_t gather_policy() {
    uint64_t p = 0;
#if defined(SGNN_GATHER_EVICT_LAST)
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#endif
    return p;
}
__device__ __forceinline__ float4 ld_gather(const float4* ptr, uint64_t pol) {
#if defined(SGNN_GATHER_EVICT_LAST)
    float4 v;
#if defined(SGNN_GATHER_L1_NO_ALLOCATE)
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(ptr), "l"(pol));
#else
    asm("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(ptr), "l"(pol));
#endif
    return v;
#elif SGNN_LD_MODE == 1  // A/B: coherent path, L1-allocating
    (void)pol;
    float4 v;
    asm("ld.global.ca.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(ptr));
    return v;
#elif SGNN_LD_MODE == 2  // A/B: L2 only (no L1 allocation)
    (void)pol;
    float4 v;
    asm("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(ptr));
    return v;
#elif SGNN_LD_MODE == 3  // A/B: read-only path without L1 allocation
    (void)pol;
    float4 v;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(ptr));
    return v;
#else
    (void)pol;
    return __ldg(ptr);
#endif
}
__device__ __forceinline__ float ld_gather(const float* ptr, uint64_t pol) {
#if defined(SGNN_GATHER_EVICT_LAST)
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(ptr), "l"(pol));
    return v;
#else
    (void)pol;
    return __ldg(ptr);
#endif
}

}  // namespace dev
}  // namespace sgnn
