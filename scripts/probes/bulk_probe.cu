// bulk_probe.cu -- can TMA bulk copies (cp.async.bulk, one instruction per
// gathered row, completion on an mbarrier) keep more gathered rows in
// flight per SM than register gathers (LDG.128, bounded by registers x
// resident warps)?  Same work as gather_probe.cu's FULL mode over a real
// col_idx sequence (dump_cols.py): per nonzero a streamed value and a
// separately rounded fold acc += v * X[col, :] (K = 128: 512-byte rows).
//   ldg<U>       : register gathers, U in flight per warp (the SpMM today)
//   bulk<U, S>   : each warp's elected lane issues U bulk row copies per
//                  batch into an S-stage shared-memory ring; lanes read
//                  their float4 back with LDS.128 after the stage's mbarrier
// ./bulk_probe <u32 col file> <n_cols>
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_probe bulk_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ void fold(float4& acc, float a, const float4& t) {
    acc.x = __fadd_rn(acc.x, __fmul_rn(a, t.x));
    acc.y = __fadd_rn(acc.y, __fmul_rn(a, t.y));
    acc.z = __fadd_rn(acc.z, __fmul_rn(a, t.z));
    acc.w = __fadd_rn(acc.w, __fmul_rn(a, t.w));
}

template <int U>
__global__ void __launch_bounds__(128) ldg_kernel(const float4* __restrict__ tab, const uint32_t* __restrict__ idx,
                                                  const float* __restrict__ vals, uint64_t n, float* out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t per = (n + n_warps - 1) / n_warps;
    const uint64_t b = warp * per, e = b + per < n ? b + per : n;
    float4 acc = make_float4(0, 0, 0, 0);
    for (uint64_t i = b; i < e; i += 32) {
        const uint32_t my = (i + lane < e) ? __ldcs(idx + i + lane) : 0u;
        const float myv = (i + lane < e) ? __ldcs(vals + i + lane) : 0.0f;
        const int cnt = int(e - i < 32 ? e - i : 32);
        for (int j = 0; j < cnt; j += U) {
            float4 t[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t r = __shfl_sync(0xffffffffu, my, (j + u) & 31);
                t[u] = __ldg(tab + uint64_t(r) * 32 + lane);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const float a = __shfl_sync(0xffffffffu, myv, (j + u) & 31);
                if (j + u < cnt) fold(acc, a, t[u]);
            }
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// One warp = one consumer with its own S-stage ring of U rows.
template <int U, int S>
__global__ void __launch_bounds__(128) bulk_kernel(const float4* __restrict__ tab, const uint32_t* __restrict__ idx,
                                                   const float* __restrict__ vals, uint64_t n, float* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float4* ring = reinterpret_cast<float4*>(smem) + size_t(wid) * S * U * 32;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(blockDim.x >> 5) * S * U * 512) + wid * S;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t per = (n + n_warps - 1) / n_warps;
    const uint64_t b = min(warp * per, n), e = min(b + per, n);
    const uint64_t nb = (e - b + U - 1) / U;  // batches of U nonzeros
    float4 acc = make_float4(0, 0, 0, 0);
    // issue batch q (nonzeros b + qU ..) into stage q % S
    auto issue = [&](uint64_t q) {
        const uint64_t base = b + q * U;
        const uint32_t c = (lane < U && base + lane < e) ? __ldcs(idx + base + lane) : 0xffffffffu;
        const int s = int(q % S);
        if (lane == 0) {
            const int cnt = int((e - base < uint64_t(U) ? e - base : uint64_t(U)));
            mbar_expect_tx(bars + s, uint32_t(cnt) * 512u);
        }
        __syncwarp();
        // each of the first U lanes copies its own row (compiler serialises the uniform op)
        if (c != 0xffffffffu) bulk_row(ring + size_t(s) * U * 32 + lane * 32, tab + uint64_t(c) * 32, 512u, bars + s);
    };
    for (uint64_t q = 0; q < (nb < uint64_t(S - 1) ? nb : uint64_t(S - 1)); ++q) issue(q);
    for (uint64_t q = 0; q < nb; ++q) {
        if (q + S - 1 < nb) issue(q + S - 1);
        const uint64_t base = b + q * U;
        const float v = (lane < U && base + lane < e) ? __ldcs(vals + base + lane) : 0.0f;
        const int s = int(q % S);
        mbar_wait(bars + s, uint32_t((q / S) & 1));
        const int cnt = int((e - base < uint64_t(U) ? e - base : uint64_t(U)));
        const float4* st = ring + size_t(s) * U * 32;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float a = __shfl_sync(0xffffffffu, v, u);
            if (u < cnt) fold(acc, a, st[u * 32 + lane]);
        }
        __syncwarp();
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}

template <class F>
float timeit(F launch, void* flush) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
        cudaMemsetAsync(flush, r, 256 << 20);
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
        exit(1);
    }
    return best;
}

template <int U, int S>
void run_bulk(const float4* tab, const uint32_t* idx, const float* vals, uint64_t n, float* out, int sms, void* flush,
              const char* path) {
    const size_t smem = size_t(4) * S * U * 512 + 4 * S * 8;
    cudaFuncSetAttribute(bulk_kernel<U, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bulk_kernel<U, S>, 128, smem);
    for (int occ = 1; occ <= per_sm; ++occ) {
        const float t = timeit([&] { bulk_kernel<U, S><<<sms * occ, 128, smem>>>(tab, idx, vals, n, out); }, flush);
        printf("{\"file\": \"%s\", \"kind\": \"bulk\", \"U\": %d, \"S\": %d, \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.0f}\n",
               path, U, S, occ, t, n * 512.0 / t / 1e6);
    }
}

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    FILE* f = fopen(argv[1], "rb");
    if (!f) return 1;
    std::vector<uint32_t> h;
    {
        std::vector<uint32_t> buf(1 << 20);
        size_t got;
        while ((got = fread(buf.data(), 4, buf.size(), f)) > 0) h.insert(h.end(), buf.begin(), buf.begin() + got);
        fclose(f);
    }
    const uint64_t n_cols = strtoull(argv[2], nullptr, 10);
    const uint64_t n = h.size();
    float4* tab;
    cudaMalloc(&tab, n_cols * 512);
    cudaMemset(tab, 0, n_cols * 512);
    uint32_t* idx;
    cudaMalloc(&idx, n * 4);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    float* vals;
    cudaMalloc(&vals, n * 4);
    cudaMemset(vals, 0, n * 4);
    float* out;
    cudaMalloc(&out, 4);
    void* flush;
    cudaMalloc(&flush, 256 << 20);
    for (int occ : {4, 5, 6, 8}) {
        const float t = timeit([&] { ldg_kernel<8><<<sms * occ, 128>>>(tab, idx, vals, n, out); }, flush);
        printf("{\"file\": \"%s\", \"kind\": \"ldg\", \"U\": 8, \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.0f}\n",
               argv[1], occ, t, n * 512.0 / t / 1e6);
    }
    run_bulk<8, 2>(tab, idx, vals, n, out, sms, flush, argv[1]);
    run_bulk<8, 3>(tab, idx, vals, n, out, sms, flush, argv[1]);
    run_bulk<4, 4>(tab, idx, vals, n, out, sms, flush, argv[1]);
    run_bulk<16, 2>(tab, idx, vals, n, out, sms, flush, argv[1]);
    printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
