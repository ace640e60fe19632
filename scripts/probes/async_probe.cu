// async_probe.cu -- does staging gathered rows in shared memory (cp.async,
// S-deep per-warp ring) raise the gather rate over register gathers when the
// table does not fit L2?  Rows of 256 B (K=64 fp32, cfg4's Y), one 16-byte
// piece per lane of a 16-lane group, two groups per warp, each group walking
// a contiguous slice of an index sequence (cfg4's col_idx).  Prints ms.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int G = 16;

// register version: U gathers in flight per group, then consume
template <int U>
__global__ void __launch_bounds__(128) reg_gather(const float4* __restrict__ tab, const uint32_t* __restrict__ idx,
                                                  uint64_t n, float* out) {
    const int lane = threadIdx.x & 31, gl = lane & (G - 1);
    const uint64_t grp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    const uint64_t ngrp = uint64_t(gridDim.x) * blockDim.x / G;
    const uint64_t per = (n + ngrp - 1) / ngrp, b = grp * per, e = (b + per < n ? b + per : n);
    float4 acc = make_float4(0, 0, 0, 0);
    for (uint64_t i = b; i < e; i += U) {
        float4 t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t r = (i + u < e) ? __ldg(idx + i + u) : 0u;
            t[u] = __ldg(tab + uint64_t(r) * G + gl);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += t[u].x; acc.y += t[u].y; acc.z += t[u].z; acc.w += t[u].w; }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}

__device__ __forceinline__ void cp16(void* smem, const void* g) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// async version: S stages of U rows per group staged in shared memory
template <int U, int S>
__global__ void __launch_bounds__(128) async_gather(const float4* __restrict__ tab, const uint32_t* __restrict__ idx,
                                                    uint64_t n, float* out) {
    extern __shared__ float4 smem[];
    const int lane = threadIdx.x & 31, gl = lane & (G - 1);
    const int gib = threadIdx.x / G;  // group in block
    float4* ring = smem + size_t(gib) * S * U * G;
    const uint64_t grp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    const uint64_t ngrp = uint64_t(gridDim.x) * blockDim.x / G;
    const uint64_t per = (n + ngrp - 1) / ngrp, b = grp * per, e = (b + per < n ? b + per : n);
    const uint64_t nb = (e > b) ? (e - b + U - 1) / U : 0;
    auto issue = [&](uint64_t bi) {
        float4* st = ring + (bi % S) * U * G;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = b + bi * U + u;
            const uint32_t r = (i < e) ? __ldg(idx + i) : 0u;
            cp16(st + u * G + gl, tab + uint64_t(r) * G + gl);
        }
    };
    float4 acc = make_float4(0, 0, 0, 0);
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
        if (uint64_t(s) < nb) issue(s);
        commit();
    }
    for (uint64_t bi = 0; bi < nb; ++bi) {
        if (bi + S - 1 < nb) issue(bi + S - 1);
        commit();
        wait_group<S - 1>();
        __syncwarp();
        const float4* st = ring + (bi % S) * U * G;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float4 t = st[u * G + gl];
            acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
        }
        __syncwarp();
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}

template <class K>
float timeit(K k, int blocks, size_t smem, const float4* tab, const uint32_t* idx, uint64_t n, float* out) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<blocks, 128, smem>>>(tab, idx, n, out);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) k<<<blocks, 128, smem>>>(tab, idx, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("err %s\n", cudaGetErrorString(err)); return -1; }
    return ms / 10;
}

int main(int argc, char** argv) {
    if (argc < 3) { printf("usage: async_probe <u32 idx file> <rows>\n"); return 1; }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    FILE* f = fopen(argv[1], "rb");
    std::vector<uint32_t> h;
    uint32_t buf[1 << 16]; size_t got;
    while ((got = fread(buf, 4, 1 << 16, f)) > 0) h.insert(h.end(), buf, buf + got);
    fclose(f);
    const uint64_t n = h.size(), rows = strtoull(argv[2], nullptr, 10);
    float4* tab; cudaMalloc(&tab, rows * 256); cudaMemset(tab, 0, rows * 256);
    uint32_t* idx; cudaMalloc(&idx, n * 4); cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    float* out; cudaMalloc(&out, 4);
    auto k_s4 = async_gather<8, 4>; auto k_s6 = async_gather<8, 6>; auto k_s8u4 = async_gather<4, 8>;
    const size_t sm4 = 4 * 8 * G * 16 * 8, sm6 = 6 * 8 * G * 16 * 8, sm8 = 8 * 4 * G * 16 * 8;  // per 128-thread block (8 groups)
    cudaFuncSetAttribute(k_s4, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm4));
    cudaFuncSetAttribute(k_s6, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm6));
    cudaFuncSetAttribute(k_s8u4, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm8));
    for (int occ : {4, 5, 6, 8, 12, 16}) {
        const int blocks = sms * occ;
        printf("{\"ctas_per_sm\": %d, \"reg_U8_ms\": %.4f, \"reg_U16_ms\": %.4f, \"async_U8_S4_ms\": %.4f, \"async_U8_S6_ms\": %.4f, \"async_U4_S8_ms\": %.4f}\n",
               occ, timeit(reg_gather<8>, blocks, 0, tab, idx, n, out), timeit(reg_gather<16>, blocks, 0, tab, idx, n, out),
               timeit(k_s4, blocks, sm4, tab, idx, n, out), timeit(k_s6, blocks, sm6, tab, idx, n, out),
               timeit(k_s8u4, blocks, sm8, tab, idx, n, out));
    }
    return 0;
}
