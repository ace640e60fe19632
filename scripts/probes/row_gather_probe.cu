// row_gather_probe.cu -- the ceiling of row-gather traffic by row size on this
// GPU: groups of G = RB / 16 lanes gather RB-byte rows (one float4 per lane),
// 32 / G rows per warp instruction, U rows in flight per group, summed into
// registers.  Uniform random row indices over tables of 32 MiB (L2-resident),
// 256 MiB (cfg4's Y) and 2 GiB (cfg5's X).  Prints GB/s of gathered bytes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o row_gather_probe row_gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

template <int G, int U>
__global__ void __launch_bounds__(128) gather(const float4* __restrict__ tab, const uint32_t* __restrict__ idx,
                                              uint64_t n, float* out) {
    const int lane = threadIdx.x & 31, gl = lane & (G - 1), grp = lane / G;
    constexpr int NG = 32 / G;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t per = (n + n_warps - 1) / n_warps;
    const uint64_t b = warp * per, e = b + per < n ? b + per : n;
    float4 acc = make_float4(0, 0, 0, 0);
    // each warp step: NG groups x U rows
    for (uint64_t i = b; i < e; i += NG * U) {
        float4 t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t k = i + uint64_t(grp) * U + u;
            const uint32_t r = k < e ? __ldg(idx + k) : 0u;
            t[u] = __ldg(tab + uint64_t(r) * G + gl);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += t[u].x; acc.y += t[u].y; acc.z += t[u].z; acc.w += t[u].w; }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}

template <int G, int U>
float run(const float4* tab, const uint32_t* idx, uint64_t n, float* out, int blocks) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    gather<G, U><<<blocks, 128>>>(tab, idx, n, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) gather<G, U><<<blocks, 128>>>(tab, idx, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

template <int G>
void sweep(const float4* tab, const uint32_t* idx, uint64_t n, float* out, int sms, uint64_t table_bytes) {
    const double bytes = double(n) * 16 * G;
    for (int occ : {4, 8, 16}) {
        const int blocks = sms * occ;
        const float t4 = run<G, 4>(tab, idx, n, out, blocks), t8 = run<G, 8>(tab, idx, n, out, blocks),
                    t16 = run<G, 16>(tab, idx, n, out, blocks);
        printf("{\"row_bytes\": %d, \"table_MiB\": %llu, \"ctas_per_sm\": %d, \"GBps_U4\": %.0f, \"GBps_U8\": %.0f, \"GBps_U16\": %.0f}\n",
               16 * G, (unsigned long long)(table_bytes >> 20), occ, bytes / t4 / 1e6, bytes / t8 / 1e6,
               bytes / t16 / 1e6);
        fflush(stdout);
    }
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t n = 32u << 20;  // 32M gathers (cfg4 has 31.4M)
    float* out; cudaMalloc(&out, 4);
    std::mt19937_64 g(1);
    for (uint64_t table_bytes : {32ull << 20, 256ull << 20, 2048ull << 20}) {
        float4* tab; cudaMalloc(&tab, table_bytes);
        cudaMemset(tab, 0, table_bytes);
        for (int rb : {256, 512}) {
            const uint64_t rows = table_bytes / rb;
            std::vector<uint32_t> h(n);
            for (auto& v : h) v = uint32_t(g() % rows);
            uint32_t* idx; cudaMalloc(&idx, n * 4);
            cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
            if (rb == 256) sweep<16>(tab, idx, n, out, sms, table_bytes);
            else sweep<32>(tab, idx, n, out, sms, table_bytes);
            cudaFree(idx);
        }
        cudaFree(tab);
    }
    return 0;
}
