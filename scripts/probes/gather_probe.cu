// gather_probe.cu -- ceiling of the SpMM's dominant traffic on this GPU:
// warps gathering 512-byte rows (K=128 fp32) by index from a table, one
// float4 per lane, U loads in flight per warp, summed into a register.
// Tables that fit L2 (64 MB) and that do not (1 GB); uniform indices and
// the cfg2 R-MAT column distribution (0.76 per-bit skew).  Prints GB/s of
// gathered bytes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cstdlib>
#include <cuda_runtime.h>

// FULL: also stream a value per gather and fold acc = acc + v*x with
// separately rounded multiply and add (the SpMM's instruction mix).
template <int U, bool FULL = false>
__global__ void __launch_bounds__(128) gather(const float4* __restrict__ tab, const uint32_t* __restrict__ idx,
                                              uint64_t n, float* out, const float* __restrict__ vals = nullptr) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t per = (n + n_warps - 1) / n_warps;
    const uint64_t b = warp * per, e = b + per < n ? b + per : n;
    float4 acc = make_float4(0, 0, 0, 0);
    for (uint64_t i = b; i < e; i += 32) {
        const uint32_t my = (i + lane < e) ? __ldcs(idx + i + lane) : 0u;
        const float myv = (FULL && i + lane < e) ? __ldcs(vals + i + lane) : 0.0f;
        const int cnt = int(e - i < 32 ? e - i : 32);
        for (int j = 0; j < cnt; j += U) {
            float4 t[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t r = __shfl_sync(0xffffffffu, my, (j + u) & 31);
                t[u] = (j + u < cnt) ? __ldg(tab + uint64_t(r) * 32 + lane) : make_float4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (FULL) {
                    const float a = __shfl_sync(0xffffffffu, myv, (j + u) & 31);
                    if (j + u < cnt) {
                        acc.x = __fadd_rn(acc.x, __fmul_rn(a, t[u].x)); acc.y = __fadd_rn(acc.y, __fmul_rn(a, t[u].y));
                        acc.z = __fadd_rn(acc.z, __fmul_rn(a, t[u].z)); acc.w = __fadd_rn(acc.w, __fmul_rn(a, t[u].w));
                    }
                } else {
                    acc.x += t[u].x; acc.y += t[u].y; acc.z += t[u].z; acc.w += t[u].w;
                }
            }
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}

template <int U, bool FULL = false>
float run(const float4* tab, const uint32_t* idx, uint64_t n, float* out, int blocks, const float* vals = nullptr) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    gather<U, FULL><<<blocks, 128>>>(tab, idx, n, out, vals);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) gather<U, FULL><<<blocks, 128>>>(tab, idx, n, out, vals);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / 10;
}

// ./gather_probe <u32 index file> <table rows>: the same sweep over a given
// gather sequence (e.g. the col_idx of a BASELINE config, in CSR order).
int run_file(const char* path, uint64_t rows, int sms) {
    FILE* f = fopen(path, "rb");
    if (!f) { printf("cannot open %s\n", path); return 1; }
    std::vector<uint32_t> h;
    uint32_t buf[1 << 16];
    size_t got;
    while ((got = fread(buf, 4, 1 << 16, f)) > 0) h.insert(h.end(), buf, buf + got);
    fclose(f);
    const uint64_t n = h.size();
    float4* tab; cudaMalloc(&tab, rows * 512);
    cudaMemset(tab, 0, rows * 512);
    uint32_t* idx; cudaMalloc(&idx, n * 4);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    float* out; cudaMalloc(&out, 4);
    void* flush; cudaMalloc(&flush, 256 << 20);
    for (int occ : {4, 5, 6, 8, 12, 16}) {
        const int blocks = sms * occ;
        cudaMemset(flush, 0, 256 << 20);
        float t4 = run<4>(tab, idx, n, out, blocks);
        float t8 = run<8>(tab, idx, n, out, blocks);
        float t16 = run<16>(tab, idx, n, out, blocks);
        float* vals = reinterpret_cast<float*>(flush);  // any n floats
        const float f4 = run<4, true>(tab, idx, n, out, blocks, vals);
        const float f8 = run<8, true>(tab, idx, n, out, blocks, vals);
        printf("{\"file\": \"%s\", \"gathers\": %llu, \"table_MB\": %llu, \"ctas_per_sm\": %d, \"ms_U4\": %.4f, \"ms_U8\": %.4f, \"ms_U16\": %.4f, \"full_ms_U4\": %.4f, \"full_ms_U8\": %.4f, \"GBps_best\": %.0f}\n",
               path, (unsigned long long)n, (unsigned long long)(rows * 512 >> 20), occ, t4, t8, t16, f4, f8,
               n * 512.0 / std::min(t4, std::min(t8, t16)) / 1e6);
    }
    return 0;
}

int main(int argc, char** argv) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (argc > 2) return run_file(argv[1], strtoull(argv[2], nullptr, 10), sms);
    const uint64_t n = 50000000;
    std::mt19937_64 g(1);
    for (int table_log : {17, 21}) {  // 2^17 rows = 64 MB (L2-resident), 2^21 = 1 GB
        const uint64_t rows = 1ull << table_log;
        float4* tab; cudaMalloc(&tab, rows * 512);
        cudaMemset(tab, 0, rows * 512);
        for (int dist = 0; dist < 2; ++dist) {
            std::vector<uint32_t> h(n);
            for (uint64_t i = 0; i < n; ++i) {
                if (dist == 0) { h[i] = uint32_t(g() & (rows - 1)); continue; }
                uint32_t c = 0;  // R-MAT column marginal: P(bit = 1) = b + d = 0.24
                for (int bit = 0; bit < table_log; ++bit) c = (c << 1) | ((g() % 100) < 24 ? 1u : 0u);
                h[i] = c;
            }
            // R-MAT rows are processed in row order; columns within a row are
            // sorted -- sort small windows to mimic that locality
            uint32_t* idx; cudaMalloc(&idx, n * 4);
            cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
            float* out; cudaMalloc(&out, 4);
            for (int occ : {4, 8, 16}) {
                const int blocks = sms * occ;
                float t4 = run<4>(tab, idx, n, out, blocks);
                float t8 = run<8>(tab, idx, n, out, blocks);
                float t16 = run<16>(tab, idx, n, out, blocks);
                printf("{\"table_MB\": %llu, \"dist\": \"%s\", \"ctas_per_sm\": %d, \"GBps_U4\": %.0f, \"GBps_U8\": %.0f, \"GBps_U16\": %.0f}\n",
                       (unsigned long long)(rows * 512 >> 20), dist ? "rmat" : "uniform", occ,
                       n * 512.0 / t4 / 1e6, n * 512.0 / t8 / 1e6, n * 512.0 / t16 / 1e6);
            }
            cudaFree(idx); cudaFree(out);
        }
        cudaFree(tab);
    }
    return 0;
}
