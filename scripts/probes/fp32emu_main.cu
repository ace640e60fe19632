// Probe driver for fp32emu.cu (tensor-core FP32 GEMM vs cuBLAS SGEMM, 4M x 128 x 128): nvcc ... fp32emu_main.cu fp32emu.o -lcublas
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cublas_v2.h>
#include <cuda_runtime.h>
extern "C" int emu_gemm(int m, int n, int k, const float* A, const float* B, float* C, float beta, void* ws, size_t ws_bytes, cudaStream_t s);
int main() {
  for (int m : {1000, 4194304}) {
    const int n = 128, k = 128;
    std::vector<float> ha(size_t(m) * k), hb(size_t(k) * n);
    srand(1);
    for (auto& v : ha) v = rand() / float(RAND_MAX) * 2 - 1;
    for (auto& v : hb) v = (rand() / float(RAND_MAX) * 2 - 1) * 0.1f;
    float *a, *b, *c, *c2; void* ws;
    cudaMalloc(&a, ha.size() * 4); cudaMalloc(&b, hb.size() * 4);
    cudaMalloc(&c, size_t(m) * n * 4); cudaMalloc(&c2, size_t(m) * n * 4); cudaMalloc(&ws, 64 << 20);
    cudaMemcpy(a, ha.data(), ha.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(b, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
    int rc = emu_gemm(m, n, k, a, b, c, 0.0f, ws, 64 << 20, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("m=%d rc=%d err=%s\n", m, rc, cudaGetErrorString(e));
    if (rc || e) return 1;
    cublasHandle_t h; cublasCreate(&h); cublasSetMathMode(h, CUBLAS_PEDANTIC_MATH);
    const float one = 1, zero = 0;
    cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, m, k, &one, b, n, a, k, &zero, c2, n);
    cudaDeviceSynchronize();
    std::vector<float> hc(size_t(m) * n), hc2(size_t(m) * n);
    cudaMemcpy(hc.data(), c, hc.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc2.data(), c2, hc.size() * 4, cudaMemcpyDeviceToHost);
    // double reference on the first 1000 rows
    double me = 0, me2 = 0;
    for (int i = 0; i < 1000; ++i) for (int j = 0; j < n; ++j) {
      double s = 0, den = 0;
      for (int q = 0; q < k; ++q) { s += double(ha[size_t(i)*k+q]) * hb[size_t(q)*n+j]; den += fabs(double(ha[size_t(i)*k+q]) * hb[size_t(q)*n+j]); }
      me = fmax(me, fabs(hc[size_t(i)*n+j] - s) / den); me2 = fmax(me2, fabs(hc2[size_t(i)*n+j] - s) / den);
    }
    printf("max err/den: emu %.3e  cublas-sgemm %.3e\n", me, me2);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int r = 0; r < 3; ++r) emu_gemm(m, n, k, a, b, c, 0.0f, ws, 64 << 20, 0);
    cudaEventRecord(e0); for (int r = 0; r < 10; ++r) emu_gemm(m, n, k, a, b, c, 0.0f, ws, 64 << 20, 0); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float t; cudaEventElapsedTime(&t, e0, e1);
    cudaEventRecord(e0); for (int r = 0; r < 10; ++r) cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, m, k, &one, b, n, a, k, &zero, c2, n); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float t2; cudaEventElapsedTime(&t2, e0, e1);
    printf("m=%d: emu %.3f ms, cublas sgemm %.3f ms (%.1f / %.1f TFLOP/s)\n", m, t / 10, t2 / 10, 2.0*m*n*k/(t/10)/1e9, 2.0*m*n*k/(t2/10)/1e9);
  }
  return 0;
}
