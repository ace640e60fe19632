// Probe driver for fp32emu_tn.cu (split-K A^T B over 4M rows vs cuBLAS SGEMM)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cublas_v2.h>
#include <cuda_runtime.h>
extern "C" int emu_gemm_tn(int m, int n, int k, const float* A, const float* B, float* C, int splits, void* ws, size_t ws_bytes, size_t* need, cudaStream_t s);
int main() {
  const int rows = 4194304, f = 128;  // C[f x f] = A[rows x f]^T B[rows x f]
  std::vector<float> ha(size_t(rows) * f), hb(size_t(rows) * f);
  srand(1);
  for (auto& v : ha) v = rand() / float(RAND_MAX) * 2 - 1;
  for (auto& v : hb) v = rand() / float(RAND_MAX) * 2 - 1;
  float *a, *b, *c, *c2; void* ws; size_t wsb = size_t(512) << 20;
  cudaMalloc(&a, ha.size() * 4); cudaMalloc(&b, hb.size() * 4); cudaMalloc(&c, f * f * 4); cudaMalloc(&c2, f * f * 4); cudaMalloc(&ws, wsb);
  cudaMemcpy(a, ha.data(), ha.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(b, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
  cublasHandle_t h; cublasCreate(&h); cublasSetMathMode(h, CUBLAS_PEDANTIC_MATH);
  const float one = 1, zero = 0;
  cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, f, f, rows, &one, b, f, a, f, &zero, c2, f);
  std::vector<float> hc2(f * f); cudaMemcpy(hc2.data(), c2, f * f * 4, cudaMemcpyDeviceToHost);
  // double reference for a few outputs
  for (int splits : {16, 64, 148, 296}) {
    size_t need = 0;
    int rc = emu_gemm_tn(f, f, rows, a, b, c, splits, ws, wsb, &need, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("splits=%d rc=%d ws=%zu err=%s\n", splits, rc, need, cudaGetErrorString(e));
    if (rc || e) continue;
    std::vector<float> hc(f * f); cudaMemcpy(hc.data(), c, f * f * 4, cudaMemcpyDeviceToHost);
    double me = 0, me2 = 0;
    for (int i = 0; i < f; i += 17) for (int j = 0; j < f; j += 13) {
      double s = 0, den = 0;
      for (int q = 0; q < rows; ++q) { double p = double(ha[size_t(q)*f+i]) * hb[size_t(q)*f+j]; s += p; den += fabs(p); }
      me = fmax(me, fabs(hc[i*f+j] - s) / den); me2 = fmax(me2, fabs(hc2[i*f+j] - s) / den);
    }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); for (int r = 0; r < 10; ++r) emu_gemm_tn(f, f, rows, a, b, c, splits, ws, wsb, &need, 0); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float t; cudaEventElapsedTime(&t, e0, e1);
    // determinism
    std::vector<float> hd(f * f); cudaMemcpy(hd.data(), c, f * f * 4, cudaMemcpyDeviceToHost);
    bool same = memcmp(hd.data(), hc.data(), f * f * 4) == 0;
    printf("  max err/den emu %.3e cublas %.3e  emu %.3f ms  deterministic %d\n", me, me2, t / 10, same);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); for (int r = 0; r < 10; ++r) cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, f, f, rows, &one, b, f, a, f, &zero, c2, f); cudaEventRecord(e1);
  cudaEventSynchronize(e1); float t2; cudaEventElapsedTime(&t2, e0, e1);
  printf("cublas sgemm %.3f ms\n", t2 / 10);
  return 0;
}
