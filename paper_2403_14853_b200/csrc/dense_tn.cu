// dense_tn.cu -- C[k x n] = A[m x k]^T B[m x n], row-major fp32, split over
// m with a deterministic reduction (dense_common.cuh): the engine's weight
// gradients over all rows.
#include "dense_common.cuh"

// C (k x n) = A' (k x m) B (m x n) with A' = A^T: column-major in A's buffer
SGNN_DENSE_GEMM(SgnnGemmTN, cutlass::layout::ColumnMajor, cutlass::layout::RowMajor, cutlass::gemm::StreamKScheduler)

namespace sgnn {
int dense_mm_tn(int m, int n, int k, const float* a, const float* b, float* c, int splits, void* ws, size_t ws_bytes,
                cudaStream_t s) {
    return dense::run_gemm<SgnnGemmTN, true>(k, n, m, a, b, c, 0.0f, splits, ws, ws_bytes, s);
}
int dense_mm_tn_workspace(int m, int n, int k, int splits, size_t* bytes) {
    return dense::run_gemm<SgnnGemmTN, true>(k, n, m, nullptr, nullptr, nullptr, 0.0f, splits, nullptr, 0, nullptr,
                                             bytes);
}
}  // namespace sgnn
