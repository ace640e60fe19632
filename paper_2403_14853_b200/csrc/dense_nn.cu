// dense_nn.cu -- C = A B (+ beta C), row-major fp32, on the tensor cores
// (dense_common.cuh): the engine's X W products.
#include "dense_common.cuh"

SGNN_DENSE_GEMM(SgnnGemmNN, cutlass::layout::RowMajor, cutlass::layout::RowMajor, void)

namespace sgnn {
int dense_mm_nn(int m, int n, int k, const float* a, const float* b, float* c, float beta, void* ws, size_t ws_bytes,
                cudaStream_t s) {
    return dense::run_gemm<SgnnGemmNN, false>(m, n, k, a, b, c, beta, 1, ws, ws_bytes, s);
}
}  // namespace sgnn
