// dense_nn.cu -- C = A B (+ beta C), row-major fp32, on the tensor cores
// (dense_common.cuh): the engine's X W products.
#include "dense_common.cuh"


// 256 x 128 tiles on SM pairs (cta_group::2): 1.64 vs 1.73 ms for 1SM 128 x 128
// on 4M x 128 x 128 (scripts/probes/fp32emu*.cu)
SGNN_DENSE_GEMM_CFG(SgnnGemmNN, cutlass::layout::RowMajor, cutlass::layout::RowMajor, void, sgnn::dense::Tile2Sm,
                    sgnn::dense::Cluster2Sm, cutlass::epilogue::TmaWarpSpecialized2Sm,
                    cutlass::gemm::KernelTmaWarpSpecialized2SmFastFP32Sm100)

// the same product with relu applied in the epilogue (D = relu(A B)): SAGE's
// h1 = relu([a1 | X] [W1; W1s]) without a separate pass
SGNN_DENSE_GEMM_FUSED(SgnnGemmNNRelu, cutlass::layout::RowMajor, cutlass::layout::RowMajor, void,
                      sgnn::dense::Tile2Sm, sgnn::dense::Cluster2Sm, cutlass::epilogue::TmaWarpSpecialized2Sm,
                      cutlass::gemm::KernelTmaWarpSpecialized2SmFastFP32Sm100, sgnn::dense::LinCombRelu)

namespace sgnn {
int dense_mm_nn_relu(int m, int n, int k, const float* a, const float* b, float* c, void* ws, size_t ws_bytes,
                     cudaStream_t s) {
    return dense::run_gemm<SgnnGemmNNRelu, false>(m, n, k, a, b, c, 0.0f, 1, ws, ws_bytes, s);
}
int dense_mm_nn(int m, int n, int k, const float* a, const float* b, float* c, float beta, void* ws, size_t ws_bytes,
                cudaStream_t s) {
    return dense::run_gemm<SgnnGemmNN, false>(m, n, k, a, b, c, beta, 1, ws, ws_bytes, s);
}
int dense_mm_nn_workspace(int m, int n, int k, size_t* bytes) {
    return dense::run_gemm<SgnnGemmNN, false>(m, n, k, nullptr, nullptr, nullptr, 0.0f, 1, nullptr, 0, nullptr, bytes);
}
}  // namespace sgnn
