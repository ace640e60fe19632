// dense_stub.cu -- built instead of dense_nn.cu / dense_tn.cu when the CUTLASS
// header tree is absent (Makefile): the tensor-core FP32 products report
// "unsupported" and every caller (the GNN engines, sgnn_dense_mm_f32) falls
// back to cuBLAS SGEMM.
#include <cuda_runtime.h>

#include <cstddef>

namespace sgnn {
int dense_mm_nn(int, int, int, const float*, const float*, float*, float, void*, size_t, cudaStream_t) { return 1; }
int dense_mm_tn(int, int, int, const float*, const float*, float*, int, void*, size_t, cudaStream_t) { return 1; }
int dense_mm_nn_relu(int, int, int, const float*, const float*, float*, void*, size_t, cudaStream_t) { return 1; }
int dense_mm_nn_workspace(int, int, int, size_t*) { return 1; }
int dense_mm_tn_workspace(int, int, int, int, size_t*) { return 1; }
}  // namespace sgnn
