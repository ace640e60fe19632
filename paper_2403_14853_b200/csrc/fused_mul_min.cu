// fused_mul_min.cu -- FusedMM worker kernels, edge op MUL, ReduceOp::Min
// (kernels.hpp:216-270).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_FUSED_LOOKUP(fused_lookup_mul_min, SGNN_REDUCE_MIN, dev::OP_FUSED_MUL)
}  // namespace sgnn
