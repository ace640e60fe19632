// fused_sig_sum.cu -- FusedMM worker kernels, edge op SIGMOID, ReduceOp::Sum
// (kernels.hpp:216-270).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_FUSED_LOOKUP(fused_lookup_sig_sum, SGNN_REDUCE_SUM, dev::OP_FUSED_SIGMOID)
}  // namespace sgnn
