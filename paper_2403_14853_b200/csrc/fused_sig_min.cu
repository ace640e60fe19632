// fused_sig_min.cu -- FusedMM worker kernels, edge op SIGMOID, ReduceOp::Min
// (kernels.hpp:216-270).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_FUSED_LOOKUP(fused_lookup_sig_min, SGNN_REDUCE_MIN, dev::OP_FUSED_SIGMOID)
}  // namespace sgnn
