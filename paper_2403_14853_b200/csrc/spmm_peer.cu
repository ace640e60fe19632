// spmm_peer.cu -- SpMM worker kernels reading the gathered operand from the
// row blocks of a partition (peer mappings over NVLink / NVSwitch), Sum (and
// hence Mean).
#include "spmm_inst.cuh"

namespace sgnn {
SGNN_DEFINE_PEER_LOOKUP(spmm_peer_lookup_sum, SGNN_REDUCE_SUM)
}  // namespace sgnn
