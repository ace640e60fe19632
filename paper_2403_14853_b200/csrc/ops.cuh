// ops.cuh -- internal host entry points shared by the C ABI (capi.cu).
#pragma once

#include "common.cuh"

struct sgnn_plan_s;
struct sgnn_cache_s;
struct sgnn_gnn_s;

namespace sgnn {

// TrainingCache (cache.cu)
sgnn_status cache_create(const sgnn_csr* a_hat, int use_cache, sgnn_cache_s** out, cudaStream_t s);
void cache_destroy(sgnn_cache_s* c);
sgnn_status cache_sum_operand(sgnn_cache_s* c, sgnn_csr* out, cudaStream_t s);
sgnn_status cache_mean_operand(sgnn_cache_s* c, sgnn_csr* out, cudaStream_t s);
sgnn_status cache_spmm_backward(sgnn_cache_s* c, const float* dc, uint32_t dc_rows, uint32_t k,
                                float* dx, int reduce, cudaStream_t s);
sgnn_status cache_counters(sgnn_cache_s* c, uint64_t* tb, uint64_t* nb, uint64_t* hits, int* sym);
sgnn_status cache_create_model(const sgnn_csr* a, int model_kind, int use_cache, int add_loops,
                               sgnn_cache_s** out, cudaStream_t s);
sgnn_status cache_a_hat(sgnn_cache_s* c, sgnn_csr* out);
sgnn_status cache_spmm_with_operand(sgnn_cache_s* c, const sgnn_csr* op, const float* dc, uint32_t k, float* dx,
                                    cudaStream_t s);

// normalize_adjacency (normalize.cu); trp == nullptr -> count only.
sgnn_status run_normalize(const sgnn_csr* a, int add_loops, uint64_t* out_nnz, uint64_t* trp,
                          uint32_t* tci, float* tv, cudaStream_t s);

sgnn_status run_spmm(const sgnn_csr* a, const float* x, uint32_t k, float* c, int reduce,
                     const sgnn_plan_s* plan, cudaStream_t s);
// the same with row strides of X and C (floats, >= K): operands that are
// column slices of wider row-major buffers
sgnn_status run_spmm_ld(const sgnn_csr* a, const float* x, uint64_t ldx, uint32_t k, float* c, uint64_t ldc,
                        int reduce, const sgnn_plan_s* plan, cudaStream_t s);
// SpMM reading X from the row blocks `parts` of a partition (peer memory).
sgnn_status run_spmm_peer(const sgnn_csr* a, const float* const* parts, uint32_t n_parts,
                          uint32_t part_shift, uint32_t k, float* c, int reduce,
                          const sgnn_plan_s* plan, cudaStream_t s);
// Mean epilogue: C[r, :k] /= deg(r) (kernels.hpp:60-63, :263-266).
sgnn_status run_mean_divide(const uint64_t* rp, uint32_t m, float* c, uint64_t ldc, uint32_t k,
                            cudaStream_t s);

sgnn_status selftest_count_division(uint64_t d0, uint64_t d1, uint32_t samples, uint64_t seed, uint64_t* mismatches,
                                    uint64_t* first_deg, uint32_t* first_bits);
sgnn_status run_transpose(const sgnn_csr* a, uint64_t* trp, uint32_t* tci, float* tv, void* ws,
                          size_t ws_bytes, cudaStream_t s);
size_t transpose_workspace_bytes(const sgnn_csr* a);
// values_out[p] = values_in[p] / deg[col_idx[p]]  (gnn.hpp:158-159)
sgnn_status run_mean_scale(const uint32_t* col_idx, const float* vin, const uint32_t* deg,
                           uint64_t nnz, float* vout, cudaStream_t s);
sgnn_status run_row_degrees(const sgnn_csr* a, uint32_t* deg, cudaStream_t s);
sgnn_status run_is_symmetric(const sgnn_csr* a, int* out, cudaStream_t s);

sgnn_status tune_spmm(const sgnn_csr* a, const float* x, uint32_t k, int reduce, int reps,
                      sgnn_plan_s** best_out, sgnn_tune_entry* entries, int max_entries,
                      int* n_entries, cudaStream_t s);

sgnn_status run_sddmm(const sgnn_csr* p, const float* x, const float* y, uint32_t k, float* out,
                      const sgnn_plan_s* plan, cudaStream_t s);
sgnn_status run_fusedmm(const sgnn_csr* p, const float* x, const float* y, uint32_t k,
                        int edge_op, int reduce, float* out, const sgnn_plan_s* plan,
                        cudaStream_t s);

// GNN training engine (gnn.cu)
sgnn_status gnn_create(const sgnn_csr* a, int kind, uint32_t in, uint32_t hidden, uint32_t classes,
                       const float* x, const uint32_t* labels, const uint8_t* mask, int use_cache,
                       int add_self_loops, uint32_t max_epochs, sgnn_gnn_s** out, cudaStream_t s);
sgnn_status gnn_set_weights(sgnn_gnn_s* g, const float* w1, const float* w2, const float* w1s, const float* w2s,
                            float eps, cudaStream_t s);
sgnn_status gnn_get_weights(sgnn_gnn_s* g, float* w1, float* w2, float* w1s, float* w2s, float* eps,
                            cudaStream_t s);
sgnn_status gnn_train(sgnn_gnn_s* g, uint32_t epochs, float lr, int cuda_graph, double* loss, double* acc,
                      double* seconds, cudaStream_t s);
sgnn_status gnn_counters(sgnn_gnn_s* g, uint64_t* tb, uint64_t* nb, uint64_t* hits, int* sym);
void gnn_destroy(sgnn_gnn_s* g);
// Tensor-core FP32 GEMMs (dense_nn.cu / dense_tn.cu, dense_common.cuh): 0 on
// success.  nn: C[m,n] = A[m,k] B[k,n] + beta C; tn: C[k,n] = A[m,k]^T B[m,n].
int dense_mm_nn(int m, int n, int k, const float* a, const float* b, float* c, float beta, void* ws, size_t ws_bytes,
                cudaStream_t s);
int dense_mm_tn(int m, int n, int k, const float* a, const float* b, float* c, int splits, void* ws, size_t ws_bytes,
                cudaStream_t s);
// C = relu(A B) (the activation in the product's epilogue)
int dense_mm_nn_relu(int m, int n, int k, const float* a, const float* b, float* c, void* ws, size_t ws_bytes,
                     cudaStream_t s);
// workspace bytes the products need for this shape (nonzero return: shape refused)
int dense_mm_nn_workspace(int m, int n, int k, size_t* bytes);
int dense_mm_tn_workspace(int m, int n, int k, int splits, size_t* bytes);
// SAGE layer glue (gnn.cu), see sgnn_b200.h
sgnn_status glue_add_relu(const float* a, const float* b, uint64_t n, float* h, cudaStream_t s);
sgnn_status glue_relu(const float* x, uint64_t n, float* y, cudaStream_t s);
sgnn_status glue_sage_logits(const float* a2, const float* h1, const float* w2, const float* w2s, uint32_t n,
                             uint32_t h, uint32_t c, float* logits, cudaStream_t s);
sgnn_status glue_softmax_xent(const float* logits, uint32_t n, uint32_t c, const uint32_t* labels,
                              const uint8_t* mask, double inv_count, float* grad, double* loss_sum,
                              uint32_t* correct, cudaStream_t s);
sgnn_status glue_sage_wgrad(const float* a2, const float* h1, const float* grad, uint32_t n, uint32_t h, uint32_t c,
                            float* g2, float* g2s, cudaStream_t s);
sgnn_status glue_sage_grad_wt(const float* grad, const float* w, uint32_t n, uint32_t h, uint32_t c, const float* u,
                              const float* act, float* out, cudaStream_t s);
// softmax_xent into caller-owned per-block partials (fixed block shape for n)
uint32_t softmax_block_count(uint32_t n);
sgnn_status softmax_xent_partials(const float* logits, uint32_t n, uint32_t c, const uint32_t* labels,
                                  const uint8_t* mask, double inv_count, float* grad, double* blk_loss,
                                  uint32_t* blk_ok, cudaStream_t s);
// SAGE layer-2 head in one pass: logits, softmax_xent + accuracy (per-block
// partials as softmax_xent_partials), grad rows, ds2 = grad W2^T
sgnn_status sage_head_partials(const float* a2, const float* h1, const float* w2, const float* w2s, uint32_t n,
                               uint32_t h, uint32_t c, const uint32_t* labels, const uint8_t* mask, double inv_count,
                               float* grad, float* ds2, double* blk_loss, uint32_t* blk_ok, cudaStream_t s);
// SAGE classes-wide weight gradients into caller-owned partials [nblk][2][h][16]
sgnn_status sage_wgrad_launch(const float* a2, const float* h1, const float* grad, uint32_t n, uint32_t h,
                              uint32_t c, uint32_t rpb, uint32_t nblk, float* part, float* g2, float* g2s,
                              cudaStream_t s);

}  // namespace sgnn
