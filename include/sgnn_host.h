/*
 * sgnn_host.h -- host-side (CPU, C++) services around the hot path:
 * deterministic synthetic inputs for the BASELINE configs and the
 * nnz-balanced 1D row partition used to shard a graph over GPUs.
 * None of this is on the device hot path; it is the harness and the
 * multi-GPU partitioner (parallel.hpp:28-41 at GPU granularity).
 *
 * All generators are counter-based (splitmix64 of (seed, stream, index)), so
 * their output is bit-identical for any thread count.
 */
#ifndef SGNN_HOST_H
#define SGNN_HOST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Uniform [lo, hi) / normal(mean, std) fp32 fills, element i drawn from
 * counter (seed, stream, i). threads <= 0: all cores. */
void sgnn_host_fill_uniform(float* out, uint64_t n, double lo, double hi, uint64_t seed,
                            uint64_t stream, int threads);
void sgnn_host_fill_normal(float* out, uint64_t n, double mean, double std, uint64_t seed,
                           uint64_t stream, int threads);

/* Erdos-Renyi with exactly `deg` distinct uniformly random columns per row
 * (rejection sampling, like Rng::below, rng.hpp:48-56), sorted per row.
 * rp: u64[n_rows+1]; ci: u32[n_rows*deg]. BASELINE cfg1. */
int sgnn_host_er(uint32_t n_rows, uint32_t n_cols, uint32_t deg, uint64_t seed, uint64_t* rp,
                 uint32_t* ci, int threads);

/* R-MAT graph on 2^scale nodes from n_samples edge draws with quadrant
 * probabilities (a, b, c, 1-a-b-c), no vertex permutation; optionally
 * symmetrised (every draw (i,j) also adds (j,i)) and with all self loops
 * (i,i); duplicates removed; columns sorted.  Two calls: the build returns
 * an opaque handle, export copies into caller arrays rp[2^scale+1], ci[nnz]. */
void* sgnn_host_rmat_build(uint32_t scale, uint64_t n_samples, double a, double b, double c,
                           uint64_t seed, int symmetrize, int self_loops, int threads);
uint64_t sgnn_host_rmat_nnz(void* h);
void sgnn_host_rmat_export(void* h, uint64_t* rp, uint32_t* ci);
void sgnn_host_rmat_free(void* h);

/* balanced_row_partition (parallel.hpp:28-41): contiguous row blocks of equal
 * (nnz + rows) cost; bounds has n_chunks+1 entries. */
void sgnn_host_balanced_row_partition(const uint64_t* rp, uint32_t n_rows, int n_chunks,
                                      uint32_t* bounds);

/* The same rule with cost(i) = nnz(rows < i) + row_weight * i: the GPU row
 * partition weights the row-proportional work of a training step (dense
 * products, element-wise passes: ~30x a nonzero's SpMM work on the cfg5
 * step) against the nonzeros.  row_weight = 1 reproduces
 * sgnn_host_balanced_row_partition exactly. */
void sgnn_host_weighted_row_partition(const uint64_t* rp, uint32_t n_rows, int n_chunks, uint32_t row_weight,
                                      uint32_t* bounds);

/* Row block `part` of a square CSR A (n x n) split at `bounds` (n_parts+1
 * entries, e.g. from sgnn_host_balanced_row_partition), with every column id
 * remapped to the padded owner layout used by the multi-GPU exchange:
 *     col' = owner(col) * stride + (col - bounds[owner])
 * so the all-gathered feature buffer [n_parts * stride, K] (rank q's block at
 * rows q*stride..) can be indexed directly.  stride >= max block size.  The
 * remap is monotone, so each row keeps its nonzero order (results are
 * bitwise those of the unpartitioned SpMM).  out_rp: bounds[part+1] -
 * bounds[part] + 1 entries; out_ci / out_v: the block's nonzeros (out_v and
 * v may be NULL).  Returns the block's nnz. */
uint64_t sgnn_host_partition_block(const uint64_t* rp, const uint32_t* ci, const float* v,
                                   const uint32_t* bounds, int n_parts, int part, uint32_t stride,
                                   uint64_t* out_rp, uint32_t* out_ci, float* out_v, int threads);

/* ---- on-disk formats either side of the path (io.hpp:80-262) ------------
 * Status: 0 ok, 3 config (dimensions / memory), 5 IoError, 6 ParseError.
 * On failure `err` receives the reference's message (without the "line N: "
 * prefix ParseError adds) and *err_line the 1-based line (0 when none). */

/* load_mtx (io.hpp:80-165): coordinate real|integer|pattern,
 * general|symmetric; 1-based -> 0-based, pattern values 1, symmetric files
 * expanded to both triangles, duplicates summed (fp32, in file order).  Entry
 * lines are parsed by `threads` host threads (<= 0: all cores).  The CSR is
 * held behind the handle: sgnn_host_csr_dims / _export / _free. */
int sgnn_host_mtx_load(const char* path, int threads, void** out, char* err, size_t err_len, long* err_line);
void sgnn_host_csr_dims(void* h, uint32_t* n_rows, uint32_t* n_cols, uint64_t* nnz);
void sgnn_host_csr_export(void* h, uint64_t* rp, uint32_t* ci, float* v);
void sgnn_host_csr_free(void* h);

/* save_mtx (io.hpp:168-185): coordinate real general, values "%.9g" (fp32
 * max_digits10), so a load round trip is exact. */
int sgnn_host_mtx_save(const char* path, uint32_t n_rows, uint32_t n_cols, const uint64_t* rp,
                       const uint32_t* ci, const float* v, int threads, char* err, size_t err_len);

/* load_features (io.hpp:187-205): header "n k", then n non-empty lines of k
 * decimals. */
int sgnn_host_features_load(const char* path, int threads, void** out, char* err, size_t err_len,
                            long* err_line);
void sgnn_host_dense_dims(void* h, uint32_t* rows, uint32_t* cols);
void sgnn_host_dense_export(void* h, float* out);
void sgnn_host_dense_free(void* h);

/* load_labels (kind 0, io.hpp:243-251) / load_mask (kind 1, :254-262):
 * header "n", then n integers.  out == NULL: count only (*n). */
int sgnn_host_int_column_load(const char* path, int kind, uint64_t max_n, uint32_t* out, uint64_t* n,
                              char* err, size_t err_len, long* err_line);

#ifdef __cplusplus
}
#endif

#endif /* SGNN_HOST_H */
