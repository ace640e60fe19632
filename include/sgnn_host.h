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

#ifdef __cplusplus
}
#endif

#endif /* SGNN_HOST_H */
