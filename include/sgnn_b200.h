/*
 * sgnn_b200.h -- C ABI of the B200-native (sm_100a) sparse GNN hot path.
 *
 * This is the drop-in boundary for the operator API of the iSpLib
 * re-creation (/root/reference/proj/include/sparsegnn/).  Every entry point
 * names the reference interface it replaces (file:line, relative to
 * proj/include/sparsegnn/ unless a src/ path is given).  INTEGRATION.md shows
 * the reference-side binding (the C++ shim include/sparsegnn_b200.hpp and a
 * ctypes stub).
 *
 * Conventions
 *  - All array pointers passed to compute entry points are DEVICE pointers
 *    (cudaMalloc / torch CUDA storage).  Layout is the reference's:
 *    row_ptr u64[n_rows+1], col_idx u32[nnz], values f32[nnz]
 *    (types.hpp:15-18,26-79); dense matrices row-major f32 (types.hpp:82-112).
 *  - Every call is asynchronous on `stream` (NULL = legacy default stream),
 *    except where noted ("synchronous").  No C++ exception crosses the ABI:
 *    errors are returned as sgnn_status codes that map 1:1 to the
 *    reference's exception classes (error.hpp:9-61); sgnn_last_error()
 *    returns the message of the calling thread's last failure.
 *  - There is no CPU fallback.  Without a usable sm_100 device every compute
 *    entry point returns SGNN_ERR_CUDA.
 *  - Numerics contract (fp32): every SpMM/FusedMM output element accumulates
 *    its row's nonzeros in ascending order with separately rounded multiply
 *    and add (no FMA contraction), exactly like spmm_rows_trusted
 *    (kernels.hpp:45-91) built without FMA -- except that rows with more than
 *    SGNN_SEGMENT nonzeros are accumulated in canonical segments of
 *    SGNN_SEGMENT nonzeros that are then added left to right.  The segment
 *    length is a library constant, so results are bitwise independent of the
 *    plan/tuning (the dispatch-transparency invariant), of the
 *    number of GPUs of a row partition, and of run-to-run scheduling.
 */
#ifndef SGNN_B200_H
#define SGNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGNN_ABI_VERSION 1
#define SGNN_SEGMENT 256 /* canonical accumulation segment (nonzeros) */

typedef struct CUstream_st* sgnn_stream; /* == cudaStream_t */

/* Status codes <-> reference exceptions (error.hpp). */
typedef enum sgnn_status {
    SGNN_OK = 0,
    SGNN_ERR_SHAPE = 1,       /* ShapeError      error.hpp:15-18 */
    SGNN_ERR_DISPATCH = 2,    /* DispatchError   error.hpp:22-25 */
    SGNN_ERR_CONFIG = 3,      /* ConfigError     error.hpp:28-31 */
    SGNN_ERR_TAPE = 4,        /* TapeError       error.hpp:34-37 */
    SGNN_ERR_IO = 5,          /* IoError         error.hpp:40-43 */
    SGNN_ERR_PARSE = 6,       /* ParseError      error.hpp:46-55 */
    SGNN_ERR_INTERNAL = 7,    /* InternalError   error.hpp:58-61 */
    SGNN_ERR_CUDA = 8,        /* CUDA runtime / device failure (no reference analogue) */
    SGNN_ERR_NOMEM = 9,       /* device allocation failed */
    SGNN_ERR_UNSUPPORTED = 10 /* configuration this build does not implement */
} sgnn_status;

/* ReduceOp, in the order of types.hpp:116. */
enum { SGNN_REDUCE_SUM = 0, SGNN_REDUCE_MIN = 1, SGNN_REDUCE_MAX = 2, SGNN_REDUCE_MEAN = 3 };

/* FusedMM edge ops: the GPU-expressible Semiring::combine (types.hpp:139-145).
 * MUL = the default combine (p*dot, kernels.hpp:239);
 * SIGMOID_MUL = p * 1/(1+exp(-dot)) (BASELINE cfg4). */
enum { SGNN_EDGE_MUL = 0, SGNN_EDGE_SIGMOID_MUL = 1 };

/* KernelKind::Tag (kernels.hpp:16-25). */
enum { SGNN_KERNEL_TRUSTED = 0, SGNN_KERNEL_SPECIALIZED = 1 };

/* CsrMatrix<float> view over device memory (types.hpp:26-79). */
typedef struct sgnn_csr {
    uint32_t n_rows;
    uint32_t n_cols;
    uint64_t nnz;
    const uint64_t* row_ptr; /* device, n_rows+1 */
    const uint32_t* col_idx; /* device, nnz */
    const float* values;     /* device, nnz */
} sgnn_csr;

/* Tunable launch parameters of a SpMM plan (the on-device tuner's search
 * space; replaces the K-sweep of autotune.hpp:99-164).  Zero fields mean
 * "library default". */
typedef struct sgnn_plan_params {
    uint32_t lanes;        /* lanes per worker group: 4, 8, 16 or 32 */
    uint32_t vec;          /* float4 (or float, scalar path) registers per lane: 1,2,4,8 */
    uint32_t unroll;       /* neighbor-row gathers in flight per lane: 2, 4 or 8 */
    uint32_t path_items;   /* rows+nonzeros per worker (nnz-balanced split), >= 1 */
    uint32_t split_rows_over; /* rows with more nonzeros than this may be split across
                                 workers (rounded up to a multiple of SGNN_SEGMENT) */
    uint32_t k_tile;       /* floats of K per pass over the matrix (0 = all of K) */
    uint32_t block;        /* threads per CTA: 64 or 128 */
    uint32_t scalar;       /* 1 = force the scalar-load ("trusted") path */
    uint32_t occupancy;    /* register cap as resident 128-thread CTAs per SM the kernel must
                              fit: 0/1 = compiler's choice, 4, 6 or 8 (float4 path) */
} sgnn_plan_params;

typedef struct sgnn_plan_s* sgnn_plan;

/* ---------------------------------------------------------------- library */
int sgnn_abi_version(void);
/* Message of the calling thread's most recent failure ("" if none). */
const char* sgnn_last_error(void);
/* Device query used by the tuner (hardware.cpp:8-34 analogue): SM count,
 * L2 bytes, compute capability.  Synchronous. */
sgnn_status sgnn_device_info(int* sm_count, int* l2_bytes, int* cc_major, int* cc_minor);
/* Workspace (plan builds, transposes, cache operands' scratch) comes from the
 * device's default stream-ordered memory pool, which the library sets to keep
 * freed blocks for reuse.  This returns all but keep_bytes of the pool's
 * unused memory to the driver (cudaMemPoolTrimTo).  Synchronous. */
sgnn_status sgnn_release_scratch(size_t keep_bytes);

/* ------------------------------------------------------------------ plans */
/* Precompute the nnz-balanced work split of A for embedding width K
 * (parallel.hpp:28-65 balanced_row_partition, at GPU-worker granularity,
 * with hub rows split in SGNN_SEGMENT units).  params == NULL -> defaults.
 * Synchronous (reads back two counts).  The plan borrows A's row_ptr; it is
 * valid while that array is unchanged.  A plan owns a workspace: do not use
 * one plan from two streams concurrently. */
sgnn_status sgnn_plan_create(const sgnn_csr* a, uint32_t k, const sgnn_plan_params* params,
                             sgnn_plan* out, sgnn_stream stream);
sgnn_status sgnn_plan_destroy(sgnn_plan plan);
sgnn_status sgnn_plan_get_params(sgnn_plan plan, sgnn_plan_params* out);
/* Plan statistics: workers, split rows, workspace slots. */
sgnn_status sgnn_plan_stats(sgnn_plan plan, uint64_t* workers, uint64_t* split_rows,
                            uint64_t* slots);

/* ------------------------------------------------------------------- SpMM */
/* C = reduce_j a_ij * X[j,:]   (spmm / spmm_with / detail::spmm_into,
 * kernels.hpp:141-182; row kernel kernels.hpp:45-91; mean divide :60-63).
 * X is x_rows x k with x_rows == a.n_cols (else SGNN_ERR_SHAPE, as
 * check_spmm_shapes, kernels.hpp:131-136); C is a.n_rows x k; both row-major
 * and caller-owned (the spmm_into convention).  plan may be NULL (a temporary default plan is
 * built, synchronously).  A plan built for another matrix or K ->
 * SGNN_ERR_DISPATCH. */
sgnn_status sgnn_spmm_f32(const sgnn_csr* a, const float* x, uint32_t x_rows, uint32_t k,
                          float* c, int reduce, sgnn_plan plan, sgnn_stream stream);

/* spmm_with(a, b, reduce, kind) (kernels.hpp:157-173): kind SPECIALIZED
 * demands reduce == Sum, spec_k in the specialization sweep
 * {16,...,1024} (kernels.hpp:27) and spec_k == k, else SGNN_ERR_DISPATCH,
 * exactly like the reference.  On the GPU "trusted" runs the default plan,
 * "specialized" the tuned plan registered for (a, k) (or `plan`); results are
 * bitwise identical either way. */
sgnn_status sgnn_spmm_with_f32(const sgnn_csr* a, const float* x, uint32_t x_rows, uint32_t k,
                               float* c, int reduce, int kind, uint32_t spec_k, sgnn_plan plan,
                               sgnn_stream stream);

/* On-device autotuner (replaces run_tuning, autotune.hpp:99-164): times every
 * candidate launch geometry for (a, k, reduce) -- lanes x float4s per lane
 * (the K-tile), gathers in flight, path items per worker, split threshold,
 * CTA size -- with CUDA events (median of `reps` >= 3, else
 * SGNN_ERR_CONFIG), asserts each candidate's output is bit-identical to the
 * default plan's (else SGNN_ERR_INTERNAL, as autotune.hpp:131-133) and
 * returns the fastest as a new plan.  x may be NULL (a seeded uniform [0,1)
 * operand is generated, as autotune.hpp:119-121).  entries (optional)
 * receives up to max_entries timings.  Synchronous. */
typedef struct sgnn_tune_entry {
    sgnn_plan_params params;
    float ms; /* median time of one SpMM with these params */
    float reserved;
} sgnn_tune_entry;
sgnn_status sgnn_tune_spmm(const sgnn_csr* a, const float* x, uint32_t k, int reduce, int reps,
                           sgnn_plan* best, sgnn_tune_entry* entries, int max_entries,
                           int* n_entries, sgnn_stream stream);

/* resolve_kernel(k, reduce) (kernels.hpp:38, src/dispatch.cpp:21-28) and the
 * dispatch toggle set_dispatch/get_dispatch (autotune.hpp:36-37,
 * src/dispatch.cpp:12-19).  Returns the kind; *spec_k receives K for
 * SPECIALIZED, 0 for TRUSTED. */
int sgnn_resolve_kernel(uint32_t k, int reduce, uint32_t* spec_k);
void sgnn_set_dispatch(int enabled);
int sgnn_get_dispatch(void);

/* ------------------------------------------------- row-partitioned SpMM */
/* The multi-GPU row partition's SpMM with the feature exchange fused in:
 * the gathered operand X is NOT materialised -- it is the union of the
 * n_parts row blocks `parts[q]` (each [2^part_shift, k] row-major, e.g. the
 * ranks' own feature blocks mapped over NVLink peer access / CUDA IPC), and
 * A's column ids are in the padded owner layout col' = q << part_shift |
 * local (sgnn_host_partition_block with stride = 2^part_shift).  Each gather
 * reads the owner block directly, replacing all-gather + SpMM.  Sum and Mean;
 * n_parts <= 8; results are bitwise those of sgnn_spmm_f32 on the gathered
 * matrix.  plan: a plan of A (required). */
sgnn_status sgnn_spmm_peer_f32(const sgnn_csr* a, const float* const* parts, uint32_t n_parts,
                               uint32_t part_shift, uint32_t k, float* c, int reduce,
                               sgnn_plan plan, sgnn_stream stream);
/* CUDA IPC plumbing for the peer mappings (cudaIpcGetMemHandle /
 * cudaIpcOpenMemHandle with peer access enabled / cudaIpcCloseMemHandle).
 * handle is 64 bytes. */
sgnn_status sgnn_peer_alloc(size_t bytes, void** dev_ptr); /* own cudaMalloc: IPC handle == pointer */
sgnn_status sgnn_peer_free(void* dev_ptr);
sgnn_status sgnn_ipc_get_handle(void* dev_ptr, void* handle64);
sgnn_status sgnn_ipc_open_handle(const void* handle64, void** dev_ptr);
sgnn_status sgnn_ipc_close_handle(void* dev_ptr);

/* Built-in self-test of the mean epilogue's division (the exact
 * reciprocal-and-round path that replaces __fdiv_rn inside the SpMM kernels,
 * kernels.hpp:60-63): every degree in [d0, d1) x `samples` values (specials,
 * random bit patterns over all exponents) compared bitwise with IEEE
 * division.  *mismatches = 0 on success.  Synchronous. */
sgnn_status sgnn_selftest_count_division(uint64_t d0, uint64_t d1, uint32_t samples, uint64_t seed,
                                         uint64_t* mismatches, uint64_t* first_deg, uint32_t* first_sample);

/* ------------------------------------------------------------- transpose */
/* transpose(a) (sparse.hpp:72-89): CSR(A) -> CSR(A^T), bit-exact with the
 * reference's stable counting sort (rows ascending within each column).
 * Outputs are device arrays: t_row_ptr u64[n_cols+1], t_col_idx u32[nnz],
 * t_values f32[nnz] (t_values may be NULL: structure only).
 * ws/ws_bytes: scratch from sgnn_transpose_workspace (ws may be NULL: the
 * call allocates stream-ordered scratch itself). */
sgnn_status sgnn_transpose_workspace(const sgnn_csr* a, size_t* ws_bytes);
sgnn_status sgnn_csr_transpose(const sgnn_csr* a, uint64_t* t_row_ptr, uint32_t* t_col_idx,
                               float* t_values, void* ws, size_t ws_bytes, sgnn_stream stream);

/* row_degrees (sparse.hpp:105-109): deg[i] = row_ptr[i+1]-row_ptr[i]. */
sgnn_status sgnn_row_degrees(const sgnn_csr* a, uint32_t* deg, sgnn_stream stream);
/* is_symmetric (sparse.hpp:179-192), exact structure + value check.
 * Synchronous; *out = 1 symmetric, 0 not. */
sgnn_status sgnn_is_symmetric(const sgnn_csr* a, int* out, sgnn_stream stream);

/* normalize_adjacency(a, add_self_loops) (sparse.hpp:116-174) on the device,
 * bit-exact: A_hat = D^-1/2 (A [+ I]) D^-1/2 with degrees and scaling in
 * double.  Two calls: with t_row_ptr == NULL only *out_nnz is computed;
 * then pass arrays of n+1 / out_nnz / out_nnz entries.  Non-square ->
 * SGNN_ERR_SHAPE, a negative value -> SGNN_ERR_CONFIG.  Synchronous. */
sgnn_status sgnn_normalize_adjacency(const sgnn_csr* a, int add_self_loops, uint64_t* out_nnz,
                                     uint64_t* t_row_ptr, uint32_t* t_col_idx, float* t_values,
                                     sgnn_stream stream);

/* ------------------------------------------------ backward cache (TrainingCache) */
/* TrainingCache<float> (gnn.hpp:113-173) + build_cache (gnn.hpp:180-196)
 * for a propagation operand that is already on the device (a_hat).  The
 * cache borrows a_hat's arrays (they must outlive it) and owns the lazily
 * built transpose / mean operand.  check_symmetric mirrors
 * `cache.symmetric = use_cache && is_symmetric(a_hat)` (gnn.hpp:194).
 * Synchronous. */
typedef struct sgnn_cache_s* sgnn_cache;
sgnn_status sgnn_cache_create(const sgnn_csr* a_hat, int use_cache, sgnn_cache* out,
                              sgnn_stream stream);
/* build_cache(kind, a, use_cache, add_self_loops) (gnn.hpp:180-196) proper:
 * model_kind 0 = GCN normalizes A on the device into a cache-owned A_hat
 * (normalize_builds = 1); 1 = SAGE-sum, 2 = SAGE-mean, 3 = GIN propagate
 * over A itself (borrowed).  Synchronous. */
sgnn_status sgnn_cache_create_model(const sgnn_csr* a, int model_kind, int use_cache,
                                    int add_self_loops, sgnn_cache* out, sgnn_stream stream);
/* The cache's propagation operand a_hat (for the forward SpMMs). */
sgnn_status sgnn_cache_a_hat(sgnn_cache cache, sgnn_csr* out);
sgnn_status sgnn_cache_destroy(sgnn_cache cache);
/* sum_operand() (gnn.hpp:127-144) / mean_operand() (gnn.hpp:149-172):
 * fills *out with a device view of the operand (valid until the next fetch
 * with use_cache == 0, or until destroy).  Counts builds/hits like the
 * reference. */
sgnn_status sgnn_cache_sum_operand(sgnn_cache cache, sgnn_csr* out, sgnn_stream stream);
sgnn_status sgnn_cache_mean_operand(sgnn_cache cache, sgnn_csr* out, sgnn_stream stream);
/* Counters (gnn.hpp:121-123) and flags: transpose_builds, normalize_builds,
 * cache_hits, symmetric. */
sgnn_status sgnn_cache_counters(sgnn_cache cache, uint64_t* transpose_builds,
                                uint64_t* normalize_builds, uint64_t* cache_hits,
                                int* symmetric);
/* SpMM backward ("spmm_backward", gnn.hpp:275,279,290,303):
 * dX = spmm(op, dC, Sum) where op = mean_operand() if reduce == Mean, else
 * sum_operand().  dC is a_hat.n_rows x k, dX is a_hat.n_cols x k.  The plan
 * for the operand is built once per K and cached inside the cache. */
sgnn_status sgnn_spmm_backward_f32(sgnn_cache cache, const float* dc, uint32_t dc_rows,
                                   uint32_t k, float* dx, int reduce, sgnn_stream stream);

/* ------------------------------------------------------- SDDMM / FusedMM */
/* sddmm(p, x, y) (kernels.hpp:187-210): out_values[e] = p_e * <X_i, Y_j>.
 * The output pattern is P's own (row_ptr/col_idx are not copied).
 * X is p.n_rows x k, Y is p.n_cols x k. */
sgnn_status sgnn_sddmm_f32(const sgnn_csr* p, const float* x, uint32_t x_rows, const float* y,
                           uint32_t y_rows, uint32_t k, float* out_values, sgnn_stream stream);
/* sddmm reusing a plan of P for its nnz-balanced work split (no per-worker
 * row search); results are identical to sgnn_sddmm_f32. */
sgnn_status sgnn_sddmm_plan_f32(const sgnn_csr* p, const float* x, uint32_t x_rows, const float* y,
                                uint32_t y_rows, uint32_t k, float* out_values, sgnn_plan plan,
                                sgnn_stream stream);
/* fusedmm(p, x, y, semiring) (kernels.hpp:216-270): out_i = reduce_j
 * combine(p_ij, <X_i,Y_j>) * Y_j in one pass (Y_j read once per edge).
 * out is p.n_rows x k. */
sgnn_status sgnn_fusedmm_f32(const sgnn_csr* p, const float* x, uint32_t x_rows, const float* y,
                             uint32_t y_rows, uint32_t k, int edge_op, int reduce, float* out,
                             sgnn_stream stream);
/* fusedmm with a caller-owned plan of P (reused work split; its lanes x vec
 * register layout is used when it holds all of K and a fused kernel exists
 * for it).  The plan must be built with k_tile = 0 (all of K). */
sgnn_status sgnn_fusedmm_plan_f32(const sgnn_csr* p, const float* x, uint32_t x_rows,
                                  const float* y, uint32_t y_rows, uint32_t k, int edge_op,
                                  int reduce, float* out, sgnn_plan plan, sgnn_stream stream);

/* ---------------------------------------------------- GNN training engine
 * train() of gnn.hpp:414-438 on the device: build_cache (GCN normalizes A),
 * forward (gnn.hpp:212-256), softmax_xent + masked_accuracy (:318-370),
 * backward through the TrainingCache (:261-313), sgd_step (:374-386).
 * Sparse propagation on this library's SpMM, dense products in cuBLAS SGEMM
 * (fp32, no TF32).  model_kind: 0 GCN, 1 SAGE-sum, 2 SAGE-mean, 3 GIN.
 * a, x [n x in], labels [n] (u32), mask [n] (u8) are device arrays (copied);
 * max_epochs sizes the per-epoch statistics.  Synchronous. */
typedef struct sgnn_gnn_s* sgnn_gnn;
sgnn_status sgnn_gnn_create(const sgnn_csr* a, int model_kind, uint32_t in_features, uint32_t hidden,
                            uint32_t classes, const float* x, const uint32_t* labels, const uint8_t* mask,
                            int use_cache, int add_self_loops, uint32_t max_epochs, sgnn_gnn* out,
                            sgnn_stream stream);
/* Weights, row-major: w1 [in x hidden], w2 [hidden x classes], and for SAGE
 * w1_self / w2_self of the same shapes (NULL otherwise); epsilon for GIN.
 * Host or device pointers.  Synchronous. */
sgnn_status sgnn_gnn_set_weights(sgnn_gnn g, const float* w1, const float* w2, const float* w1_self,
                                 const float* w2_self, float epsilon, sgnn_stream stream);
sgnn_status sgnn_gnn_get_weights(sgnn_gnn g, float* w1, float* w2, float* w1_self, float* w2_self,
                                 float* epsilon, sgnn_stream stream);
/* `epochs` training epochs at learning rate lr.  Per epoch: loss[e] (mean
 * masked cross-entropy), accuracy[e], seconds[e] (device time); any of them
 * may be NULL.  cuda_graph != 0: epoch 1 runs eagerly, later epochs replay
 * its CUDA-graph capture (needs use_cache; operand fetches are then counted
 * at capture only).  Synchronous. */
sgnn_status sgnn_gnn_train(sgnn_gnn g, uint32_t epochs, float lr, int cuda_graph, double* loss,
                           double* accuracy, double* seconds, sgnn_stream stream);
/* The engine's TrainingCache counters (gnn.hpp:121-123). */
sgnn_status sgnn_gnn_counters(sgnn_gnn g, uint64_t* transpose_builds, uint64_t* normalize_builds,
                              uint64_t* cache_hits, int* symmetric);
sgnn_status sgnn_gnn_destroy(sgnn_gnn g);

/* ------------------------------------- multi-GPU: communicator + row-partitioned trainer
 * The 1D row partition of SURVEY 8e for the partitioned config (BASELINE
 * cfg5, 2-layer GraphSAGE): the reference's thread fan-out over contiguous
 * row chunks (parallel.hpp:28-65, balanced_row_partition) lifted to GPUs, and
 * train() (gnn.hpp:414-438) for SAGE-sum / SAGE-mean on each rank's rows.
 * The layer-1 products are one fp32 product [a1 | X] [W1; W1s] (and one
 * [a1 | X]^T dz1 for the weight gradients) instead of the reference's two
 * products and an add: the same values within fp32 rounding of the sum.
 *
 * Communicator: one process per GPU, NCCL (ncclCommInitRank on the calling
 * thread's current device; libnccl.so.2 is loaded at run time -- the one the
 * process already has, e.g. torch's, else the system's).  Rank 0 makes the
 * 128-byte id, the host distributes it (any channel), every rank inits.
 * A *loopback* communicator runs P virtual ranks in one process on one
 * stream, phase by phase (device copies instead of NCCL): the partition and
 * exchange logic and each rank's share of the work, measured on one GPU.
 * NULL comm = one rank, no exchange.  Synchronous. */
typedef struct sgnn_comm_s* sgnn_comm;
#define SGNN_COMM_ID_BYTES 128
sgnn_status sgnn_comm_get_unique_id(void* id /* SGNN_COMM_ID_BYTES */);
sgnn_status sgnn_comm_init_rank(const void* id, int nranks, int rank, sgnn_comm* out);
sgnn_status sgnn_comm_init_loopback(int nranks, sgnn_comm* out);
/* kind: 0 NCCL, 1 loopback */
sgnn_status sgnn_comm_info(sgnn_comm c, int* nranks, int* rank, int* kind);
sgnn_status sgnn_comm_destroy(sgnn_comm c);

/* Rank `rank` (NCCL: the communicator's own rank, argument ignored) of the
 * row-partitioned trainer.  bounds (host, P+1 entries, bounds[0] = 0,
 * bounds[P] = n): rank r owns rows [bounds[r], bounds[r+1]).  block: those
 * rows of A as a device CSR with GLOBAL column ids (rows x n; borrowed -- it
 * must outlive the engine).  bwd_block: NULL for a symmetric A (the backward
 * operand is A's own rows, gnn.hpp:133-136,152-153), else the same rows of
 * A^T (borrowed); for SAGE-mean the engine scales its values by 1/deg of the
 * column (gnn.hpp:158-159) with the all-gathered global degrees.
 * model_kind 1 SAGE-sum, 2 SAGE-mean (others SGNN_ERR_UNSUPPORTED); needs
 * in % 4 == 0, hidden % 4 == 0, hidden <= 128, classes <= 16.  x_local
 * [rows x in], labels_local [rows] (u32), mask_local [rows] (u8): host or
 * device, copied.  Labels are range-checked here (ConfigError, gnn.hpp:327);
 * a rank that fails must abort the job (its peers would wait).  Weights are
 * zero until sgnn_dist_set_weights.  Synchronous. */
typedef struct sgnn_dist_s* sgnn_dist;
sgnn_status sgnn_dist_create(sgnn_comm comm, int rank, const uint32_t* bounds, const sgnn_csr* block,
                             const sgnn_csr* bwd_block, int model_kind, uint32_t in_features, uint32_t hidden,
                             uint32_t classes, const float* x_local, const uint32_t* labels_local,
                             const uint8_t* mask_local, uint32_t max_epochs, sgnn_dist* out, sgnn_stream stream);
/* w1, w1_self [in x hidden], w2, w2_self [hidden x classes], row-major, host
 * or device; identical on every rank.  Synchronous. */
sgnn_status sgnn_dist_set_weights(sgnn_dist g, const float* w1, const float* w2, const float* w1_self,
                                  const float* w2_self, sgnn_stream stream);
sgnn_status sgnn_dist_get_weights(sgnn_dist g, float* w1, float* w2, float* w1_self, float* w2_self,
                                  sgnn_stream stream);
/* New features for the rank's rows (host or device pointer [rows x in]),
 * copied into the engine's [a1 | X_r] row buffer and, with P ranks, into the
 * gathered feature buffer (re-exchanged at the next epoch).  `borrow` is
 * accepted for compatibility and ignored (the features are always copied).
 * Stream-asynchronous. */
sgnn_status sgnn_dist_set_features(sgnn_dist g, const float* x_local, int borrow, sgnn_stream stream);
/* `epochs` training epochs at learning rate lr (forward, softmax_xent +
 * masked_accuracy, backward, sgd_step; the loss is the global masked mean).
 * NCCL / one rank: engines = {own engine}; loopback: all P engines, in rank
 * order.  The first call also runs the one-time collective setup (global
 * degrees, mean operand values, the global masked-row count; synchronous
 * once).  Stream-asynchronous otherwise (no host sync per epoch). */
sgnn_status sgnn_dist_epochs(sgnn_dist* engines, int n_engines, uint32_t epochs, float lr, sgnn_stream stream);
/* Statistics of epochs [first, first+count) since the last reset:
 * loss[i], accuracy[i], and times[i*SGNN_DIST_TIMES + j] in device ms:
 * j=0 epoch, 1 the three SpMMs, 2 this rank's compute phases, 3 = epoch - compute
 * (exchanges and waiting for peers; loopback: also the other virtual ranks'
 * phases), 4/5/6 the layer-1 / layer-2 / backward SpMM, 7 the two dense
 * products ([a1 | X] [W1; W1s] and its weight gradient; timed apart from
 * the sparse path as BASELINE asks).  Any output may be NULL.  Synchronizes
 * the stream. */
#define SGNN_DIST_TIMES 8
sgnn_status sgnn_dist_stats(sgnn_dist g, uint32_t first, uint32_t count, double* loss, double* accuracy,
                            double* times, sgnn_stream stream);
/* (loss, accuracy) pairs of epochs [first, first+count) copied to dst
 * (host or device, 2*count doubles), stream-asynchronous: the per-step
 * result read of a pipelined caller. */
sgnn_status sgnn_dist_stats_copy(sgnn_dist g, uint32_t first, uint32_t count, double* dst, sgnn_stream stream);
/* Restart the epoch counter (statistics slots) at 0. */
sgnn_status sgnn_dist_reset(sgnn_dist g);
/* The rank's first row, row count, block nnz, global masked count (after the
 * first epoch) and the device address of its feature rows (row stride
 * 2 * in_features: the right half of the [a1 | X_r] buffer). */
sgnn_status sgnn_dist_info(sgnn_dist g, uint32_t* row0, uint32_t* rows, uint64_t* nnz, uint64_t* n_masked,
                           float** x_local);
sgnn_status sgnn_dist_destroy(sgnn_dist g);

/* ------------------------------------------------- dense FP32 products
 * The GNN layers' tall products on the 5th-gen tensor cores in FP32
 * emulation (each operand split into three bf16 terms, fp32 accumulation;
 * max |err| / sum|a*b| ~1e-7, below SGEMM's): op 0: C[m x n] = A[m x k] B[k x n];
 * op 1: C[k x n] = A[m x k]^T B[m x n] (split over m, deterministic).  Row-
 * major device arrays, 16-byte aligned, k and n multiples of 4 (SGNN_ERR_
 * UNSUPPORTED otherwise -- callers then use their own GEMM).  The engine
 * above uses these for m >= 4096.  Stream-asynchronous. */
sgnn_status sgnn_dense_mm_f32(int op, uint32_t m, uint32_t n, uint32_t k, const float* a, const float* b, float* c,
                              sgnn_stream stream);

/* ------------------------------------------------------ SAGE layer glue
 * The element-wise and classes-wide steps of a SAGE layer pair as device
 * passes, for hosts that sequence the layers themselves (the row-partitioned
 * trainer calls them on each rank's rows; the engine above uses the same
 * kernels).  Forward gnn.hpp:236-244, softmax_xent + masked_accuracy
 * :318-370, backward :283-292.  Device arrays, row-major, 16-byte aligned;
 * the classes-wide products need hidden % 4 == 0, hidden <= 128 and
 * 1 <= classes <= 16 (SGNN_ERR_SHAPE otherwise).  Stream-asynchronous. */
/* h = relu(a + b) over n elements (z1 = a1 W1 + X W1s, then relu) */
sgnn_status sgnn_add_relu_f32(const float* a, const float* b, uint64_t n, float* h, sgnn_stream stream);
/* logits[i, :] = [a2 | h1][i, :] . [w2; w2s]  (a2, h1: n x hidden; w2, w2s:
 * hidden x classes; one fp32 accumulation over the 2*hidden inputs) */
sgnn_status sgnn_sage_logits_f32(const float* a2, const float* h1, const float* w2, const float* w2s,
                                 uint32_t n, uint32_t hidden, uint32_t classes, float* logits,
                                 sgnn_stream stream);
/* softmax_xent + masked_accuracy over n rows: grad[i, :] = (softmax - onehot)
 * * inv_count on masked rows, 0 elsewhere; *loss_sum (double) = sum of the
 * masked rows' cross-entropy, *correct = masked rows whose argmax (first
 * index on ties) is the label.  Labels are not range-checked here. */
sgnn_status sgnn_softmax_xent_f32(const float* logits, uint32_t n, uint32_t classes, const uint32_t* labels,
                                  const uint8_t* mask, double inv_count, float* grad, double* loss_sum,
                                  uint32_t* correct, sgnn_stream stream);
/* g2 = a2^T grad, g2s = h1^T grad  (hidden x classes; block partials added
 * in a fixed order: deterministic for given n) */
sgnn_status sgnn_sage_wgrad_f32(const float* a2, const float* h1, const float* grad, uint32_t n,
                                uint32_t hidden, uint32_t classes, float* g2, float* g2s, sgnn_stream stream);
/* out = grad w^T (u == act == NULL), or out = relu_backward(u + grad w^T, act):
 * ds2 = grad W2^T, and dz1 from dh1 = A^T ds2 + grad W2s^T */
sgnn_status sgnn_sage_grad_wt_f32(const float* grad, const float* w, uint32_t n, uint32_t hidden,
                                  uint32_t classes, const float* u, const float* act, float* out,
                                  sgnn_stream stream);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* SGNN_B200_H */
