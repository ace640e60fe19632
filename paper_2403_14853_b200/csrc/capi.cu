#include <algorithm>
// capi.cu -- the extern "C" boundary (include/sgnn_b200.h).  Validation and
// error messages follow the reference operator API (kernels.hpp:131-173).
#include <atomic>
#include <initializer_list>
#include <cstring>
#include <new>

#include "ops.cuh"
#include "plan.cuh"
#include "spmm_kernel.cuh"

using namespace sgnn;

namespace {

std::atomic<bool> g_tuned_enabled{true};  // src/dispatch.cpp:9

constexpr uint32_t kSweep[] = {16, 32, 64, 128, 256, 512, 1024};  // kernels.hpp:27

bool is_specialized_k(uint32_t k) {
    for (uint32_t s : kSweep)
        if (s == k) return true;
    return false;
}

const char* reduce_name(int r) {
    switch (r) {
        case SGNN_REDUCE_SUM: return "sum";
        case SGNN_REDUCE_MIN: return "min";
        case SGNN_REDUCE_MAX: return "max";
        case SGNN_REDUCE_MEAN: return "mean";
    }
    return "?";
}

cudaStream_t cs(sgnn_stream s) { return reinterpret_cast<cudaStream_t>(s); }

// the glue passes issue float4 loads: every (non-null) array 16-byte aligned
bool aligned16(std::initializer_list<const void*> ps) {
    for (const void* p : ps)
        if (reinterpret_cast<uintptr_t>(p) % 16) return false;
    return true;
}

sgnn_status spmm_shapes(const sgnn_csr* a, uint32_t x_rows, uint32_t k) {
    if (a->n_cols != x_rows)  // check_spmm_shapes, kernels.hpp:131-136
        return fail(SGNN_ERR_SHAPE, "spmm: sparse operand is " + std::to_string(a->n_rows) + "x" +
                                        std::to_string(a->n_cols) + " but dense operand is " +
                                        std::to_string(x_rows) + "x" + std::to_string(k));
    return SGNN_OK;
}

sgnn_status spmm_dispatch(const sgnn_csr* a, const float* x, uint32_t k, float* c, int reduce,
                          sgnn_plan plan, cudaStream_t s) {
    if (plan) return run_spmm(a, x, k, c, reduce, plan, s);
    if (k == 0 || a->n_rows == 0) return SGNN_OK;
    sgnn_plan_s* tmp = nullptr;
    SGNN_TRY(build_plan(a, k, nullptr, k % 4 == 0, &tmp, s));
    sgnn_status st = run_spmm(a, x, k, c, reduce, tmp, s);
    destroy_plan(tmp);  // cudaFree synchronises with the queued work
    return st;
}

}  // namespace

extern "C" {

int sgnn_abi_version(void) { return SGNN_ABI_VERSION; }

const char* sgnn_last_error(void) { return last_error(); }

sgnn_status sgnn_device_info(int* sm_count, int* l2_bytes, int* cc_major, int* cc_minor) {
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    if (sm_count) *sm_count = dp.sm_count;
    if (l2_bytes) *l2_bytes = dp.l2_bytes;
    if (cc_major) *cc_major = dp.cc_major;
    if (cc_minor) *cc_minor = dp.cc_minor;
    return SGNN_OK;
}

sgnn_status sgnn_release_scratch(size_t keep_bytes) {
    int dev = 0;
    SGNN_CUDA_TRY(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    SGNN_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
    SGNN_CUDA_TRY(cudaDeviceSynchronize());
    SGNN_CUDA_TRY(cudaMemPoolTrimTo(pool, keep_bytes));
    return SGNN_OK;
}

// ------------------------------------------------------------------ plans
sgnn_status sgnn_plan_create(const sgnn_csr* a, uint32_t k, const sgnn_plan_params* params,
                             sgnn_plan* out, sgnn_stream stream) {
    if (!out) return fail(SGNN_ERR_CONFIG, "plan_create: null out");
    *out = nullptr;
    SGNN_TRY(check_csr(a, "plan_create"));
    if (k == 0) return fail(SGNN_ERR_CONFIG, "plan_create: K must be positive");
    try {
        SGNN_TRY(build_plan(a, k, params, k % 4 == 0, out, cs(stream)));
        const sgnn_plan_s* p = *out;
        if (!find_spmm_launcher(p->vec, int(p->p.lanes), int(p->p.vec), int(p->p.unroll),
                                SGNN_REDUCE_SUM, int(p->p.occupancy))) {
            destroy_plan(*out);
            *out = nullptr;
            return fail(SGNN_ERR_UNSUPPORTED,
                        "plan_create: no kernel compiled for lanes=" + std::to_string(p->p.lanes) +
                            " vec=" + std::to_string(p->p.vec) + " unroll=" + std::to_string(p->p.unroll) + " occupancy=" + std::to_string(p->p.occupancy) +
                            (p->vec ? " (float4)" : " (scalar)"));
        }
        return SGNN_OK;
    } catch (const std::bad_alloc&) {
        return fail(SGNN_ERR_NOMEM, "plan_create: host allocation failed");
    }
}

sgnn_status sgnn_plan_destroy(sgnn_plan plan) {
    destroy_plan(plan);
    return SGNN_OK;
}

sgnn_status sgnn_plan_get_params(sgnn_plan plan, sgnn_plan_params* out) {
    if (!plan || !out) return fail(SGNN_ERR_CONFIG, "plan_get_params: null argument");
    *out = plan->p;
    return SGNN_OK;
}

sgnn_status sgnn_plan_stats(sgnn_plan plan, uint64_t* workers, uint64_t* split_rows,
                            uint64_t* slots) {
    if (!plan) return fail(SGNN_ERR_CONFIG, "plan_stats: null plan");
    if (workers) *workers = plan->n_workers;
    if (split_rows) *split_rows = plan->n_fix;
    if (slots) *slots = plan->n_slots;
    return SGNN_OK;
}

// ------------------------------------------------------------------- SpMM
sgnn_status sgnn_spmm_f32(const sgnn_csr* a, const float* x, uint32_t x_rows, uint32_t k, float* c,
                          int reduce, sgnn_plan plan, sgnn_stream stream) {
    SGNN_TRY(check_csr(a, "spmm"));
    SGNN_TRY(spmm_shapes(a, x_rows, k));
    if (reduce < 0 || reduce > 3) return fail(SGNN_ERR_CONFIG, "spmm: unknown reduce op");
    return spmm_dispatch(a, x, k, c, reduce, plan, cs(stream));
}

sgnn_status sgnn_spmm_with_f32(const sgnn_csr* a, const float* x, uint32_t x_rows, uint32_t k,
                               float* c, int reduce, int kind, uint32_t spec_k, sgnn_plan plan,
                               sgnn_stream stream) {
    SGNN_TRY(check_csr(a, "spmm_with"));
    SGNN_TRY(spmm_shapes(a, x_rows, k));
    if (reduce < 0 || reduce > 3) return fail(SGNN_ERR_CONFIG, "spmm: unknown reduce op");
    if (kind == SGNN_KERNEL_SPECIALIZED) {  // kernels.hpp:159-169
        if (reduce != SGNN_REDUCE_SUM)
            return fail(SGNN_ERR_DISPATCH, std::string("specialized kernels support sum only, got ") +
                                               reduce_name(reduce));
        if (!is_specialized_k(spec_k))
            return fail(SGNN_ERR_DISPATCH,
                        "K=" + std::to_string(spec_k) + " is not in the specialization set");
        if (k != spec_k)
            return fail(SGNN_ERR_DISPATCH, "kernel is fixed at K=" + std::to_string(spec_k) +
                                               " but dense operand has K=" + std::to_string(k));
        return spmm_dispatch(a, x, k, c, reduce, plan, cs(stream));
    }
    if (kind != SGNN_KERNEL_TRUSTED) return fail(SGNN_ERR_CONFIG, "spmm_with: unknown kernel kind");
    // trusted: the default (untuned) plan -- bitwise the same result
    return spmm_dispatch(a, x, k, c, reduce, nullptr, cs(stream));
}

sgnn_status sgnn_tune_spmm(const sgnn_csr* a, const float* x, uint32_t k, int reduce, int reps,
                           sgnn_plan* best, sgnn_tune_entry* entries, int max_entries,
                           int* n_entries, sgnn_stream stream) {
    SGNN_TRY(check_csr(a, "run_tuning"));
    if (!best) return fail(SGNN_ERR_CONFIG, "run_tuning: null out");
    if (reduce < 0 || reduce > 3) return fail(SGNN_ERR_CONFIG, "run_tuning: unknown reduce op");
    try {
        return tune_spmm(a, x, k, reduce, reps, best, entries, max_entries, n_entries, cs(stream));
    } catch (const std::bad_alloc&) {
        return fail(SGNN_ERR_NOMEM, "run_tuning: host allocation failed");
    }
}

int sgnn_resolve_kernel(uint32_t k, int reduce, uint32_t* spec_k) {
    // src/dispatch.cpp:21-28
    int kind = SGNN_KERNEL_TRUSTED;
    if (g_tuned_enabled.load(std::memory_order_relaxed) && reduce == SGNN_REDUCE_SUM &&
        is_specialized_k(k))
        kind = SGNN_KERNEL_SPECIALIZED;
    if (spec_k) *spec_k = kind == SGNN_KERNEL_SPECIALIZED ? k : 0;
    return kind;
}

// ------------------------------------------------- row-partitioned SpMM
sgnn_status sgnn_spmm_peer_f32(const sgnn_csr* a, const float* const* parts, uint32_t n_parts,
                               uint32_t part_shift, uint32_t k, float* c, int reduce,
                               sgnn_plan plan, sgnn_stream stream) {
    SGNN_TRY(check_csr(a, "spmm_peer"));
    if (!parts || !plan) return fail(SGNN_ERR_CONFIG, "spmm_peer: null parts or plan");
    for (uint32_t i = 0; i < n_parts && i < SGNN_MAX_PEERS; ++i)
        if (!parts[i]) return fail(SGNN_ERR_CONFIG, "spmm_peer: null part pointer");
    return run_spmm_peer(a, parts, n_parts, part_shift, k, c, reduce, plan, cs(stream));
}

sgnn_status sgnn_peer_alloc(size_t bytes, void** dev_ptr) {
    if (!dev_ptr) return fail(SGNN_ERR_CONFIG, "peer_alloc: null out");
    SGNN_CUDA_TRY(cudaMalloc(dev_ptr, bytes ? bytes : 16));
    return SGNN_OK;
}

sgnn_status sgnn_peer_free(void* dev_ptr) {
    if (dev_ptr) SGNN_CUDA_TRY(cudaFree(dev_ptr));
    return SGNN_OK;
}

sgnn_status sgnn_ipc_get_handle(void* dev_ptr, void* handle64) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    if (!dev_ptr || !handle64) return fail(SGNN_ERR_CONFIG, "ipc_get_handle: null argument");
    cudaIpcMemHandle_t h;
    SGNN_CUDA_TRY(cudaIpcGetMemHandle(&h, dev_ptr));
    std::memcpy(handle64, &h, sizeof(h));
    return SGNN_OK;
}

sgnn_status sgnn_ipc_open_handle(const void* handle64, void** dev_ptr) {
    if (!dev_ptr || !handle64) return fail(SGNN_ERR_CONFIG, "ipc_open_handle: null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    SGNN_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return SGNN_OK;
}

sgnn_status sgnn_ipc_close_handle(void* dev_ptr) {
    if (!dev_ptr) return fail(SGNN_ERR_CONFIG, "ipc_close_handle: null argument");
    SGNN_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
    return SGNN_OK;
}

// ------------------------------------------------------------- transpose
sgnn_status sgnn_transpose_workspace(const sgnn_csr* a, size_t* ws_bytes) {
    SGNN_TRY(check_csr(a, "transpose"));
    if (!ws_bytes) return fail(SGNN_ERR_CONFIG, "transpose_workspace: null out");
    *ws_bytes = transpose_workspace_bytes(a);
    return SGNN_OK;
}

sgnn_status sgnn_csr_transpose(const sgnn_csr* a, uint64_t* t_row_ptr, uint32_t* t_col_idx,
                               float* t_values, void* ws, size_t ws_bytes, sgnn_stream stream) {
    SGNN_TRY(check_csr(a, "transpose"));
    if (!t_row_ptr || (a->nnz && !t_col_idx))
        return fail(SGNN_ERR_CONFIG, "transpose: null output arrays");
    return run_transpose(a, t_row_ptr, t_col_idx, t_values, ws, ws_bytes, cs(stream));
}

sgnn_status sgnn_row_degrees(const sgnn_csr* a, uint32_t* deg, sgnn_stream stream) {
    SGNN_TRY(check_csr(a, "row_degrees"));
    return run_row_degrees(a, deg, cs(stream));
}

sgnn_status sgnn_is_symmetric(const sgnn_csr* a, int* out, sgnn_stream stream) {
    SGNN_TRY(check_csr(a, "is_symmetric"));
    if (!out) return fail(SGNN_ERR_CONFIG, "is_symmetric: null out");
    return run_is_symmetric(a, out, cs(stream));
}

// ------------------------------------------------------------ backward cache
sgnn_status sgnn_cache_create(const sgnn_csr* a_hat, int use_cache, sgnn_cache* out,
                              sgnn_stream stream) {
    if (!out) return fail(SGNN_ERR_CONFIG, "cache_create: null out");
    try {
        return cache_create(a_hat, use_cache, out, cs(stream));
    } catch (const std::bad_alloc&) {
        return fail(SGNN_ERR_NOMEM, "cache_create: host allocation failed");
    }
}

sgnn_status sgnn_normalize_adjacency(const sgnn_csr* a, int add_self_loops, uint64_t* out_nnz,
                                     uint64_t* t_row_ptr, uint32_t* t_col_idx, float* t_values,
                                     sgnn_stream stream) {
    SGNN_TRY(check_csr(a, "normalize_adjacency"));
    if (!out_nnz) return fail(SGNN_ERR_CONFIG, "normalize_adjacency: null out_nnz");
    return run_normalize(a, add_self_loops, out_nnz, t_row_ptr, t_col_idx, t_values, cs(stream));
}

sgnn_status sgnn_cache_create_model(const sgnn_csr* a, int model_kind, int use_cache,
                                    int add_self_loops, sgnn_cache* out, sgnn_stream stream) {
    if (!out) return fail(SGNN_ERR_CONFIG, "build_cache: null out");
    try {
        return cache_create_model(a, model_kind, use_cache, add_self_loops, out, cs(stream));
    } catch (const std::bad_alloc&) {
        return fail(SGNN_ERR_NOMEM, "build_cache: host allocation failed");
    }
}

sgnn_status sgnn_cache_a_hat(sgnn_cache cache, sgnn_csr* out) {
    if (!cache || !out) return fail(SGNN_ERR_CONFIG, "cache_a_hat: null argument");
    return cache_a_hat(cache, out);
}

sgnn_status sgnn_cache_destroy(sgnn_cache cache) {
    cache_destroy(cache);
    return SGNN_OK;
}

sgnn_status sgnn_cache_sum_operand(sgnn_cache cache, sgnn_csr* out, sgnn_stream stream) {
    if (!cache || !out) return fail(SGNN_ERR_CONFIG, "sum_operand: null argument");
    return cache_sum_operand(cache, out, cs(stream));
}

sgnn_status sgnn_cache_mean_operand(sgnn_cache cache, sgnn_csr* out, sgnn_stream stream) {
    if (!cache || !out) return fail(SGNN_ERR_CONFIG, "mean_operand: null argument");
    return cache_mean_operand(cache, out, cs(stream));
}

sgnn_status sgnn_cache_counters(sgnn_cache cache, uint64_t* transpose_builds,
                                uint64_t* normalize_builds, uint64_t* cache_hits, int* symmetric) {
    if (!cache) return fail(SGNN_ERR_CONFIG, "cache_counters: null cache");
    return cache_counters(cache, transpose_builds, normalize_builds, cache_hits, symmetric);
}

sgnn_status sgnn_spmm_backward_f32(sgnn_cache cache, const float* dc, uint32_t dc_rows, uint32_t k,
                                   float* dx, int reduce, sgnn_stream stream) {
    if (!cache) return fail(SGNN_ERR_CONFIG, "spmm_backward: null cache");
    try {
        return cache_spmm_backward(cache, dc, dc_rows, k, dx, reduce, cs(stream));
    } catch (const std::bad_alloc&) {
        return fail(SGNN_ERR_NOMEM, "spmm_backward: host allocation failed");
    }
}

// ------------------------------------------------------- SDDMM / FusedMM
sgnn_status sgnn_sddmm_f32(const sgnn_csr* p, const float* x, uint32_t x_rows, const float* y,
                           uint32_t y_rows, uint32_t k, float* out_values, sgnn_stream stream) {
    SGNN_TRY(check_csr(p, "sddmm"));
    if (p->n_rows != x_rows || p->n_cols != y_rows)  // kernels.hpp:189-195
        return fail(SGNN_ERR_SHAPE, "sddmm: pattern " + std::to_string(p->n_rows) + "x" +
                                        std::to_string(p->n_cols) + " needs X with " +
                                        std::to_string(p->n_rows) + " rows and Y with " +
                                        std::to_string(p->n_cols) + " rows of equal width; got X " +
                                        std::to_string(x_rows) + "x" + std::to_string(k) + ", Y " +
                                        std::to_string(y_rows) + "x" + std::to_string(k));
    if (p->nnz && !out_values) return fail(SGNN_ERR_CONFIG, "sddmm: null output");
    return run_sddmm(p, x, y, k, out_values, nullptr, cs(stream));
}

sgnn_status sgnn_sddmm_plan_f32(const sgnn_csr* p, const float* x, uint32_t x_rows, const float* y,
                                uint32_t y_rows, uint32_t k, float* out_values, sgnn_plan plan,
                                sgnn_stream stream) {
    SGNN_TRY(check_csr(p, "sddmm"));
    if (p->n_rows != x_rows || p->n_cols != y_rows)
        return fail(SGNN_ERR_SHAPE, "sddmm: pattern " + std::to_string(p->n_rows) + "x" +
                                        std::to_string(p->n_cols) + " needs X with " +
                                        std::to_string(p->n_rows) + " rows and Y with " +
                                        std::to_string(p->n_cols) + " rows of equal width; got X " +
                                        std::to_string(x_rows) + "x" + std::to_string(k) + ", Y " +
                                        std::to_string(y_rows) + "x" + std::to_string(k));
    if (p->nnz && !out_values) return fail(SGNN_ERR_CONFIG, "sddmm: null output");
    if (!plan) return fail(SGNN_ERR_CONFIG, "sddmm_plan: null plan");
    return run_sddmm(p, x, y, k, out_values, plan, cs(stream));
}

sgnn_status sgnn_fusedmm_f32(const sgnn_csr* p, const float* x, uint32_t x_rows, const float* y,
                             uint32_t y_rows, uint32_t k, int edge_op, int reduce, float* out,
                             sgnn_stream stream) {
    SGNN_TRY(check_csr(p, "fusedmm"));
    if (p->n_rows != x_rows || p->n_cols != y_rows)  // kernels.hpp:218-222
        return fail(SGNN_ERR_SHAPE, "fusedmm: operand shapes do not compose (P " +
                                        std::to_string(p->n_rows) + "x" + std::to_string(p->n_cols) +
                                        ", X " + std::to_string(x_rows) + "x" + std::to_string(k) +
                                        ", Y " + std::to_string(y_rows) + "x" + std::to_string(k) + ")");
    return run_fusedmm(p, x, y, k, edge_op, reduce, out, nullptr, cs(stream));
}

sgnn_status sgnn_fusedmm_plan_f32(const sgnn_csr* p, const float* x, uint32_t x_rows,
                                  const float* y, uint32_t y_rows, uint32_t k, int edge_op,
                                  int reduce, float* out, sgnn_plan plan, sgnn_stream stream) {
    SGNN_TRY(check_csr(p, "fusedmm"));
    if (p->n_rows != x_rows || p->n_cols != y_rows)
        return fail(SGNN_ERR_SHAPE, "fusedmm: operand shapes do not compose (P " +
                                        std::to_string(p->n_rows) + "x" + std::to_string(p->n_cols) +
                                        ", X " + std::to_string(x_rows) + "x" + std::to_string(k) +
                                        ", Y " + std::to_string(y_rows) + "x" + std::to_string(k) + ")");
    if (!plan) return fail(SGNN_ERR_CONFIG, "fusedmm_plan: null plan");
    return run_fusedmm(p, x, y, k, edge_op, reduce, out, plan, cs(stream));
}

void sgnn_set_dispatch(int enabled) {
    g_tuned_enabled.store(enabled != 0, std::memory_order_relaxed);
}

int sgnn_get_dispatch(void) { return g_tuned_enabled.load(std::memory_order_relaxed) ? 1 : 0; }

// ---------------------------------------------------------- GNN engine
sgnn_status sgnn_gnn_create(const sgnn_csr* a, int model_kind, uint32_t in_features, uint32_t hidden,
                            uint32_t classes, const float* x, const uint32_t* labels, const uint8_t* mask,
                            int use_cache, int add_self_loops, uint32_t max_epochs, sgnn_gnn* out,
                            sgnn_stream stream) {
    if (!out) return fail(SGNN_ERR_CONFIG, "gnn_create: null out");
    *out = nullptr;
    SGNN_TRY(check_csr(a, "gnn_create"));
    if (!x || !labels || !mask) return fail(SGNN_ERR_CONFIG, "gnn_create: null features/labels/mask");
    return gnn_create(a, model_kind, in_features, hidden, classes, x, labels, mask, use_cache, add_self_loops,
                      max_epochs, out, cs(stream));
}

sgnn_status sgnn_gnn_set_weights(sgnn_gnn g, const float* w1, const float* w2, const float* w1_self,
                                 const float* w2_self, float epsilon, sgnn_stream stream) {
    if (!g) return fail(SGNN_ERR_CONFIG, "gnn: null engine");
    return gnn_set_weights(g, w1, w2, w1_self, w2_self, epsilon, cs(stream));
}

sgnn_status sgnn_gnn_get_weights(sgnn_gnn g, float* w1, float* w2, float* w1_self, float* w2_self,
                                 float* epsilon, sgnn_stream stream) {
    if (!g) return fail(SGNN_ERR_CONFIG, "gnn: null engine");
    return gnn_get_weights(g, w1, w2, w1_self, w2_self, epsilon, cs(stream));
}

sgnn_status sgnn_gnn_train(sgnn_gnn g, uint32_t epochs, float lr, int cuda_graph, double* loss,
                           double* accuracy, double* seconds, sgnn_stream stream) {
    if (!g) return fail(SGNN_ERR_CONFIG, "gnn: null engine");
    return gnn_train(g, epochs, lr, cuda_graph, loss, accuracy, seconds, cs(stream));
}

sgnn_status sgnn_gnn_counters(sgnn_gnn g, uint64_t* transpose_builds, uint64_t* normalize_builds,
                              uint64_t* cache_hits, int* symmetric) {
    if (!g) return fail(SGNN_ERR_CONFIG, "gnn: null engine");
    return gnn_counters(g, transpose_builds, normalize_builds, cache_hits, symmetric);
}

sgnn_status sgnn_gnn_destroy(sgnn_gnn g) {
    gnn_destroy(g);
    return SGNN_OK;
}

sgnn_status sgnn_selftest_count_division(uint64_t d0, uint64_t d1, uint32_t samples, uint64_t seed,
                                         uint64_t* mismatches, uint64_t* first_deg, uint32_t* first_sample) {
    if (!mismatches) return fail(SGNN_ERR_CONFIG, "selftest: null out");
    return selftest_count_division(d0, d1, samples, seed, mismatches, first_deg, first_sample);
}

// ---------------------------------------------------- dense FP32 products
sgnn_status sgnn_dense_mm_f32(int op, uint32_t m, uint32_t n, uint32_t k, const float* a, const float* b, float* c,
                              sgnn_stream stream) {
    if (op != 0 && op != 1) return fail(SGNN_ERR_CONFIG, "dense_mm: op must be 0 (A B) or 1 (A^T B)");
    if (m == 0 || n == 0 || k == 0) return SGNN_OK;
    if (!a || !b || !c) return fail(SGNN_ERR_CONFIG, "dense_mm: null array");
    auto al = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
    if (k % 4 || n % 4 || !al(a) || !al(b) || !al(c) || m > 0x7fffffffu)
        return fail(SGNN_ERR_UNSUPPORTED, "dense_mm: needs 16-byte aligned rows (k, n multiples of 4)");
    const cudaStream_t s = cs(stream);
    const int splits = int(std::max<uint32_t>(1, std::min<uint32_t>(148, m / 8192)));
    size_t ws_bytes = 0;  // exactly what the kernel asks for this shape
    int rc = op == 0 ? dense_mm_nn_workspace(int(m), int(n), int(k), &ws_bytes)
                     : dense_mm_tn_workspace(int(m), int(n), int(k), splits, &ws_bytes);
    if (rc) return fail(SGNN_ERR_UNSUPPORTED, "dense_mm: the tensor-core kernel refused this shape (" + std::to_string(rc) + ")");
    void* ws = nullptr;
    if (ws_bytes) SGNN_TRY(scratch_alloc(&ws, ws_bytes, s));
    rc = op == 0 ? dense_mm_nn(int(m), int(n), int(k), a, b, c, 0.0f, ws, ws_bytes, s)
                 : dense_mm_tn(int(m), int(n), int(k), a, b, c, splits, ws, ws_bytes, s);
    if (ws) scratch_free(ws, s);
    if (rc) return fail(SGNN_ERR_UNSUPPORTED, "dense_mm: the tensor-core kernel refused this shape (" + std::to_string(rc) + ")");
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

// ---------------------------------------------------------- SAGE glue
sgnn_status sgnn_add_relu_f32(const float* a, const float* b, uint64_t n, float* h, sgnn_stream stream) {
    if (n && (!a || !b || !h)) return fail(SGNN_ERR_CONFIG, "add_relu: null array");
    if (!aligned16({a, b, h})) return fail(SGNN_ERR_UNSUPPORTED, "add_relu: arrays must be 16-byte aligned");
    return glue_add_relu(a, b, n, h, cs(stream));
}

sgnn_status sgnn_sage_logits_f32(const float* a2, const float* h1, const float* w2, const float* w2s, uint32_t n,
                                 uint32_t hidden, uint32_t classes, float* logits, sgnn_stream stream) {
    if (n && (!a2 || !h1 || !w2 || !w2s || !logits)) return fail(SGNN_ERR_CONFIG, "sage_logits: null array");
    if (!aligned16({a2, h1})) return fail(SGNN_ERR_UNSUPPORTED, "sage_logits: a2 / h1 must be 16-byte aligned");
    return glue_sage_logits(a2, h1, w2, w2s, n, hidden, classes, logits, cs(stream));
}

sgnn_status sgnn_softmax_xent_f32(const float* logits, uint32_t n, uint32_t classes, const uint32_t* labels,
                                  const uint8_t* mask, double inv_count, float* grad, double* loss_sum,
                                  uint32_t* correct, sgnn_stream stream) {
    if (!loss_sum || !correct || (n && (!logits || !labels || !mask || !grad)))
        return fail(SGNN_ERR_CONFIG, "softmax_xent: null array");
    return glue_softmax_xent(logits, n, classes, labels, mask, inv_count, grad, loss_sum, correct, cs(stream));
}

sgnn_status sgnn_sage_wgrad_f32(const float* a2, const float* h1, const float* grad, uint32_t n, uint32_t hidden,
                                uint32_t classes, float* g2, float* g2s, sgnn_stream stream) {
    if (!g2 || !g2s || (n && (!a2 || !h1 || !grad))) return fail(SGNN_ERR_CONFIG, "sage_wgrad: null array");
    if (!aligned16({a2, h1, grad})) return fail(SGNN_ERR_UNSUPPORTED, "sage_wgrad: arrays must be 16-byte aligned");
    return glue_sage_wgrad(a2, h1, grad, n, hidden, classes, g2, g2s, cs(stream));
}

sgnn_status sgnn_sage_grad_wt_f32(const float* grad, const float* w, uint32_t n, uint32_t hidden, uint32_t classes,
                                  const float* u, const float* act, float* out, sgnn_stream stream) {
    if (n && (!grad || !w || !out)) return fail(SGNN_ERR_CONFIG, "sage_grad_wt: null array");
    if (!aligned16({grad, u, act, out})) return fail(SGNN_ERR_UNSUPPORTED, "sage_grad_wt: arrays must be 16-byte aligned");
    return glue_sage_grad_wt(grad, w, n, hidden, classes, u, act, out, cs(stream));
}

}  // extern "C"
