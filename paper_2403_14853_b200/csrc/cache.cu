// cache.cu -- the device-resident backward cache: TrainingCache<float>
// (gnn.hpp:113-173) and build_cache (gnn.hpp:180-196) for an a_hat that is
// already on the device.  The transpose is built once (on the device, bit-exact)
// and reused; a symmetric a_hat is used as its own transpose; the mean operand
// carries 1/deg-scaled values (gnn.hpp:149-172).  Counters mirror gnn.hpp:121-123.
#include <map>
#include <utility>

#include "ops.cuh"
#include "plan.cuh"

namespace {

struct DevCsr {
    uint64_t* rp = nullptr;
    uint32_t* ci = nullptr;
    float* v = nullptr;
    void* mem = nullptr;

    sgnn_status alloc(uint32_t n_rows, uint64_t nnz, bool with_structure) {
        if (mem) return SGNN_OK;
        auto a = [](size_t b) { return (b + 255) & ~size_t(255); };
        const size_t brp = with_structure ? a(sizeof(uint64_t) * (size_t(n_rows) + 1)) : 0;
        const size_t bci = with_structure ? a(sizeof(uint32_t) * nnz) : 0;
        const size_t bv = a(sizeof(float) * nnz) + 256;
        cudaError_t e = cudaMalloc(&mem, brp + bci + bv);
        if (e != cudaSuccess) return sgnn::fail(SGNN_ERR_NOMEM, "cache alloc failed");
        char* p = static_cast<char*>(mem);
        if (with_structure) {
            rp = reinterpret_cast<uint64_t*>(p);
            ci = reinterpret_cast<uint32_t*>(p + brp);
        }
        v = reinterpret_cast<float*>(p + brp + bci);
        return SGNN_OK;
    }
    void release() {
        if (mem) cudaFree(mem);
        mem = nullptr;
        rp = nullptr;
        ci = nullptr;
        v = nullptr;
    }
};

}  // namespace

struct sgnn_cache_s {
    sgnn_csr a_hat{};  // borrowed, or a view of `own` (GCN: normalized on the device)
    DevCsr own;
    bool use_cache = true;
    bool symmetric = false;
    uint64_t transpose_builds = 0, normalize_builds = 0, cache_hits = 0;
    DevCsr at;            // a_hat^T (sum operand) when built
    bool have_at = false;
    DevCsr mean;          // mean operand: own transpose (or a_hat's structure) + scaled values
    bool have_mean = false;
    uint32_t* deg = nullptr;  // row_degrees(a_hat)  (gnn.hpp:193)
    std::map<std::pair<const uint64_t*, uint32_t>, sgnn_plan_s*> plans;

    ~sgnn_cache_s() {
        own.release();
        at.release();
        mean.release();
        if (deg) cudaFree(deg);
        for (auto& kv : plans) sgnn::destroy_plan(kv.second);
    }
};

namespace sgnn {
namespace {

sgnn_csr view(uint32_t rows, uint32_t cols, uint64_t nnz, const uint64_t* rp, const uint32_t* ci,
              const float* v) {
    sgnn_csr c;
    c.n_rows = rows;
    c.n_cols = cols;
    c.nnz = nnz;
    c.row_ptr = rp;
    c.col_idx = ci;
    c.values = v;
    return c;
}

sgnn_status build_transpose(sgnn_cache_s* c, DevCsr* dst, cudaStream_t s) {
    SGNN_TRY(dst->alloc(c->a_hat.n_cols, c->a_hat.nnz, true));
    SGNN_TRY(run_transpose(&c->a_hat, dst->rp, dst->ci, dst->v, nullptr, 0, s));
    ++c->transpose_builds;
    return SGNN_OK;
}

}  // namespace

sgnn_status cache_create(const sgnn_csr* a_hat, int use_cache, sgnn_cache_s** out, cudaStream_t s) {
    *out = nullptr;
    SGNN_TRY(check_csr(a_hat, "build_cache"));
    if (a_hat->n_rows != a_hat->n_cols)  // gnn.hpp:183-185
        return fail(SGNN_ERR_SHAPE, "build_cache: adjacency is " + std::to_string(a_hat->n_rows) + "x" +
                                        std::to_string(a_hat->n_cols) + ", expected square");
    auto* c = new sgnn_cache_s;
    c->a_hat = *a_hat;
    c->use_cache = use_cache != 0;
    sgnn_status st = SGNN_OK;
    if (cudaMalloc(&c->deg, sizeof(uint32_t) * (size_t(a_hat->n_rows) + 1)) != cudaSuccess)
        st = fail(SGNN_ERR_NOMEM, "build_cache: degree alloc failed");
    if (st == SGNN_OK) st = run_row_degrees(a_hat, c->deg, s);
    if (st == SGNN_OK && c->use_cache) {  // gnn.hpp:194
        int sym = 0;
        st = run_is_symmetric(a_hat, &sym, s);
        c->symmetric = sym != 0;
    }
    if (st != SGNN_OK) {
        delete c;
        return st;
    }
    *out = c;
    return SGNN_OK;
}

void cache_destroy(sgnn_cache_s* c) { delete c; }

// build_cache (gnn.hpp:180-196): GCN normalizes (counted), others borrow A.
sgnn_status cache_create_model(const sgnn_csr* a, int model_kind, int use_cache, int add_loops,
                               sgnn_cache_s** out, cudaStream_t s) {
    *out = nullptr;
    SGNN_TRY(check_csr(a, "build_cache"));
    if (a->n_rows != a->n_cols)
        return fail(SGNN_ERR_SHAPE, "build_cache: adjacency is " + std::to_string(a->n_rows) + "x" +
                                        std::to_string(a->n_cols) + ", expected square");
    if (model_kind < 0 || model_kind > 3) return fail(SGNN_ERR_CONFIG, "build_cache: unknown model kind");
    if (model_kind != 0) return cache_create(a, use_cache, out, s);
    DevCsr norm;
    uint64_t nnz = 0;
    SGNN_TRY(run_normalize(a, add_loops, &nnz, nullptr, nullptr, nullptr, s));
    SGNN_TRY(norm.alloc(a->n_rows, nnz, true));
    sgnn_status st = run_normalize(a, add_loops, &nnz, norm.rp, norm.ci, norm.v, s);
    if (st != SGNN_OK) {
        norm.release();
        return st;
    }
    sgnn_csr ah = view(a->n_rows, a->n_cols, nnz, norm.rp, norm.ci, norm.v);
    st = cache_create(&ah, use_cache, out, s);
    if (st != SGNN_OK) {
        norm.release();
        return st;
    }
    (*out)->own = norm;  // the cache owns A_hat from here on
    norm.mem = nullptr;
    (*out)->normalize_builds = 1;  // gnn.hpp:189
    return SGNN_OK;
}

sgnn_status cache_a_hat(sgnn_cache_s* c, sgnn_csr* out) {
    *out = c->a_hat;
    return SGNN_OK;
}

// gnn.hpp:127-144
sgnn_status cache_sum_operand(sgnn_cache_s* c, sgnn_csr* out, cudaStream_t s) {
    const sgnn_csr& a = c->a_hat;
    if (!c->use_cache) {
        SGNN_TRY(build_transpose(c, &c->at, s));
        c->have_at = true;
    } else if (c->symmetric) {
        ++c->cache_hits;
        *out = a;
        return SGNN_OK;
    } else if (!c->have_at) {
        SGNN_TRY(build_transpose(c, &c->at, s));
        c->have_at = true;
    } else {
        ++c->cache_hits;
    }
    *out = view(a.n_cols, a.n_rows, a.nnz, c->at.rp, c->at.ci, c->at.v);
    return SGNN_OK;
}

// gnn.hpp:149-172
sgnn_status cache_mean_operand(sgnn_cache_s* c, sgnn_csr* out, cudaStream_t s) {
    const sgnn_csr& a = c->a_hat;
    const bool shared_structure = c->use_cache && c->symmetric;
    auto build = [&]() -> sgnn_status {
        if (shared_structure) {
            SGNN_TRY(c->mean.alloc(a.n_rows, a.nnz, false));
            SGNN_TRY(run_mean_scale(a.col_idx, a.values, c->deg, a.nnz, c->mean.v, s));
        } else {
            SGNN_TRY(build_transpose(c, &c->mean, s));
            SGNN_TRY(run_mean_scale(c->mean.ci, c->mean.v, c->deg, a.nnz, c->mean.v, s));
        }
        c->have_mean = true;
        return SGNN_OK;
    };
    if (!c->use_cache || !c->have_mean) {
        SGNN_TRY(build());
    } else {
        ++c->cache_hits;
    }
    if (shared_structure)
        *out = view(a.n_rows, a.n_cols, a.nnz, a.row_ptr, a.col_idx, c->mean.v);
    else
        *out = view(a.n_cols, a.n_rows, a.nnz, c->mean.rp, c->mean.ci, c->mean.v);
    return SGNN_OK;
}

sgnn_status cache_spmm_backward(sgnn_cache_s* c, const float* dc, uint32_t dc_rows, uint32_t k,
                                float* dx, int reduce, cudaStream_t s) {
    if (dc_rows != c->a_hat.n_rows)
        return fail(SGNN_ERR_TAPE, "backward: gradient has " + std::to_string(dc_rows) +
                                       " rows but graph has " + std::to_string(c->a_hat.n_rows) +
                                       " nodes");
    if (reduce < 0 || reduce > 3) return fail(SGNN_ERR_CONFIG, "backward: unknown reduce op");
    if (reduce == SGNN_REDUCE_MIN || reduce == SGNN_REDUCE_MAX)  // SPEC.md:317 (forward only)
        return fail(SGNN_ERR_DISPATCH, "backward: min/max reductions have no backward");
    sgnn_csr op;
    if (reduce == SGNN_REDUCE_MEAN) SGNN_TRY(cache_mean_operand(c, &op, s));
    else SGNN_TRY(cache_sum_operand(c, &op, s));
    if (k == 0 || op.n_rows == 0) return SGNN_OK;
    auto key = std::make_pair(op.row_ptr, k);
    auto it = c->plans.find(key);
    sgnn_plan_s* plan = nullptr;
    if (it == c->plans.end()) {
        SGNN_TRY(build_plan(&op, k, nullptr, k % 4 == 0, &plan, s));
        c->plans[key] = plan;
    } else {
        plan = it->second;
    }
    return run_spmm(&op, dc, k, dx, SGNN_REDUCE_SUM, plan, s);
}

// dX = spmm(op, dC, Sum) for an operand already fetched from this cache (the
// GCN backward fetches sum_operand once and applies it twice, gnn.hpp:274-279)
sgnn_status cache_spmm_with_operand(sgnn_cache_s* c, const sgnn_csr* op, const float* dc, uint32_t k, float* dx,
                                    cudaStream_t s) {
    if (k == 0 || op->n_rows == 0) return SGNN_OK;
    auto key = std::make_pair(op->row_ptr, k);
    auto it = c->plans.find(key);
    sgnn_plan_s* plan = nullptr;
    if (it == c->plans.end()) {
        SGNN_TRY(build_plan(op, k, nullptr, k % 4 == 0, &plan, s));
        c->plans[key] = plan;
    } else {
        plan = it->second;
    }
    return run_spmm(op, dc, k, dx, SGNN_REDUCE_SUM, plan, s);
}

sgnn_status cache_counters(sgnn_cache_s* c, uint64_t* tb, uint64_t* nb, uint64_t* hits, int* sym) {
    if (tb) *tb = c->transpose_builds;
    if (nb) *nb = c->normalize_builds;
    if (hits) *hits = c->cache_hits;
    if (sym) *sym = c->symmetric ? 1 : 0;
    return SGNN_OK;
}

}  // namespace sgnn
