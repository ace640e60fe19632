// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// headers (/root/reference/proj/include/sparsegnn/*.hpp) and sources
// (/root/reference/proj/src/*.cpp), compiled by oracle/Makefile into
// oracle/_ref/libsgnn_ref_<flags>.so.
//
// TEST / BASELINE INFRASTRUCTURE ONLY: this is the reference itself, used
// (a) to pin the C restatement in oracle/sgnn_oracle.c and to generate the
// golden fixtures in tests/golden/, and (b) as bench.py's CPU reference arm
// (cpu_baseline kind "reference").  Nothing in paper_2403_14853_b200/ links it.
//
// gnn.hpp uses DispatchGuard without including autotune.hpp (gnn.hpp:424,
// autotune.hpp:40-51), so autotune.hpp is included first.
#include "sparsegnn/autotune.hpp"
#include "sparsegnn/gnn.hpp"
#include "sparsegnn/io.hpp"
#include "sparsegnn/kernels.hpp"
#include "sparsegnn/parallel.hpp"
#include "sparsegnn/sparse.hpp"

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>

using namespace sparsegnn;

namespace {

template <class T>
CsrMatrix<T> make_csr(uint32_t m, uint32_t n, const uint64_t* rp, const uint32_t* ci, const T* v) {
    CsrMatrix<T> a(m, n);
    a.row_ptr.assign(rp, rp + m + 1);
    const uint64_t nnz = rp[m];
    a.col_idx.assign(ci, ci + nnz);
    a.values.assign(v, v + nnz);
    return a;
}

template <class T>
DenseMatrix<T> make_dense(uint32_t r, uint32_t c, const T* x) {
    DenseMatrix<T> d(r, c);
    std::memcpy(d.data.data(), x, sizeof(T) * size_t(r) * c);
    return d;
}

// Status codes mirror include/sgnn_b200.h (sgnn_status).
int status_of(const std::exception& e) {
    if (dynamic_cast<const ShapeError*>(&e)) return 1;
    if (dynamic_cast<const DispatchError*>(&e)) return 2;
    if (dynamic_cast<const ConfigError*>(&e)) return 3;
    if (dynamic_cast<const TapeError*>(&e)) return 4;
    if (dynamic_cast<const InternalError*>(&e)) return 7;
    return 7;
}

template <class T>
Semiring<T> semiring(int edge_op, int reduce) {
    Semiring<T> sr;
    sr.reduce = static_cast<ReduceOp>(reduce);
    if (edge_op == 1) sr.combine = [](T p, T d) { return p * (T(1) / (T(1) + std::exp(-d))); };
    return sr;
}

}  // namespace

#define GUARD_BEGIN try {
#define GUARD_END                              \
    }                                          \
    catch (const std::exception& e) {          \
        return status_of(e);                   \
    }                                          \
    return 0;

extern "C" {

// spmm_with(a, b, reduce, kind, threads)  (kernels.hpp:157-173)
// kind: 0 = KernelKind::trusted(), 1 = KernelKind::specialized(spec_k)
int ref_spmm_f32(uint32_t m, uint32_t n, const uint64_t* rp, const uint32_t* ci, const float* v,
                 const float* x, uint32_t k, int reduce, int kind, uint32_t spec_k, int threads,
                 float* out) {
    GUARD_BEGIN
    auto a = make_csr<float>(m, n, rp, ci, v);
    auto b = make_dense<float>(n, k, x);
    auto c = spmm_with(a, b, static_cast<ReduceOp>(reduce),
                       kind ? KernelKind::specialized(spec_k) : KernelKind::trusted(), threads);
    std::memcpy(out, c.data.data(), sizeof(float) * size_t(m) * k);
    GUARD_END
}

// spmm(a, b, reduce) (kernels.hpp:179-182), fp64 instantiation = the oracle.
int ref_spmm_f64(uint32_t m, uint32_t n, const uint64_t* rp, const uint32_t* ci, const double* v,
                 const double* x, uint32_t k, int reduce, int threads, double* out) {
    GUARD_BEGIN
    auto a = make_csr<double>(m, n, rp, ci, v);
    auto b = make_dense<double>(n, k, x);
    auto c = spmm(a, b, static_cast<ReduceOp>(reduce), threads);
    std::memcpy(out, c.data.data(), sizeof(double) * size_t(m) * k);
    GUARD_END
}

// transpose (sparse.hpp:72-89)
int ref_transpose_f32(uint32_t m, uint32_t n, const uint64_t* rp, const uint32_t* ci,
                      const float* v, uint64_t* trp, uint32_t* tci, float* tv) {
    GUARD_BEGIN
    auto t = transpose(make_csr<float>(m, n, rp, ci, v));
    std::memcpy(trp, t.row_ptr.data(), sizeof(uint64_t) * (size_t(n) + 1));
    std::memcpy(tci, t.col_idx.data(), sizeof(uint32_t) * t.nnz());
    std::memcpy(tv, t.values.data(), sizeof(float) * t.nnz());
    GUARD_END
}

// sddmm (kernels.hpp:187-210)
int ref_sddmm_f32(uint32_t m, uint32_t n, const uint64_t* rp, const uint32_t* ci, const float* v,
                  const float* x, const float* y, uint32_t k, int threads, float* out) {
    GUARD_BEGIN
    auto s = sddmm(make_csr<float>(m, n, rp, ci, v), make_dense<float>(m, k, x),
                   make_dense<float>(n, k, y), threads);
    std::memcpy(out, s.values.data(), sizeof(float) * s.nnz());
    GUARD_END
}
int ref_sddmm_f64(uint32_t m, uint32_t n, const uint64_t* rp, const uint32_t* ci, const double* v,
                  const double* x, const double* y, uint32_t k, int threads, double* out) {
    GUARD_BEGIN
    auto s = sddmm(make_csr<double>(m, n, rp, ci, v), make_dense<double>(m, k, x),
                   make_dense<double>(n, k, y), threads);
    std::memcpy(out, s.values.data(), sizeof(double) * s.nnz());
    GUARD_END
}

// fusedmm (kernels.hpp:216-270); edge_op 0 = plus_times(), 1 = sigmoid combine
int ref_fusedmm_f32(uint32_t m, uint32_t n, const uint64_t* rp, const uint32_t* ci, const float* v,
                    const float* x, const float* y, uint32_t k, int edge_op, int reduce,
                    int threads, float* out) {
    GUARD_BEGIN
    auto c = fusedmm(make_csr<float>(m, n, rp, ci, v), make_dense<float>(m, k, x),
                     make_dense<float>(n, k, y), semiring<float>(edge_op, reduce), threads);
    std::memcpy(out, c.data.data(), sizeof(float) * size_t(m) * k);
    GUARD_END
}
int ref_fusedmm_f64(uint32_t m, uint32_t n, const uint64_t* rp, const uint32_t* ci,
                    const double* v, const double* x, const double* y, uint32_t k, int edge_op,
                    int reduce, int threads, double* out) {
    GUARD_BEGIN
    auto c = fusedmm(make_csr<double>(m, n, rp, ci, v), make_dense<double>(m, k, x),
                     make_dense<double>(n, k, y), semiring<double>(edge_op, reduce), threads);
    std::memcpy(out, c.data.data(), sizeof(double) * size_t(m) * k);
    GUARD_END
}

// is_symmetric (sparse.hpp:179-192)
int ref_is_symmetric_f32(uint32_t m, uint32_t n, const uint64_t* rp, const uint32_t* ci,
                         const float* v) {
    return is_symmetric(make_csr<float>(m, n, rp, ci, v)) ? 1 : 0;
}

// normalize_adjacency (sparse.hpp:116-174); trp == nullptr -> returns nnz of the result
int64_t ref_normalize_adjacency_f32(uint32_t n, const uint64_t* rp, const uint32_t* ci,
                                    const float* v, int add_self_loops, uint64_t* trp,
                                    uint32_t* tci, float* tv) {
    try {
        auto t = normalize_adjacency(make_csr<float>(n, n, rp, ci, v), add_self_loops != 0);
        if (trp) {
            std::memcpy(trp, t.row_ptr.data(), sizeof(uint64_t) * (size_t(n) + 1));
            std::memcpy(tci, t.col_idx.data(), sizeof(uint32_t) * t.nnz());
            std::memcpy(tv, t.values.data(), sizeof(float) * t.nnz());
        }
        return static_cast<int64_t>(t.nnz());
    } catch (const std::exception& e) {
        return -status_of(e);
    }
}

// balanced_row_partition (parallel.hpp:28-41)
void ref_balanced_row_partition(const uint64_t* rp, uint32_t n_rows, int n_chunks,
                                uint32_t* bounds) {
    auto b = balanced_row_partition(std::span<const offset_t>(rp, size_t(n_rows) + 1), n_rows,
                                    n_chunks);
    std::memcpy(bounds, b.data(), sizeof(uint32_t) * b.size());
}

// resolve_kernel (dispatch.cpp:21-28) under a given dispatch state.
// Returns tag*65536 + k  (tag 0 trusted, 1 specialized).
int ref_resolve_kernel(uint32_t k, int reduce, int tuned_enabled) {
    DispatchGuard g(tuned_enabled != 0);
    auto kk = resolve_kernel(k, static_cast<ReduceOp>(reduce));
    return (kk.is_specialized() ? 65536 : 0) + static_cast<int>(kk.k);
}

// TrainingCache semantics (gnn.hpp:113-196): build the cache for `model_kind`
// (0 gcn, 1 sage-sum, 2 sage-mean, 3 gin), fetch the requested operand
// `n_fetches` times (which: 0 sum_operand, 1 mean_operand), export the last
// operand and the counters {transpose_builds, normalize_builds, cache_hits, symmetric}.
int ref_cache_operand_f32(uint32_t n, const uint64_t* rp, const uint32_t* ci, const float* v,
                          int model_kind, int use_cache, int which, int n_fetches,
                          uint64_t* out_nnz, uint64_t* trp, uint32_t* tci, float* tv,
                          uint64_t* counters) {
    GUARD_BEGIN
    auto cache = build_cache(static_cast<ModelKind>(model_kind), make_csr<float>(n, n, rp, ci, v),
                             use_cache != 0, true);
    const CsrMatrix<float>* op = nullptr;
    for (int f = 0; f < n_fetches; ++f) op = which ? &cache.mean_operand() : &cache.sum_operand();
    *out_nnz = op ? op->nnz() : 0;
    if (op && trp) {
        std::memcpy(trp, op->row_ptr.data(), sizeof(uint64_t) * op->row_ptr.size());
        std::memcpy(tci, op->col_idx.data(), sizeof(uint32_t) * op->nnz());
        std::memcpy(tv, op->values.data(), sizeof(float) * op->nnz());
    }
    counters[0] = cache.transpose_builds;
    counters[1] = cache.normalize_builds;
    counters[2] = cache.cache_hits;
    counters[3] = cache.symmetric ? 1 : 0;
    GUARD_END
}

// ---- bench arm: one SpMM fwd + cached-transpose bwd "step" (gnn.hpp:290 shape) ----
struct RefBench {
    CsrMatrix<float> a, at;
    DenseMatrix<float> x, g, c, dx;
    int reduce = 0;
};

void* ref_bench_create(uint32_t m, uint32_t n, const uint64_t* rp, const uint32_t* ci,
                       const float* v, const float* x, const float* g, uint32_t k, int reduce) {
    auto* b = new RefBench;
    b->a = make_csr<float>(m, n, rp, ci, v);
    b->at = transpose(b->a);  // built once, outside the timed step (TrainingCache)
    if (reduce == 3) {        // mean backward operand, gnn.hpp:149-172
        const auto deg = row_degrees(b->a);
        for (offset_t e = 0; e < b->at.nnz(); ++e)
            b->at.values[e] = b->at.values[e] / static_cast<float>(deg[b->at.col_idx[e]]);
    }
    b->x = make_dense<float>(n, k, x);
    b->g = make_dense<float>(m, k, g);
    b->c = DenseMatrix<float>(m, k);
    b->dx = DenseMatrix<float>(n, k);
    b->reduce = reduce;
    return b;
}

// Runs fwd spmm_into(A, X) and bwd spmm_into(A^T, G) (kernels.hpp:141-149).
// kind 0 trusted, 1 specialized (Sum only, K in the sweep); which: 1 fwd, 2 bwd, 3 both.
int ref_bench_step(void* h, int kind, int threads, int which) {
    GUARD_BEGIN
    auto* b = static_cast<RefBench*>(h);
    const KernelKind kk =
        kind ? KernelKind::specialized(b->x.n_cols) : KernelKind::trusted();
    const ReduceOp red = static_cast<ReduceOp>(b->reduce);
    if (which & 1) detail::spmm_into(b->a, b->x, red, kk, threads, b->c);
    if (which & 2) detail::spmm_into(b->at, b->g, ReduceOp::Sum, kk, threads, b->dx);
    GUARD_END
}

const float* ref_bench_out(void* h, int which) {
    auto* b = static_cast<RefBench*>(h);
    return which == 2 ? b->dx.data.data() : b->c.data.data();
}

void ref_bench_free(void* h) { delete static_cast<RefBench*>(h); }

int ref_hw_cores() { return detect_hardware().cores; }

// ---- bench arm for the GNN epoch: train() (gnn.hpp:414-438) split so that
// each call runs exactly one iteration of its epoch loop (gnn.hpp:427-435:
// forward, softmax_xent, masked_accuracy, backward, sgd_step).  The one-time
// part of train() -- build_cache (gnn.hpp:423) -- runs in create, outside the
// timed region, like the reference's own per-epoch clock (gnn.hpp:428,434).
struct RefTrainer {
    GnnModel<float> model;
    TrainingCache<float> cache;
    DenseMatrix<float> x;
    std::vector<index_t> labels;
    std::vector<std::uint8_t> mask;
    float lr = 0.05f;
    int threads = 0;
    bool use_tuned = true;
};

void* ref_trainer_create(int kind, uint32_t n, const uint64_t* rp, const uint32_t* ci, const float* v,
                         uint32_t in, const float* x, const uint32_t* labels, const uint8_t* mask,
                         uint32_t hidden, uint32_t classes, const float* w_init, double lr, int threads) {
    try {
        auto* t = new RefTrainer{init_model<float>(static_cast<ModelKind>(kind), in, hidden, classes, 1)};
        size_t o = 0;
        auto get = [&](DenseMatrix<float>& w) {
            std::memcpy(w.data.data(), w_init + o, sizeof(float) * w.data.size());
            o += w.data.size();
        };
        get(t->model.w1);
        get(t->model.w2);
        if (t->model.has_self_weights()) {
            get(t->model.w1_self);
            get(t->model.w2_self);
        }
        {
            CsrMatrix<float> a = make_csr<float>(n, n, rp, ci, v);
            t->cache = build_cache(t->model.kind, a, true, true);  // TrainOptions defaults
        }
        t->x = make_dense<float>(n, in, x);
        t->labels.assign(labels, labels + n);
        t->mask.assign(mask, mask + n);
        t->lr = static_cast<float>(lr);
        t->threads = threads;
        return t;
    } catch (const std::exception&) {
        return nullptr;
    }
}

int ref_trainer_epoch(void* h, double* loss, double* acc) {
    GUARD_BEGIN
    auto* t = static_cast<RefTrainer*>(h);
    DispatchGuard dispatch(t->use_tuned);
    auto [logits, tape] = forward(t->model, t->cache, t->x, t->threads);
    auto [l, grad] = softmax_xent(logits, std::span<const index_t>(t->labels), std::span<const std::uint8_t>(t->mask));
    const double a = masked_accuracy(logits, std::span<const index_t>(t->labels), std::span<const std::uint8_t>(t->mask));
    Gradients<float> grads = backward(t->model, t->cache, tape, grad, t->threads);
    sgd_step(t->model, grads, t->lr);
    if (loss) *loss = l;
    if (acc) *acc = a;
    GUARD_END
}

void ref_trainer_free(void* h) { delete static_cast<RefTrainer*>(h); }

// ---- a ROW SAMPLE of the SAGE epoch: the same sequence of reference calls
// as forward + softmax_xent + masked_accuracy + backward + sgd_step for
// SAGE (gnn.hpp:234-244, :318-370, :283-296, :374-386), restricted to a row
// set R: every row-proportional operand has |R| rows and the three SpMMs
// run over rows R of A_hat / of the backward operand (|R| x n, all columns),
// gathering from full-height [n x K] operands.  The layer-2 and backward
// SpMM operands (h1, ds2 of ALL rows, which a sample cannot compute) are
// full-height stand-ins of the same shape.  Work (and time) scales with |R|
// and nnz(R): the bounded CPU baseline for an epoch that takes minutes.
struct RefSageSample {
    GnnModel<float> model;
    CsrMatrix<float> a_r, m_r;
    DenseMatrix<float> x, x_r, h_full, ds_full;
    std::vector<index_t> labels;
    std::vector<std::uint8_t> mask;
    float lr = 0.05f;
    int threads = 0;
};

void* ref_sage_sample_create(int kind, uint32_t n, uint32_t in, uint32_t n_r, const uint64_t* rp_a,
                             const uint32_t* ci_a, const float* v_a, const uint64_t* rp_m, const uint32_t* ci_m,
                             const float* v_m, const float* x, const float* x_r, const float* stand_in,
                             const uint32_t* labels_r, const uint8_t* mask_r, uint32_t hidden, uint32_t classes,
                             const float* w_init, double lr, int threads) {
    try {
        auto* t = new RefSageSample{init_model<float>(static_cast<ModelKind>(kind), in, hidden, classes, 1)};
        size_t o = 0;
        auto get = [&](DenseMatrix<float>& w) {
            std::memcpy(w.data.data(), w_init + o, sizeof(float) * w.data.size());
            o += w.data.size();
        };
        get(t->model.w1);
        get(t->model.w2);
        get(t->model.w1_self);
        get(t->model.w2_self);
        t->a_r = make_csr<float>(n_r, n, rp_a, ci_a, v_a);
        t->m_r = make_csr<float>(n_r, n, rp_m, ci_m, v_m);
        t->x = make_dense<float>(n, in, x);
        t->x_r = make_dense<float>(n_r, in, x_r);
        t->h_full = make_dense<float>(n, hidden, stand_in);
        t->ds_full = make_dense<float>(n, hidden, stand_in);
        t->labels.assign(labels_r, labels_r + n_r);
        t->mask.assign(mask_r, mask_r + n_r);
        t->lr = static_cast<float>(lr);
        t->threads = threads;
        return t;
    } catch (const std::exception&) {
        return nullptr;
    }
}

int ref_sage_sample_epoch(void* h, double* loss) {
    GUARD_BEGIN
    auto* t = static_cast<RefSageSample*>(h);
    const GnnModel<float>& m = t->model;
    const ReduceOp red = m.propagate_reduce();
    const int th = t->threads;
    const std::span<const index_t> lab(t->labels);
    const std::span<const std::uint8_t> msk(t->mask);
    // forward (gnn.hpp:236-244)
    DenseMatrix<float> a1 = spmm(t->a_r, t->x, red, th);
    DenseMatrix<float> z1 = matmul(a1, m.w1, th);
    add_inplace(z1, matmul(t->x_r, m.w1_self, th));
    DenseMatrix<float> h1 = relu(z1);
    DenseMatrix<float> a2 = spmm(t->a_r, t->h_full, red, th);
    DenseMatrix<float> logits = matmul(a2, m.w2, th);
    add_inplace(logits, matmul(h1, m.w2_self, th));
    // softmax_xent + masked_accuracy (gnn.hpp:318-370)
    auto [l, grad] = softmax_xent(logits, lab, msk);
    (void)masked_accuracy(logits, lab, msk);
    // backward (gnn.hpp:283-296)
    Gradients<float> g;
    g.w2 = matmul_tn(a2, grad, th);
    g.w2_self = matmul_tn(h1, grad, th);
    DenseMatrix<float> ds2 = matmul_nt(grad, m.w2, th);
    DenseMatrix<float> dh1 = spmm(t->m_r, t->ds_full, ReduceOp::Sum, th);
    add_inplace(dh1, matmul_nt(grad, m.w2_self, th));
    DenseMatrix<float> dz1 = relu_backward(dh1, h1);
    g.w1 = matmul_tn(a1, dz1, th);
    g.w1_self = matmul_tn(t->x_r, dz1, th);
    sgd_step(t->model, g, t->lr);
    (void)ds2;  // its full-height counterpart is the stand-in ds_full
    if (loss) *loss = l;
    GUARD_END
}

void ref_sage_sample_free(void* h) { delete static_cast<RefSageSample*>(h); }

// load_report (src/report.cpp:76-145): parses `path` with the reference's own
// loader; returns 0 and best_k / #entries / #skipped, or a status (6 = ParseError).
int ref_load_report(const char* path, uint32_t* best_k, uint32_t* n_entries, uint32_t* n_skipped) {
    try {
        auto r = load_report(path);
        *best_k = r.best_k;
        *n_entries = uint32_t(r.entries.size());
        *n_skipped = uint32_t(r.skipped.size());
        return 0;
    } catch (const ParseError&) {
        return 6;
    } catch (const IoError&) {
        return 5;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// ---- GNN training (gnn.hpp:75-438), the callers of the hot path --------------
// init_model (gnn.hpp:75-99): writes w1, w2 (and w1_self, w2_self for SAGE) in
// that order into `out` (sizes in*h, h*c, in*h, h*c).
int ref_init_model(int kind, uint32_t in, uint32_t hidden, uint32_t classes, uint64_t seed, float* out) {
    GUARD_BEGIN
    auto m = init_model<float>(static_cast<ModelKind>(kind), in, hidden, classes, seed);
    size_t o = 0;
    auto put = [&](const DenseMatrix<float>& w) {
        std::memcpy(out + o, w.data.data(), sizeof(float) * w.data.size());
        o += w.data.size();
    };
    put(m.w1);
    put(m.w2);
    if (m.has_self_weights()) {
        put(m.w1_self);
        put(m.w2_self);
    }
    GUARD_END
}

// train (gnn.hpp:414-438) from the given initial weights; returns per-epoch
// loss/accuracy, the final weights (same packing as ref_init_model) and the
// cache counters {transpose_builds, normalize_builds, cache_hits}.
int ref_train(int kind, uint32_t n, const uint64_t* rp, const uint32_t* ci, const float* v,
              uint32_t in, const float* x, const uint32_t* labels, const uint8_t* mask,
              uint32_t hidden, uint32_t classes, const float* w_init, int epochs, double lr,
              int use_cache, int threads, double* losses, double* accs, float* w_out,
              uint64_t* counters) {
    GUARD_BEGIN
    GnnModel<float> m = init_model<float>(static_cast<ModelKind>(kind), in, hidden, classes, 1);
    size_t o = 0;
    auto get = [&](DenseMatrix<float>& w) {
        std::memcpy(w.data.data(), w_init + o, sizeof(float) * w.data.size());
        o += w.data.size();
    };
    get(m.w1);
    get(m.w2);
    if (m.has_self_weights()) {
        get(m.w1_self);
        get(m.w2_self);
    }
    TrainOptions opts;
    opts.epochs = epochs;
    opts.lr = lr;
    opts.threads = threads;
    opts.use_cache = use_cache != 0;
    std::vector<index_t> lab(labels, labels + n);
    std::vector<std::uint8_t> msk(mask, mask + n);
    auto res = train(m, make_csr<float>(n, n, rp, ci, v), make_dense<float>(n, in, x), lab, msk, opts);
    for (int e = 0; e < epochs; ++e) {
        losses[e] = res.stats[e].loss;
        accs[e] = res.stats[e].train_accuracy;
    }
    o = 0;
    auto put = [&](const DenseMatrix<float>& w) {
        std::memcpy(w_out + o, w.data.data(), sizeof(float) * w.data.size());
        o += w.data.size();
    };
    put(m.w1);
    put(m.w2);
    if (m.has_self_weights()) {
        put(m.w1_self);
        put(m.w2_self);
    }
    counters[0] = res.cache.transpose_builds;
    counters[1] = res.cache.normalize_builds;
    counters[2] = res.cache.cache_hits;
    GUARD_END
}

// synth_planted (io.hpp:315-378): the reference's seeded node-classification set.
// Two calls: features/labels/mask sized by n/feat_dim; the graph via out_nnz + arrays.
void* ref_synth_planted(uint32_t n, uint32_t classes, double p_intra, double p_inter, uint32_t feat_dim,
                        double noise, uint64_t seed) {
    try {
        return new Dataset<float>(synth_planted<float>(n, classes, p_intra, p_inter, feat_dim, noise, seed));
    } catch (...) {
        return nullptr;
    }
}
uint64_t ref_dataset_nnz(void* h) { return static_cast<Dataset<float>*>(h)->adjacency.nnz(); }
void ref_dataset_export(void* h, uint64_t* rp, uint32_t* ci, float* v, float* x, uint32_t* labels,
                        uint8_t* mask) {
    auto* d = static_cast<Dataset<float>*>(h);
    std::memcpy(rp, d->adjacency.row_ptr.data(), sizeof(uint64_t) * d->adjacency.row_ptr.size());
    std::memcpy(ci, d->adjacency.col_idx.data(), sizeof(uint32_t) * d->adjacency.nnz());
    std::memcpy(v, d->adjacency.values.data(), sizeof(float) * d->adjacency.nnz());
    std::memcpy(x, d->features.data.data(), sizeof(float) * d->features.data.size());
    std::memcpy(labels, d->labels.data(), sizeof(uint32_t) * d->labels.size());
    std::memcpy(mask, d->train_mask.data(), d->train_mask.size());
}
void ref_dataset_free(void* h) { delete static_cast<Dataset<float>*>(h); }

// ---- on-disk formats (io.hpp:80-262) ------------------------------------------
// Each loader returns 0, 5 (IoError) or 6 (ParseError, *line = e.line()), with
// e.what() copied into err.
namespace {
int io_status(const std::exception& e, char* err, size_t err_len, long* line) {
    if (err && err_len) {
        std::strncpy(err, e.what(), err_len - 1);
        err[err_len - 1] = 0;
    }
    if (auto* p = dynamic_cast<const ParseError*>(&e)) {
        if (line) *line = p->line();
        return 6;
    }
    if (line) *line = 0;
    if (dynamic_cast<const IoError*>(&e)) return 5;
    return status_of(e);
}
}  // namespace

int ref_load_mtx(const char* path, void** out, char* err, size_t err_len, long* line) {
    try {
        *out = new CsrMatrix<float>(load_mtx<float>(path));
        return 0;
    } catch (const std::exception& e) {
        *out = nullptr;
        return io_status(e, err, err_len, line);
    }
}

void ref_csr_dims(void* h, uint32_t* m, uint32_t* n, uint64_t* nnz) {
    auto* a = static_cast<CsrMatrix<float>*>(h);
    *m = a->n_rows;
    *n = a->n_cols;
    *nnz = a->nnz();
}

void ref_csr_export(void* h, uint64_t* rp, uint32_t* ci, float* v) {
    auto* a = static_cast<CsrMatrix<float>*>(h);
    std::memcpy(rp, a->row_ptr.data(), sizeof(uint64_t) * a->row_ptr.size());
    std::memcpy(ci, a->col_idx.data(), sizeof(uint32_t) * a->col_idx.size());
    std::memcpy(v, a->values.data(), sizeof(float) * a->values.size());
}

void ref_csr_free(void* h) { delete static_cast<CsrMatrix<float>*>(h); }

int ref_save_mtx(const char* path, uint32_t m, uint32_t n, const uint64_t* rp, const uint32_t* ci, const float* v,
                 char* err, size_t err_len) {
    try {
        save_mtx(make_csr<float>(m, n, rp, ci, v), path);
        return 0;
    } catch (const std::exception& e) {
        return io_status(e, err, err_len, nullptr);
    }
}

int ref_load_features(const char* path, void** out, char* err, size_t err_len, long* line) {
    try {
        *out = new DenseMatrix<float>(load_features<float>(path));
        return 0;
    } catch (const std::exception& e) {
        *out = nullptr;
        return io_status(e, err, err_len, line);
    }
}

void ref_dense_dims(void* h, uint32_t* r, uint32_t* c) {
    auto* d = static_cast<DenseMatrix<float>*>(h);
    *r = d->n_rows;
    *c = d->n_cols;
}

void ref_dense_export(void* h, float* out) {
    auto* d = static_cast<DenseMatrix<float>*>(h);
    std::memcpy(out, d->data.data(), sizeof(float) * d->data.size());
}

void ref_dense_free(void* h) { delete static_cast<DenseMatrix<float>*>(h); }

// kind 0: load_labels, 1: load_mask; out may be NULL (count only)
int ref_load_int_column(const char* path, int kind, uint32_t* out, uint64_t* n, char* err, size_t err_len,
                        long* line) {
    try {
        if (kind == 0) {
            auto l = load_labels(path);
            *n = l.size();
            if (out) std::memcpy(out, l.data(), sizeof(uint32_t) * l.size());
        } else {
            auto m = load_mask(path);
            *n = m.size();
            if (out)
                for (size_t i = 0; i < m.size(); ++i) out[i] = m[i];
        }
        return 0;
    } catch (const std::exception& e) {
        return io_status(e, err, err_len, line);
    }
}

}  // extern "C"
