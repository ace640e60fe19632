// test_compat_ref.cpp -- the C++ drop-in compiled against the REFERENCE's own
// headers (a git-ignored copy of /root/reference/proj/include in
// baseline/_ref/include, made by __graft_entry__.build()) with
// SGNN_B200_ERROR_NS=sparsegnn: the caller's sparsegnn::CsrMatrix<float> /
// DenseMatrix<float> objects go straight into sparsegnn_b200's operators and
// the reference's exception classes come back out.  The reference's own CPU
// spmm / transpose (linked from oracle/_ref, test infrastructure) run on the
// same objects in the same process as the checker.
#include <cmath>
#include <cstdio>
#include <random>

#include "sparsegnn/autotune.hpp"  // (gnn.hpp needs DispatchGuard from here)
#include "sparsegnn/error.hpp"
#include "sparsegnn/kernels.hpp"
#include "sparsegnn/sparse.hpp"
#include "sparsegnn/types.hpp"

#define SGNN_B200_ERROR_NS sparsegnn
#include "sparsegnn_b200.hpp"
#include "sparsegnn_b200_io.hpp"
#include "sparsegnn_b200_tune.hpp"

namespace ref = sparsegnn;
namespace sg = sparsegnn_b200;

static int failures = 0;
#define EXPECT(cond)                                                             \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                          \
        }                                                                        \
    } while (0)

template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    std::mt19937_64 g(3);
    std::uniform_real_distribution<float> u(-1.f, 1.f);
    std::bernoulli_distribution keep(0.02);
    const ref::index_t m = 900, n = 700, k = 64;
    ref::CsrMatrix<float> a(m, n);
    for (ref::index_t i = 0; i < m; ++i) {
        for (ref::index_t j = 0; j < n; ++j)
            if (keep(g) || (i == 5 && j % 2 == 0)) {  // row 5: a 350-nonzero hub (two segments)
                a.col_idx.push_back(j);
                a.values.push_back(u(g));
            }
        a.row_ptr[i + 1] = a.col_idx.size();
    }
    ref::DenseMatrix<float> x(n, k);
    for (float& v : x.data) v = u(g);

    // the reference's operator API, answered on the GPU
    for (auto red : {ref::ReduceOp::Sum, ref::ReduceOp::Mean, ref::ReduceOp::Min, ref::ReduceOp::Max}) {
        const ref::DenseMatrix<float> want = ref::spmm(a, x, red, 1);
        const ref::DenseMatrix<float> got = sg::spmm(a, x, red);
        EXPECT(got.n_rows == m && got.n_cols == k);
        for (ref::index_t i = 0; i < m; ++i) {
            double denom_max = 0.0, err_max = 0.0;
            for (ref::index_t c = 0; c < k; ++c) {
                double den = 0.0;
                for (auto e = a.row_ptr[i]; e < a.row_ptr[i + 1]; ++e)
                    den += std::fabs(double(a.values[e]) * x(a.col_idx[e], c));
                if (red == ref::ReduceOp::Mean && a.row_ptr[i + 1] > a.row_ptr[i]) den /= double(a.row_ptr[i + 1] - a.row_ptr[i]);
                err_max = std::max(err_max, std::fabs(double(got(i, c)) - double(want(i, c))) - 1e-5 * den);
                denom_max = std::max(denom_max, den);
            }
            EXPECT(err_max <= 0.0);
        }
    }
    // transpose bit-exact against the reference's own
    {
        const ref::CsrMatrix<float> t_ref = ref::transpose(a);
        const ref::CsrMatrix<float> t = sg::transpose(a);
        EXPECT(t.row_ptr == t_ref.row_ptr && t.col_idx == t_ref.col_idx && t.values == t_ref.values);
        EXPECT(sg::is_symmetric(a) == ref::is_symmetric(a));
    }
    // the reference's exception classes come back out
    {
        ref::DenseMatrix<float> bad(n + 1, k);
        EXPECT(throws<ref::ShapeError>([&] { (void)sg::spmm(a, bad); }));
        EXPECT(throws<ref::DispatchError>([&] {
            (void)sg::spmm_with(a, x, ref::ReduceOp::Mean, ref::KernelKind::specialized(k));
        }));
        EXPECT(throws<ref::DispatchError>([&] {
            (void)sg::spmm_with(a, x, ref::ReduceOp::Sum, ref::KernelKind::specialized(48));
        }));
        EXPECT(throws<ref::Error>([&] { (void)sg::load_mtx<ref::CsrMatrix<float>>("/nonexistent.mtx"); }));
        EXPECT(throws<ref::IoError>([&] { (void)sg::load_report("/nonexistent.csv"); }));
    }
    // a report written by the drop-in is read by the reference's load_report
    {
        const std::vector<ref::index_t> ks{32, 64};
        sg::TuningReport r = sg::run_tuning(a, std::span<const ref::index_t>(ks), 3);
        sg::save_report(r, "/tmp/sgnn_ref_report.csv");
        const ref::TuningReport q = ref::load_report("/tmp/sgnn_ref_report.csv");
        EXPECT(q.best_k == r.best_k && q.entries.size() == r.entries.size() && q.profile.vlen == 32);
        std::remove("/tmp/sgnn_ref_report.csv");
        std::remove("/tmp/sgnn_ref_report.csv.plans.csv");
    }
    if (failures) {
        std::fprintf(stderr, "%d failures\n", failures);
        return 1;
    }
    std::printf("compat-ref OK\n");
    return 0;
}
