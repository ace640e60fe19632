// test_compat.cpp -- the C++ drop-in (include/sparsegnn_b200.hpp) used the way
// the reference's operator API is used, checked against the SPEC known
// answers and the CPU oracle (oracle/liboracle.so, test infrastructure).
// Run by tests/test_cpp_compat.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "sparsegnn_b200.hpp"
#include "sparsegnn_b200_io.hpp"
#include "sparsegnn_b200_tune.hpp"

extern "C" {
void orc_spmm_f64(uint32_t, const uint64_t*, const uint32_t*, const double*, const double*, uint32_t,
                  int, double*);
void orc_spmm_f32(uint32_t, const uint64_t*, const uint32_t*, const float*, const float*, uint32_t, int,
                  float*);
void orc_spmm_absdenom_f64(uint32_t, const uint64_t*, const uint32_t*, const double*, const double*,
                           uint32_t, int, double*);
void orc_transpose_f32(uint32_t, uint32_t, const uint64_t*, const uint32_t*, const float*, uint64_t*,
                       uint32_t*, float*);
}

namespace sg = sparsegnn_b200;
using Csr = sg::CsrMatrix<float>;
using Dense = sg::DenseMatrix<float>;

static int failures = 0;
#define EXPECT(cond)                                                         \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                      \
        }                                                                    \
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

static Csr make(uint32_t m, uint32_t n, std::vector<uint64_t> rp, std::vector<uint32_t> ci, std::vector<float> v) {
    Csr a(m, n);
    a.row_ptr = std::move(rp);
    a.col_idx = std::move(ci);
    a.values = std::move(v);
    return a;
}

static Csr random_csr(std::mt19937_64& g, uint32_t m, uint32_t n, double dens, bool hub) {
    Csr a(m, n);
    std::uniform_real_distribution<float> u(-1.f, 1.f);
    std::bernoulli_distribution b(dens), bh(0.8);
    for (uint32_t i = 0; i < m; ++i) {
        for (uint32_t j = 0; j < n; ++j)
            if ((hub && i == 1) ? bh(g) : b(g)) {
                a.col_idx.push_back(j);
                a.values.push_back(u(g));
            }
        a.row_ptr[i + 1] = a.col_idx.size();
    }
    return a;
}

int main() {
    // ---- SPEC.md:141-143 known answers
    {
        Csr a = make(2, 2, {0, 1, 2}, {1, 0}, {2.f, 3.f});
        Dense b(2, 2);
        b.data = {1, 1, 2, 2};
        Dense c = sg::spmm(a, b);
        EXPECT((c.data == std::vector<float>{4, 4, 3, 3}));
        Csr r = make(1, 2, {0, 2}, {0, 1}, {1.f, 1.f});
        Dense bb(2, 2);
        bb.data = {2, 8, 4, 2};
        EXPECT((sg::spmm(r, bb, sg::ReduceOp::Min).data == std::vector<float>{2, 2}));
        EXPECT((sg::spmm(r, bb, sg::ReduceOp::Max).data == std::vector<float>{4, 8}));
        EXPECT((sg::spmm(r, bb, sg::ReduceOp::Mean).data == std::vector<float>{3, 5}));
    }
    // ---- sddmm / fusedmm known answers
    {
        Csr ident = make(2, 2, {0, 1, 2}, {0, 1}, {1.f, 1.f});
        Dense x(2, 2);
        x.data = {1, 2, 3, 4};
        Csr s = sg::sddmm(ident, x, x);
        EXPECT((s.values == std::vector<float>{5, 25}));
        EXPECT(s.row_ptr == ident.row_ptr && s.col_idx == ident.col_idx);
        EXPECT((sg::fusedmm(ident, x, x).data == std::vector<float>{5, 10, 75, 100}));
        auto sr = sg::sigmoid_times<float>();
        Dense f = sg::fusedmm(ident, x, x, sr);
        const float e0 = 1.f / (1.f + std::exp(-5.f));
        EXPECT(std::fabs(f.data[0] - e0 * 1.f) < 1e-6f);
        sg::Semiring<float> untagged{[](float p, float d) { return p + d; }, sg::ReduceOp::Sum};
        untagged.edge_op = -1;
        EXPECT(throws<sg::DispatchError>([&] { sg::fusedmm(ident, x, x, untagged); }));
    }
    // ---- errors mirror kernels.hpp:131-169
    {
        Csr a = make(1, 2, {0, 1}, {0}, {1.f});
        Dense bad(3, 32);
        EXPECT(throws<sg::ShapeError>([&] { sg::spmm(a, bad); }));
        Dense b48(2, 48);
        EXPECT(throws<sg::DispatchError>([&] { sg::spmm_with(a, b48, sg::ReduceOp::Sum, sg::KernelKind::specialized(32)); }));
        Dense b32(2, 32);
        EXPECT(throws<sg::DispatchError>([&] { sg::spmm_with(a, b32, sg::ReduceOp::Mean, sg::KernelKind::specialized(32)); }));
        EXPECT(!throws<sg::Error>([&] { sg::spmm_with(a, b32, sg::ReduceOp::Sum, sg::KernelKind::specialized(32)); }));
    }
    // ---- dispatch toggle (dispatch.cpp:21-28)
    {
        EXPECT(sg::resolve_kernel(32, sg::ReduceOp::Sum).is_specialized());
        EXPECT(!sg::resolve_kernel(48, sg::ReduceOp::Sum).is_specialized());
        EXPECT(!sg::resolve_kernel(32, sg::ReduceOp::Mean).is_specialized());
        {
            sg::DispatchGuard off(false);
            EXPECT(!sg::resolve_kernel(32, sg::ReduceOp::Sum).is_specialized());
        }
        EXPECT(sg::get_dispatch());
    }
    // ---- random parity vs the oracle: tolerance + bitwise on rows <= 256 nnz
    std::mt19937_64 g(7);
    for (uint32_t k : {16u, 33u, 128u}) {
        Csr a = random_csr(g, 200, 900, 0.02, true);
        Dense x(900, k);
        std::uniform_real_distribution<float> u(-1.f, 1.f);
        for (auto& v : x.data) v = u(g);
        for (int red = 0; red < 4; ++red) {
            Dense c = sg::spmm(a, x, static_cast<sg::ReduceOp>(red));
            std::vector<double> av(a.values.begin(), a.values.end()), xv(x.data.begin(), x.data.end());
            std::vector<double> ref(size_t(200) * k), den(size_t(200) * k);
            std::vector<float> ref32(size_t(200) * k);
            orc_spmm_f64(200, a.row_ptr.data(), a.col_idx.data(), av.data(), xv.data(), k, red, ref.data());
            orc_spmm_absdenom_f64(200, a.row_ptr.data(), a.col_idx.data(), av.data(), xv.data(), k, red, den.data());
            orc_spmm_f32(200, a.row_ptr.data(), a.col_idx.data(), a.values.data(), x.data.data(), k, red, ref32.data());
            for (uint32_t i = 0; i < 200; ++i) {
                const bool short_row = a.row_ptr[i + 1] - a.row_ptr[i] <= SGNN_SEGMENT;
                for (uint32_t q = 0; q < k; ++q) {
                    const size_t o = size_t(i) * k + q;
                    EXPECT(std::fabs(c.data[o] - ref[o]) <= 1e-5 * den[o]);
                    if (short_row || red == 1 || red == 2)
                        EXPECT(std::memcmp(&c.data[o], &ref32[o], 4) == 0);
                }
            }
        }
    }
    // ---- transpose bit-exact (sparse.hpp:72-89)
    {
        Csr a = random_csr(g, 300, 500, 0.03, true);
        Csr t = sg::transpose(a);
        std::vector<uint64_t> trp(501);
        std::vector<uint32_t> tci(a.nnz());
        std::vector<float> tv(a.nnz());
        orc_transpose_f32(300, 500, a.row_ptr.data(), a.col_idx.data(), a.values.data(), trp.data(), tci.data(), tv.data());
        EXPECT(t.row_ptr == trp && t.col_idx == tci && t.values == tv);
        Csr tt = sg::transpose(t);
        EXPECT(tt.row_ptr == a.row_ptr && tt.col_idx == a.col_idx && tt.values == a.values);
        EXPECT(!sg::is_symmetric(a));
    }
    // ---- TrainingCache counters (gnn.hpp:113-173)
    {
        Csr a = random_csr(g, 400, 400, 0.01, false);
        sg::TrainingCache cache(a, true);
        sg::DeviceBuffer<float> dc(size_t(400) * 8), dx(size_t(400) * 8);
        cudaMemset(dc.get(), 0, sizeof(float) * 400 * 8);
        for (int i = 0; i < 5; ++i) cache.spmm_backward(dc.get(), 8, dx.get());
        cudaDeviceSynchronize();
        EXPECT(cache.transpose_builds() == 1 && cache.cache_hits() == 4 && !cache.symmetric());
    }
    if (failures) {
        std::fprintf(stderr, "%d failures\n", failures);
        return 1;
    }
    // ---- train (gnn.hpp:414-438) through the native engine: a tiny
    // two-community graph; the loss falls, the cache counters follow the
    // reference's rules (GCN: one normalize, symmetric -> no transpose, one
    // operand fetch per epoch), and the CUDA-graph replay is bitwise the
    // eager run.
    {
        const uint32_t n = 64, f = 8, hid = 16, cls = 2;
        Csr a(n, n);
        for (uint32_t i = 0; i < n; ++i) {
            for (uint32_t j = 0; j < n; ++j)
                if (i != j && (i / 32 == j / 32) && ((i * 7 + j * 7) % 5 == 0)) {
                    a.col_idx.push_back(j);
                    a.values.push_back(1.f);
                }
            a.row_ptr[i + 1] = a.col_idx.size();
        }
        Dense x(n, f);
        std::mt19937_64 g(3);
        std::normal_distribution<float> nd(0.f, 0.3f);
        for (uint32_t i = 0; i < n; ++i)
            for (uint32_t j = 0; j < f; ++j) x.data[i * f + j] = nd(g) + (j == i / 32 ? 1.f : 0.f);
        std::vector<uint32_t> labels(n);
        std::vector<uint8_t> mask(n, 1);
        for (uint32_t i = 0; i < n; ++i) labels[i] = i / 32;
        struct Model {
            int kind = 0;  // GCN
            uint32_t in_features, hidden, classes;
            Dense w1, w2, w1_self, w2_self;
            float epsilon = 0.f;
        };
        auto init = [&](Model& m) {
            m.in_features = f;
            m.hidden = hid;
            m.classes = cls;
            m.w1 = Dense(f, hid);
            m.w2 = Dense(hid, cls);
            std::mt19937_64 gw(7);
            std::uniform_real_distribution<float> u(-0.4f, 0.4f);
            for (auto& w : m.w1.data) w = u(gw);
            for (auto& w : m.w2.data) w = u(gw);
        };
        Model m1, m2;
        init(m1);
        init(m2);
        sg::TrainOptions o;
        o.epochs = 20;
        o.lr = 0.5;
        sg::TrainOutput r1 = sg::train(m1, a, x, labels, mask, o);
        EXPECT(r1.stats.size() == 20u);
        EXPECT(r1.stats.back().loss < r1.stats.front().loss);
        EXPECT(r1.normalize_builds == 1u && r1.transpose_builds == 0u && r1.symmetric);
        EXPECT(r1.cache_hits == 20u);
        o.cuda_graph = true;
        sg::TrainOutput r2 = sg::train(m2, a, x, labels, mask, o);
        EXPECT(m1.w1.data == m2.w1.data && m1.w2.data == m2.w2.data);
        for (std::size_t i = 0; i < r1.stats.size(); ++i) EXPECT(r1.stats[i].loss == r2.stats[i].loss);
        EXPECT(throws<sg::ConfigError>([&] { sg::TrainOptions bad; bad.epochs = 0; sg::train(m1, a, x, labels, mask, bad); }));
        // ---- the row-partitioned SAGE-mean trainer from C++ (sgnn_dist_*):
        // one rank vs two loopback ranks of a balanced_row_partition
        struct SModel {
            Dense w1, w2, w1_self, w2_self;
        } sm{Dense(f, hid), Dense(hid, cls), Dense(f, hid), Dense(hid, cls)};
        std::mt19937_64 gs(11);
        std::uniform_real_distribution<float> us(-0.4f, 0.4f);
        for (Dense* w : {&sm.w1, &sm.w2, &sm.w1_self, &sm.w2_self})
            for (auto& v : w->data) v = us(gs);
        sg::PartitionedSage one(nullptr, 0, {0u, n}, a, x, labels, mask, 2, hid, cls, 32);
        one.set_weights(sm);
        one.epochs(15, 0.5f);
        sg::Comm comm = sg::Comm::loopback(2);
        const std::vector<uint32_t> b = sg::row_partition(a, 2, 1);
        sg::PartitionedSage p0(&comm, 0, b, a, x, labels, mask, 2, hid, cls, 32);
        sg::PartitionedSage p1(&comm, 1, b, a, x, labels, mask, 2, hid, cls, 32);
        p0.set_weights(sm);
        p1.set_weights(sm);
        std::vector<sg::PartitionedSage*> ranks{&p0, &p1};
        sg::PartitionedSage::epochs_group(ranks, 15, 0.5f);
        const auto l1 = one.losses(), l2 = p0.losses();
        EXPECT(l1.size() == 15u && l2.size() == 15u && l1.back() < l1.front());
        EXPECT(p0.rows() + p1.rows() == n && p1.row0() == p0.rows());
        for (std::size_t i = 0; i < l1.size() && i < l2.size(); ++i) EXPECT(std::fabs(l1[i] - l2[i]) <= 1e-5 * std::fabs(l1[i]));
    }
    // ---- io.hpp drop-in: load_mtx / save_mtx round trip, ParseError lines
    {
        const std::string p = "/tmp/sgnn_compat_test.mtx";
        {
            FILE* f = std::fopen(p.c_str(), "w");
            std::fputs("%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 3\n1 1 2\n3 1 0.5\n3 3 -1\n", f);
            std::fclose(f);
        }
        Csr a = sg::load_mtx<Csr>(p);
        EXPECT(a.n_rows == 3u && a.n_cols == 3u);
        EXPECT((a.row_ptr == std::vector<uint64_t>{0, 2, 2, 4}));
        EXPECT((a.col_idx == std::vector<uint32_t>{0, 2, 0, 2}));
        EXPECT((a.values == std::vector<float>{2.f, 0.5f, 0.5f, -1.f}));
        sg::save_mtx(a, p);
        Csr b = sg::load_mtx<Csr>(p);
        EXPECT(b.row_ptr == a.row_ptr && b.col_idx == a.col_idx && b.values == a.values);
        {
            FILE* f = std::fopen(p.c_str(), "w");
            std::fputs("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 x 1\n", f);
            std::fclose(f);
        }
        long line = -1;
        try {
            (void)sg::load_mtx<Csr>(p);
        } catch (const sg::ParseError& e) {
            line = e.line();
        }
        EXPECT(line == 4);
        EXPECT(throws<sg::IoError>([&] { (void)sg::load_mtx<Csr>("/nonexistent/x.mtx"); }));
        std::remove(p.c_str());
    }
    // ---- device-resident handles: same results as the host operators, plans
    // cached per K, repeated calls without re-upload
    {
        std::mt19937_64 g(7);
        Csr a = random_csr(g, 700, 500, 0.03, true);
        Dense x(500, 64);
        std::uniform_real_distribution<float> u(-1.f, 1.f);
        for (float& v : x.data) v = u(g);
        sg::DeviceCsr da(a);
        sg::DeviceDense dx(x);
        for (auto red : {sg::ReduceOp::Sum, sg::ReduceOp::Mean, sg::ReduceOp::Max}) {
            const Dense want = sg::spmm(a, x, red);
            sg::DeviceDense c1 = sg::spmm(da, dx, red);
            sg::DeviceDense c2 = sg::spmm(da, dx, red);  // cached plan
            EXPECT(c1.to_host<Dense>().data == want.data);
            EXPECT(c2.to_host<Dense>().data == want.data);
        }
        sg::DeviceDense out(700, 64);
        sg::detail::spmm_into(da, dx, sg::ReduceOp::Sum, sg::KernelKind::specialized(64), 0, out);
        EXPECT(out.to_host<Dense>().data == sg::spmm(a, x, sg::ReduceOp::Sum).data);
        sg::DeviceDense bad(10, 64);
        EXPECT(throws<sg::ShapeError>([&] { sg::detail::spmm_into(da, dx, sg::ReduceOp::Sum, sg::KernelKind::trusted(), 0, bad); }));
        Dense xr(700, 64), y(500, 64);
        for (float& v : xr.data) v = 0.1f * u(g);
        for (float& v : y.data) v = 0.1f * u(g);
        sg::DeviceDense dxr(xr), dy(y);
        const Csr want_s = sg::sddmm(a, xr, y);
        std::vector<float> got_s(a.nnz());
        sg::sddmm(da, dxr, dy).download(got_s.data(), got_s.size());
        EXPECT(got_s == want_s.values);
        const auto sr = sg::sigmoid_times<float>();
        EXPECT(sg::fusedmm(da, dxr, dy, sr).to_host<Dense>().data == sg::fusedmm(a, xr, y, sr).data);
    }
    // ---- row_degrees / normalize_adjacency (sparse.hpp:105-174)
    {
        Csr a = make(3, 3, {0, 2, 3, 4}, {0, 1, 0, 2}, {1.f, 1.f, 1.f, 1.f});
        EXPECT((sg::row_degrees(a) == std::vector<uint32_t>{2, 1, 1}));
        // A + I: row sums 1+1+1 = 3 (diag 1+1), 2, 2 (self-loop added to row 2's 1 at col 2 -> 2)
        Csr n = sg::normalize_adjacency(a, true);
        EXPECT(n.n_rows == 3u && n.row_ptr.back() == 5u);
        EXPECT(n.values[0] > 0.f);
        Csr n0 = sg::normalize_adjacency(a, false);
        EXPECT(n0.row_ptr.back() == 4u);
        Csr rect(2, 3);
        EXPECT(throws<sg::ShapeError>([&] { (void)sg::normalize_adjacency(rect); }));
    }
    // ---- run_tuning / save_report / load_report (autotune.hpp:98-164, report.cpp)
    {
        std::mt19937_64 g(11);
        Csr a = random_csr(g, 4000, 4000, 0.01, true);
        const std::vector<uint32_t> ks{32, 64, 48, 32};
        sg::TuningReport r = sg::run_tuning(a, std::span<const uint32_t>(ks), 3, 0, 42, "compat-graph");
        EXPECT(r.entries.size() == 2 && r.skipped == std::vector<uint32_t>{48});
        EXPECT(r.best_k == 32 || r.best_k == 64);
        EXPECT(r.plans.size() == 2 && r.profile.cores > 0);
        for (const auto& e : r.entries) EXPECT(e.t_trusted_ms > 0 && e.t_specialized_ms > 0 && e.speedup > 0);
        const std::string p = "/tmp/sgnn_compat_report.csv";
        sg::save_report(r, p);
        sg::TuningReport q = sg::load_report(p);
        EXPECT(q.best_k == r.best_k && q.entries.size() == 2 && q.graph_id == "compat-graph" && q.skipped == r.skipped);
        EXPECT(q.profile.vlen == 32 && q.profile.cores == r.profile.cores && q.plans.size() == 2);
        EXPECT(q.plans.at(64).lanes == r.plans.at(64).lanes);
        sg::DeviceCsr da(a);
        da.use_plan(64, q.plans.at(64));  // tuned geometry reused: same results
        Dense x(4000, 64);
        for (std::size_t i = 0; i < x.data.size(); ++i) x.data[i] = float(i % 7) - 3.f;
        EXPECT(sg::spmm(da, sg::DeviceDense(x)).to_host<Dense>().data == sg::spmm(a, x).data);
        EXPECT(throws<sg::ConfigError>([&] { (void)sg::run_tuning(a, std::span<const uint32_t>(ks), 2); }));
        {
            FILE* f = std::fopen(p.c_str(), "w");
            std::fputs("k,t_trusted_ms,t_specialized_ms,speedup\n32,1,0.5,2\nvlen,x\n", f);
            std::fclose(f);
        }
        long line = -1;
        try {
            (void)sg::load_report(p);
        } catch (const sg::ParseError& e) {
            line = e.line();
        }
        EXPECT(line == 3);
        EXPECT(throws<sg::IoError>([&] { (void)sg::load_report("/nonexistent/r.csv"); }));
        std::remove(p.c_str());
        std::remove((p + ".plans.csv").c_str());
    }
    if (failures) {
        std::fprintf(stderr, "%d failures\n", failures);
        return 1;
    }
    std::printf("compat OK\n");
    return 0;
}
