// sparsegnn_b200_tune.hpp -- C++ drop-in for the reference's tuning API
// (autotune.hpp:17-164, src/report.cpp:12-145, src/hardware.cpp:8-43):
//
//   HardwareProfile / detect_hardware     autotune.hpp:17-26 (the GPU's profile)
//   TuningEntry / TuningReport            autotune.hpp:58-74 (+ the tuned plans)
//   run_tuning(a, ks, reps, threads, seed, graph_id)   autotune.hpp:98-164
//   save_report / load_report             report.cpp:59-145, same text dialect
//
// run_tuning times, per K of the specialization sweep, the library's default
// ("trusted") SpMM plan against the on-device tuner's best ("specialized")
// plan on a seeded uniform [0,1) operand -- CUDA events, median of `reps`
// after a warm-up -- and inherits the tuner's bitwise check of every
// candidate against the default plan (InternalError on a mismatch, as
// autotune.hpp:128-133).  best_k = argmax speedup, ties to the smaller K.
// Ks outside the sweep go to `skipped`; an empty list or reps < 3 is a
// ConfigError.  The report also keeps the tuned plan of every K so it can be
// registered for later calls (`plans`).
//
// The report file is exactly report.cpp's format -- the reference's own
// load_report reads it back (tests/test_report.py) -- with the GPU mapped
// onto the profile footers: vlen = 32 (warp lanes), simd_bits = 1024,
// cores = SM count, description = device name.  Plans go to <path>.plans.csv.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <map>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "sparsegnn_b200.hpp"
#include "sparsegnn_b200_io.hpp"

namespace sparsegnn_b200 {

struct HardwareProfile {  // autotune.hpp:17-22
    int simd_bits = 1024;
    int vlen = 32;
    int cores = 1;
    std::string description = "cuda";
};

/// The device's profile (sgnn_device_info + the runtime's device name).
inline HardwareProfile detect_hardware() {
    HardwareProfile p;
    int sm = 0, l2 = 0, ma = 0, mi = 0;
    if (sgnn_device_info(&sm, &l2, &ma, &mi) == SGNN_OK) {
        p.cores = sm;
        int dev = 0;
        cudaDeviceProp prop{};
        if (cudaGetDevice(&dev) == cudaSuccess && cudaGetDeviceProperties(&prop, dev) == cudaSuccess)
            p.description = prop.name;
    }
    return p;
}

struct TuningEntry {  // autotune.hpp:58-63
    index_t k = 0;
    double t_trusted_ms = 0;
    double t_specialized_ms = 0;
    double speedup = 0;
};

struct TuningReport {  // autotune.hpp:67-74
    std::vector<TuningEntry> entries;
    index_t best_k = 0;
    HardwareProfile profile;
    std::string graph_id;
    std::vector<index_t> skipped;
    std::map<index_t, sgnn_plan_params> plans;  // K -> tuned launch geometry
};

inline constexpr index_t kSpecializationSweep[] = {16, 32, 64, 128, 256, 512, 1024};  // kernels.hpp:27

namespace tune_detail {
inline double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const std::size_t n = v.size();
    return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}
// median device time of `reps` SpMMs with `plan`
inline double time_plan(const sgnn_csr& v, const float* x, index_t k, float* c, sgnn_plan plan, int reps) {
    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
    std::vector<double> ts;
    for (int r = 0; r < reps; ++r) {
        cuda_check(cudaEventRecord(e0, nullptr), "event");
        check(sgnn_spmm_f32(&v, x, v.n_cols, k, c, SGNN_REDUCE_SUM, plan, nullptr));
        cuda_check(cudaEventRecord(e1, nullptr), "event");
        cuda_check(cudaEventSynchronize(e1), "event");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        ts.push_back(ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return median(std::move(ts));
}
inline std::string fmt(double v) {  // report.cpp's "%.9g"
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.9g", v);
    return buf;
}
inline bool u32(const std::string& s, index_t& out) {
    if (s.empty() || s.size() > 10) return false;
    std::uint64_t v = 0;
    for (char ch : s) {
        if (ch < '0' || ch > '9') return false;
        v = v * 10 + std::uint64_t(ch - '0');
    }
    if (v > 0xffffffffull) return false;
    out = index_t(v);
    return true;
}
inline bool f64(const std::string& s, double& out) {
    if (s.empty()) return false;
    char* end = nullptr;
    out = std::strtod(s.c_str(), &end);
    return end == s.c_str() + s.size();
}
inline std::vector<std::string> fields(const std::string& line) {
    std::vector<std::string> f;
    std::size_t a = 0;
    for (std::size_t b; (b = line.find(',', a)) != std::string::npos; a = b + 1) f.push_back(line.substr(a, b - a));
    f.push_back(line.substr(a));
    return f;
}
}  // namespace tune_detail

/// run_tuning (autotune.hpp:98-164) on the device.  `a` is a host CSR
/// (uploaded once) or a DeviceCsr; `threads` is accepted and ignored.
template <class Csr>
TuningReport run_tuning(const Csr& a, std::span<const index_t> ks, int reps = 5, int /*threads*/ = 0,
                        std::uint64_t seed = 42, const std::string& graph_id = "") {
    if (ks.empty()) throw SGNN_B200_ERR(ConfigError)("run_tuning: candidate list is empty");
    if (reps < 3) throw SGNN_B200_ERR(ConfigError)("run_tuning: reps must be >= 3");
    const DeviceCsr* dev_a = nullptr;
    DeviceCsr owned;
    if constexpr (std::is_same_v<Csr, DeviceCsr>) {
        dev_a = &a;
    } else {
        owned = DeviceCsr(a);
        dev_a = &owned;
    }
    const sgnn_csr v = dev_a->view();
    TuningReport report;
    report.profile = detect_hardware();
    report.graph_id = graph_id;
    std::vector<index_t> seen;
    for (index_t k : ks) {
        if (std::find(seen.begin(), seen.end(), k) != seen.end()) continue;
        seen.push_back(k);
        if (std::find(std::begin(kSpecializationSweep), std::end(kSpecializationSweep), k) ==
            std::end(kSpecializationSweep)) {
            report.skipped.push_back(k);
            continue;
        }
        std::vector<float> hb(std::size_t(v.n_cols) * k);
        std::mt19937_64 rng(seed ^ (0x9e3779b97f4a7c15ull * k));
        std::uniform_real_distribution<float> u01(0.0f, 1.0f);
        for (float& x : hb) x = u01(rng);
        DeviceBuffer<float> b(hb.data(), hb.size());
        DeviceBuffer<float> c(std::size_t(v.n_rows) * k);
        sgnn_plan best = nullptr, dflt = nullptr;
        check(sgnn_tune_spmm(&v, b.get(), k, SGNN_REDUCE_SUM, reps, &best, nullptr, 0, nullptr, nullptr));
        check(sgnn_plan_create(&v, k, nullptr, &dflt, nullptr));
        TuningEntry e;
        e.k = k;
        check(sgnn_spmm_f32(&v, b.get(), v.n_cols, k, c.get(), SGNN_REDUCE_SUM, dflt, nullptr));  // warm-up
        e.t_trusted_ms = tune_detail::time_plan(v, b.get(), k, c.get(), dflt, reps);
        e.t_specialized_ms = tune_detail::time_plan(v, b.get(), k, c.get(), best, reps);
        e.speedup = e.t_trusted_ms / e.t_specialized_ms;
        sgnn_plan_params pp{};
        check(sgnn_plan_get_params(best, &pp));
        report.plans[k] = pp;
        sgnn_plan_destroy(best);
        sgnn_plan_destroy(dflt);
        report.entries.push_back(e);
    }
    if (report.entries.empty()) throw SGNN_B200_ERR(ConfigError)("run_tuning: no requested K has a specialized kernel");
    const TuningEntry* top = &report.entries.front();
    for (const TuningEntry& e : report.entries)
        if (e.speedup > top->speedup || (e.speedup == top->speedup && e.k < top->k)) top = &e;
    report.best_k = top->k;
    return report;
}

inline constexpr const char* kReportHeader = "k,t_trusted_ms,t_specialized_ms,speedup";
inline constexpr const char* kPlanFields[] = {"lanes", "vec", "unroll", "path_items", "split_rows_over",
                                              "k_tile", "block", "scalar", "occupancy"};

/// save_report (report.cpp:59-74) + the plans sidecar.
inline void save_report(const TuningReport& r, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw SGNN_B200_IO_ERR(IoError)("cannot open '" + path + "' for writing");
    out << kReportHeader << '\n';
    for (const TuningEntry& e : r.entries)
        out << e.k << ',' << tune_detail::fmt(e.t_trusted_ms) << ',' << tune_detail::fmt(e.t_specialized_ms) << ','
            << tune_detail::fmt(e.speedup) << '\n';
    out << "best_k," << r.best_k << "\nvlen," << r.profile.vlen << "\nsimd_bits," << r.profile.simd_bits
        << "\ncores," << r.profile.cores << "\ndescription," << r.profile.description << "\ngraph_id," << r.graph_id
        << '\n';
    for (index_t k : r.skipped) out << "skipped," << k << '\n';
    if (!out) throw SGNN_B200_IO_ERR(IoError)("write to '" + path + "' failed");
    std::ofstream side(path + ".plans.csv");
    side << 'k';
    for (const char* f : kPlanFields) side << ',' << f;
    side << '\n';
    for (const auto& [k, p] : r.plans)
        side << k << ',' << p.lanes << ',' << p.vec << ',' << p.unroll << ',' << p.path_items << ','
             << p.split_rows_over << ',' << p.k_tile << ',' << p.block << ',' << p.scalar << ',' << p.occupancy
             << '\n';
}

/// load_report (report.cpp:76-145): same acceptance rules, messages and
/// 1-based line numbers; reads the plans sidecar when present.
inline TuningReport load_report(const std::string& path) {
    using tune_detail::u32;
    std::ifstream in(path);
    if (!in) throw SGNN_B200_IO_ERR(IoError)("cannot open '" + path + "'");
    TuningReport r;
    r.profile = HardwareProfile{256, 8, 1, "fallback"};  // the reference's defaults
    std::string line;
    long n = 0;
    if (!std::getline(in, line)) throw SGNN_B200_IO_ERR(ParseError)("empty report file", 1);
    ++n;
    if (line != kReportHeader)
        throw SGNN_B200_IO_ERR(ParseError)("expected header '" + std::string(kReportHeader) + "'", n);
    bool best = false, vlen = false;
    while (std::getline(in, line)) {
        ++n;
        if (line.empty()) continue;
        const auto f = tune_detail::fields(line);
        const std::string& key = f[0];
        index_t v = 0;
        auto footer = [&](const char* name) {
            if (f.size() != 2 || !u32(f[1], v))
                throw SGNN_B200_IO_ERR(ParseError)(std::string("malformed ") + name + " footer", n);
        };
        if (key == "best_k") {
            footer("best_k");
            r.best_k = v;
            best = true;
        } else if (key == "vlen") {
            footer("vlen");
            r.profile.vlen = int(v);
            r.profile.simd_bits = r.profile.vlen * 32;
            vlen = true;
        } else if (key == "simd_bits") {
            footer("simd_bits");
            r.profile.simd_bits = int(v);
        } else if (key == "cores") {
            footer("cores");
            r.profile.cores = int(v);
        } else if (key == "description") {
            r.profile.description = line.substr(key.size() + 1);
        } else if (key == "graph_id") {
            r.graph_id = line.substr(key.size() + 1);
        } else if (key == "skipped") {
            footer("skipped");
            r.skipped.push_back(v);
        } else {
            TuningEntry e;
            if (f.size() != 4 || !u32(f[0], e.k) || !tune_detail::f64(f[1], e.t_trusted_ms) ||
                !tune_detail::f64(f[2], e.t_specialized_ms) || !tune_detail::f64(f[3], e.speedup))
                throw SGNN_B200_IO_ERR(ParseError)("malformed data line '" + line + "'", n);
            if (e.t_trusted_ms <= 0 || e.t_specialized_ms <= 0 || e.speedup <= 0)
                throw SGNN_B200_IO_ERR(ParseError)("times and speedup must be positive", n);
            r.entries.push_back(e);
        }
    }
    if (r.entries.empty()) throw SGNN_B200_IO_ERR(ParseError)("report has no data lines", n + 1);
    if (!best) throw SGNN_B200_IO_ERR(ParseError)("missing best_k footer", n + 1);
    if (!vlen) throw SGNN_B200_IO_ERR(ParseError)("missing vlen footer", n + 1);
    if (std::none_of(r.entries.begin(), r.entries.end(), [&](const TuningEntry& e) { return e.k == r.best_k; }))
        throw SGNN_B200_IO_ERR(ParseError)("best_k does not match any data line", n + 1);
    std::ifstream side(path + ".plans.csv");
    if (side && std::getline(side, line)) {
        while (std::getline(side, line)) {
            if (line.empty()) continue;
            const auto f = tune_detail::fields(line);
            if (f.size() != 10) continue;
            index_t k = 0, p[9];
            bool ok = u32(f[0], k);
            for (int i = 0; i < 9 && ok; ++i) ok = u32(f[i + 1], p[i]);
            if (ok) r.plans[k] = sgnn_plan_params{p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7], p[8]};
        }
    }
    return r;
}

}  // namespace sparsegnn_b200
