// sparsegnn_b200_io.hpp -- C++ drop-in for the reference's io.hpp loaders
// (load_mtx / save_mtx / load_features / load_labels / load_mask,
// io.hpp:80-262) over libsgnn_host.so (include/sgnn_host.h).  Same
// acceptance rules, messages and 1-based line numbers; the entry lines are
// parsed by all host cores.  Errors: IoError(msg) / ParseError(msg, line) of
// SGNN_B200_ERROR_NS when defined (e.g. sparsegnn), else the classes below.
//
// Link: -L<repo>/paper_2403_14853_b200 -lsgnn_host
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sgnn_host.h"

namespace sparsegnn_b200 {

#ifndef SGNN_B200_ERROR_NS
class IoError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& what, long line)
        : std::runtime_error("line " + std::to_string(line) + ": " + what), line_(line) {}
    long line() const noexcept { return line_; }

private:
    long line_;
};
#define SGNN_B200_IO_ERR(cls) ::sparsegnn_b200::cls
#else
#define SGNN_B200_IO_ERR(cls) ::SGNN_B200_ERROR_NS::cls
#endif

namespace io_detail {
inline void raise(int st, const char* err, long line) {
    if (st == 6) throw SGNN_B200_IO_ERR(ParseError)(err, line);
    if (st == 5) throw SGNN_B200_IO_ERR(IoError)(err);
    throw std::runtime_error(err);
}
}  // namespace io_detail

/// load_mtx<float> (io.hpp:80-165) into any CsrMatrix-like type with
/// n_rows, n_cols, row_ptr, col_idx, values (a (rows, cols) constructor).
template <class Csr>
Csr load_mtx(const std::string& path, int threads = 0) {
    void* h = nullptr;
    char err[4096] = {0};
    long line = 0;
    const int st = sgnn_host_mtx_load(path.c_str(), threads, &h, err, sizeof err, &line);
    if (st) io_detail::raise(st, err, line);
    uint32_t m = 0, n = 0;
    uint64_t nnz = 0;
    sgnn_host_csr_dims(h, &m, &n, &nnz);
    Csr a(m, n);
    std::vector<uint64_t> rp(std::size_t(m) + 1);
    std::vector<uint32_t> ci(nnz);
    std::vector<float> v(nnz);
    sgnn_host_csr_export(h, rp.data(), ci.data(), v.data());
    sgnn_host_csr_free(h);
    a.row_ptr.assign(rp.begin(), rp.end());
    a.col_idx.assign(ci.begin(), ci.end());
    a.values.assign(v.begin(), v.end());
    return a;
}

/// save_mtx (io.hpp:168-185): coordinate real general, "%.9g" values.
template <class Csr>
void save_mtx(const Csr& a, const std::string& path, int threads = 0) {
    std::vector<uint64_t> rp(a.row_ptr.begin(), a.row_ptr.end());
    std::vector<uint32_t> ci(a.col_idx.begin(), a.col_idx.end());
    std::vector<float> v(a.values.begin(), a.values.end());
    char err[4096] = {0};
    const int st = sgnn_host_mtx_save(path.c_str(), uint32_t(a.n_rows), uint32_t(a.n_cols), rp.data(), ci.data(),
                                      v.data(), threads, err, sizeof err);
    if (st) io_detail::raise(st, err, 0);
}

/// load_features<float> (io.hpp:187-205) into a DenseMatrix-like type.
template <class Dense>
Dense load_features(const std::string& path, int threads = 0) {
    void* h = nullptr;
    char err[4096] = {0};
    long line = 0;
    const int st = sgnn_host_features_load(path.c_str(), threads, &h, err, sizeof err, &line);
    if (st) io_detail::raise(st, err, line);
    uint32_t r = 0, c = 0;
    sgnn_host_dense_dims(h, &r, &c);
    Dense d(r, c);
    std::vector<float> f(std::size_t(r) * c);
    sgnn_host_dense_export(h, f.data());
    sgnn_host_dense_free(h);
    d.data.assign(f.begin(), f.end());
    return d;
}

namespace io_detail {
inline std::vector<uint32_t> int_column(const std::string& path, int kind) {
    char err[4096] = {0};
    long line = 0;
    uint64_t n = 0;
    int st = sgnn_host_int_column_load(path.c_str(), kind, 0, nullptr, &n, err, sizeof err, &line);
    if (st) raise(st, err, line);
    std::vector<uint32_t> out(n);
    st = sgnn_host_int_column_load(path.c_str(), kind, n, out.data(), &n, err, sizeof err, &line);
    if (st) raise(st, err, line);
    return out;
}
}  // namespace io_detail

/// load_labels (io.hpp:243-251)
inline std::vector<uint32_t> load_labels(const std::string& path) { return io_detail::int_column(path, 0); }

/// load_mask (io.hpp:254-262)
inline std::vector<uint8_t> load_mask(const std::string& path) {
    const auto v = io_detail::int_column(path, 1);
    return std::vector<uint8_t>(v.begin(), v.end());
}

}  // namespace sparsegnn_b200
