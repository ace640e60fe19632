// sparsegnn_b200.hpp -- C++ drop-in over the C ABI (sgnn_b200.h) with the
// operator API of the iSpLib re-creation (proj/include/sparsegnn/):
//
//   spmm / spmm_with / detail::spmm_into   kernels.hpp:141-182
//   sddmm / fusedmm                        kernels.hpp:187-270
//   transpose / row_degrees / is_symmetric sparse.hpp:72-109,179-192
//   normalize_adjacency                    sparse.hpp:116-174
//   resolve_kernel, set_dispatch, get_dispatch, DispatchGuard
//                                          kernels.hpp:38, autotune.hpp:36-51
//   TrainingCache / build_cache            gnn.hpp:113-196
//
// Every function is a template over the matrix types, so the caller's own
// sparsegnn::CsrMatrix<float> / DenseMatrix<float> (or the look-alikes below)
// pass straight in: same names, same argument meaning, same result
// semantics, same exception classes by name.  Host operands are uploaded per
// call; for repeated calls keep operands resident: the same operators take
// DeviceCsr / DeviceDense handles (plans cached per K, stream-asynchronous,
// no upload), and TrainingCache keeps the backward operand on the device.
// Tuning (run_tuning, save_report, load_report): sparsegnn_b200_tune.hpp.
// `threads` is accepted and ignored (the GPU decides its own parallelism).
//
// Errors: sgnn_status codes become exceptions.  By default the classes below
// are thrown; define SGNN_B200_ERROR_NS to a namespace that has the
// reference's classes (e.g. `sparsegnn`, after including its error.hpp) to
// throw those instead.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sgnn_b200.h"
#include "sgnn_host.h"

namespace sparsegnn_b200 {

// ------------------------------------------------------------- errors
#ifndef SGNN_B200_ERROR_NS
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class ShapeError : public Error { public: using Error::Error; };
class DispatchError : public Error { public: using Error::Error; };
class ConfigError : public Error { public: using Error::Error; };
class TapeError : public Error { public: using Error::Error; };
class InternalError : public Error { public: using Error::Error; };
#define SGNN_B200_ERR(cls) ::sparsegnn_b200::cls
#else
#define SGNN_B200_ERR(cls) ::SGNN_B200_ERROR_NS::cls
#endif
/// CUDA runtime / device failure (no reference analogue).
class CudaError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline void check(sgnn_status st) {
    if (st == SGNN_OK) return;
    const std::string msg = sgnn_last_error();
    switch (st) {
        case SGNN_ERR_SHAPE: throw SGNN_B200_ERR(ShapeError)(msg);
        case SGNN_ERR_DISPATCH: throw SGNN_B200_ERR(DispatchError)(msg);
        case SGNN_ERR_CONFIG: throw SGNN_B200_ERR(ConfigError)(msg);
        case SGNN_ERR_TAPE: throw SGNN_B200_ERR(TapeError)(msg);
        case SGNN_ERR_INTERNAL: throw SGNN_B200_ERR(InternalError)(msg);
        default: throw CudaError(msg);
    }
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------- host types (look-alikes)
using index_t = std::uint32_t;   // types.hpp:15
using offset_t = std::uint64_t;  // types.hpp:18
enum class ReduceOp { Sum, Min, Max, Mean };  // types.hpp:116 (same order)

template <class T>
struct CsrMatrix {
    index_t n_rows = 0, n_cols = 0;
    std::vector<offset_t> row_ptr{0};
    std::vector<index_t> col_idx;
    std::vector<T> values;
    CsrMatrix() = default;
    CsrMatrix(index_t r, index_t c) : n_rows(r), n_cols(c), row_ptr(std::size_t(r) + 1, 0) {}
    offset_t nnz() const { return row_ptr.empty() ? 0 : row_ptr.back(); }
};

template <class T>
struct DenseMatrix {
    index_t n_rows = 0, n_cols = 0;
    std::vector<T> data;
    DenseMatrix() = default;
    DenseMatrix(index_t r, index_t c) : n_rows(r), n_cols(c), data(std::size_t(r) * c, T(0)) {}
    T& operator()(index_t i, index_t j) { return data[std::size_t(i) * n_cols + j]; }
    T operator()(index_t i, index_t j) const { return data[std::size_t(i) * n_cols + j]; }
};

/// KernelKind (kernels.hpp:14-25).
struct KernelKind {
    enum class Tag : std::uint8_t { Trusted, Specialized };
    Tag tag = Tag::Trusted;
    index_t k = 0;
    static constexpr KernelKind trusted() { return {Tag::Trusted, 0}; }
    static constexpr KernelKind specialized(index_t k) { return {Tag::Specialized, k}; }
    bool is_specialized() const { return tag == Tag::Specialized; }
};

/// Semiring (types.hpp:139-145) with the GPU edge-op tag.  `combine` keeps
/// the CPU meaning; the GPU runs `edge_op`.  A semiring with a combine but no
/// tag cannot run on the GPU and raises DispatchError (no CPU fallback).
template <class T>
struct Semiring {
    std::function<T(T, T)> combine;
    ReduceOp reduce = ReduceOp::Sum;
    int edge_op = -1;  // -1: derive (empty combine -> MUL)
    static Semiring plus_times() { return {nullptr, ReduceOp::Sum, SGNN_EDGE_MUL}; }
};

/// combine(p, d) = p * sigmoid(d)  (BASELINE cfg4 edge op), CPU + GPU forms.
template <class T>
Semiring<T> sigmoid_times(ReduceOp reduce = ReduceOp::Sum) {
    return {[](T p, T d) { return p * (T(1) / (T(1) + std::exp(-d))); }, reduce, SGNN_EDGE_SIGMOID_MUL};
}

// ------------------------------------------------------- device buffers
template <class T>
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t n) : n_(n) {
        if (n) cuda_check(cudaMalloc(&p_, n * sizeof(T)), "cudaMalloc");
    }
    DeviceBuffer(const T* host, std::size_t n) : DeviceBuffer(n) { upload(host, n); }
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
        return *this;
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    ~DeviceBuffer() { if (p_) cudaFree(p_); }
    void upload(const T* host, std::size_t n) {
        if (n) cuda_check(cudaMemcpy(p_, host, n * sizeof(T), cudaMemcpyHostToDevice), "upload");
    }
    void download(T* host, std::size_t n) const {
        if (n) cuda_check(cudaMemcpy(host, p_, n * sizeof(T), cudaMemcpyDeviceToHost), "download");
    }
    T* get() const { return p_; }
    std::size_t size() const { return n_; }

private:
    T* p_ = nullptr;
    std::size_t n_ = 0;
};

/// A CSR matrix resident on the device (uploaded once), with the SpMM plans
/// (work splits) built for it cached per K: the device-handle operators
/// below reuse them, so repeated calls neither re-upload nor re-plan.
class DeviceCsr {
public:
    DeviceCsr() = default;
    template <class Csr>
    explicit DeviceCsr(const Csr& a)
        : n_rows_(a.n_rows), n_cols_(a.n_cols), nnz_(a.row_ptr.empty() ? 0 : a.row_ptr.back()),
          rp_(a.row_ptr.data(), a.row_ptr.size()), ci_(a.col_idx.data(), a.col_idx.size()),
          v_(nullptr, 0), plans_(std::make_shared<Plans>()) {
        std::vector<float> vf(a.values.begin(), a.values.end());
        v_ = DeviceBuffer<float>(vf.data(), vf.size());
    }
    sgnn_csr view() const {
        return sgnn_csr{n_rows_, n_cols_, nnz_, rp_.get(), ci_.get(), v_.get()};
    }
    index_t n_rows() const { return n_rows_; }
    index_t n_cols() const { return n_cols_; }
    offset_t nnz() const { return nnz_; }

    /// The cached plan for width k (built on first use).
    sgnn_plan plan(index_t k) const {
        auto& m = plans_->map;
        auto it = m.find(k);
        if (it != m.end()) return it->second;
        const sgnn_csr v = view();
        sgnn_plan p = nullptr;
        check(sgnn_plan_create(&v, k, nullptr, &p, nullptr));
        m[k] = p;
        return p;
    }
    /// Use these launch parameters for width k from now on (e.g. a tuned
    /// plan of run_tuning / load_report: TuningReport::plans).
    void use_plan(index_t k, const sgnn_plan_params& params) {
        const sgnn_csr v = view();
        sgnn_plan p = nullptr;
        check(sgnn_plan_create(&v, k, &params, &p, nullptr));
        auto& m = plans_->map;
        if (m.count(k)) sgnn_plan_destroy(m[k]);
        m[k] = p;
    }

private:
    struct Plans {
        std::map<index_t, sgnn_plan> map;
        ~Plans() {
            for (auto& kv : map) sgnn_plan_destroy(kv.second);
        }
    };
    index_t n_rows_ = 0, n_cols_ = 0;
    offset_t nnz_ = 0;
    DeviceBuffer<offset_t> rp_;
    DeviceBuffer<index_t> ci_;
    DeviceBuffer<float> v_;
    std::shared_ptr<Plans> plans_ = std::make_shared<Plans>();
};

/// A row-major fp32 dense matrix resident on the device.
class DeviceDense {
public:
    DeviceDense() = default;
    DeviceDense(index_t r, index_t c) : n_rows(r), n_cols(c), buf_(std::size_t(r) * c) {}
    template <class Dense>
    explicit DeviceDense(const Dense& h) : n_rows(h.n_rows), n_cols(h.n_cols) {
        std::vector<float> f(h.data.begin(), h.data.end());
        buf_ = DeviceBuffer<float>(f.data(), f.size());
    }
    float* data() const { return buf_.get(); }
    std::size_t size() const { return std::size_t(n_rows) * n_cols; }
    /// Copies to a host DenseMatrix-like object (synchronous).
    template <class Dense>
    void download(Dense& h) const {
        std::vector<float> f(size());
        buf_.download(f.data(), f.size());
        h.n_rows = n_rows;
        h.n_cols = n_cols;
        h.data.assign(f.begin(), f.end());
    }
    template <class Dense = DenseMatrix<float>>
    Dense to_host() const {
        Dense h(n_rows, n_cols);
        download(h);
        return h;
    }
    index_t n_rows = 0, n_cols = 0;

private:
    DeviceBuffer<float> buf_;
};

/// Copies a device CSR view back into a host CsrMatrix-like object.
template <class Csr>
void download_csr(const sgnn_csr& v, Csr& out) {
    out.n_rows = v.n_rows;
    out.n_cols = v.n_cols;
    out.row_ptr.resize(std::size_t(v.n_rows) + 1);
    out.col_idx.resize(v.nnz);
    std::vector<float> vals(v.nnz);
    cuda_check(cudaMemcpy(out.row_ptr.data(), v.row_ptr, sizeof(offset_t) * out.row_ptr.size(),
                          cudaMemcpyDeviceToHost), "download");
    if (v.nnz) {
        cuda_check(cudaMemcpy(out.col_idx.data(), v.col_idx, sizeof(index_t) * v.nnz, cudaMemcpyDeviceToHost), "download");
        cuda_check(cudaMemcpy(vals.data(), v.values, sizeof(float) * v.nnz, cudaMemcpyDeviceToHost), "download");
    }
    out.values.assign(vals.begin(), vals.end());
}

namespace internal {
template <class Dense>
DeviceBuffer<float> upload_dense(const Dense& b) {
    std::vector<float> f(b.data.begin(), b.data.end());
    return DeviceBuffer<float>(f.data(), f.size());
}
template <class Dense>
void download_dense(const DeviceBuffer<float>& d, Dense& c) {
    std::vector<float> f(c.data.size());
    d.download(f.data(), f.size());
    c.data.assign(f.begin(), f.end());
}
template <class R>
int reduce_code(R r) { return static_cast<int>(r); }  // same order as types.hpp:116
}  // namespace internal

// --------------------------------------------------------- dispatch toggle
inline void set_dispatch(bool enabled) { sgnn_set_dispatch(enabled ? 1 : 0); }
inline bool get_dispatch() { return sgnn_get_dispatch() != 0; }
class DispatchGuard {  // autotune.hpp:40-51
public:
    explicit DispatchGuard(bool enabled) : prev_(get_dispatch()) { set_dispatch(enabled); }
    ~DispatchGuard() { set_dispatch(prev_); }
    DispatchGuard(const DispatchGuard&) = delete;
    DispatchGuard& operator=(const DispatchGuard&) = delete;

private:
    bool prev_;
};
template <class R = ReduceOp>
KernelKind resolve_kernel(index_t k, R reduce) {
    std::uint32_t sk = 0;
    const int tag = sgnn_resolve_kernel(k, internal::reduce_code(reduce), &sk);
    return tag == SGNN_KERNEL_SPECIALIZED ? KernelKind::specialized(sk) : KernelKind::trusted();
}

// -------------------------------------------------------------- operators
namespace detail {
/// detail::spmm_into (kernels.hpp:141-149): caller-owned output.
template <class Csr, class Dense, class R, class Kind>
void spmm_into(const Csr& a, const Dense& b, R reduce, Kind kind, int /*threads*/, Dense& c) {
    DeviceCsr da(a);
    auto db = internal::upload_dense(b);
    DeviceBuffer<float> dc(std::size_t(a.n_rows) * b.n_cols);
    const sgnn_csr v = da.view();
    check(sgnn_spmm_with_f32(&v, db.get(), b.n_rows, b.n_cols, dc.get(), internal::reduce_code(reduce),
                             kind.is_specialized() ? SGNN_KERNEL_SPECIALIZED : SGNN_KERNEL_TRUSTED,
                             kind.k, nullptr, nullptr));
    cuda_check(cudaDeviceSynchronize(), "spmm");
    internal::download_dense(dc, c);
}
}  // namespace detail

/// spmm_with (kernels.hpp:157-173).
template <class Csr, class Dense, class R, class Kind>
Dense spmm_with(const Csr& a, const Dense& b, R reduce, Kind kind, int threads = 0) {
    Dense c(a.n_rows, b.n_cols);
    detail::spmm_into(a, b, reduce, kind, threads, c);
    return c;
}

/// spmm (kernels.hpp:179-182): kernel picked by the dispatch state.
template <class Csr, class Dense, class R = ReduceOp>
Dense spmm(const Csr& a, const Dense& b, R reduce = R::Sum, int threads = 0) {
    return spmm_with(a, b, reduce, resolve_kernel(b.n_cols, reduce), threads);
}

/// transpose (sparse.hpp:72-89), bit-exact, computed on the device.
template <class Csr>
Csr transpose(const Csr& a) {
    DeviceCsr da(a);
    const sgnn_csr v = da.view();
    DeviceBuffer<offset_t> trp(std::size_t(a.n_cols) + 1);
    DeviceBuffer<index_t> tci(v.nnz);
    DeviceBuffer<float> tv(v.nnz);
    check(sgnn_csr_transpose(&v, trp.get(), tci.get(), tv.get(), nullptr, 0, nullptr));
    cuda_check(cudaDeviceSynchronize(), "transpose");
    Csr t;
    download_csr(sgnn_csr{a.n_cols, a.n_rows, v.nnz, trp.get(), tci.get(), tv.get()}, t);
    return t;
}

/// is_symmetric (sparse.hpp:179-192).
template <class Csr>
bool is_symmetric(const Csr& a) {
    DeviceCsr da(a);
    const sgnn_csr v = da.view();
    int out = 0;
    check(sgnn_is_symmetric(&v, &out, nullptr));
    return out != 0;
}

/// sddmm (kernels.hpp:187-210): P's pattern, values p_e * <X_i, Y_j>.
template <class Csr, class Dense>
Csr sddmm(const Csr& p, const Dense& x, const Dense& y, int /*threads*/ = 0) {
    DeviceCsr dp(p);
    auto dx = internal::upload_dense(x);
    auto dy = internal::upload_dense(y);
    DeviceBuffer<float> out(dp.nnz());
    const sgnn_csr v = dp.view();
    check(sgnn_sddmm_f32(&v, dx.get(), x.n_rows, dy.get(), y.n_rows, x.n_cols, out.get(), nullptr));
    cuda_check(cudaDeviceSynchronize(), "sddmm");
    Csr r = p;  // the reference returns a copy of P with new values (kernels.hpp:196)
    std::vector<float> f(dp.nnz());
    out.download(f.data(), f.size());
    r.values.assign(f.begin(), f.end());
    return r;
}

/// fusedmm (kernels.hpp:216-270).  Accepts the reference's Semiring (empty
/// combine = plus_times) or this header's (tagged edge op).
template <class Csr, class Dense, class SR>
Dense fusedmm(const Csr& p, const Dense& x, const Dense& y, const SR& sr, int /*threads*/ = 0) {
    int edge = SGNN_EDGE_MUL;
    if constexpr (requires { sr.edge_op; }) {
        if (sr.edge_op >= 0) edge = sr.edge_op;
        else if (sr.combine) throw SGNN_B200_ERR(DispatchError)("fusedmm: untagged combine cannot run on the GPU");
    } else {
        if (sr.combine) throw SGNN_B200_ERR(DispatchError)("fusedmm: untagged combine cannot run on the GPU");
    }
    DeviceCsr dp(p);
    auto dx = internal::upload_dense(x);
    auto dy = internal::upload_dense(y);
    DeviceBuffer<float> out(std::size_t(p.n_rows) * y.n_cols);
    const sgnn_csr v = dp.view();
    check(sgnn_fusedmm_f32(&v, dx.get(), x.n_rows, dy.get(), y.n_rows, x.n_cols, edge,
                           internal::reduce_code(sr.reduce), out.get(), nullptr));
    cuda_check(cudaDeviceSynchronize(), "fusedmm");
    Dense c(p.n_rows, y.n_cols);
    internal::download_dense(out, c);
    return c;
}
template <class Csr, class Dense>
Dense fusedmm(const Csr& p, const Dense& x, const Dense& y) {
    return fusedmm(p, x, y, Semiring<float>::plus_times());
}

// ---------------------------------------------- device-resident operators
// Same names and argument meaning as the host operators, over DeviceCsr /
// DeviceDense handles: nothing is uploaded or re-planned per call, calls are
// asynchronous on `stream` (default: the legacy stream) -- synchronise or
// download to read results.
namespace detail {
/// detail::spmm_into (kernels.hpp:141-149) on device handles.
template <class R, class Kind>
void spmm_into(const DeviceCsr& a, const DeviceDense& b, R reduce, Kind kind, int /*threads*/, DeviceDense& c,
               cudaStream_t stream = nullptr) {
    if (c.n_rows != a.n_rows() || c.n_cols != b.n_cols)
        throw SGNN_B200_ERR(ShapeError)("spmm_into: output is " + std::to_string(c.n_rows) + "x" +
                                        std::to_string(c.n_cols) + ", expected " + std::to_string(a.n_rows()) + "x" +
                                        std::to_string(b.n_cols));
    const sgnn_csr v = a.view();
    check(sgnn_spmm_with_f32(&v, b.data(), b.n_rows, b.n_cols, c.data(), internal::reduce_code(reduce),
                             kind.is_specialized() ? SGNN_KERNEL_SPECIALIZED : SGNN_KERNEL_TRUSTED, kind.k,
                             a.n_cols() == b.n_rows && b.n_cols ? a.plan(b.n_cols) : nullptr,
                             reinterpret_cast<sgnn_stream>(stream)));
}
}  // namespace detail

template <class R, class Kind>
DeviceDense spmm_with(const DeviceCsr& a, const DeviceDense& b, R reduce, Kind kind, int threads = 0,
                      cudaStream_t stream = nullptr) {
    DeviceDense c(a.n_rows(), b.n_cols);
    detail::spmm_into(a, b, reduce, kind, threads, c, stream);
    return c;
}

template <class R = ReduceOp>
DeviceDense spmm(const DeviceCsr& a, const DeviceDense& b, R reduce = R::Sum, int threads = 0,
                 cudaStream_t stream = nullptr) {
    return spmm_with(a, b, reduce, resolve_kernel(b.n_cols, reduce), threads, stream);
}

/// sddmm on device handles: the values of P's pattern (device, nnz floats).
inline DeviceBuffer<float> sddmm(const DeviceCsr& p, const DeviceDense& x, const DeviceDense& y, int /*threads*/ = 0,
                                 cudaStream_t stream = nullptr) {
    DeviceBuffer<float> out(p.nnz());
    const sgnn_csr v = p.view();
    check(sgnn_sddmm_plan_f32(&v, x.data(), x.n_rows, y.data(), y.n_rows, x.n_cols, out.get(),
                              x.n_cols && p.n_rows() == x.n_rows ? p.plan(x.n_cols) : nullptr,
                              reinterpret_cast<sgnn_stream>(stream)));
    return out;
}

template <class SR>
DeviceDense fusedmm(const DeviceCsr& p, const DeviceDense& x, const DeviceDense& y, const SR& sr, int /*threads*/ = 0,
                    cudaStream_t stream = nullptr) {
    int edge = SGNN_EDGE_MUL;
    if constexpr (requires { sr.edge_op; }) {
        if (sr.edge_op >= 0) edge = sr.edge_op;
        else if (sr.combine) throw SGNN_B200_ERR(DispatchError)("fusedmm: untagged combine cannot run on the GPU");
    } else {
        if (sr.combine) throw SGNN_B200_ERR(DispatchError)("fusedmm: untagged combine cannot run on the GPU");
    }
    DeviceDense c(p.n_rows(), y.n_cols);
    const sgnn_csr v = p.view();
    check(sgnn_fusedmm_f32(&v, x.data(), x.n_rows, y.data(), y.n_rows, x.n_cols, edge,
                           internal::reduce_code(sr.reduce), c.data(), reinterpret_cast<sgnn_stream>(stream)));
    return c;
}

// ------------------------------------------------------ structure helpers
/// row_degrees (sparse.hpp:105-109): nnz of every row.
template <class Csr>
std::vector<index_t> row_degrees(const Csr& a) {
    DeviceCsr da(a);
    const sgnn_csr v = da.view();
    DeviceBuffer<index_t> d(a.n_rows);
    check(sgnn_row_degrees(&v, d.get(), nullptr));
    std::vector<index_t> out(a.n_rows);
    cuda_check(cudaDeviceSynchronize(), "row_degrees");
    d.download(out.data(), out.size());
    return out;
}

/// normalize_adjacency (sparse.hpp:116-174) on the device, bit-exact:
/// D^-1/2 (A [+ I]) D^-1/2.
template <class Csr>
Csr normalize_adjacency(const Csr& a, bool add_self_loops = true) {
    DeviceCsr da(a);
    const sgnn_csr v = da.view();
    std::uint64_t nnz = 0;
    check(sgnn_normalize_adjacency(&v, add_self_loops ? 1 : 0, &nnz, nullptr, nullptr, nullptr, nullptr));
    DeviceBuffer<offset_t> rp(std::size_t(a.n_rows) + 1);
    DeviceBuffer<index_t> ci(nnz);
    DeviceBuffer<float> vals(nnz);
    check(sgnn_normalize_adjacency(&v, add_self_loops ? 1 : 0, &nnz, rp.get(), ci.get(), vals.get(), nullptr));
    Csr out;
    download_csr(sgnn_csr{a.n_rows, a.n_cols, nnz, rp.get(), ci.get(), vals.get()}, out);
    return out;
}

// --------------------------------------------------- backward cache (gnn.hpp)
/// TrainingCache + build_cache (gnn.hpp:113-196) with a device-resident a_hat.
/// sum_operand()/mean_operand() return device views; spmm_backward() runs
/// dX = spmm(operand, dC, Sum) on the device.
class TrainingCache {
public:
    template <class Csr>
    explicit TrainingCache(const Csr& a_hat, bool use_cache = true) : a_(a_hat) {
        const sgnn_csr v = a_.view();
        check(sgnn_cache_create(&v, use_cache ? 1 : 0, &h_, nullptr));
    }
    ~TrainingCache() { if (h_) sgnn_cache_destroy(h_); }
    TrainingCache(const TrainingCache&) = delete;
    TrainingCache& operator=(const TrainingCache&) = delete;

    sgnn_csr sum_operand() { sgnn_csr o; check(sgnn_cache_sum_operand(h_, &o, nullptr)); return o; }
    sgnn_csr mean_operand() { sgnn_csr o; check(sgnn_cache_mean_operand(h_, &o, nullptr)); return o; }

    std::uint64_t transpose_builds() const { return counter(0); }
    std::uint64_t normalize_builds() const { return counter(1); }
    std::uint64_t cache_hits() const { return counter(2); }
    bool symmetric() const { std::uint64_t a, b, c; int s; sgnn_cache_counters(h_, &a, &b, &c, &s); return s != 0; }

    /// dX = op^T-style backward SpMM for a device dC (rows = a_hat.n_rows).
    void spmm_backward(const float* dc_dev, index_t k, float* dx_dev, ReduceOp reduce = ReduceOp::Sum,
                       cudaStream_t stream = nullptr) {
        check(sgnn_spmm_backward_f32(h_, dc_dev, a_.n_rows(), k, dx_dev, static_cast<int>(reduce),
                                     reinterpret_cast<sgnn_stream>(stream)));
    }
    const DeviceCsr& a_hat() const { return a_; }

private:
    std::uint64_t counter(int i) const {
        std::uint64_t v[3];
        int s;
        check(sgnn_cache_counters(h_, &v[0], &v[1], &v[2], &s));
        return v[i];
    }
    DeviceCsr a_;
    sgnn_cache h_ = nullptr;
};

// ------------------------------------------------------ GNN training (gnn.hpp)
/// EpochStats / TrainOptions / train (gnn.hpp:389-438) over the native engine
/// (sgnn_gnn_*): the whole epoch runs on the device (SpMM, cuBLAS SGEMM,
/// device softmax-xent and SGD).  `Model` is the caller's GnnModel-like
/// object (kind, in_features, hidden, classes, w1, w2, w1_self, w2_self with
/// a `data` vector, epsilon); its parameters are updated in place, as in the
/// reference.  `cuda_graph` replays a captured epoch after the first.
struct EpochStats {
    int epoch = 0;  // 1-based
    double loss = 0;
    double train_accuracy = 0;
    double epoch_seconds = 0;
};

struct TrainOptions {
    int epochs = 100;
    double lr = 0.05;
    int threads = 0;  // accepted for signature compatibility; unused on the GPU
    bool use_tuned = true;
    bool use_cache = true;
    bool add_self_loops = true;
    bool cuda_graph = false;
};

struct TrainOutput {
    std::vector<EpochStats> stats;
    std::uint64_t transpose_builds = 0, normalize_builds = 0, cache_hits = 0;
    bool symmetric = false;
};

template <class Model, class Csr, class Dense, class Labels, class Mask>
TrainOutput train(Model& model, const Csr& a, const Dense& x, const Labels& labels, const Mask& mask,
                  const TrainOptions& opts = {}) {
    if (opts.epochs < 1) throw SGNN_B200_ERR(ConfigError)("train: epochs must be >= 1");
    if (labels.size() != a.n_rows || mask.size() != a.n_rows)
        throw SGNN_B200_ERR(ShapeError)("train: labels/mask length must equal the node count");
    const int kind = static_cast<int>(model.kind);
    const bool self_w = kind == 1 || kind == 2;
    DeviceCsr da(a);
    auto dx = internal::upload_dense(x);
    std::vector<std::uint32_t> lab(labels.begin(), labels.end());
    std::vector<std::uint8_t> msk(mask.begin(), mask.end());
    DeviceBuffer<std::uint32_t> dlab(lab.data(), lab.size());
    DeviceBuffer<std::uint8_t> dmsk(msk.data(), msk.size());
    const sgnn_csr v = da.view();
    sgnn_gnn g = nullptr;
    check(sgnn_gnn_create(&v, kind, model.in_features, model.hidden, model.classes, dx.get(), dlab.get(),
                          dmsk.get(), opts.use_cache ? 1 : 0, opts.add_self_loops ? 1 : 0,
                          static_cast<std::uint32_t>(opts.epochs), &g, nullptr));
    struct Guard {
        sgnn_gnn g;
        ~Guard() { sgnn_gnn_destroy(g); }
    } guard{g};
    auto f32 = [](const auto& m) { return std::vector<float>(m.data.begin(), m.data.end()); };
    std::vector<float> w1 = f32(model.w1), w2 = f32(model.w2), w1s, w2s;
    if (self_w) {
        w1s = f32(model.w1_self);
        w2s = f32(model.w2_self);
    }
    check(sgnn_gnn_set_weights(g, w1.data(), w2.data(), self_w ? w1s.data() : nullptr,
                               self_w ? w2s.data() : nullptr, static_cast<float>(model.epsilon), nullptr));
    const std::size_t e = static_cast<std::size_t>(opts.epochs);
    std::vector<double> loss(e), acc(e), secs(e);
    check(sgnn_gnn_train(g, static_cast<std::uint32_t>(opts.epochs), static_cast<float>(opts.lr),
                         opts.cuda_graph ? 1 : 0, loss.data(), acc.data(), secs.data(), nullptr));
    float eps = 0.0f;
    check(sgnn_gnn_get_weights(g, w1.data(), w2.data(), self_w ? w1s.data() : nullptr,
                               self_w ? w2s.data() : nullptr, &eps, nullptr));
    auto put = [](auto& m, const std::vector<float>& f) { std::copy(f.begin(), f.end(), m.data.begin()); };
    put(model.w1, w1);
    put(model.w2, w2);
    if (self_w) {
        put(model.w1_self, w1s);
        put(model.w2_self, w2s);
    }
    model.epsilon = eps;
    TrainOutput out;
    for (std::size_t i = 0; i < e; ++i) out.stats.push_back({int(i) + 1, loss[i], acc[i], secs[i]});
    int sym = 0;
    check(sgnn_gnn_counters(g, &out.transpose_builds, &out.normalize_builds, &out.cache_hits, &sym));
    out.symmetric = sym != 0;
    return out;
}

// ------------------------------------------- multi-GPU: row-partitioned SAGE
/// The communicator of the row partition (sgnn_comm_*): one process per GPU
/// over NCCL (the 128-byte id from rank 0 travels over the caller's channel),
/// or P virtual ranks in one process (loopback).
class Comm {
public:
    static std::vector<std::uint8_t> unique_id() {
        std::vector<std::uint8_t> id(SGNN_COMM_ID_BYTES);
        check(sgnn_comm_get_unique_id(id.data()));
        return id;
    }
    static Comm nccl(const std::vector<std::uint8_t>& id, int nranks, int rank) {
        Comm c;
        check(sgnn_comm_init_rank(id.data(), nranks, rank, &c.h_));
        return c;
    }
    static Comm loopback(int nranks) {
        Comm c;
        check(sgnn_comm_init_loopback(nranks, &c.h_));
        return c;
    }
    Comm() = default;
    Comm(Comm&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    Comm& operator=(Comm&& o) noexcept {
        std::swap(h_, o.h_);
        return *this;
    }
    ~Comm() { if (h_) sgnn_comm_destroy(h_); }
    sgnn_comm get() const { return h_; }

private:
    sgnn_comm h_ = nullptr;
};

/// Contiguous row bounds of equal nnz + row_weight * rows cost
/// (balanced_row_partition, parallel.hpp:28-41, at GPU granularity).
template <class Csr>
std::vector<std::uint32_t> row_partition(const Csr& a, int parts, std::uint32_t row_weight = 30) {
    std::vector<std::uint32_t> b(std::size_t(parts) + 1);
    sgnn_host_weighted_row_partition(a.row_ptr.data(), a.n_rows, parts, row_weight, b.data());
    return b;
}

/// One rank of the row-partitioned SAGE trainer (train(), gnn.hpp:414-438,
/// on rows [bounds[rank], bounds[rank+1]) of a symmetric A): the rank's
/// block is uploaded from the caller's host CSR and features.
class PartitionedSage {
public:
    template <class Csr, class Dense, class Labels, class Mask>
    PartitionedSage(const Comm* comm, int rank, const std::vector<std::uint32_t>& bounds, const Csr& a, const Dense& x,
                    const Labels& labels, const Mask& mask, int model_kind /* 1 sum, 2 mean */, index_t hidden,
                    index_t classes, std::uint32_t max_epochs = 128)
        : r0_(bounds.at(std::size_t(rank))), rows_(bounds.at(std::size_t(rank) + 1) - r0_) {
        const offset_t e0 = a.row_ptr[r0_], e1 = a.row_ptr[r0_ + rows_];
        std::vector<offset_t> rp(rows_ + 1);
        for (index_t i = 0; i <= rows_; ++i) rp[i] = a.row_ptr[r0_ + i] - e0;
        std::vector<float> v(a.values.begin() + std::ptrdiff_t(e0), a.values.begin() + std::ptrdiff_t(e1));
        rp_ = DeviceBuffer<offset_t>(rp.data(), rp.size());
        ci_ = DeviceBuffer<index_t>(a.col_idx.data() + e0, std::size_t(e1 - e0));
        v_ = DeviceBuffer<float>(v.data(), v.size());
        const sgnn_csr blk{rows_, a.n_cols, e1 - e0, rp_.get(), ci_.get(), v_.get()};
        std::vector<float> xr(x.data.begin() + std::ptrdiff_t(std::size_t(r0_) * x.n_cols),
                              x.data.begin() + std::ptrdiff_t(std::size_t(r0_ + rows_) * x.n_cols));
        std::vector<std::uint32_t> lab(labels.begin() + r0_, labels.begin() + r0_ + rows_);
        std::vector<std::uint8_t> msk(mask.begin() + r0_, mask.begin() + r0_ + rows_);
        check(sgnn_dist_create(comm ? comm->get() : nullptr, rank, bounds.data(), &blk, nullptr, model_kind, x.n_cols,
                               hidden, classes, xr.data(), lab.data(), msk.data(), max_epochs, &h_, nullptr));
    }
    ~PartitionedSage() { if (h_) sgnn_dist_destroy(h_); }
    PartitionedSage(const PartitionedSage&) = delete;
    PartitionedSage& operator=(const PartitionedSage&) = delete;

    /// Weights in the model's layout (w1, w2, w1_self, w2_self with `data`).
    template <class Model>
    void set_weights(const Model& m) {
        auto f = [](const auto& w) { return std::vector<float>(w.data.begin(), w.data.end()); };
        const auto w1 = f(m.w1), w2 = f(m.w2), w1s = f(m.w1_self), w2s = f(m.w2_self);
        check(sgnn_dist_set_weights(h_, w1.data(), w2.data(), w1s.data(), w2s.data(), nullptr));
    }
    /// `epochs` epochs on this rank alone (NCCL rank or one rank).
    void epochs(std::uint32_t n, float lr) {
        sgnn_dist g = h_;
        check(sgnn_dist_epochs(&g, 1, n, lr, nullptr));
        run_ += n;
    }
    /// Loopback: all P ranks of one communicator, in rank order.
    static void epochs_group(std::vector<PartitionedSage*>& ranks, std::uint32_t n, float lr) {
        std::vector<sgnn_dist> hs;
        for (auto* r : ranks) hs.push_back(r->h_);
        check(sgnn_dist_epochs(hs.data(), int(hs.size()), n, lr, nullptr));
        for (auto* r : ranks) r->run_ += n;
    }
    /// Per-epoch loss (the global masked mean) of the epochs run so far.
    std::vector<double> losses() const {
        std::vector<double> l(run_);
        if (run_) check(sgnn_dist_stats(h_, 0, run_, l.data(), nullptr, nullptr, nullptr));
        return l;
    }
    index_t row0() const { return r0_; }
    index_t rows() const { return rows_; }

private:
    index_t r0_ = 0, rows_ = 0;
    DeviceBuffer<offset_t> rp_;
    DeviceBuffer<index_t> ci_;
    DeviceBuffer<float> v_;
    sgnn_dist h_ = nullptr;
    std::uint32_t run_ = 0;
};

}  // namespace sparsegnn_b200
