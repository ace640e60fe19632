// dist.cu -- the row-partitioned GraphSAGE trainer (BASELINE cfg5, SURVEY
// 8e): train() of gnn.hpp:414-438 for SAGE-sum / SAGE-mean with the graph's
// rows split into P contiguous blocks, one block per GPU, and the C ABI
// (sgnn_comm_*, sgnn_dist_*) that owns the NCCL communicator.
//
// Rank r owns rows [b_r, b_{r+1}) of A (global column ids, no remap), the
// same rows of X, of every activation and of the labels/mask.  The SpMM
// gathers rows of a *full-height* operand buffer ([n, K], rank r's rows at
// b_r); the only sparse-path exchange is an in-place all-gather-v of those
// buffers (grouped ncclSend/ncclRecv: each rank receives exactly the other
// ranks' rows, no padding), so the gathered buffer IS the operand in its own
// row order and each local row is accumulated exactly as on one GPU.  Dense
// weight gradients and the (loss, correct) pair are all-reduced.
//
// One epoch = compute phases separated by exchanges:
//   [X all-gather, when features changed]
//   phase 0  a1 = A_r X (mean), h1_r = relu([a1 | X_r] [W1; W1s])  (gnn.hpp:237-240)
//   exch     all-gather h1
//   phase 1  a2 = A_r h1; logits, softmax_xent + accuracy and ds2_r = grad W2^T
//            in one pass (sage_head_kernel); W2/W2s gradients     (:241-244, :318-370, :283-289)
//   exch     all-gather grad (16 floats a row, not ds2's 128)
//   phase 2  the other ranks' ds2 rows = their grad rows W2^T (bitwise the
//            owners'), dh1 = M_r ds2 (M = mean/sum backward operand rows), dz1 =
//            relu_backward(dh1 + grad W2s^T), W1/W1s gradients    (:290-296)
//   exch     all-reduce gradients + (loss, correct)
//   phase 3  sgd_step (:374-386), epoch stats
// The symmetric short-circuit (gnn.hpp:152-153) gives M_r from A_r itself
// (mean: values / deg[col] with the all-gathered global degrees); a
// non-symmetric graph passes rows of A^T as the backward block.
//
// Communicators: NCCL (one process per GPU, ncclCommInitRank; libnccl is
// dlopen'ed, so the library itself does not depend on it), or *loopback*:
// P virtual ranks in one process and on one stream, phase by phase, so the
// partition logic and the per-rank work balance can be measured on one GPU.
#include <cublas_v2.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "ops.cuh"
#include "plan.cuh"

namespace {

using sgnn::fail;

// ------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
    bool loaded = false;
    std::string why;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclGetVersion) GetVersion = nullptr;
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        // reuse the NCCL the process already has (torch's), else the system one
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return a;
        }
#define SGNN_NCCL_SYM(name)                                                         \
    a.name = reinterpret_cast<decltype(a.name)>(dlsym(h, "nccl" #name));          \
    if (!a.name) {                                                                \
        a.why = "libnccl lacks nccl" #name;                                       \
        return a;                                                                 \
    }
        SGNN_NCCL_SYM(GetUniqueId)
        SGNN_NCCL_SYM(CommInitRank)
        SGNN_NCCL_SYM(CommDestroy)
        SGNN_NCCL_SYM(Send)
        SGNN_NCCL_SYM(Recv)
        SGNN_NCCL_SYM(GroupStart)
        SGNN_NCCL_SYM(GroupEnd)
        SGNN_NCCL_SYM(AllReduce)
        SGNN_NCCL_SYM(GetErrorString)
        SGNN_NCCL_SYM(GetVersion)
#undef SGNN_NCCL_SYM
        a.loaded = true;
        return a;
    }();
    return api;
}

sgnn_status nccl_ok(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return SGNN_OK;
    return fail(SGNN_ERR_CUDA, std::string("NCCL ") + what + ": " + nccl().GetErrorString(r));
}

constexpr int kCommNccl = 0, kCommLoopback = 1;
constexpr int kSageSum = 1, kSageMean = 2;  // ModelKind order, gnn.hpp:17

// ------------------------------------------------------------------ kernels
unsigned ew_grid(uint64_t n) {
    const uint64_t b = (n + 255) / 256;
    return unsigned(b < 2368 ? (b ? b : 1) : 2368);  // 16 CTAs per SM at most
}

// w -= lr * g over the packed weights (sgd_step, gnn.hpp:374-386)
__global__ void pack_sgd_kernel(float* __restrict__ w, const float* __restrict__ g, uint64_t n, float lr) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        w[i] = __fsub_rn(w[i], __fmul_rn(lr, g[i]));
}

// dst += src (loopback all-reduce, ranks added in rank order)
template <class T>
__global__ void add_into_kernel(T* __restrict__ dst, const T* __restrict__ src, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        dst[i] += src[i];
}

// (loss_sum, correct) of this rank's rows from softmax_xent's per-block
// partials, in block order (deterministic for a given partition)
// (one block of 256: strided partial sums, then a fixed tree)
__global__ void __launch_bounds__(256) rank_stats_kernel(const double* __restrict__ blk_loss,
                                                         const uint32_t* __restrict__ blk_ok, uint32_t nblk,
                                                         double* __restrict__ out) {
    __shared__ double sl[256], sk[256];
    double l = 0.0, k = 0.0;
    for (uint32_t b = threadIdx.x; b < nblk; b += 256) {
        l += blk_loss[b];
        k += double(blk_ok[b]);
    }
    sl[threadIdx.x] = l;
    sk[threadIdx.x] = k;
    __syncthreads();
    for (uint32_t h = 128; h >= 1; h >>= 1) {
        if (threadIdx.x < h) {
            sl[threadIdx.x] += sl[threadIdx.x + h];
            sk[threadIdx.x] += sk[threadIdx.x + h];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = sl[0];
        out[1] = sk[0];
    }
}

__global__ void epoch_record_kernel(const double* __restrict__ red, double inv_n, double* __restrict__ stats) {
    stats[0] = red[0] * inv_n;  // mean masked cross-entropy (softmax_xent's loss * inv_n)
    stats[1] = red[1] * inv_n;  // masked accuracy
}

// mean operand values: v[e] / deg[col[e]] (gnn.hpp:158-159), IEEE divide
__global__ void mean_values_kernel(const uint32_t* __restrict__ ci, const float* __restrict__ vin,
                                   const uint32_t* __restrict__ deg, uint64_t nnz, float* __restrict__ vout) {
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz; e += uint64_t(gridDim.x) * blockDim.x)
        vout[e] = __fdiv_rn(vin[e], float(deg[ci[e]]));
}

// deg[r] = row_ptr[r+1] - row_ptr[r] for the block's rows (written at the
// rank's offset of the global degree array)
__global__ void block_degrees_kernel(const uint64_t* __restrict__ rp, uint32_t rows, uint32_t* __restrict__ deg) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
        deg[r] = uint32_t(rp[r + 1] - rp[r]);
}

}  // namespace

// -------------------------------------------------------------- communicator
struct sgnn_comm_s {
    int kind = kCommNccl;
    int nranks = 1, rank = 0;
    ncclComm_t comm = nullptr;
    std::vector<sgnn_dist_s*> members;  // loopback: engine of each virtual rank

    ~sgnn_comm_s() {
        if (comm) nccl().CommDestroy(comm);
    }
};

// ------------------------------------------------------------------- engine
enum Mark {  // per-epoch event markers (P*_S / P*_E: a compute phase of this rank)
    M_BEGIN, M_X, M_P0_S, M_SPMM1_0, M_SPMM1_1, M_GEMM1_1, M_P0_E, M_EX1, M_P1_S, M_SPMM2_0, M_SPMM2_1, M_P1_E, M_EX2,
    M_P2_S, M_SPMMB_0, M_SPMMB_1, M_GEMM2_0, M_P2_E, M_EX3, M_P3_S, M_END, M_COUNT
};

struct sgnn_dist_s {
    sgnn_comm_s* comm = nullptr;  // null: one rank
    int P = 1, rank = 0;
    std::vector<uint32_t> bounds;  // P+1
    uint32_t n = 0, r0 = 0, rows = 0;
    int kind = kSageMean;
    uint32_t in = 0, hid = 0, cls = 0;
    sgnn_csr fwd{};       // A_r (borrowed)
    sgnn_csr bwd{};       // M_r (borrowed structure; values owned for mean)
    bool bwd_given = false;
    float* bwd_vals = nullptr;
    sgnn_plan_s* plan_in = nullptr;   // A_r at K = in
    sgnn_plan_s* plan_hid = nullptr;  // A_r at K = hid (== plan_in when in == hid)
    sgnn_plan_s* plan_bwd = nullptr;  // M_r at K = hid
    cublasHandle_t blas = nullptr;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    bool dense_tc = true;
    std::vector<void*> owned;
    // full-height operands (gathered) and rank-local activations
    // ax = [a1 | X_r] (R x 2 in): the layer-1 aggregate beside the rank's
    // own features, so a1 W1 + X_r W1s is ONE product with [W1; W1s] (and the
    // weight gradient one A^T B); with one rank X_r is also the SpMM operand
    // (row stride 2 in), with P ranks the gathered x_full [n x in] is.
    float *ax = nullptr, *x_full = nullptr, *h1_full = nullptr, *ds2_full = nullptr;
    float *a2 = nullptr, *z1 = nullptr, *dh1 = nullptr;
    float* grad_full = nullptr;  // [n x classes]: the rank's rows at r0, the others gathered
    float* grad() const { return grad_full + uint64_t(r0) * cls; }
    uint32_t* labels = nullptr;
    uint8_t* mask = nullptr;
    uint32_t* deg = nullptr;  // global degrees [n] (gathered)
    uint64_t n_masked_local = 0, n_masked = 0;
    double inv_n = 0.0;
    // packs: weights and gradients [w1 | w2 | w1s | w2s], each slice 64-float aligned
    float *wpack = nullptr, *gpack = nullptr;
    uint64_t off_w1 = 0, off_w2 = 0, off_w1s = 0, off_w2s = 0, pack_n = 0;
    uint32_t sm_blocks = 0;  // softmax partial blocks
    double* blk_loss = nullptr;
    uint32_t* blk_ok = nullptr;
    uint32_t wg_rpb = 0, wg_blocks = 0;
    float* wg_part = nullptr;
    double* red = nullptr;    // (loss_sum, correct), all-reduced
    double* stats = nullptr;  // [2 * max_epochs]
    uint32_t max_epochs = 0, epoch = 0;
    bool prepared = false, x_dirty = true;
    std::vector<cudaEvent_t> ev;  // [max_epochs * M_COUNT]

    const float* x_operand() const { return P == 1 ? ax + in : x_full; }
    uint64_t x_ld() const { return P == 1 ? 2ull * in : uint64_t(in); }
    cudaEvent_t mark(uint32_t e, int m) { return ev[size_t(e) * M_COUNT + m]; }

    ~sgnn_dist_s() {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
        if (plan_hid && plan_hid != plan_in) sgnn::destroy_plan(plan_hid);
        if (plan_in) sgnn::destroy_plan(plan_in);
        if (plan_bwd) sgnn::destroy_plan(plan_bwd);
        if (blas) cublasDestroy(blas);
        for (void* p : owned) cudaFree(p);
    }
};

namespace {

template <class T>
sgnn_status dalloc(sgnn_dist_s* g, T** p, uint64_t count) {
    void* m = nullptr;
    SGNN_CUDA_TRY(cudaMalloc(&m, sizeof(T) * (count ? count : 1)));
    g->owned.push_back(m);
    *p = static_cast<T*>(m);
    return SGNN_OK;
}

sgnn_status blas_ok(cublasStatus_t st, const char* what) {
    if (st != CUBLAS_STATUS_SUCCESS) return fail(SGNN_ERR_CUDA, std::string("cuBLAS ") + what + " failed");
    return SGNN_OK;
}

bool tall_ok(const sgnn_dist_s* g, uint32_t m, uint32_t k, uint32_t n, std::initializer_list<const void*> ptrs) {
    if (!g->dense_tc || m < 4096 || k < 32 || n < 32 || k % 4 || n % 4) return false;
    for (const void* p : ptrs)
        if (reinterpret_cast<uintptr_t>(p) % 16) return false;
    return true;
}

// C[m,n] = A[m,k] B[k,n] (row-major): tensor-core FP32 product, else SGEMM
sgnn_status mm(sgnn_dist_s* g, const float* A, const float* B, float* Cm, uint32_t m, uint32_t k, uint32_t n,
               cudaStream_t s) {
    if (m == 0) return SGNN_OK;
    if (tall_ok(g, m, k, n, {A, B, Cm}) &&
        sgnn::dense_mm_nn(int(m), int(n), int(k), A, B, Cm, 0.0f, g->ws, g->ws_bytes, s) == 0)
        return SGNN_OK;
    const float one = 1.0f, zero = 0.0f;
    cublasSetStream(g->blas, s);
    return blas_ok(cublasSgemm(g->blas, CUBLAS_OP_N, CUBLAS_OP_N, int(n), int(m), int(k), &one, B, int(n), A, int(k),
                               &zero, Cm, int(n)),
                   "mm");
}

// C[k,n] = A[m,k]^T B[m,n]
sgnn_status mm_tn(sgnn_dist_s* g, const float* A, const float* B, float* Cm, uint32_t m, uint32_t k, uint32_t n,
                  cudaStream_t s) {
    if (m == 0) return cudaMemsetAsync(Cm, 0, sizeof(float) * k * n, s) == cudaSuccess
                           ? SGNN_OK
                           : fail(SGNN_ERR_CUDA, "dist: memset");
    if (tall_ok(g, m, k, n, {A, B, Cm})) {
        const int splits = int(std::max<uint32_t>(1, std::min<uint32_t>(148, m / 8192)));
        if (sgnn::dense_mm_tn(int(m), int(n), int(k), A, B, Cm, splits, g->ws, g->ws_bytes, s) == 0) return SGNN_OK;
    }
    const float one = 1.0f, zero = 0.0f;
    cublasSetStream(g->blas, s);
    return blas_ok(cublasSgemm(g->blas, CUBLAS_OP_N, CUBLAS_OP_T, int(n), int(k), int(m), &one, B, int(n), A, int(k),
                               &zero, Cm, int(n)),
                   "mm_tn");
}

// ---- exchanges over the engines this call drives (NCCL: one; loopback: P)
// In-place all-gather-v: rank q's rows [b_q, b_{q+1}) of buf(q) (width w
// 4-byte words) to every other rank's buffer at the same rows.
template <class BufOf>
sgnn_status allgather_rows(sgnn_dist_s* const* gs, int ng, BufOf buf, uint64_t w, cudaStream_t s) {
    sgnn_dist_s* g0 = gs[0];
    const int P = g0->P;
    if (P == 1) return SGNN_OK;
    const auto& b = g0->bounds;
    if (g0->comm->kind == kCommNccl) {
        NcclApi& api = nccl();
        const int me = g0->rank;
        float* base = reinterpret_cast<float*>(buf(g0));
        SGNN_TRY(nccl_ok(api.GroupStart(), "group start"));
        for (int q = 0; q < P; ++q) {
            if (q == me) continue;
            const uint64_t mine = uint64_t(b[me + 1] - b[me]) * w, theirs = uint64_t(b[q + 1] - b[q]) * w;
            if (mine) {
                const ncclResult_t r = api.Send(base + uint64_t(b[me]) * w, mine, ncclFloat, q, g0->comm->comm, s);
                if (r != ncclSuccess) {
                    api.GroupEnd();
                    return nccl_ok(r, "send");
                }
            }
            if (theirs) {
                const ncclResult_t r = api.Recv(base + uint64_t(b[q]) * w, theirs, ncclFloat, q, g0->comm->comm, s);
                if (r != ncclSuccess) {
                    api.GroupEnd();
                    return nccl_ok(r, "recv");
                }
            }
        }
        return nccl_ok(api.GroupEnd(), "group end");
    }
    // loopback: device copies between the virtual ranks' buffers
    for (int q = 0; q < ng; ++q) {
        const uint64_t off = uint64_t(b[q]) * w * 4, bytes = uint64_t(b[q + 1] - b[q]) * w * 4;
        if (!bytes) continue;
        const char* src = reinterpret_cast<const char*>(buf(gs[q])) + off;
        for (int r = 0; r < ng; ++r)
            if (r != q)
                SGNN_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<char*>(buf(gs[r])) + off, src, bytes,
                                              cudaMemcpyDeviceToDevice, s));
    }
    return SGNN_OK;
}

// Sum of the gradient pack and the (loss, correct) pair over the ranks.
sgnn_status allreduce_grads(sgnn_dist_s* const* gs, int ng, cudaStream_t s) {
    sgnn_dist_s* g0 = gs[0];
    if (g0->P == 1) return SGNN_OK;
    if (g0->comm->kind == kCommNccl) {
        NcclApi& api = nccl();
        SGNN_TRY(nccl_ok(api.GroupStart(), "group start"));
        ncclResult_t r = api.AllReduce(g0->gpack, g0->gpack, g0->pack_n, ncclFloat, ncclSum, g0->comm->comm, s);
        if (r == ncclSuccess) r = api.AllReduce(g0->red, g0->red, 2, ncclDouble, ncclSum, g0->comm->comm, s);
        const ncclResult_t e = api.GroupEnd();
        SGNN_TRY(nccl_ok(r, "all-reduce"));
        return nccl_ok(e, "group end");
    }
    for (int r = 1; r < ng; ++r) {
        add_into_kernel<float><<<ew_grid(g0->pack_n), 256, 0, s>>>(g0->gpack, gs[r]->gpack, g0->pack_n);
        add_into_kernel<double><<<1, 32, 0, s>>>(g0->red, gs[r]->red, 2);
    }
    SGNN_LAUNCH_CHECK();
    for (int r = 1; r < ng; ++r) {
        SGNN_CUDA_TRY(cudaMemcpyAsync(gs[r]->gpack, g0->gpack, sizeof(float) * g0->pack_n, cudaMemcpyDeviceToDevice, s));
        SGNN_CUDA_TRY(cudaMemcpyAsync(gs[r]->red, g0->red, 2 * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    return SGNN_OK;
}

// ---- one-time collective preparation (first epochs call): global degrees
// and the mean backward operand, the global masked-row count.
sgnn_status prepare(sgnn_dist_s* const* gs, int ng, cudaStream_t s) {
    for (int i = 0; i < ng; ++i) {
        sgnn_dist_s* g = gs[i];
        if (g->rows)
            block_degrees_kernel<<<ew_grid(g->rows), 256, 0, s>>>(g->fwd.row_ptr, g->rows, g->deg + g->r0);
        SGNN_LAUNCH_CHECK();
    }
    SGNN_TRY(allgather_rows(gs, ng, [](sgnn_dist_s* g) { return static_cast<void*>(g->deg); }, 1, s));
    // global masked count
    uint64_t total = 0;
    if (gs[0]->P > 1 && gs[0]->comm->kind == kCommNccl) {
        double* tmp = nullptr;
        SGNN_TRY(sgnn::scratch_alloc(reinterpret_cast<void**>(&tmp), sizeof(double), s));
        const double local = double(gs[0]->n_masked_local);
        SGNN_CUDA_TRY(cudaMemcpyAsync(tmp, &local, sizeof(double), cudaMemcpyHostToDevice, s));
        SGNN_TRY(nccl_ok(nccl().AllReduce(tmp, tmp, 1, ncclDouble, ncclSum, gs[0]->comm->comm, s), "all-reduce"));
        double got = 0.0;
        SGNN_CUDA_TRY(cudaMemcpyAsync(&got, tmp, sizeof(double), cudaMemcpyDeviceToHost, s));
        SGNN_CUDA_TRY(cudaStreamSynchronize(s));
        sgnn::scratch_free(tmp, s);
        total = uint64_t(got);
    } else {
        for (int i = 0; i < ng; ++i) total += gs[i]->n_masked_local;
    }
    if (total == 0) return fail(SGNN_ERR_CONFIG, "softmax_xent: mask selects no rows");
    for (int i = 0; i < ng; ++i) {
        sgnn_dist_s* g = gs[i];
        g->n_masked = total;
        g->inv_n = 1.0 / double(total);
        if (g->kind == kSageMean && g->bwd.nnz)  // mean operand values (gnn.hpp:149-172)
            mean_values_kernel<<<ew_grid(g->bwd.nnz), 256, 0, s>>>(
                g->bwd.col_idx, g->bwd_given ? g->bwd.values : g->fwd.values, g->deg, g->bwd.nnz, g->bwd_vals);
        SGNN_LAUNCH_CHECK();
        if (g->kind == kSageMean) g->bwd.values = g->bwd_vals;
        g->prepared = true;
    }
    return SGNN_OK;
}

#define DIST_MARK(g, m) SGNN_CUDA_TRY(cudaEventRecord((g)->mark(e, (m)), s))

// phase 0: a1 = A_r X, h1_r = relu(a1 W1 + X_r W1s)
sgnn_status phase0(sgnn_dist_s* g, uint32_t e, cudaStream_t s) {
    const int red = g->kind == kSageMean ? SGNN_REDUCE_MEAN : SGNN_REDUCE_SUM;
    DIST_MARK(g, M_P0_S);
    DIST_MARK(g, M_SPMM1_0);
    if (g->rows)  // a1 into the left half of ax
        SGNN_TRY(sgnn::run_spmm_ld(&g->fwd, g->x_operand(), g->x_ld(), g->in, g->ax, 2ull * g->in, red, g->plan_in, s));
    DIST_MARK(g, M_SPMM1_1);
    // h1_r = relu([a1 | X_r] [W1; W1s]): relu in the product's epilogue, or a separate pass
    float* h1r = g->h1_full + uint64_t(g->r0) * g->hid;
    const float* w1cat = g->wpack + g->off_w1;
    if (!(tall_ok(g, g->rows, 2 * g->in, g->hid, {g->ax, w1cat, h1r}) &&
          sgnn::dense_mm_nn_relu(int(g->rows), int(g->hid), int(2 * g->in), g->ax, w1cat, h1r, g->ws, g->ws_bytes,
                                 s) == 0)) {
        SGNN_TRY(mm(g, g->ax, w1cat, g->z1, g->rows, 2 * g->in, g->hid, s));
        SGNN_TRY(sgnn::glue_relu(g->z1, uint64_t(g->rows) * g->hid, h1r, s));
    }
    DIST_MARK(g, M_GEMM1_1);
    DIST_MARK(g, M_P0_E);
    return SGNN_OK;
}

// phase 1: a2 = A_r h1, logits, softmax_xent, W2 / W2s gradients, ds2_r
sgnn_status phase1(sgnn_dist_s* g, uint32_t e, cudaStream_t s) {
    const int red = g->kind == kSageMean ? SGNN_REDUCE_MEAN : SGNN_REDUCE_SUM;
    const float* h1r = g->h1_full + uint64_t(g->r0) * g->hid;
    DIST_MARK(g, M_P1_S);
    DIST_MARK(g, M_SPMM2_0);
    if (g->rows) SGNN_TRY(sgnn::run_spmm(&g->fwd, g->h1_full, g->hid, g->a2, red, g->plan_hid, s));
    DIST_MARK(g, M_SPMM2_1);
    // logits, softmax_xent + accuracy, grad, ds2_r = grad W2^T in one pass
    SGNN_TRY(sgnn::sage_head_partials(g->a2, h1r, g->wpack + g->off_w2, g->wpack + g->off_w2s, g->rows, g->hid,
                                      g->cls, g->labels, g->mask, g->inv_n, g->grad(),
                                      g->ds2_full + uint64_t(g->r0) * g->hid, g->blk_loss, g->blk_ok, s));
    rank_stats_kernel<<<1, 256, 0, s>>>(g->blk_loss, g->blk_ok, g->rows ? g->sm_blocks : 0, g->red);
    SGNN_LAUNCH_CHECK();
    if (g->rows) {
        SGNN_TRY(sgnn::sage_wgrad_launch(g->a2, h1r, g->grad(), g->rows, g->hid, g->cls, g->wg_rpb, g->wg_blocks,
                                         g->wg_part, g->gpack + g->off_w2, g->gpack + g->off_w2s, s));
    } else {
        SGNN_CUDA_TRY(cudaMemsetAsync(g->gpack + g->off_w2, 0, sizeof(float) * (g->pack_n - g->off_w2), s));
    }
    DIST_MARK(g, M_P1_E);
    return SGNN_OK;
}

// phase 2: dh1 = M_r ds2, dz1 = relu_backward(dh1 + grad W2s^T, h1), W1 / W1s gradients
sgnn_status phase2(sgnn_dist_s* g, uint32_t e, cudaStream_t s) {
    const float* h1r = g->h1_full + uint64_t(g->r0) * g->hid;
    DIST_MARK(g, M_P2_S);
    if (g->P > 1) {
        // the other ranks' ds2 rows from their gathered gradient rows (16
        // floats a row on the wire instead of 128): the head's own chain
        // (sage_grad_wt_kernel), so every ds2 row is bitwise the owner's
        const uint64_t r1 = uint64_t(g->r0) + g->rows;
        SGNN_TRY(sgnn::glue_sage_grad_wt(g->grad_full, g->wpack + g->off_w2, g->r0, g->hid, g->cls, nullptr, nullptr,
                                         g->ds2_full, s));
        SGNN_TRY(sgnn::glue_sage_grad_wt(g->grad_full + r1 * g->cls, g->wpack + g->off_w2, uint32_t(g->n - r1), g->hid,
                                         g->cls, nullptr, nullptr, g->ds2_full + r1 * g->hid, s));
    }
    DIST_MARK(g, M_SPMMB_0);
    if (g->rows) SGNN_TRY(sgnn::run_spmm(&g->bwd, g->ds2_full, g->hid, g->dh1, SGNN_REDUCE_SUM, g->plan_bwd, s));
    DIST_MARK(g, M_SPMMB_1);
    SGNN_TRY(sgnn::glue_sage_grad_wt(g->grad(), g->wpack + g->off_w2s, g->rows, g->hid, g->cls, g->dh1, h1r, g->z1, s));
    DIST_MARK(g, M_GEMM2_0);
    SGNN_TRY(mm_tn(g, g->ax, g->z1, g->gpack + g->off_w1, g->rows, 2 * g->in, g->hid, s));  // [g1; g1s] = ax^T dz1
    DIST_MARK(g, M_P2_E);
    return SGNN_OK;
}

// phase 3: sgd_step on every weight, epoch statistics
sgnn_status phase3(sgnn_dist_s* g, uint32_t e, float lr, cudaStream_t s) {
    DIST_MARK(g, M_P3_S);
    pack_sgd_kernel<<<ew_grid(g->pack_n), 256, 0, s>>>(g->wpack, g->gpack, g->pack_n, lr);
    epoch_record_kernel<<<1, 1, 0, s>>>(g->red, g->inv_n, g->stats + 2 * uint64_t(e));
    SGNN_LAUNCH_CHECK();
    DIST_MARK(g, M_END);
    return SGNN_OK;
}

#undef DIST_MARK

sgnn_status run_epochs(sgnn_dist_s* const* gs, int ng, uint32_t epochs, float lr, cudaStream_t s) {
    sgnn_dist_s* g0 = gs[0];
    for (int i = 0; i < ng; ++i) {
        if (gs[i]->epoch + epochs > gs[i]->max_epochs)
            return fail(SGNN_ERR_CONFIG, "dist: more epochs than the engine was sized for (call sgnn_dist_reset)");
        if (gs[i]->ev.empty()) {
            gs[i]->ev.resize(size_t(gs[i]->max_epochs) * M_COUNT);
            for (auto& ev : gs[i]->ev) SGNN_CUDA_TRY(cudaEventCreate(&ev));
        }
    }
    if (!g0->prepared) SGNN_TRY(prepare(gs, ng, s));
    auto each = [&](auto&& fn) -> sgnn_status {
        for (int i = 0; i < ng; ++i) SGNN_TRY(fn(gs[i]));
        return SGNN_OK;
    };
    for (uint32_t it = 0; it < epochs; ++it) {
        const uint32_t e = g0->epoch;
        SGNN_TRY(each([&](sgnn_dist_s* g) { return cudaEventRecord(g->mark(e, M_BEGIN), s) == cudaSuccess ? SGNN_OK : fail(SGNN_ERR_CUDA, "event"); }));
        if (g0->x_dirty && g0->P > 1)
            SGNN_TRY(allgather_rows(gs, ng, [](sgnn_dist_s* g) { return static_cast<void*>(g->x_full); }, g0->in, s));
        SGNN_TRY(each([&](sgnn_dist_s* g) {
            g->x_dirty = false;
            return cudaEventRecord(g->mark(e, M_X), s) == cudaSuccess ? SGNN_OK : fail(SGNN_ERR_CUDA, "event");
        }));
        SGNN_TRY(each([&](sgnn_dist_s* g) { return phase0(g, e, s); }));
        SGNN_TRY(allgather_rows(gs, ng, [](sgnn_dist_s* g) { return static_cast<void*>(g->h1_full); }, g0->hid, s));
        SGNN_TRY(each([&](sgnn_dist_s* g) { return cudaEventRecord(g->mark(e, M_EX1), s) == cudaSuccess ? SGNN_OK : fail(SGNN_ERR_CUDA, "event"); }));
        SGNN_TRY(each([&](sgnn_dist_s* g) { return phase1(g, e, s); }));
        SGNN_TRY(allgather_rows(gs, ng, [](sgnn_dist_s* g) { return static_cast<void*>(g->grad_full); }, g0->cls, s));
        SGNN_TRY(each([&](sgnn_dist_s* g) { return cudaEventRecord(g->mark(e, M_EX2), s) == cudaSuccess ? SGNN_OK : fail(SGNN_ERR_CUDA, "event"); }));
        SGNN_TRY(each([&](sgnn_dist_s* g) { return phase2(g, e, s); }));
        SGNN_TRY(allreduce_grads(gs, ng, s));
        SGNN_TRY(each([&](sgnn_dist_s* g) { return cudaEventRecord(g->mark(e, M_EX3), s) == cudaSuccess ? SGNN_OK : fail(SGNN_ERR_CUDA, "event"); }));
        SGNN_TRY(each([&](sgnn_dist_s* g) { return phase3(g, e, lr, s); }));
        for (int i = 0; i < ng; ++i) ++gs[i]->epoch;
    }
    return SGNN_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {
sgnn_status sgnn_dist_set_features(sgnn_dist g, const float* x_local, int borrow, sgnn_stream stream);

sgnn_status sgnn_comm_get_unique_id(void* id) {
    if (!id) return fail(SGNN_ERR_CONFIG, "comm_get_unique_id: null id");
    NcclApi& api = nccl();
    if (!api.loaded) return fail(SGNN_ERR_UNSUPPORTED, "NCCL unavailable: " + api.why);
    ncclUniqueId u;
    SGNN_TRY(nccl_ok(api.GetUniqueId(&u), "get unique id"));
    std::memcpy(id, &u, sizeof(u));
    return SGNN_OK;
}

sgnn_status sgnn_comm_init_rank(const void* id, int nranks, int rank, sgnn_comm* out) {
    if (!out || !id) return fail(SGNN_ERR_CONFIG, "comm_init_rank: null argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SGNN_ERR_CONFIG, "comm_init_rank: bad rank / nranks");
    auto* c = new sgnn_comm_s;
    c->kind = kCommNccl;
    c->nranks = nranks;
    c->rank = rank;
    if (nranks > 1) {
        NcclApi& api = nccl();
        if (!api.loaded) {
            delete c;
            return fail(SGNN_ERR_UNSUPPORTED, "NCCL unavailable: " + api.why);
        }
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        const sgnn_status st = nccl_ok(api.CommInitRank(&c->comm, nranks, u, rank), "comm init rank");
        if (st != SGNN_OK) {
            c->comm = nullptr;
            delete c;
            return st;
        }
    }
    *out = c;
    return SGNN_OK;
}

sgnn_status sgnn_comm_init_loopback(int nranks, sgnn_comm* out) {
    if (!out) return fail(SGNN_ERR_CONFIG, "comm_init_loopback: null out");
    *out = nullptr;
    if (nranks < 1 || nranks > 64) return fail(SGNN_ERR_CONFIG, "comm_init_loopback: 1..64 ranks");
    auto* c = new sgnn_comm_s;
    c->kind = kCommLoopback;
    c->nranks = nranks;
    c->members.assign(size_t(nranks), nullptr);
    *out = c;
    return SGNN_OK;
}

sgnn_status sgnn_comm_info(sgnn_comm c, int* nranks, int* rank, int* kind) {
    if (!c) return fail(SGNN_ERR_CONFIG, "comm_info: null comm");
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
    if (kind) *kind = c->kind;
    return SGNN_OK;
}

sgnn_status sgnn_comm_destroy(sgnn_comm c) {
    delete c;
    return SGNN_OK;
}

sgnn_status sgnn_dist_create(sgnn_comm comm, int rank, const uint32_t* bounds, const sgnn_csr* block,
                             const sgnn_csr* bwd_block, int model_kind, uint32_t in_features, uint32_t hidden,
                             uint32_t classes, const float* x_local, const uint32_t* labels_local,
                             const uint8_t* mask_local, uint32_t max_epochs, sgnn_dist* out, sgnn_stream stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!out) return fail(SGNN_ERR_CONFIG, "dist_create: null out");
    *out = nullptr;
    if (!bounds || !block) return fail(SGNN_ERR_CONFIG, "dist_create: null bounds / block");
    if (model_kind != kSageSum && model_kind != kSageMean)
        return fail(SGNN_ERR_UNSUPPORTED, "dist_create: the row-partitioned trainer runs SAGE-sum / SAGE-mean");
    if (in_features == 0 || hidden == 0 || classes == 0)
        return fail(SGNN_ERR_CONFIG, "init_model: in_features, hidden, and classes must be positive");
    if (hidden % 4 || hidden > 128 || classes > 16 || in_features % 4)
        return fail(SGNN_ERR_UNSUPPORTED, "dist_create: needs in % 4 == 0, hidden % 4 == 0, hidden <= 128, classes <= 16");
    const int P = comm ? comm->nranks : 1;
    if (comm && comm->kind == kCommNccl) rank = comm->rank;
    if (rank < 0 || rank >= P) return fail(SGNN_ERR_CONFIG, "dist_create: rank out of range");
    if (comm && comm->kind == kCommLoopback && comm->members[size_t(rank)])
        return fail(SGNN_ERR_CONFIG, "dist_create: loopback rank already has an engine");
    const uint32_t n = bounds[P];
    if (bounds[0] != 0) return fail(SGNN_ERR_CONFIG, "dist_create: bounds[0] must be 0");
    for (int q = 0; q < P; ++q)
        if (bounds[q + 1] < bounds[q]) return fail(SGNN_ERR_CONFIG, "dist_create: bounds must be non-decreasing");
    const uint32_t r0 = bounds[rank], rows = bounds[rank + 1] - r0;
    if (block->n_rows != rows || block->n_cols != n)
        return fail(SGNN_ERR_SHAPE, "dist_create: block is " + std::to_string(block->n_rows) + "x" +
                                        std::to_string(block->n_cols) + ", expected " + std::to_string(rows) + "x" +
                                        std::to_string(n) + " (rank rows x global columns)");
    SGNN_TRY(sgnn::check_csr(block, "dist_create"));
    if (bwd_block) {
        SGNN_TRY(sgnn::check_csr(bwd_block, "dist_create"));
        if (bwd_block->n_rows != rows || bwd_block->n_cols != n)
            return fail(SGNN_ERR_SHAPE, "dist_create: backward block must be rank rows x global columns");
    }
    if (rows && (!x_local || !labels_local || !mask_local))
        return fail(SGNN_ERR_CONFIG, "dist_create: null features/labels/mask");
    auto* g = new sgnn_dist_s;
    auto bail = [&](sgnn_status st) {
        delete g;
        return st;
    };
    g->comm = comm;
    g->P = P;
    g->rank = rank;
    g->bounds.assign(bounds, bounds + P + 1);
    g->n = n;
    g->r0 = r0;
    g->rows = rows;
    g->kind = model_kind;
    g->in = in_features;
    g->hid = hidden;
    g->cls = classes;
    g->max_epochs = max_epochs ? max_epochs : 1;
    g->fwd = *block;
    g->bwd_given = bwd_block != nullptr;
    g->bwd = bwd_block ? *bwd_block : *block;
    g->dense_tc = !std::getenv("SGNN_GNN_CUBLAS_DENSE");
    if (cublasCreate(&g->blas) != CUBLAS_STATUS_SUCCESS) return bail(fail(SGNN_ERR_CUDA, "cuBLAS create failed"));
    cublasSetMathMode(g->blas, CUBLAS_PEDANTIC_MATH);  // fp32, no TF32
    g->ws_bytes = size_t(32) << 20;
    sgnn_status st = SGNN_OK;
    void* wsp = nullptr;
    if (cudaMalloc(&wsp, g->ws_bytes) != cudaSuccess) return bail(fail(SGNN_ERR_NOMEM, "dist: workspace"));
    g->ws = wsp;
    g->owned.push_back(wsp);
    cublasSetWorkspace(g->blas, g->ws, g->ws_bytes);
    const uint64_t N = n, R = rows;
    auto al = [](uint64_t v) { return (v + 63) / 64 * 64; };
    g->off_w1 = 0;  // [W1; W1s] contiguous: the layer-1 product's B operand
    g->off_w1s = uint64_t(in_features) * hidden;
    g->off_w2 = al(2ull * in_features * hidden);
    g->off_w2s = g->off_w2 + al(uint64_t(hidden) * classes);
    g->pack_n = g->off_w2s + al(uint64_t(hidden) * classes);
    g->sm_blocks = sgnn::softmax_block_count(rows ? rows : 1);
    g->wg_blocks = std::min<uint32_t>(592, std::max<uint32_t>(1, rows));
    g->wg_rpb = (std::max<uint32_t>(1, rows) + g->wg_blocks - 1) / g->wg_blocks;
    g->wg_blocks = (std::max<uint32_t>(1, rows) + g->wg_rpb - 1) / g->wg_rpb;
    if ((P > 1 && (st = dalloc(g, &g->x_full, N * in_features)) != SGNN_OK) ||
        (st = dalloc(g, &g->h1_full, N * hidden)) != SGNN_OK || (st = dalloc(g, &g->ds2_full, N * hidden)) != SGNN_OK ||
        (st = dalloc(g, &g->ax, R * 2 * in_features)) != SGNN_OK || (st = dalloc(g, &g->a2, R * hidden)) != SGNN_OK ||
        (st = dalloc(g, &g->z1, R * hidden)) != SGNN_OK || (st = dalloc(g, &g->dh1, R * hidden)) != SGNN_OK ||
        (st = dalloc(g, &g->grad_full, N * classes)) != SGNN_OK ||
        (st = dalloc(g, &g->labels, R)) != SGNN_OK || (st = dalloc(g, &g->mask, R)) != SGNN_OK ||
        (st = dalloc(g, &g->deg, N)) != SGNN_OK || (st = dalloc(g, &g->wpack, g->pack_n)) != SGNN_OK ||
        (st = dalloc(g, &g->gpack, g->pack_n)) != SGNN_OK || (st = dalloc(g, &g->blk_loss, g->sm_blocks)) != SGNN_OK ||
        (st = dalloc(g, &g->blk_ok, g->sm_blocks)) != SGNN_OK ||
        (st = dalloc(g, &g->wg_part, uint64_t(g->wg_blocks) * 2 * hidden * 16)) != SGNN_OK ||
        (st = dalloc(g, &g->red, 2)) != SGNN_OK || (st = dalloc(g, &g->stats, 2ull * g->max_epochs)) != SGNN_OK)
        return bail(st);
    if (model_kind == kSageMean && (st = dalloc(g, &g->bwd_vals, g->bwd.nnz)) != SGNN_OK) return bail(st);
    if (cudaMemsetAsync(g->wpack, 0, sizeof(float) * g->pack_n, s) != cudaSuccess ||
        cudaMemsetAsync(g->gpack, 0, sizeof(float) * g->pack_n, s) != cudaSuccess)
        return bail(fail(SGNN_ERR_CUDA, "dist: memset"));
    if (rows) {
        if (sgnn_dist_set_features(g, x_local, 0, reinterpret_cast<sgnn_stream>(s)) != SGNN_OK ||
            cudaMemcpyAsync(g->labels, labels_local, sizeof(uint32_t) * R, cudaMemcpyDefault, s) != cudaSuccess ||
            cudaMemcpyAsync(g->mask, mask_local, R, cudaMemcpyDefault, s) != cudaSuccess)
            return bail(fail(SGNN_ERR_CUDA, "dist: input upload failed"));
        // local masked count and the label range check (softmax_xent, gnn.hpp:322-331)
        std::vector<uint8_t> hm(R);
        std::vector<uint32_t> hl(R);
        if (cudaMemcpyAsync(hm.data(), g->mask, R, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaMemcpyAsync(hl.data(), g->labels, sizeof(uint32_t) * R, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return bail(fail(SGNN_ERR_CUDA, "dist: label readback failed"));
        for (uint64_t i = 0; i < R; ++i) {
            if (!hm[i]) continue;
            ++g->n_masked_local;
            if (hl[i] >= classes)
                return bail(fail(SGNN_ERR_CONFIG, "softmax_xent: label " + std::to_string(hl[i]) + " out of range for " +
                                                      std::to_string(classes) + " classes"));
        }
        if ((st = sgnn::build_plan(&g->fwd, in_features, nullptr, true, &g->plan_in, s)) != SGNN_OK) return bail(st);
        if (hidden == in_features) {
            g->plan_hid = g->plan_in;
        } else if ((st = sgnn::build_plan(&g->fwd, hidden, nullptr, true, &g->plan_hid, s)) != SGNN_OK) {
            return bail(st);
        }
        sgnn_csr bplan = g->bwd;
        if ((st = sgnn::build_plan(&bplan, hidden, nullptr, true, &g->plan_bwd, s)) != SGNN_OK) return bail(st);
    }
    if (cudaStreamSynchronize(s) != cudaSuccess) return bail(fail(SGNN_ERR_CUDA, "dist: create failed"));
    if (comm && comm->kind == kCommLoopback) comm->members[size_t(rank)] = g;
    *out = g;
    return SGNN_OK;
}

sgnn_status sgnn_dist_set_weights(sgnn_dist g, const float* w1, const float* w2, const float* w1s, const float* w2s,
                                  sgnn_stream stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!g || !w1 || !w2 || !w1s || !w2s) return fail(SGNN_ERR_CONFIG, "dist_set_weights: missing weights");
    const uint64_t a = uint64_t(g->in) * g->hid, b = uint64_t(g->hid) * g->cls;
    if (cudaMemcpyAsync(g->wpack + g->off_w1, w1, sizeof(float) * a, cudaMemcpyDefault, s) != cudaSuccess ||
        cudaMemcpyAsync(g->wpack + g->off_w2, w2, sizeof(float) * b, cudaMemcpyDefault, s) != cudaSuccess ||
        cudaMemcpyAsync(g->wpack + g->off_w1s, w1s, sizeof(float) * a, cudaMemcpyDefault, s) != cudaSuccess ||
        cudaMemcpyAsync(g->wpack + g->off_w2s, w2s, sizeof(float) * b, cudaMemcpyDefault, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return fail(SGNN_ERR_CUDA, "dist: weight upload failed");
    return SGNN_OK;
}

sgnn_status sgnn_dist_get_weights(sgnn_dist g, float* w1, float* w2, float* w1s, float* w2s, sgnn_stream stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!g) return fail(SGNN_ERR_CONFIG, "dist_get_weights: null engine");
    const uint64_t a = uint64_t(g->in) * g->hid, b = uint64_t(g->hid) * g->cls;
    if ((w1 && cudaMemcpyAsync(w1, g->wpack + g->off_w1, sizeof(float) * a, cudaMemcpyDefault, s) != cudaSuccess) ||
        (w2 && cudaMemcpyAsync(w2, g->wpack + g->off_w2, sizeof(float) * b, cudaMemcpyDefault, s) != cudaSuccess) ||
        (w1s && cudaMemcpyAsync(w1s, g->wpack + g->off_w1s, sizeof(float) * a, cudaMemcpyDefault, s) != cudaSuccess) ||
        (w2s && cudaMemcpyAsync(w2s, g->wpack + g->off_w2s, sizeof(float) * b, cudaMemcpyDefault, s) != cudaSuccess) ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return fail(SGNN_ERR_CUDA, "dist: weight download failed");
    return SGNN_OK;
}

sgnn_status sgnn_dist_set_features(sgnn_dist g, const float* x_local, int borrow, sgnn_stream stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!g) return fail(SGNN_ERR_CONFIG, "dist_set_features: null engine");
    if (!x_local && g->rows) return fail(SGNN_ERR_CONFIG, "dist_set_features: null features");
    (void)borrow;  // the features are always copied: into the right half of [a1 | X_r] and, with P ranks,
                   // into the rank's rows of the gathered operand
    if (g->rows) {
        const size_t row = sizeof(float) * g->in;
        SGNN_CUDA_TRY(cudaMemcpy2DAsync(g->ax + g->in, 2 * row, x_local, row, row, g->rows, cudaMemcpyDefault, s));
        if (g->P > 1)
            SGNN_CUDA_TRY(cudaMemcpyAsync(g->x_full + uint64_t(g->r0) * g->in, x_local, row * g->rows,
                                          cudaMemcpyDefault, s));
    }
    g->x_dirty = true;
    return SGNN_OK;
}

sgnn_status sgnn_dist_epochs(sgnn_dist* engines, int n_engines, uint32_t epochs, float lr, sgnn_stream stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!engines || n_engines < 1) return fail(SGNN_ERR_CONFIG, "dist_epochs: no engines");
    if (epochs == 0) return fail(SGNN_ERR_CONFIG, "train: epochs must be >= 1");
    sgnn_dist_s* g0 = engines[0];
    if (!g0) return fail(SGNN_ERR_CONFIG, "dist_epochs: null engine");
    if (g0->P == 1 || (g0->comm && g0->comm->kind == kCommNccl)) {
        if (n_engines != 1) return fail(SGNN_ERR_CONFIG, "dist_epochs: an NCCL rank drives exactly its own engine");
    } else {
        if (n_engines != g0->P) return fail(SGNN_ERR_CONFIG, "dist_epochs: loopback needs all P engines in rank order");
        for (int i = 0; i < n_engines; ++i)
            if (!engines[i] || engines[i]->comm != g0->comm || engines[i]->rank != i || engines[i]->epoch != g0->epoch)
                return fail(SGNN_ERR_CONFIG, "dist_epochs: loopback engines must be ranks 0..P-1 of one comm, in step");
    }
    return run_epochs(engines, n_engines, epochs, lr, s);
}

sgnn_status sgnn_dist_stats(sgnn_dist g, uint32_t first, uint32_t count, double* loss, double* accuracy,
                            double* times, sgnn_stream stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!g) return fail(SGNN_ERR_CONFIG, "dist_stats: null engine");
    if (first + count > g->epoch) return fail(SGNN_ERR_CONFIG, "dist_stats: epochs not run yet");
    SGNN_CUDA_TRY(cudaStreamSynchronize(s));
    if (count == 0) return SGNN_OK;
    std::vector<double> hs(2ull * count);
    SGNN_CUDA_TRY(cudaMemcpy(hs.data(), g->stats + 2ull * first, sizeof(double) * hs.size(), cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < count; ++i) {
        if (loss) loss[i] = hs[2 * i];
        if (accuracy) accuracy[i] = hs[2 * i + 1];
        if (times) {
            const uint32_t e = first + i;
            auto el = [&](int a, int b) {
                float ms = 0.0f;
                cudaEventElapsedTime(&ms, g->mark(e, a), g->mark(e, b));
                return double(ms);
            };
            double* t = times + size_t(i) * SGNN_DIST_TIMES;
            t[0] = el(M_BEGIN, M_END);                                                    // epoch
            t[1] = el(M_SPMM1_0, M_SPMM1_1) + el(M_SPMM2_0, M_SPMM2_1) + el(M_SPMMB_0, M_SPMMB_1);  // 3 SpMMs
            t[2] = el(M_P0_S, M_P0_E) + el(M_P1_S, M_P1_E) + el(M_P2_S, M_P2_E) + el(M_P3_S, M_END);  // own compute
            t[3] = t[0] - t[2];  // exchanges + waiting for peers (loopback: + the other ranks' phases)
            t[4] = el(M_SPMM1_0, M_SPMM1_1);
            t[5] = el(M_SPMM2_0, M_SPMM2_1);
            t[6] = el(M_SPMMB_0, M_SPMMB_1);
            t[7] = el(M_SPMM1_1, M_GEMM1_1) + el(M_GEMM2_0, M_P2_E);  // the two dense products
        }
    }
    return SGNN_OK;
}

sgnn_status sgnn_dist_stats_copy(sgnn_dist g, uint32_t first, uint32_t count, double* dst, sgnn_stream stream) {
    if (!g || (!dst && count)) return fail(SGNN_ERR_CONFIG, "dist_stats_copy: null argument");
    if (first + count > g->epoch) return fail(SGNN_ERR_CONFIG, "dist_stats_copy: epochs not run yet");
    if (count)
        SGNN_CUDA_TRY(cudaMemcpyAsync(dst, g->stats + 2ull * first, sizeof(double) * 2 * count, cudaMemcpyDefault,
                                      reinterpret_cast<cudaStream_t>(stream)));
    return SGNN_OK;
}

sgnn_status sgnn_dist_reset(sgnn_dist g) {
    if (!g) return fail(SGNN_ERR_CONFIG, "dist_reset: null engine");
    g->epoch = 0;
    return SGNN_OK;
}

sgnn_status sgnn_dist_info(sgnn_dist g, uint32_t* row0, uint32_t* rows, uint64_t* nnz, uint64_t* n_masked,
                           float** x_local) {
    if (!g) return fail(SGNN_ERR_CONFIG, "dist_info: null engine");
    if (row0) *row0 = g->r0;
    if (rows) *rows = g->rows;
    if (nnz) *nnz = g->fwd.nnz;
    if (n_masked) *n_masked = g->n_masked;
    if (x_local) *x_local = g->ax + g->in;  // row stride 2 * in
    return SGNN_OK;
}

sgnn_status sgnn_dist_destroy(sgnn_dist g) {
    if (g && g->comm && g->comm->kind == kCommLoopback) g->comm->members[size_t(g->rank)] = nullptr;
    delete g;
    return SGNN_OK;
}

}  // extern "C"
