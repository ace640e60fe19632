// gnn.cu -- the native GNN training engine: train() of gnn.hpp:414-438 with
// forward (gnn.hpp:212-256), backward (:261-313), softmax_xent (:318-349),
// masked_accuracy (:353-370) and sgd_step (:374-386) on the device.  Sparse
// propagation runs on this library's SpMM through the TrainingCache
// (cache.cu); the dense products are cuBLAS SGEMMs (fp32, no TF32); the rest
// are small element-wise kernels below.  An epoch never synchronises with the
// host (loss / accuracy land in device memory), so it can be captured once
// and replayed as a CUDA graph.
#include <cublas_v2.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <vector>

#include "ops.cuh"
#include "plan.cuh"

namespace {

constexpr int kGcn = 0, kSageSum = 1, kSageMean = 2, kGin = 3;  // ModelKind order, gnn.hpp:17

// Element-wise passes over n floats: float4 body (every buffer here is a
// whole cudaMalloc allocation or a 16-byte aligned offset into one) plus a
// scalar tail; grid-stride over at most grid_for(n / 4) blocks.
template <class Op>
__device__ __forceinline__ void ew_loop(uint64_t n, Op op) {
    const uint64_t n4 = n / 4, stride = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t t0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (uint64_t i = t0; i < n4; i += stride) op.vec(i);
    for (uint64_t i = 4 * n4 + t0; i < n; i += stride) op.one(i);
}

// relu (dense.hpp): x > 0 ? x : 0
__device__ __forceinline__ float relu1(float x) { return x > 0.0f ? x : 0.0f; }
// relu_backward: grad where act > 0, else 0
__device__ __forceinline__ float relu_bwd1(float g, float act) { return act <= 0.0f ? 0.0f : g; }

__global__ void relu_kernel(const float* __restrict__ x, uint64_t n, float* __restrict__ y) {
    struct {
        const float* x; float* y;
        __device__ void vec(uint64_t i) const {
            const float4 a = reinterpret_cast<const float4*>(x)[i];
            reinterpret_cast<float4*>(y)[i] = make_float4(relu1(a.x), relu1(a.y), relu1(a.z), relu1(a.w));
        }
        __device__ void one(uint64_t i) const { y[i] = relu1(x[i]); }
    } op{x, y};
    ew_loop(n, op);
}

__global__ void relu_backward_kernel(const float* __restrict__ g, const float* __restrict__ act, uint64_t n,
                                     float* __restrict__ out) {
    struct {
        const float *g, *act; float* out;
        __device__ void vec(uint64_t i) const {
            const float4 a = reinterpret_cast<const float4*>(g)[i], h = reinterpret_cast<const float4*>(act)[i];
            reinterpret_cast<float4*>(out)[i] =
                make_float4(relu_bwd1(a.x, h.x), relu_bwd1(a.y, h.y), relu_bwd1(a.z, h.z), relu_bwd1(a.w, h.w));
        }
        __device__ void one(uint64_t i) const { out[i] = relu_bwd1(g[i], act[i]); }
    } op{g, act, out};
    ew_loop(n, op);
}

// y += x (add_inplace)
__global__ void add_kernel(float* __restrict__ y, const float* __restrict__ x, uint64_t n) {
    struct {
        float* y; const float* x;
        __device__ void vec(uint64_t i) const {
            float4 a = reinterpret_cast<float4*>(y)[i];
            const float4 b = reinterpret_cast<const float4*>(x)[i];
            a.x = __fadd_rn(a.x, b.x); a.y = __fadd_rn(a.y, b.y); a.z = __fadd_rn(a.z, b.z); a.w = __fadd_rn(a.w, b.w);
            reinterpret_cast<float4*>(y)[i] = a;
        }
        __device__ void one(uint64_t i) const { y[i] = __fadd_rn(y[i], x[i]); }
    } op{y, x};
    ew_loop(n, op);
}

// h = relu(a + b): SAGE's z1 = a1 W1 + X W1s followed by relu (gnn.hpp:238-239)
// in one pass; z1 itself is not needed later (relu_backward tests h1).
__global__ void add_relu_kernel(const float* __restrict__ a, const float* __restrict__ b, uint64_t n,
                                float* __restrict__ h) {
    struct {
        const float *a, *b; float* h;
        __device__ void vec(uint64_t i) const {
            const float4 u = reinterpret_cast<const float4*>(a)[i], v = reinterpret_cast<const float4*>(b)[i];
            reinterpret_cast<float4*>(h)[i] = make_float4(relu1(__fadd_rn(u.x, v.x)), relu1(__fadd_rn(u.y, v.y)),
                                                          relu1(__fadd_rn(u.z, v.z)), relu1(__fadd_rn(u.w, v.w)));
        }
        __device__ void one(uint64_t i) const { h[i] = relu1(__fadd_rn(a[i], b[i])); }
    } op{a, b, h};
    ew_loop(n, op);
}

// out = relu_backward(g + u, act): SAGE's dh1 = A^T ds2 + grad W2s^T then
// dz1 (gnn.hpp:290-292) in one pass.
__global__ void add_relu_backward_kernel(const float* __restrict__ g, const float* __restrict__ u,
                                         const float* __restrict__ act, uint64_t n, float* __restrict__ out) {
    struct {
        const float *g, *u, *act; float* out;
        __device__ void vec(uint64_t i) const {
            const float4 a = reinterpret_cast<const float4*>(g)[i], b = reinterpret_cast<const float4*>(u)[i];
            const float4 h = reinterpret_cast<const float4*>(act)[i];
            reinterpret_cast<float4*>(out)[i] =
                make_float4(relu_bwd1(__fadd_rn(a.x, b.x), h.x), relu_bwd1(__fadd_rn(a.y, b.y), h.y),
                            relu_bwd1(__fadd_rn(a.z, b.z), h.z), relu_bwd1(__fadd_rn(a.w, b.w), h.w));
        }
        __device__ void one(uint64_t i) const { out[i] = relu_bwd1(__fadd_rn(g[i], u[i]), act[i]); }
    } op{g, u, act, out};
    ew_loop(n, op);
}

// out = (1 + eps) * x + y  (scaled_add with the GIN scale, eps on the device)
__global__ void scaled_add_kernel(const float* __restrict__ eps, const float* __restrict__ x,
                                  const float* __restrict__ y, uint64_t n, float* __restrict__ out) {
    const float s = __fadd_rn(1.0f, *eps);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = __fadd_rn(__fmul_rn(s, x[i]), y[i]);
}

// w -= lr * g
__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g, uint64_t n, float lr) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        w[i] = __fsub_rn(w[i], __fmul_rn(lr, g[i]));
}

// softmax_xent + masked_accuracy (gnn.hpp:318-370).  A group of G lanes
// (G = the power of two >= classes, at most 32) owns a row; lane j holds
// class j (and j + G, ... when classes > 32).  Per row: the gradient row
// (zero outside the mask), and the row's loss (double) and correct flag
// folded into the group's running sums.  Block b covers the contiguous rows
// [b*rpb, (b+1)*rpb); its groups' sums are added in group order and written
// to blk_loss[b] / blk_ok[b] -- a fixed order for a given n, so the epoch's
// loss is deterministic (epoch_stats_kernel adds the block sums).
constexpr int kSoftmaxThreads = 256;
template <int G>
__global__ void __launch_bounds__(kSoftmaxThreads) softmax_xent_kernel(
    const float* __restrict__ logits, uint32_t n, uint32_t c, const uint32_t* __restrict__ labels,
    const uint8_t* __restrict__ mask, double inv_n, uint32_t rpb, float* __restrict__ grad,
    double* __restrict__ blk_loss, uint32_t* __restrict__ blk_ok) {
    constexpr int NG = kSoftmaxThreads / G;
    __shared__ double s_loss[NG];
    __shared__ uint32_t s_ok[NG];
    const uint32_t gl = threadIdx.x % G, grp = threadIdx.x / G;
    const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
    const uint32_t r0 = blockIdx.x * rpb, r1 = min(n, r0 + rpb);
    double lsum = 0.0;
    uint32_t oks = 0;
    for (uint32_t i = r0 + grp; i < r1; i += NG) {  // group-uniform trip count
        const float* row = logits + uint64_t(i) * c;
        float* grow = grad + uint64_t(i) * c;
        if (!mask[i]) {
            for (uint32_t j = gl; j < c; j += G) grow[j] = 0.0f;
            continue;
        }
        float mxf = -1.0f / 0.0f, bestv = -1.0f / 0.0f;
        uint32_t best = 0;
        for (uint32_t j = gl; j < c; j += G) {
            const float v = row[j];
            mxf = fmaxf(mxf, v);
            if (v > bestv) {  // ties: smallest class index
                bestv = v;
                best = j;
            }
        }
#pragma unroll
        for (int o = G / 2; o >= 1; o >>= 1) {
            mxf = fmaxf(mxf, __shfl_xor_sync(gmask, mxf, o, G));
            const float ov = __shfl_xor_sync(gmask, bestv, o, G);
            const uint32_t oj = __shfl_xor_sync(gmask, best, o, G);
            if (ov > bestv || (ov == bestv && oj < best)) {
                bestv = ov;
                best = oj;
            }
        }
        const double mx = double(mxf);  // max in double of the float logits
        double e0 = 0.0, den = 0.0;
        for (uint32_t j = gl; j < c; j += G) {
            const double e = exp(double(row[j]) - mx);
            if (j == gl) e0 = e;
            den += e;
        }
#pragma unroll
        for (int o = G / 2; o >= 1; o >>= 1) den += __shfl_xor_sync(gmask, den, o, G);
        const uint32_t lab = labels[i];
        for (uint32_t j = gl; j < c; j += G) {
            const double p = (j == gl ? e0 : exp(double(row[j]) - mx)) / den;
            grow[j] = float((p - (j == lab ? 1.0 : 0.0)) * inv_n);
        }
        if (gl == 0) {
            lsum += (mx + log(den)) - double(row[lab]);
            oks += best == lab ? 1u : 0u;
        }
    }
    if (gl == 0) {
        s_loss[grp] = lsum;
        s_ok[grp] = oks;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double l = 0.0;
        uint32_t k = 0;
        for (int q = 0; q < NG; ++q) {
            l += s_loss[q];
            k += s_ok[q];
        }
        blk_loss[blockIdx.x] = l;
        blk_ok[blockIdx.x] = k;
    }
}

// Sum of the per-block losses / correct counts in a fixed order (one
// block), and the epoch's stats written to stats[2 * (*epoch)]; epoch
// counter advanced.
__global__ void __launch_bounds__(1024) epoch_stats_kernel(const double* __restrict__ row_loss,
                                                           const uint32_t* __restrict__ row_ok, uint32_t n,
                                                           double inv_n, double* __restrict__ stats,
                                                           uint32_t* __restrict__ epoch, uint32_t max_epochs) {
    __shared__ double sl[1024];
    __shared__ unsigned long long sc[1024];
    double l = 0.0;
    unsigned long long cnt = 0;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        l += row_loss[i];
        cnt += row_ok[i];
    }
    sl[threadIdx.x] = l;
    sc[threadIdx.x] = cnt;
    __syncthreads();
    for (uint32_t s = blockDim.x / 2; s >= 1; s >>= 1) {
        if (threadIdx.x < s) {
            sl[threadIdx.x] += sl[threadIdx.x + s];
            sc[threadIdx.x] += sc[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const uint32_t e = *epoch;
        if (e < max_epochs) {
            stats[2 * e] = sl[0] * inv_n;
            stats[2 * e + 1] = double(sc[0]) * inv_n;
        }
        *epoch = e + 1;
    }
}

// Masked loss sum and correct count over the per-block sums, in block order
// (the ABI's softmax_xent; the engine's epoch_stats_kernel does the same
// and divides).
__global__ void softmax_finish_kernel(const double* __restrict__ blk_loss, const uint32_t* __restrict__ blk_ok,
                                      uint32_t nblk, double* __restrict__ loss_sum, uint32_t* __restrict__ correct) {
    if (threadIdx.x != 0) return;
    double l = 0.0;
    uint32_t k = 0;
    for (uint32_t b = 0; b < nblk; ++b) {
        l += blk_loss[b];
        k += blk_ok[b];
    }
    *loss_sum = l;
    *correct = k;
}

// ---- SAGE's classes-wide products (hidden h <= 128, h % 4 == 0, classes
// c <= CP): memory-bound passes of their own instead of cuBLAS calls that
// run far below HBM speed at this shape.  A warp owns a row; lane l holds
// hidden features 4l..4l+3 (lanes l >= h/4 idle in the loads).  Each
// product is rounded on its own and the two are added like the reference
// (matmul, matmul, add: gnn.hpp:241-244 and :285-292).

// grad[i, 0..CP) (zero past c); float4 loads when rows are 16-byte aligned
template <int CP>
__device__ __forceinline__ void load_grad_row(const float* __restrict__ grad, uint32_t i, uint32_t c, float (&g)[CP]) {
    if (c % 4 == 0) {
        const float4* r = reinterpret_cast<const float4*>(grad + uint64_t(i) * c);
#pragma unroll
        for (int j4 = 0; j4 < CP / 4; ++j4) {
            const float4 v = 4 * j4 < int(c) ? __ldg(r + j4) : make_float4(0.f, 0.f, 0.f, 0.f);
            g[4 * j4] = v.x; g[4 * j4 + 1] = v.y; g[4 * j4 + 2] = v.z; g[4 * j4 + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < CP; ++j) g[j] = j < int(c) ? __ldg(grad + uint64_t(i) * c + j) : 0.0f;
    }
}

// the same row from a shared-memory copy (c % 4 == 0)
template <int CP>
__device__ __forceinline__ void load_grad_row_smem(const float* grad, uint32_t i, uint32_t c, float (&g)[CP]) {
    const float4* r = reinterpret_cast<const float4*>(grad + uint64_t(i) * c);
#pragma unroll
    for (int j4 = 0; j4 < CP / 4; ++j4) {
        const float4 v = 4 * j4 < int(c) ? r[j4] : make_float4(0.f, 0.f, 0.f, 0.f);
        g[4 * j4] = v.x; g[4 * j4 + 1] = v.y; g[4 * j4 + 2] = v.z; g[4 * j4 + 3] = v.w;
    }
}

// W (row-major h x c) staged in shared memory for lane l's rows 4l..4l+3:
// float4 (q, j4) of lane l = W[4l + q][4 j4 .. 4 j4 + 3] at index
// (q * CP/4 + j4) * 32 + l, so a warp's LDS.128 hits consecutive addresses.
template <int CP>
__device__ __forceinline__ void stage_w(const float* __restrict__ w, uint32_t h, uint32_t c, float4* sw) {
    for (uint32_t t = threadIdx.x; t < 4 * (CP / 4) * 32; t += blockDim.x) {
        const uint32_t l = t % 32, qj = t / 32, q = qj / (CP / 4), j4 = qj % (CP / 4), k = 4 * l + q;
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (k < h && 4 * j4 + e < c) ? w[k * c + 4 * j4 + e] : 0.0f;
        sw[t] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

// logits[i, :] = [a2 | h1][i, :] . [W2; W2s]: one fp32 accumulation over the
// concatenated 2h inputs (the usual SAGE concat form of a2 W2 + h1 W2s).
// A warp takes RU rows at a time (their loads in flight together).
template <int CP>
__global__ void __launch_bounds__(256) sage_logits_kernel(const float* __restrict__ a2, const float* __restrict__ h1,
                                                          const float* __restrict__ w2, const float* __restrict__ w2s,
                                                          uint32_t n, uint32_t h, uint32_t c,
                                                          float* __restrict__ logits) {
    constexpr int RU = 4, J4 = CP / 4;
    __shared__ float4 sw[2][4 * J4 * 32];
    stage_w<CP>(w2, h, c, sw[0]);
    stage_w<CP>(w2s, h, c, sw[1]);
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    const bool act = lane < h / 4;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * RU; i0 < n; i0 += nw * RU) {
        float4 x[2][RU];
#pragma unroll
        for (int r = 0; r < RU; ++r) {
            const bool ok = act && i0 + r < n;
            x[0][r] = ok ? __ldg(reinterpret_cast<const float4*>(a2 + uint64_t(i0 + r) * h) + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
            x[1][r] = ok ? __ldg(reinterpret_cast<const float4*>(h1 + uint64_t(i0 + r) * h) + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float p[RU][CP];
#pragma unroll
        for (int r = 0; r < RU; ++r)
#pragma unroll
            for (int j = 0; j < CP; ++j) p[r][j] = 0.0f;
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int j4 = 0; j4 < J4; ++j4) {
                    const float4 wv = sw[m][(q * J4 + j4) * 32 + lane];
#pragma unroll
                    for (int r = 0; r < RU; ++r) {
                        const float xv = q == 0 ? x[m][r].x : q == 1 ? x[m][r].y : q == 2 ? x[m][r].z : x[m][r].w;
                        p[r][4 * j4 + 0] = __fmaf_rn(xv, wv.x, p[r][4 * j4 + 0]);
                        p[r][4 * j4 + 1] = __fmaf_rn(xv, wv.y, p[r][4 * j4 + 1]);
                        p[r][4 * j4 + 2] = __fmaf_rn(xv, wv.z, p[r][4 * j4 + 2]);
                        p[r][4 * j4 + 3] = __fmaf_rn(xv, wv.w, p[r][4 * j4 + 3]);
                    }
                }
        // transpose-reduce each row's CP partials over the warp: lane l ends
        // with class l / (32 / CP)
#pragma unroll
        for (int r = 0; r < RU; ++r) {
            int sh = 16;
#pragma unroll
            for (int half = CP / 2; half >= 1; half >>= 1, sh >>= 1) {
                const bool up = (lane & sh) != 0;
#pragma unroll
                for (int j = 0; j < half; ++j) {
                    const float send = up ? p[r][j] : p[r][half + j];
                    const float keep = up ? p[r][half + j] : p[r][j];
                    p[r][j] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, sh));
                }
            }
#pragma unroll
            for (; sh >= 1; sh >>= 1) p[r][0] = __fadd_rn(p[r][0], __shfl_xor_sync(0xffffffffu, p[r][0], sh));
        }
        constexpr uint32_t PER = 32 / CP;
        const uint32_t j = lane / PER;
        if (lane % PER == 0 && j < c) {
#pragma unroll
            for (int r = 0; r < RU; ++r)
                if (i0 + r < n) logits[uint64_t(i0 + r) * c + j] = p[r][0];
        }
    }
}

// Per-block partial weight gradients of the classes-wide layer:
// part[b][m][k][j] = sum over block b's rows i of (m ? h1 : a2)[i, k] grad[i, j]
// (g2 = a2^T grad, g2s = h1^T grad).  Warps 0-3 take a2, warps 4-7 h1 (warp
// wm of a product: rows r0 + 2 wm + 8 t, +1); the four warps of a product are
// combined in warp order.  The a2 / h1 rows arrive in shared memory by bulk
// copies (cp.async.bulk, one elected thread, mbarrier completion) of
// kWgChunk-row chunks, kWgStages in flight, so the streaming read is not
// limited by the registers of loads in flight (126 registers capped this
// kernel at 16 warps/SM with 2 rows in flight each: 2.7 TB/s).  Bitwise the
// register-load version (same rows per warp, same FFMA2 order).
constexpr int kWgChunk = 32, kWgStages = 3;
template <int CP>
__global__ void __launch_bounds__(256) sage_wgrad_kernel(const float* __restrict__ a2, const float* __restrict__ h1,
                                                         const float* __restrict__ grad, uint32_t n, uint32_t h,
                                                         uint32_t c, uint32_t rpb, float* __restrict__ part) {
    constexpr int RU = 2;
    extern __shared__ __align__(128) float wsm[];  // [stages][2][kWgChunk][h] | [stages][kWgChunk][c]; then red
    __shared__ __align__(8) uint64_t full[kWgStages];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, m = w >> 2, wm = w & 3;
    const bool act = lane < h / 4;
    const uint32_t r0 = min(n, blockIdx.x * rpb), r1 = min(n, r0 + rpb);
    const uint32_t nch = (r1 - r0 + kWgChunk - 1) / kWgChunk;
    const size_t stage_floats = size_t(2) * kWgChunk * h;
    const bool sgrad = c % 4 == 0;  // grad rows staged too (16-byte multiples)
    float* gsm = wsm + kWgStages * stage_floats;  // [stages][kWgChunk][c]
    auto smem_u32 = [](const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); };
    if (threadIdx.x == 0) {
        for (int q = 0; q < kWgStages; ++q)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + q)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](uint32_t q) {  // chunk q -> stage q % kWgStages (thread 0)
        const uint32_t s = q % kWgStages, row = r0 + q * kWgChunk;
        const uint32_t rows = min(uint32_t(kWgChunk), r1 - row);
        const uint32_t bytes = rows * h * 4;
        float* dst = wsm + s * stage_floats;
        const uint32_t bar = smem_u32(full + s);
        const uint32_t gbytes = sgrad ? rows * c * 4 : 0u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * bytes + gbytes)
                     : "memory");
        if (sgrad)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(gsm + size_t(s) * kWgChunk * c)),
                         "l"(grad + uint64_t(row) * c), "r"(gbytes), "r"(bar)
                         : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(dst)),
                     "l"(a2 + uint64_t(row) * h), "r"(bytes), "r"(bar)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(dst + kWgChunk * h)),
                     "l"(h1 + uint64_t(row) * h), "r"(bytes), "r"(bar)
                     : "memory");
    };
    if (threadIdx.x == 0)
        for (uint32_t q = 0; q < min(nch, uint32_t(kWgStages)); ++q) issue(q);
    float acc[4][CP];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int j = 0; j < CP; ++j) acc[q][j] = 0.0f;
    for (uint32_t q = 0; q < nch; ++q) {
        const uint32_t s = q % kWgStages, row = r0 + q * kWgChunk;
        const uint32_t rows = min(uint32_t(kWgChunk), r1 - row);
        asm volatile(
            "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
                smem_u32(full + s)),
            "r"((q / kWgStages) & 1)
            : "memory");
        const float* src = wsm + s * stage_floats + size_t(m) * kWgChunk * h;
        if (act) {
            for (uint32_t lr = wm * RU; lr < rows; lr += 4 * RU) {
                float4 x[RU];
                float g[RU][CP];
#pragma unroll
                for (int r = 0; r < RU; ++r) {
                    const bool ok = lr + r < rows;
                    x[r] = ok ? reinterpret_cast<const float4*>(src + size_t(lr + r) * h)[lane]
                              : make_float4(0.f, 0.f, 0.f, 0.f);
                    if (sgrad) load_grad_row_smem<CP>(gsm + size_t(s) * kWgChunk * c, ok ? lr + r : lr, c, g[r]);
                    else load_grad_row<CP>(grad, ok ? row + lr + r : row + lr, c, g[r]);
                }
#pragma unroll
                for (int r = 0; r < RU; ++r) {
                    const float xs[4] = {x[r].x, x[r].y, x[r].z, x[r].w};  // zero past the block's rows
                    // packed FFMA2 over class pairs: each half an ordinary fma
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq)
#pragma unroll
                        for (int j = 0; j < CP; j += 2)
                            sgnn::dev::fma2_rn(acc[qq][j], acc[qq][j + 1], xs[qq], g[r][j], g[r][j + 1]);
                }
            }
        }
        __syncthreads();  // stage s consumed by every warp
        if (threadIdx.x == 0 && q + kWgStages < nch) issue(q + kWgStages);
    }
    float(*red)[128 * CP] = reinterpret_cast<float(*)[128 * CP]>(wsm);  // stages are free now
    for (uint32_t step = 0; step < 4; ++step) {
        if (wm == step && act) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int j = 0; j < CP; ++j) {
                    float* r = &red[m][(4 * lane + q) * CP + j];
                    *r = step == 0 ? acc[q][j] : __fadd_rn(*r, acc[q][j]);
                }
        }
        __syncthreads();
    }
    float* out = part + uint64_t(blockIdx.x) * 2 * h * CP;
    for (uint32_t t = threadIdx.x; t < 2 * h * CP; t += blockDim.x) out[t] = red[t / (h * CP)][t % (h * CP)];
}

size_t sage_wgrad_smem(uint32_t h, uint32_t c, int cp) {
    return std::max(size_t(kWgStages) * kWgChunk * (2 * h + (c % 4 == 0 ? c : 0)), size_t(2) * 128 * cp) *
           sizeof(float);
}

// g2 / g2s (h x c row-major) = sum of the block partials in block order
template <int CP>
__global__ void sage_wgrad_finish_kernel(const float* __restrict__ part, uint32_t nblk, uint32_t h, uint32_t c,
                                         float* __restrict__ g2, float* __restrict__ g2s) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * h * CP) return;
    const uint32_t m = t / (h * CP), kj = t % (h * CP), k = kj / CP, j = kj % CP;
    if (j >= c) return;
    float v = 0.0f;
    for (uint32_t b = 0; b < nblk; ++b) v = __fadd_rn(v, part[uint64_t(b) * 2 * h * CP + t]);
    (m ? g2s : g2)[k * c + j] = v;
}

// out[i, k] = grad[i, :] . W[k, :]  (grad W^T, W row-major h x c); with
// U != null: out[i, k] = relu_backward(U[i, k] + grad[i, :] . W[k, :], act[i, k])
// -- SAGE's ds2 = grad W2^T, and dz1 from dh1 = A^T ds2 + grad W2s^T
// (the second product never reaches memory).
template <int CP>
__global__ void __launch_bounds__(256) sage_grad_wt_kernel(const float* __restrict__ grad, const float* __restrict__ w,
                                                           uint32_t n, uint32_t h, uint32_t c,
                                                           const float* __restrict__ u, const float* __restrict__ act,
                                                           float* __restrict__ out) {
    constexpr int RU = 4, J4 = CP / 4;
    __shared__ float4 sw[4 * J4 * 32];
    stage_w<CP>(w, h, c, sw);
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    if (lane >= h / 4) return;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * RU; i0 < n; i0 += nw * RU) {
        float g[RU][CP];
        float4 uv[RU], hv[RU];
#pragma unroll
        for (int r = 0; r < RU; ++r) {
            const uint32_t i = i0 + r < n ? i0 + r : i0;
            load_grad_row<CP>(grad, i, c, g[r]);
            if (u) {
                uv[r] = __ldg(reinterpret_cast<const float4*>(u + uint64_t(i) * h) + lane);
                hv[r] = __ldg(reinterpret_cast<const float4*>(act + uint64_t(i) * h) + lane);
            }
        }
        float d[RU][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int j4 = 0; j4 < J4; ++j4) {
                const float4 wv = sw[(q * J4 + j4) * 32 + lane];
#pragma unroll
                for (int r = 0; r < RU; ++r) {
                    float t = j4 == 0 ? __fmul_rn(g[r][0], wv.x) : __fmaf_rn(g[r][4 * j4], wv.x, d[r][q]);
                    t = __fmaf_rn(g[r][4 * j4 + 1], wv.y, t);
                    t = __fmaf_rn(g[r][4 * j4 + 2], wv.z, t);
                    d[r][q] = __fmaf_rn(g[r][4 * j4 + 3], wv.w, t);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < RU; ++r) {
            if (i0 + r >= n) break;
            float4* o = reinterpret_cast<float4*>(out + uint64_t(i0 + r) * h) + lane;
            if (u) {
                *o = make_float4(relu_bwd1(__fadd_rn(uv[r].x, d[r][0]), hv[r].x),
                                 relu_bwd1(__fadd_rn(uv[r].y, d[r][1]), hv[r].y),
                                 relu_bwd1(__fadd_rn(uv[r].z, d[r][2]), hv[r].z),
                                 relu_bwd1(__fadd_rn(uv[r].w, d[r][3]), hv[r].w));
            } else {
                *o = make_float4(d[r][0], d[r][1], d[r][2], d[r][3]);
            }
        }
    }
}

// SAGE's layer-2 head in one pass over a2 and h1 (gnn.hpp:241-244,
// :318-370, :283-287).  A warp takes R = 32 / CP rows at a time: lane l
// accumulates the logit partials of all R x CP (row, class) pairs over its
// features (sage_logits_kernel's FMA chains), and one 32-value
// transpose-reduce (lane offsets 16, 8, 4, 2, 1 -- the same lane tree as
// sage_logits_kernel) leaves lane l with the logit of row l / CP, class
// l % CP.  Each CP-lane group then runs softmax_xent + masked_accuracy for
// its row exactly as softmax_xent_kernel<G = CP> (same double arithmetic,
// butterfly and tie rule), writes the gradient row and forms ds2 = grad W2^T
// with sage_grad_wt_kernel's FMA chain (lane gl: feature blocks gl + CP b).
// grad and ds2 are bitwise the three-kernel sequence's; a2 / h1 are read
// once and the logits never reach memory.  Block b owns rows [b*rpb,
// (b+1)*rpb); loss / correct sums go to blk_loss[b] / blk_ok[b] in a fixed
// order.
template <int CP, int H>
__global__ void __launch_bounds__(256) sage_head_kernel(
    const float* __restrict__ a2, const float* __restrict__ h1, const float* __restrict__ w2,
    const float* __restrict__ w2s, uint32_t n, uint32_t h, uint32_t c, const uint32_t* __restrict__ labels,
    const uint8_t* __restrict__ mask, double inv_n, uint32_t rpb, float* __restrict__ grad,
    float* __restrict__ ds2, double* __restrict__ blk_loss, uint32_t* __restrict__ blk_ok) {
    // H sub-steps of R rows share every weight fragment read from shared
    // memory (the pass is bound by those reads: 4 J4 + 4 J4 NB 16-byte loads
    // per lane and step), each row's arithmetic unchanged
    constexpr int R = 32 / CP, J4 = CP / 4, NB = 32 / CP;  // rows per warp sub-step; feature blocks per lane
    constexpr unsigned FULL = 0xffffffffu;
    __shared__ float4 sw[2][4 * J4 * 32];
    __shared__ double s_loss[8];
    __shared__ uint32_t s_ok[8];
    stage_w<CP>(w2, h, c, sw[0]);
    stage_w<CP>(w2s, h, c, sw[1]);
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool act = lane < h / 4;
    const uint32_t gl = lane % CP, grp = lane / CP;  // class / row-of-sub-step after the reduce
    const uint32_t r0 = blockIdx.x * rpb, r1 = min(n, r0 + rpb);
    double lsum = 0.0;
    uint32_t oks = 0;
    // the per-row log(den) is batched: a group's lane (sub % CP) keeps the
    // row's (mx, den, label logit), and every CP sub-steps all lanes take
    // their log at once (one log sequence per CP rows instead of one per row)
    uint32_t sub = 0;
    double p_mx = 0.0, p_den = 1.0;
    float p_vlab = 0.0f;
    bool p_has = false;
    auto flush = [&]() {
        if (p_has) lsum += (p_mx + log(p_den)) - double(p_vlab);
        p_has = false;
    };
    for (uint32_t i0 = r0 + wid * (R * H); i0 < r1; i0 += 8 * R * H) {
        float v[H];
        {
            float4 x[2][R * H];
#pragma unroll
            for (int r = 0; r < R * H; ++r) {
                const bool ok = act && i0 + r < r1;
                x[0][r] = ok ? __ldg(reinterpret_cast<const float4*>(a2 + uint64_t(i0 + r) * h) + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
                x[1][r] = ok ? __ldg(reinterpret_cast<const float4*>(h1 + uint64_t(i0 + r) * h) + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            float p[H][32];  // p[hh][r * CP + j]
#pragma unroll
            for (int hh = 0; hh < H; ++hh)
#pragma unroll
                for (int t = 0; t < 32; ++t) p[hh][t] = 0.0f;
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int j4 = 0; j4 < J4; ++j4) {
                        const float4 wv = sw[m][(q * J4 + j4) * 32 + lane];
#pragma unroll
                        for (int hh = 0; hh < H; ++hh)
#pragma unroll
                            for (int r = 0; r < R; ++r) {
                                const float4 xr = x[m][hh * R + r];
                                const float xv = q == 0 ? xr.x : q == 1 ? xr.y : q == 2 ? xr.z : xr.w;
                                float* pr = p[hh] + r * CP + 4 * j4;
                                // packed FFMA2 over class pairs (each half an ordinary fma)
                                sgnn::dev::fma2_rn(pr[0], pr[1], xv, wv.x, wv.y);
                                sgnn::dev::fma2_rn(pr[2], pr[3], xv, wv.z, wv.w);
                            }
                    }
            // 32-value transpose-reduce per sub-step: lane l ends with index l
#pragma unroll
            for (int hh = 0; hh < H; ++hh) {
#pragma unroll
                for (int sh = 16; sh >= 1; sh >>= 1) {
                    const bool up = (lane & sh) != 0;
#pragma unroll
                    for (int t = 0; t < sh; ++t) {
                        const float send = up ? p[hh][t] : p[hh][sh + t];
                        const float keep = up ? p[hh][sh + t] : p[hh][t];
                        p[hh][t] = __fadd_rn(keep, __shfl_xor_sync(FULL, send, sh));
                    }
                }
                v[hh] = p[hh][0];
            }
        }
        const unsigned gmask = CP == 32 ? FULL : (((1u << CP) - 1u) << (lane & ~(CP - 1)));
        const bool cl = gl < c;
        float g[H];
#pragma unroll
        for (int hh = 0; hh < H; ++hh, ++sub) {
            const uint32_t i = i0 + hh * R + grp;
            const bool row_ok = i < r1;
            g[hh] = 0.0f;
            if (row_ok && mask[i]) {  // group-uniform
                float mxf = -1.0f / 0.0f, bestv = -1.0f / 0.0f;
                uint32_t best = 0;
                if (cl) {
                    mxf = fmaxf(mxf, v[hh]);
                    if (v[hh] > bestv) {
                        bestv = v[hh];
                        best = gl;
                    }
                }
#pragma unroll
                for (int o = CP / 2; o >= 1; o >>= 1) {
                    mxf = fmaxf(mxf, __shfl_xor_sync(gmask, mxf, o, CP));
                    const float ov = __shfl_xor_sync(gmask, bestv, o, CP);
                    const uint32_t oj = __shfl_xor_sync(gmask, best, o, CP);
                    if (ov > bestv || (ov == bestv && oj < best)) {
                        bestv = ov;
                        best = oj;
                    }
                }
                const double mx = double(mxf);
                const double e = cl ? exp(double(v[hh]) - mx) : 0.0;
                double den = e;
#pragma unroll
                for (int o = CP / 2; o >= 1; o >>= 1) den += __shfl_xor_sync(gmask, den, o, CP);
                const uint32_t lab = labels[i];
                const float vlab = __shfl_sync(gmask, v[hh], int(lab), CP);
                if (cl) g[hh] = float((e / den - (gl == lab ? 1.0 : 0.0)) * inv_n);
                if (gl == sub % CP) {
                    p_mx = mx;
                    p_den = den;
                    p_vlab = vlab;
                    p_has = true;
                }
                if (gl == 0) oks += best == lab ? 1u : 0u;
            }
            if (sub % CP == CP - 1) flush();
            if (row_ok && cl) grad[uint64_t(i) * c + gl] = g[hh];
        }
        // ds2[i, k] = sum_j grad[i, j] W2[k, j] (sage_grad_wt_kernel's chain)
        float gj[H][CP];
#pragma unroll
        for (int hh = 0; hh < H; ++hh)
#pragma unroll
            for (int j = 0; j < CP; ++j) gj[hh][j] = __shfl_sync(FULL, g[hh], j, CP);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const uint32_t fb = gl + CP * b;  // feature block: features 4 fb .. 4 fb + 3
            if (fb >= h / 4) break;
            // features (4 fb + q, 4 fb + q + 1) as packed pairs: each half
            // is sage_grad_wt_kernel's chain (mul, then fmas in class order)
            float d[H][4];
#pragma unroll
            for (int q = 0; q < 4; q += 2) {
#pragma unroll
                for (int j4 = 0; j4 < J4; ++j4) {
                    const float4 wa = sw[0][(q * J4 + j4) * 32 + fb];
                    const float4 wb = sw[0][((q + 1) * J4 + j4) * 32 + fb];
#pragma unroll
                    for (int hh = 0; hh < H; ++hh) {
                        if (j4 == 0) {
                            d[hh][q] = __fmul_rn(gj[hh][0], wa.x);
                            d[hh][q + 1] = __fmul_rn(gj[hh][0], wb.x);
                        } else {
                            sgnn::dev::fma2s_rn(d[hh][q], d[hh][q + 1], gj[hh][4 * j4], wa.x, wb.x);
                        }
                        sgnn::dev::fma2s_rn(d[hh][q], d[hh][q + 1], gj[hh][4 * j4 + 1], wa.y, wb.y);
                        sgnn::dev::fma2s_rn(d[hh][q], d[hh][q + 1], gj[hh][4 * j4 + 2], wa.z, wb.z);
                        sgnn::dev::fma2s_rn(d[hh][q], d[hh][q + 1], gj[hh][4 * j4 + 3], wa.w, wb.w);
                    }
                }
            }
#pragma unroll
            for (int hh = 0; hh < H; ++hh) {
                const uint32_t i = i0 + hh * R + grp;
                if (i < r1)
                    reinterpret_cast<float4*>(ds2 + uint64_t(i) * h)[fb] = make_float4(d[hh][0], d[hh][1], d[hh][2], d[hh][3]);
            }
        }
    }
    flush();
    // per warp: the lanes' loss partials by a fixed butterfly, the groups'
    // correct counts (lane gl == 0 of each group)
    double wl = lsum;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) wl += __shfl_xor_sync(FULL, wl, o);
    uint32_t wk = 0;
#pragma unroll
    for (int q = 0; q < R; ++q) wk += __shfl_sync(FULL, oks, q * CP);
    if (lane == 0) {
        s_loss[wid] = wl;
        s_ok[wid] = wk;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double l = 0.0;
        uint32_t k = 0;
        for (int q = 0; q < 8; ++q) {
            l += s_loss[q];
            k += s_ok[q];
        }
        blk_loss[blockIdx.x] = l;
        blk_ok[blockIdx.x] = k;
    }
}

// GIN: deps += sum(a .* b) in double (dot_all), fixed order (one block)
__global__ void __launch_bounds__(1024) dot_all_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                       uint64_t n, double* __restrict__ acc) {
    __shared__ double s[1024];
    double v = 0.0;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) v += double(a[i]) * double(b[i]);
    s[threadIdx.x] = v;
    __syncthreads();
    for (uint32_t k = blockDim.x / 2; k >= 1; k >>= 1) {
        if (threadIdx.x < k) s[threadIdx.x] += s[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) *acc += s[0];
}

// GIN: eps -= lr * float(deps); deps reset
__global__ void eps_step_kernel(float* eps, double* deps, float lr) {
    *eps = __fsub_rn(*eps, __fmul_rn(lr, float(*deps)));
    *deps = 0.0;
}

unsigned grid_for(uint64_t n) {
    const uint64_t b = (n + 255) / 256;
    return unsigned(b < 4096 ? (b ? b : 1) : 4096);
}

// softmax_xent launch shape for n rows: rows per block and blocks (a fixed
// function of n, so the loss reduction order is too)
int head_substeps() {
    static const int h = [] {
        const char* e = std::getenv("SGNN_HEAD_H");
        const int v = e ? std::atoi(e) : 2;
        return (v == 1 || v == 4) ? v : 2;
    }();
    return h;
}

void softmax_shape(uint32_t n, uint32_t* rpb, uint32_t* blocks) {
    const uint32_t want = 2048;  // blocks (~14 per SM)
    uint32_t r = (n + want - 1) / want;
    r = r < 1 ? 1 : r;
    *rpb = r;
    *blocks = (n + r - 1) / r;
    if (*blocks == 0) *blocks = 1;
}

}  // namespace

struct sgnn_gnn_s {
    int kind = kGcn;
    uint32_t n = 0, in = 0, hid = 0, cls = 0;
    sgnn_cache_s* cache = nullptr;
    sgnn_csr a_hat{};
    cublasHandle_t blas = nullptr;
    void* blas_ws = nullptr;
    size_t blas_ws_bytes = 0;
    bool dense_tc = true;  // tall products on the tensor cores (mm / mm_tn)
    std::vector<void*> owned;
    // inputs
    float* x = nullptr;
    uint32_t* labels = nullptr;
    uint8_t* mask = nullptr;
    uint32_t n_masked = 0;
    // parameters and their gradients
    float *w1 = nullptr, *w2 = nullptr, *w1s = nullptr, *w2s = nullptr, *eps = nullptr;
    float *g1 = nullptr, *g2 = nullptr, *g1s = nullptr, *g2s = nullptr;
    double* deps = nullptr;
    // activations / scratch
    float *a1 = nullptr, *h1 = nullptr, *a2 = nullptr, *z1 = nullptr, *t1 = nullptr, *logits = nullptr,
          *t2 = nullptr, *grad = nullptr, *d_h = nullptr, *d_h2 = nullptr, *d_c = nullptr;
    double* row_loss = nullptr;
    uint32_t* row_ok = nullptr;
    // SAGE classes-wide products in the library's own passes (sage_*_kernel)
    bool skinny = false;
    uint32_t wg_rpb = 0, wg_blocks = 0;
    float* wg_part = nullptr;  // [wg_blocks][2][hid][16]
    double* stats = nullptr;  // [2 * max_epochs]
    uint32_t* epoch = nullptr;
    uint32_t max_epochs = 0;
    // forward plans on a_hat, per K
    std::vector<std::pair<uint32_t, sgnn_plan_s*>> plans;
    cudaGraphExec_t graph = nullptr;
    float graph_lr = 0.0f;
    bool use_cache = true;

    ~sgnn_gnn_s() {
        if (graph) cudaGraphExecDestroy(graph);
        for (auto& p : plans) sgnn::destroy_plan(p.second);
        if (cache) sgnn::cache_destroy(cache);
        if (blas) cublasDestroy(blas);
        for (void* p : owned) cudaFree(p);
    }
};

namespace sgnn {
namespace {

template <class T>
sgnn_status dalloc(sgnn_gnn_s* g, T** p, uint64_t count) {
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

// Tall products (all rows of the graph) run on the tensor cores in FP32
// emulation (dense_common.cuh: 3 bf16 terms per operand, fp32 accumulation,
// more accurate than SGEMM); the small ones, and any shape the CUTLASS
// kernels refuse, on cuBLAS SGEMM.
bool tall_ok(const sgnn_gnn_s* g, int m, int k, int n, std::initializer_list<const void*> ptrs) {
    if (!g->dense_tc || m < 4096 || k < 32 || n < 32 || k % 4 || n % 4) return false;
    for (const void* p : ptrs)
        if (reinterpret_cast<uintptr_t>(p) % 16) return false;
    return true;
}

// Row-major products through column-major cuBLAS (C^T = B^T A^T etc.).
// matmul (dense.hpp): C[m,n] = A[m,k] B[k,n]
sgnn_status mm(sgnn_gnn_s* g, const float* A, const float* B, float* Cm, int m, int k, int n, cudaStream_t s) {
    if (tall_ok(g, m, k, n, {A, B, Cm}) &&
        dense_mm_nn(m, n, k, A, B, Cm, 0.0f, g->blas_ws, g->blas_ws_bytes, s) == 0)
        return SGNN_OK;
    const float one = 1.0f, zero = 0.0f;
    return blas_ok(cublasSgemm(g->blas, CUBLAS_OP_N, CUBLAS_OP_N, n, m, k, &one, B, n, A, k, &zero, Cm, n), "mm");
}
// matmul_tn: C[k,n] = A[m,k]^T B[m,n]
sgnn_status mm_tn(sgnn_gnn_s* g, const float* A, const float* B, float* Cm, int m, int k, int n, cudaStream_t s) {
    if (tall_ok(g, m, k, n, {A, B, Cm})) {
        const int splits = std::max(1, std::min(148, m / 8192));  // one split per SM at cfg5 sizes
        if (dense_mm_tn(m, n, k, A, B, Cm, splits, g->blas_ws, g->blas_ws_bytes, s) == 0) return SGNN_OK;
    }
    const float one = 1.0f, zero = 0.0f;
    return blas_ok(cublasSgemm(g->blas, CUBLAS_OP_N, CUBLAS_OP_T, n, k, m, &one, B, n, A, k, &zero, Cm, n), "mm_tn");
}
// matmul_nt: C[m,n] = A[m,k] B[n,k]^T
sgnn_status mm_nt(sgnn_gnn_s* g, const float* A, const float* B, float* Cm, int m, int k, int n) {
    const float one = 1.0f, zero = 0.0f;
    return blas_ok(cublasSgemm(g->blas, CUBLAS_OP_T, CUBLAS_OP_N, n, m, k, &one, B, k, A, k, &zero, Cm, n), "mm_nt");
}

sgnn_status fwd_spmm(sgnn_gnn_s* g, const float* x, uint32_t k, float* out, int reduce, cudaStream_t s) {
    sgnn_plan_s* plan = nullptr;
    for (auto& p : g->plans)
        if (p.first == k) plan = p.second;
    if (!plan) return fail(SGNN_ERR_INTERNAL, "gnn: no forward plan for K=" + std::to_string(k));
    return run_spmm(&g->a_hat, x, k, out, reduce, plan, s);
}

#define LAUNCH_EW(kernel, n, ...)                                              \
    do {                                                                       \
        kernel<<<grid_for(n), 256, 0, s>>>(__VA_ARGS__);                       \
        SGNN_LAUNCH_CHECK();                                                   \
    } while (0)
// SAGE classes-wide kernels, instantiated for 4, 8 or 16 padded classes
#define SAGE_CP(kernel, cls, grid, block, args)                                \
    do {                                                                       \
        if ((cls) <= 4) kernel<4><<<(grid), (block), 0, s>>> args;            \
        else if ((cls) <= 8) kernel<8><<<(grid), (block), 0, s>>> args;       \
        else kernel<16><<<(grid), (block), 0, s>>> args;                      \
        SGNN_LAUNCH_CHECK();                                                   \
    } while (0)
// the fused head: H sub-steps per warp step (SGNN_HEAD_H = 1 / 2 / 4: A/B switch)
#define SAGE_HEAD_H(CPV, hsel, grid, args)                                                      \
    do {                                                                                        \
        if ((hsel) == 1) sage_head_kernel<CPV, 1><<<(grid), 256, 0, s>>> args;                  \
        else if ((hsel) == 4) sage_head_kernel<CPV, 4><<<(grid), 256, 0, s>>> args;             \
        else sage_head_kernel<CPV, 2><<<(grid), 256, 0, s>>> args;                              \
    } while (0)
#define SAGE_HEAD(cls, grid, args)                                             \
    do {                                                                       \
        const int hsel_ = head_substeps();                                     \
        if ((cls) <= 4) SAGE_HEAD_H(4, hsel_, grid, args);                     \
        else if ((cls) <= 8) SAGE_HEAD_H(8, hsel_, grid, args);                \
        else SAGE_HEAD_H(16, hsel_, grid, args);                               \
        SGNN_LAUNCH_CHECK();                                                   \
    } while (0)
// float4 element-wise kernels (ew_loop): a quarter of the threads
#define LAUNCH_EW4(kernel, n, ...)                                             \
    do {                                                                       \
        kernel<<<grid_for(((n) + 3) / 4), 256, 0, s>>>(__VA_ARGS__);           \
        SGNN_LAUNCH_CHECK();                                                   \
    } while (0)

// One epoch (gnn.hpp:427-435): forward, softmax_xent, accuracy, backward, sgd.
sgnn_status epoch(sgnn_gnn_s* g, float lr, cudaStream_t s) {
    const uint64_t nh = uint64_t(g->n) * g->hid, nc = uint64_t(g->n) * g->cls, ni = uint64_t(g->n) * g->in;
    const int n = int(g->n), in = int(g->in), hid = int(g->hid), cls = int(g->cls);
    const int red = g->kind == kSageMean ? SGNN_REDUCE_MEAN : SGNN_REDUCE_SUM;
    // ---- forward (gnn.hpp:212-256)
    if (g->kind == kGcn) {
        SGNN_TRY(mm(g, g->x, g->w1, g->z1, n, in, hid, s));                 // z1 = X W1
        SGNN_TRY(fwd_spmm(g, g->z1, g->hid, g->t1, SGNN_REDUCE_SUM, s));  // A_hat z1
        LAUNCH_EW4(relu_kernel, nh, g->t1, nh, g->h1);                    // h1
        SGNN_TRY(mm(g, g->h1, g->w2, g->t2, n, hid, cls, s));               // z2 = h1 W2
        SGNN_TRY(fwd_spmm(g, g->t2, g->cls, g->logits, SGNN_REDUCE_SUM, s));
    } else if (g->kind == kSageSum || g->kind == kSageMean) {
        SGNN_TRY(fwd_spmm(g, g->x, g->in, g->a1, red, s));                // a1 = A X
        SGNN_TRY(mm(g, g->a1, g->w1, g->z1, n, in, hid, s));
        SGNN_TRY(mm(g, g->x, g->w1s, g->t1, n, in, hid, s));
        LAUNCH_EW4(add_relu_kernel, nh, g->z1, g->t1, nh, g->h1);          // h1 = relu(a1 W1 + X W1s)
        SGNN_TRY(fwd_spmm(g, g->h1, g->hid, g->a2, red, s));               // a2 = A h1
        if (g->skinny) {
            // logits + softmax_xent + accuracy + ds2 = grad W2^T in one pass
            // (sage_head_kernel); the loss partials feed epoch_stats below
            uint32_t rpb = 1, nblk = 1;
            softmax_shape(g->n, &rpb, &nblk);
            SAGE_HEAD(g->cls, nblk,
                    (g->a2, g->h1, g->w2, g->w2s, g->n, g->hid, g->cls, g->labels, g->mask,
                     1.0 / double(g->n_masked), rpb, g->grad, g->d_h, g->row_loss, g->row_ok));
        } else {
            SGNN_TRY(mm(g, g->a2, g->w2, g->logits, n, hid, cls, s));
            SGNN_TRY(mm(g, g->h1, g->w2s, g->t2, n, hid, cls, s));
            LAUNCH_EW4(add_kernel, nc, g->logits, g->t2, nc);
        }
    } else {  // GIN
        SGNN_TRY(fwd_spmm(g, g->x, g->in, g->t1, SGNN_REDUCE_SUM, s));
        LAUNCH_EW(scaled_add_kernel, ni, g->eps, g->x, g->t1, ni, g->a1);  // a1 = (1+eps) X + A X
        SGNN_TRY(mm(g, g->a1, g->w1, g->z1, n, in, hid, s));
        LAUNCH_EW4(relu_kernel, nh, g->z1, nh, g->h1);
        SGNN_TRY(fwd_spmm(g, g->h1, g->hid, g->z1, SGNN_REDUCE_SUM, s));
        LAUNCH_EW(scaled_add_kernel, nh, g->eps, g->h1, g->z1, nh, g->a2);
        SGNN_TRY(mm(g, g->a2, g->w2, g->logits, n, hid, cls, s));
    }
    // ---- softmax_xent + masked_accuracy (gnn.hpp:318-370)
    const double inv_n = 1.0 / double(g->n_masked);
    uint32_t rpb = 1, nblk = 1;
    softmax_shape(g->n, &rpb, &nblk);
    if (g->skinny) {
        // (done by sage_head_kernel in the forward)
    } else if (g->cls <= 4)
        softmax_xent_kernel<4><<<nblk, kSoftmaxThreads, 0, s>>>(g->logits, g->n, g->cls, g->labels, g->mask, inv_n,
                                                                rpb, g->grad, g->row_loss, g->row_ok);
    else if (g->cls <= 8)
        softmax_xent_kernel<8><<<nblk, kSoftmaxThreads, 0, s>>>(g->logits, g->n, g->cls, g->labels, g->mask, inv_n,
                                                                rpb, g->grad, g->row_loss, g->row_ok);
    else if (g->cls <= 16)
        softmax_xent_kernel<16><<<nblk, kSoftmaxThreads, 0, s>>>(g->logits, g->n, g->cls, g->labels, g->mask, inv_n,
                                                                 rpb, g->grad, g->row_loss, g->row_ok);
    else
        softmax_xent_kernel<32><<<nblk, kSoftmaxThreads, 0, s>>>(g->logits, g->n, g->cls, g->labels, g->mask, inv_n,
                                                                 rpb, g->grad, g->row_loss, g->row_ok);
    SGNN_LAUNCH_CHECK();
    epoch_stats_kernel<<<1, 1024, 0, s>>>(g->row_loss, g->row_ok, nblk, inv_n, g->stats, g->epoch, g->max_epochs);
    SGNN_LAUNCH_CHECK();
    // ---- backward (gnn.hpp:261-313)
    if (g->kind == kGcn) {
        sgnn_csr at;  // fetched once, applied twice (gnn.hpp:274-279)
        SGNN_TRY(cache_sum_operand(g->cache, &at, s));
        SGNN_TRY(cache_spmm_with_operand(g->cache, &at, g->grad, g->cls, g->d_c, s));                 // dz2
        SGNN_TRY(mm_tn(g, g->h1, g->d_c, g->g2, n, hid, cls, s));                                        // W2 grad
        SGNN_TRY(mm_nt(g, g->d_c, g->w2, g->d_h, n, cls, hid));                                       // dh1
        LAUNCH_EW4(relu_backward_kernel, nh, g->d_h, g->h1, nh, g->d_h2);                            // dp1
        SGNN_TRY(cache_spmm_with_operand(g->cache, &at, g->d_h2, g->hid, g->d_h, s));                 // dz1
        SGNN_TRY(mm_tn(g, g->x, g->d_h, g->g1, n, in, hid, s));
    } else if (g->kind == kSageSum || g->kind == kSageMean) {
        if (g->skinny) {
            SGNN_TRY(sage_wgrad_launch(g->a2, g->h1, g->grad, g->n, g->hid, g->cls, g->wg_rpb, g->wg_blocks, g->wg_part,
                                       g->g2, g->g2s, s));
            // ds2 = grad W2^T is already in d_h (sage_head_kernel)
            SGNN_TRY(cache_spmm_backward(g->cache, g->d_h, g->n, g->hid, g->d_h2, red, s));          // dh1 (A^T part)
            // dz1 = relu_backward(dh1 + grad W2s^T, h1) into z1 (free after the forward)
            SAGE_CP(sage_grad_wt_kernel, g->cls, grid_for(uint64_t(g->n) * 32), 256,
                    (g->grad, g->w2s, g->n, g->hid, g->cls, g->d_h2, g->h1, g->z1));
        } else {
            SGNN_TRY(mm_tn(g, g->a2, g->grad, g->g2, n, hid, cls, s));
            SGNN_TRY(mm_tn(g, g->h1, g->grad, g->g2s, n, hid, cls, s));
            SGNN_TRY(mm_nt(g, g->grad, g->w2, g->d_h, n, cls, hid));                                  // ds2
            SGNN_TRY(cache_spmm_backward(g->cache, g->d_h, g->n, g->hid, g->d_h2, red, s));          // dh1
            SGNN_TRY(mm_nt(g, g->grad, g->w2s, g->d_h, n, cls, hid));
            // dz1 into z1 (free after the forward's add_relu)
            LAUNCH_EW4(add_relu_backward_kernel, nh, g->d_h2, g->d_h, g->h1, nh, g->z1);
        }
        SGNN_TRY(mm_tn(g, g->a1, g->z1, g->g1, n, in, hid, s));
        SGNN_TRY(mm_tn(g, g->x, g->z1, g->g1s, n, in, hid, s));
    } else {  // GIN
        SGNN_TRY(mm_tn(g, g->a2, g->grad, g->g2, n, hid, cls, s));
        SGNN_TRY(mm_nt(g, g->grad, g->w2, g->d_h, n, cls, hid));                                      // dm2
        dot_all_kernel<<<1, 1024, 0, s>>>(g->d_h, g->h1, nh, g->deps);
        SGNN_LAUNCH_CHECK();
        SGNN_TRY(cache_spmm_backward(g->cache, g->d_h, g->n, g->hid, g->d_h2, SGNN_REDUCE_SUM, s));
        LAUNCH_EW(scaled_add_kernel, nh, g->eps, g->d_h, g->d_h2, nh, g->z1);                        // dh1
        LAUNCH_EW4(relu_backward_kernel, nh, g->z1, g->h1, nh, g->d_h2);                             // dz1
        SGNN_TRY(mm_tn(g, g->a1, g->d_h2, g->g1, n, in, hid, s));
        SGNN_TRY(mm_nt(g, g->d_h2, g->w1, g->t1, n, hid, in));                                        // dm1
        dot_all_kernel<<<1, 1024, 0, s>>>(g->t1, g->x, ni, g->deps);
        SGNN_LAUNCH_CHECK();
    }
    // ---- sgd_step (gnn.hpp:374-386)
    LAUNCH_EW(sgd_kernel, uint64_t(in) * hid, g->w1, g->g1, uint64_t(in) * hid, lr);
    LAUNCH_EW(sgd_kernel, uint64_t(hid) * cls, g->w2, g->g2, uint64_t(hid) * cls, lr);
    if (g->kind == kSageSum || g->kind == kSageMean) {
        LAUNCH_EW(sgd_kernel, uint64_t(in) * hid, g->w1s, g->g1s, uint64_t(in) * hid, lr);
        LAUNCH_EW(sgd_kernel, uint64_t(hid) * cls, g->w2s, g->g2s, uint64_t(hid) * cls, lr);
    }
    if (g->kind == kGin) {
        eps_step_kernel<<<1, 1, 0, s>>>(g->eps, g->deps, lr);
        SGNN_LAUNCH_CHECK();
    }
    return SGNN_OK;
}

}  // namespace

sgnn_status gnn_create(const sgnn_csr* a, int kind, uint32_t in, uint32_t hidden, uint32_t classes,
                       const float* x, const uint32_t* labels, const uint8_t* mask, int use_cache,
                       int add_self_loops, uint32_t max_epochs, sgnn_gnn_s** out, cudaStream_t s) {
    *out = nullptr;
    if (kind < kGcn || kind > kGin) return fail(SGNN_ERR_CONFIG, "gnn: unknown model kind");
    if (in == 0 || hidden == 0 || classes == 0)
        return fail(SGNN_ERR_CONFIG, "init_model: in_features, hidden, and classes must be positive");
    if (a->n_rows != a->n_cols)
        return fail(SGNN_ERR_SHAPE, "build_cache: adjacency is " + std::to_string(a->n_rows) + "x" +
                                        std::to_string(a->n_cols) + ", expected square");
    auto* g = new sgnn_gnn_s;
    g->kind = kind;
    g->n = a->n_rows;
    g->in = in;
    g->hid = hidden;
    g->cls = classes;
    g->max_epochs = max_epochs ? max_epochs : 1;
    g->use_cache = use_cache != 0;
    auto bail = [&](sgnn_status st) {
        delete g;
        return st;
    };
    sgnn_status st = cache_create_model(a, kind, use_cache, add_self_loops, &g->cache, s);
    if (st != SGNN_OK) return bail(st);
    if ((st = cache_a_hat(g->cache, &g->a_hat)) != SGNN_OK) return bail(st);
    if (cublasCreate(&g->blas) != CUBLAS_STATUS_SUCCESS) return bail(fail(SGNN_ERR_CUDA, "cuBLAS create failed"));
    // fp32 products (no TF32); explicit workspace so an epoch can be graph-captured
    cublasSetMathMode(g->blas, CUBLAS_PEDANTIC_MATH);
    const size_t ws = size_t(32) << 20;
    if (cudaMalloc(&g->blas_ws, ws) != cudaSuccess) return bail(fail(SGNN_ERR_NOMEM, "gnn: cuBLAS workspace"));
    g->owned.push_back(g->blas_ws);
    cublasSetWorkspace(g->blas, g->blas_ws, ws);
    g->blas_ws_bytes = ws;  // shared with the CUTLASS GEMMs (same stream, never concurrent)
    g->dense_tc = !std::getenv("SGNN_GNN_CUBLAS_DENSE");  // A/B switch
    cublasSetStream(g->blas, s);
    const uint64_t n = g->n;
    const uint64_t wide = std::max<uint64_t>(hidden, in);
    if ((st = dalloc(g, &g->x, n * in)) != SGNN_OK || (st = dalloc(g, &g->labels, n)) != SGNN_OK ||
        (st = dalloc(g, &g->mask, n)) != SGNN_OK || (st = dalloc(g, &g->w1, uint64_t(in) * hidden)) != SGNN_OK ||
        (st = dalloc(g, &g->w2, uint64_t(hidden) * classes)) != SGNN_OK ||
        (st = dalloc(g, &g->w1s, uint64_t(in) * hidden)) != SGNN_OK ||
        (st = dalloc(g, &g->w2s, uint64_t(hidden) * classes)) != SGNN_OK || (st = dalloc(g, &g->eps, 1)) != SGNN_OK ||
        (st = dalloc(g, &g->g1, uint64_t(in) * hidden)) != SGNN_OK ||
        (st = dalloc(g, &g->g2, uint64_t(hidden) * classes)) != SGNN_OK ||
        (st = dalloc(g, &g->g1s, uint64_t(in) * hidden)) != SGNN_OK ||
        (st = dalloc(g, &g->g2s, uint64_t(hidden) * classes)) != SGNN_OK || (st = dalloc(g, &g->deps, 1)) != SGNN_OK ||
        (st = dalloc(g, &g->a1, n * in)) != SGNN_OK || (st = dalloc(g, &g->h1, n * hidden)) != SGNN_OK ||
        (st = dalloc(g, &g->a2, n * hidden)) != SGNN_OK || (st = dalloc(g, &g->z1, n * wide)) != SGNN_OK ||
        (st = dalloc(g, &g->t1, n * wide)) != SGNN_OK || (st = dalloc(g, &g->logits, n * classes)) != SGNN_OK ||
        (st = dalloc(g, &g->t2, n * classes)) != SGNN_OK || (st = dalloc(g, &g->grad, n * classes)) != SGNN_OK ||
        (st = dalloc(g, &g->d_h, n * wide)) != SGNN_OK || (st = dalloc(g, &g->d_h2, n * wide)) != SGNN_OK ||
        (st = dalloc(g, &g->d_c, n * classes)) != SGNN_OK || (st = dalloc(g, &g->row_loss, n)) != SGNN_OK ||
        (st = dalloc(g, &g->row_ok, n)) != SGNN_OK || (st = dalloc(g, &g->stats, 2ull * g->max_epochs)) != SGNN_OK ||
        (st = dalloc(g, &g->epoch, 1)) != SGNN_OK)
        return bail(st);
    g->skinny = (kind == kSageSum || kind == kSageMean) && hidden % 4 == 0 && hidden <= 128 && classes <= 16 &&
                !std::getenv("SGNN_GNN_CUBLAS_SKINNY");  // A/B switch
    if (g->skinny) {
        g->wg_blocks = std::min<uint32_t>(592, std::max<uint32_t>(1, g->n));  // 4 per SM
        g->wg_rpb = (g->n + g->wg_blocks - 1) / g->wg_blocks;
        g->wg_blocks = (g->n + g->wg_rpb - 1) / g->wg_rpb;
        if ((st = dalloc(g, &g->wg_part, uint64_t(g->wg_blocks) * 2 * hidden * 16)) != SGNN_OK) return bail(st);
    }
    if (cudaMemcpyAsync(g->x, x, sizeof(float) * n * in, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(g->labels, labels, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(g->mask, mask, n, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
        cudaMemsetAsync(g->eps, 0, sizeof(float), s) != cudaSuccess ||
        cudaMemsetAsync(g->deps, 0, sizeof(double), s) != cudaSuccess ||
        cudaMemsetAsync(g->epoch, 0, sizeof(uint32_t), s) != cudaSuccess)
        return bail(fail(SGNN_ERR_CUDA, "gnn: input upload failed"));
    // n_masked and the label range check (softmax_xent, gnn.hpp:322-331)
    std::vector<uint8_t> hm(n);
    std::vector<uint32_t> hl(n);
    if (cudaMemcpyAsync(hm.data(), mask, n, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(hl.data(), labels, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return bail(fail(SGNN_ERR_CUDA, "gnn: label readback failed"));
    for (uint64_t i = 0; i < n; ++i) {
        if (!hm[i]) continue;
        ++g->n_masked;
        if (hl[i] >= classes)
            return bail(fail(SGNN_ERR_CONFIG, "softmax_xent: label " + std::to_string(hl[i]) + " out of range for " +
                                                  std::to_string(classes) + " classes"));
    }
    if (g->n_masked == 0) return bail(fail(SGNN_ERR_CONFIG, "softmax_xent: mask selects no rows"));
    // forward plans for the widths this model propagates
    std::vector<uint32_t> ks;
    if (kind == kGcn) ks = {hidden, classes};
    else ks = {in, hidden};
    for (uint32_t k : ks) {
        bool have = false;
        for (auto& p : g->plans) have |= p.first == k;
        if (have) continue;
        sgnn_plan_s* p = nullptr;
        if ((st = build_plan(&g->a_hat, k, nullptr, k % 4 == 0, &p, s)) != SGNN_OK) return bail(st);
        g->plans.push_back({k, p});
    }
    *out = g;
    return SGNN_OK;
}

sgnn_status gnn_set_weights(sgnn_gnn_s* g, const float* w1, const float* w2, const float* w1s, const float* w2s,
                            float eps, cudaStream_t s) {
    const uint64_t a = uint64_t(g->in) * g->hid, b = uint64_t(g->hid) * g->cls;
    const bool self = g->kind == kSageSum || g->kind == kSageMean;
    if (!w1 || !w2 || (self && (!w1s || !w2s))) return fail(SGNN_ERR_CONFIG, "gnn: missing weights");
    if (cudaMemcpyAsync(g->w1, w1, sizeof(float) * a, cudaMemcpyDefault, s) != cudaSuccess ||
        cudaMemcpyAsync(g->w2, w2, sizeof(float) * b, cudaMemcpyDefault, s) != cudaSuccess ||
        (self && (cudaMemcpyAsync(g->w1s, w1s, sizeof(float) * a, cudaMemcpyDefault, s) != cudaSuccess ||
                  cudaMemcpyAsync(g->w2s, w2s, sizeof(float) * b, cudaMemcpyDefault, s) != cudaSuccess)) ||
        cudaMemcpyAsync(g->eps, &eps, sizeof(float), cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return fail(SGNN_ERR_CUDA, "gnn: weight upload failed");
    return SGNN_OK;
}

sgnn_status gnn_get_weights(sgnn_gnn_s* g, float* w1, float* w2, float* w1s, float* w2s, float* eps,
                            cudaStream_t s) {
    const uint64_t a = uint64_t(g->in) * g->hid, b = uint64_t(g->hid) * g->cls;
    const bool self = g->kind == kSageSum || g->kind == kSageMean;
    if ((w1 && cudaMemcpyAsync(w1, g->w1, sizeof(float) * a, cudaMemcpyDefault, s) != cudaSuccess) ||
        (w2 && cudaMemcpyAsync(w2, g->w2, sizeof(float) * b, cudaMemcpyDefault, s) != cudaSuccess) ||
        (self && w1s && cudaMemcpyAsync(w1s, g->w1s, sizeof(float) * a, cudaMemcpyDefault, s) != cudaSuccess) ||
        (self && w2s && cudaMemcpyAsync(w2s, g->w2s, sizeof(float) * b, cudaMemcpyDefault, s) != cudaSuccess) ||
        (eps && cudaMemcpyAsync(eps, g->eps, sizeof(float), cudaMemcpyDeviceToHost, s) != cudaSuccess) ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return fail(SGNN_ERR_CUDA, "gnn: weight download failed");
    return SGNN_OK;
}

// train (gnn.hpp:414-438): epochs of forward / xent / backward / sgd; stats
// (loss, accuracy) per epoch and per-epoch device time (CUDA events).
// cuda_graph: epoch 1 runs eagerly, epochs 2.. replay its capture.
sgnn_status gnn_train(sgnn_gnn_s* g, uint32_t epochs, float lr, int cuda_graph, double* loss, double* acc,
                      double* seconds, cudaStream_t s) {
    if (epochs == 0) return fail(SGNN_ERR_CONFIG, "train: epochs must be >= 1");
    if (epochs > g->max_epochs) return fail(SGNN_ERR_CONFIG, "train: more epochs than the engine was sized for");
    // A graph is captured on a stream of our own (capturing the legacy
    // default stream is not allowed); it is ordered after the caller's
    // stream and the caller's stream after it.
    cudaStream_t user = s;
    cudaStream_t own = nullptr;
    if (cuda_graph && g->use_cache) {
        cudaEvent_t ready;
        SGNN_CUDA_TRY(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
        SGNN_CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        SGNN_CUDA_TRY(cudaEventRecord(ready, user));
        SGNN_CUDA_TRY(cudaStreamWaitEvent(own, ready, 0));
        cudaEventDestroy(ready);
        s = own;
    }
    SGNN_CUDA_TRY(cudaMemsetAsync(g->epoch, 0, sizeof(uint32_t), s));
    cublasSetStream(g->blas, s);
    std::vector<cudaEvent_t> ev(epochs + 1);
    for (auto& e : ev) SGNN_CUDA_TRY(cudaEventCreate(&e));
    sgnn_status st = SGNN_OK;
    SGNN_CUDA_TRY(cudaEventRecord(ev[0], s));
    for (uint32_t e = 0; e < epochs && st == SGNN_OK; ++e) {
        // replays need every operand resident: with use_cache off the
        // backward operand is rebuilt (allocated) per fetch, so run eagerly
        const bool replay = cuda_graph && g->use_cache && e > 0;
        if (replay && (!g->graph || g->graph_lr != lr)) {
            if (g->graph) {
                cudaGraphExecDestroy(g->graph);
                g->graph = nullptr;
            }
            cudaGraph_t cg = nullptr;
            if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
                st = fail(SGNN_ERR_CUDA, "gnn: graph capture failed to start");
                break;
            }
            const sgnn_status cs = epoch(g, lr, s);
            const cudaError_t ce = cudaStreamEndCapture(s, &cg);
            if (cs != SGNN_OK || ce != cudaSuccess) {
                if (cg) cudaGraphDestroy(cg);
                st = cs != SGNN_OK ? cs : fail(SGNN_ERR_CUDA, "gnn: graph capture failed");
                break;
            }
            const cudaError_t ie = cudaGraphInstantiate(&g->graph, cg, 0);
            cudaGraphDestroy(cg);
            if (ie != cudaSuccess) {
                st = fail(SGNN_ERR_CUDA, "gnn: graph instantiate failed");
                break;
            }
            g->graph_lr = lr;
        }
        if (replay) {
            if (cudaGraphLaunch(g->graph, s) != cudaSuccess) st = fail(SGNN_ERR_CUDA, "gnn: graph launch failed");
        } else {
            st = epoch(g, lr, s);
        }
        if (st == SGNN_OK && cudaEventRecord(ev[e + 1], s) != cudaSuccess) st = fail(SGNN_ERR_CUDA, "gnn: event");
    }
    if (st == SGNN_OK && cudaStreamSynchronize(s) != cudaSuccess) st = fail(SGNN_ERR_CUDA, "gnn: epoch failed");
    if (st == SGNN_OK) {
        std::vector<double> hs(2ull * epochs);
        if (cudaMemcpy(hs.data(), g->stats, sizeof(double) * hs.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
            st = fail(SGNN_ERR_CUDA, "gnn: stats readback failed");
        for (uint32_t e = 0; e < epochs && st == SGNN_OK; ++e) {
            if (loss) loss[e] = hs[2 * e];
            if (acc) acc[e] = hs[2 * e + 1];
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, ev[e], ev[e + 1]);
            if (seconds) seconds[e] = double(ms) * 1e-3;
        }
    }
    for (auto& e : ev) cudaEventDestroy(e);
    if (own) {
        cudaStreamSynchronize(own);
        cudaStreamDestroy(own);
        cublasSetStream(g->blas, user);
    }
    return st;
}

sgnn_status gnn_counters(sgnn_gnn_s* g, uint64_t* tb, uint64_t* nb, uint64_t* hits, int* sym) {
    return cache_counters(g->cache, tb, nb, hits, sym);
}

void gnn_destroy(sgnn_gnn_s* g) { delete g; }

// ------------------------------------------------------------ SAGE glue (ABI)
namespace {
bool sage_shape_ok(uint32_t h, uint32_t c) { return h > 0 && h % 4 == 0 && h <= 128 && c > 0 && c <= 16; }
sgnn_status sage_shape(uint32_t h, uint32_t c, const char* what) {
    if (!sage_shape_ok(h, c))
        return fail(SGNN_ERR_SHAPE, std::string(what) + ": needs hidden % 4 == 0, hidden <= 128, 1 <= classes <= 16 (got " +
                                        std::to_string(h) + ", " + std::to_string(c) + ")");
    return SGNN_OK;
}
}  // namespace

sgnn_status glue_relu(const float* x, uint64_t n, float* y, cudaStream_t s) {
    if (n == 0) return SGNN_OK;
    LAUNCH_EW4(relu_kernel, n, x, n, y);
    return SGNN_OK;
}

sgnn_status glue_add_relu(const float* a, const float* b, uint64_t n, float* h, cudaStream_t s) {
    if (n == 0) return SGNN_OK;
    LAUNCH_EW4(add_relu_kernel, n, a, b, n, h);
    return SGNN_OK;
}

sgnn_status glue_sage_logits(const float* a2, const float* h1, const float* w2, const float* w2s, uint32_t n,
                             uint32_t h, uint32_t c, float* logits, cudaStream_t s) {
    SGNN_TRY(sage_shape(h, c, "sage_logits"));
    if (n == 0) return SGNN_OK;
    SAGE_CP(sage_logits_kernel, c, grid_for(uint64_t(n) * 32), 256, (a2, h1, w2, w2s, n, h, c, logits));
    return SGNN_OK;
}

sgnn_status glue_softmax_xent(const float* logits, uint32_t n, uint32_t c, const uint32_t* labels,
                              const uint8_t* mask, double inv_count, float* grad, double* loss_sum,
                              uint32_t* correct, cudaStream_t s) {
    if (c == 0) return fail(SGNN_ERR_SHAPE, "softmax_xent: classes must be positive");
    uint32_t rpb = 1, nblk = 1;
    softmax_shape(n, &rpb, &nblk);
    void* blk = nullptr;
    SGNN_TRY(scratch_alloc(&blk, size_t(nblk) * (sizeof(double) + sizeof(uint32_t)), s));
    double* bl = static_cast<double*>(blk);
    uint32_t* bo = reinterpret_cast<uint32_t*>(bl + nblk);
    if (n) {
        if (c <= 4)
            softmax_xent_kernel<4><<<nblk, kSoftmaxThreads, 0, s>>>(logits, n, c, labels, mask, inv_count, rpb, grad, bl, bo);
        else if (c <= 8)
            softmax_xent_kernel<8><<<nblk, kSoftmaxThreads, 0, s>>>(logits, n, c, labels, mask, inv_count, rpb, grad, bl, bo);
        else if (c <= 16)
            softmax_xent_kernel<16><<<nblk, kSoftmaxThreads, 0, s>>>(logits, n, c, labels, mask, inv_count, rpb, grad, bl, bo);
        else
            softmax_xent_kernel<32><<<nblk, kSoftmaxThreads, 0, s>>>(logits, n, c, labels, mask, inv_count, rpb, grad, bl, bo);
    }
    softmax_finish_kernel<<<1, 32, 0, s>>>(bl, bo, n ? nblk : 0, loss_sum, correct);
    const cudaError_t e = cudaGetLastError();
    scratch_free(blk, s);
    if (e != cudaSuccess) return fail(SGNN_ERR_CUDA, std::string("softmax_xent: ") + cudaGetErrorString(e));
    return SGNN_OK;
}

uint32_t softmax_block_count(uint32_t n) {
    uint32_t rpb = 1, nblk = 1;
    softmax_shape(n, &rpb, &nblk);
    return nblk;
}

sgnn_status softmax_xent_partials(const float* logits, uint32_t n, uint32_t c, const uint32_t* labels,
                                  const uint8_t* mask, double inv_count, float* grad, double* blk_loss,
                                  uint32_t* blk_ok, cudaStream_t s) {
    if (c == 0 || c > 32) return fail(SGNN_ERR_SHAPE, "softmax_xent: 1..32 classes");
    if (n == 0) return SGNN_OK;
    uint32_t rpb = 1, nblk = 1;
    softmax_shape(n, &rpb, &nblk);
    if (c <= 4)
        softmax_xent_kernel<4><<<nblk, kSoftmaxThreads, 0, s>>>(logits, n, c, labels, mask, inv_count, rpb, grad, blk_loss, blk_ok);
    else if (c <= 8)
        softmax_xent_kernel<8><<<nblk, kSoftmaxThreads, 0, s>>>(logits, n, c, labels, mask, inv_count, rpb, grad, blk_loss, blk_ok);
    else if (c <= 16)
        softmax_xent_kernel<16><<<nblk, kSoftmaxThreads, 0, s>>>(logits, n, c, labels, mask, inv_count, rpb, grad, blk_loss, blk_ok);
    else
        softmax_xent_kernel<32><<<nblk, kSoftmaxThreads, 0, s>>>(logits, n, c, labels, mask, inv_count, rpb, grad, blk_loss, blk_ok);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

sgnn_status sage_head_partials(const float* a2, const float* h1, const float* w2, const float* w2s, uint32_t n,
                               uint32_t h, uint32_t c, const uint32_t* labels, const uint8_t* mask, double inv_count,
                               float* grad, float* ds2, double* blk_loss, uint32_t* blk_ok, cudaStream_t s) {
    SGNN_TRY(sage_shape(h, c, "sage_head"));
    if (n == 0) return SGNN_OK;
    uint32_t rpb = 1, nblk = 1;
    softmax_shape(n, &rpb, &nblk);
    SAGE_HEAD(c, nblk,
            (a2, h1, w2, w2s, n, h, c, labels, mask, inv_count, rpb, grad, ds2, blk_loss, blk_ok));
    return SGNN_OK;
}

template <int CP>
sgnn_status wgrad_launch_cp(const float* a2, const float* h1, const float* grad, uint32_t n, uint32_t h, uint32_t c,
                            uint32_t rpb, uint32_t nblk, float* part, cudaStream_t s) {
    const size_t smem = sage_wgrad_smem(h, c, CP);
    SGNN_CUDA_TRY(cudaFuncSetAttribute(sage_wgrad_kernel<CP>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    sage_wgrad_kernel<CP><<<nblk, 256, smem, s>>>(a2, h1, grad, n, h, c, rpb, part);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

sgnn_status sage_wgrad_launch(const float* a2, const float* h1, const float* grad, uint32_t n, uint32_t h,
                              uint32_t c, uint32_t rpb, uint32_t nblk, float* part, float* g2, float* g2s,
                              cudaStream_t s) {
    if (c <= 4) SGNN_TRY(wgrad_launch_cp<4>(a2, h1, grad, n, h, c, rpb, nblk, part, s));
    else if (c <= 8) SGNN_TRY(wgrad_launch_cp<8>(a2, h1, grad, n, h, c, rpb, nblk, part, s));
    else SGNN_TRY(wgrad_launch_cp<16>(a2, h1, grad, n, h, c, rpb, nblk, part, s));
    SAGE_CP(sage_wgrad_finish_kernel, c, unsigned((2 * h * 16 + 127) / 128), 128, (part, nblk, h, c, g2, g2s));
    return SGNN_OK;
}

sgnn_status glue_sage_wgrad(const float* a2, const float* h1, const float* grad, uint32_t n, uint32_t h, uint32_t c,
                            float* g2, float* g2s, cudaStream_t s) {
    SGNN_TRY(sage_shape(h, c, "sage_wgrad"));
    const uint32_t want = std::min<uint32_t>(592, std::max<uint32_t>(1, n));
    const uint32_t rpb = std::max<uint32_t>(1, (n + want - 1) / want);
    const uint32_t nblk = std::max<uint32_t>(1, (n + rpb - 1) / rpb);
    float* part = nullptr;
    SGNN_TRY(scratch_alloc(reinterpret_cast<void**>(&part), sizeof(float) * nblk * 2 * h * 16, s));
    const sgnn_status st = sage_wgrad_launch(a2, h1, grad, n, h, c, rpb, nblk, part, g2, g2s, s);
    scratch_free(part, s);
    return st;
}

sgnn_status glue_sage_grad_wt(const float* grad, const float* w, uint32_t n, uint32_t h, uint32_t c, const float* u,
                              const float* act, float* out, cudaStream_t s) {
    SGNN_TRY(sage_shape(h, c, "sage_grad_wt"));
    if ((u == nullptr) != (act == nullptr)) return fail(SGNN_ERR_CONFIG, "sage_grad_wt: u and act go together");
    if (n == 0) return SGNN_OK;
    SAGE_CP(sage_grad_wt_kernel, c, grid_for(uint64_t(n) * 32), 256, (grad, w, n, h, c, u, act, out));
    return SGNN_OK;
}


}  // namespace sgnn
