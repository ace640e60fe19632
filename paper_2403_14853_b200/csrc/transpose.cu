// transpose.cu -- on-device CSR -> CSC (= CSR of A^T), bit-exact with the
// reference's serial counting sort (sparse.hpp:72-89): placement in
// ascending original row within each column, t_row_ptr = the column starts.
//
// The stable placement is an LSD radix sort of the nonzeros keyed by column
// (passes of <= 9-bit digits: 2 up to 2^18 columns, 3 up to 2^27), carrying (row, value)
// as payload.  Each tile of 4096 nonzeros is ranked warp by warp in index
// order (digit peers from one ballot per digit bit, the warp's running digit
// counts advanced by one shared-memory atomic per peer group), staged in
// shared memory in digit order and written out as contiguous runs per digit,
// so the output is exactly the counting-sort order.  The first pass derives
// the row of every nonzero from the row starts inside its tile (marks + a
// block scan, the tile's first row precomputed for all tiles at once), so no
// expanded row array is read and no per-nonzero search is made.  The column
// starts come from the sorted keys at the end (one boundary pass), not from a
// column histogram: hub columns made the histogram's global atomics the
// single slowest step (0.52 ms of 2.5 ms on cfg2).
//
// Also: row_degrees (sparse.hpp:105-109), is_symmetric (sparse.hpp:179-192)
// and the mean-operand value scaling (gnn.hpp:158-159).
#include <algorithm>
#include <cstdlib>

#include "ops.cuh"

namespace sgnn {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;                          // per thread per tile
constexpr uint64_t kTile = uint64_t(kThreads) * kItems;  // 4096 nonzeros
// <= 512 bins: 22-bit columns (cfg5) as 3 passes of 8 bits run 5.7 ms
// against 9.0 ms as 2 passes of 11 (2048-bin bookkeeping, 2 CTAs/SM), 20-bit
// (cfg4) 0.95 vs 1.02 ms as 3 x 7 against 2 x 10; 18-bit cfg2 keeps 2 x 9
// (1.22 ms; 3 x 6: 1.30)
constexpr int kMaxDigitBits = 9;
constexpr unsigned kFull = 0xffffffffu;

constexpr int kUpTiles = kWarps;  // tiles per upsweep CTA (one per warp): a 32-byte sector per digit

struct RadixPlan {
    int passes = 1;
    int dbits = 1;
    uint32_t bins = 2;
    uint64_t tiles = 0;
    uint64_t tstride = 0;  // tiles rounded up to kUpTiles: the [digit][tile] count rows
};

RadixPlan radix_plan(uint32_t n_cols, uint64_t nnz) {
    RadixPlan r;
    int nbits = 0;
    if (n_cols > 1) {
        uint32_t v = n_cols - 1;
        while (v) { ++nbits; v >>= 1; }
    }
    r.passes = std::max(1, (nbits + kMaxDigitBits - 1) / kMaxDigitBits);
    r.dbits = std::max(1, (nbits + r.passes - 1) / r.passes);
    r.bins = 1u << r.dbits;
    r.tiles = ceil_div_u64(nnz, kTile);
    r.tstride = ceil_div_u64(r.tiles, kUpTiles) * kUpTiles;
    return r;
}

struct Workspace {
    uint32_t* keys_a;
    uint32_t* keys_b;
    uint32_t* rows_a;
    float* vals_a;
    uint32_t* hist;       // bins * tiles (+1 for the scan total)
    uint32_t* tile_row0;  // tiles: row holding each tile's first nonzero
    size_t bytes;
};

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

Workspace carve(void* base, const sgnn_csr* a, const RadixPlan& rp) {
    Workspace w{};
    char* p = static_cast<char*>(base);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* q = p ? p + off : nullptr;
        off += align256(bytes);
        return q;
    };
    const size_t nnz = a->nnz;
    w.keys_a = reinterpret_cast<uint32_t*>(take(4 * nnz));
    w.keys_b = reinterpret_cast<uint32_t*>(take(4 * nnz));
    w.rows_a = reinterpret_cast<uint32_t*>(take(4 * nnz));
    w.vals_a = reinterpret_cast<float*>(take(4 * nnz));
    w.hist = reinterpret_cast<uint32_t*>(take(4 * (size_t(rp.bins) * rp.tstride + 1)));
    w.tile_row0 = reinterpret_cast<uint32_t*>(take(4 * (size_t(rp.tiles) + 1)));
    w.bytes = off;
    return w;
}

// Largest r in [lo, hi) with rp[r] <= idx (the row holding nonzero idx).
__device__ __forceinline__ uint32_t find_row(const uint64_t* __restrict__ rp, uint32_t lo,
                                             uint32_t hi, uint64_t idx) {
    while (hi - lo > 1) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (__ldg(rp + mid) <= idx) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Row range [r_lo, r_hi] covering nonzeros [base, last] of a tile.
__device__ __forceinline__ void tile_rows(const uint64_t* __restrict__ rp, uint32_t m,
                                          uint64_t base, uint64_t last, uint32_t* r_lo,
                                          uint32_t* r_hi) {
    *r_lo = find_row(rp, 0, m, base);
    *r_hi = find_row(rp, *r_lo, m, last);
}

// tile_row0[t] = the row holding nonzero t * kTile (the largest r with
// rp[r] <= t * kTile): each nonempty row names the tiles starting inside it.
__global__ void tile_row0_kernel(const uint64_t* __restrict__ rp, uint32_t m,
                                 uint32_t* __restrict__ out) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
        const uint64_t s = __ldg(rp + r), e = __ldg(rp + r + 1);
        for (uint64_t t = (s + kTile - 1) / kTile; t * kTile < e; ++t) out[t] = r;
    }
}

// t_row_ptr from the sorted column keys: position p starts every column in
// (keys[p-1], keys[p]] (empty columns included); p = nnz closes the rest.
// Four positions per thread (one 16-byte load where aligned).  Runs of more
// than kGapRun empty columns are left (only their last column, the
// nonempty one, is written) to col_gaps_kernel, so no thread walks a long run.
constexpr int64_t kGapRun = 64;
constexpr uint64_t kUnset = ~0ull;
__global__ void col_starts_kernel(const uint32_t* __restrict__ keys, uint64_t nnz, uint32_t n_cols,
                                  uint64_t* __restrict__ trp) {
    const uint64_t p0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (p0 > nnz) return;
    int64_t k[5];
    k[0] = p0 ? int64_t(__ldg(keys + p0 - 1)) : -1;
    if (p0 + 4 <= nnz && (reinterpret_cast<uintptr_t>(keys + p0) & 15) == 0) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(keys + p0));
        k[1] = v.x; k[2] = v.y; k[3] = v.z; k[4] = v.w;
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            k[i + 1] = p0 + i < nnz ? int64_t(__ldg(keys + p0 + i)) : (p0 + i == nnz ? int64_t(n_cols) : k[i]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t lo = k[i + 1] - k[i] > kGapRun ? k[i + 1] : k[i] + 1;
        for (int64_t c = lo; c <= k[i + 1]; ++c) trp[c] = p0 + i;
    }
}

// The columns col_starts_kernel left unset (inside long empty runs): the
// first position whose key is >= c (binary search of the sorted keys).
__global__ void col_gaps_kernel(const uint32_t* __restrict__ keys, uint64_t nnz, uint32_t n_cols,
                                uint64_t* __restrict__ trp) {
    for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n_cols;
         c += uint64_t(gridDim.x) * blockDim.x) {
        if (trp[c] != kUnset) continue;
        uint64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (__ldg(keys + mid) < c) lo = mid + 1;
            else hi = mid;
        }
        trp[c] = lo;
    }
}

// Per-tile digit counts, hist[d * tstride + t]: warp w of CTA b counts tile
// b * kUpTiles + w into its own shared histogram (16 loads per lane in flight
// before their shared atomics), then each digit's kUpTiles counts leave as one
// aligned 32-byte sector (one tile per CTA wrote a 4-byte partial sector per
// digit: 512 scattered writes per 4096 nonzeros).
__global__ void __launch_bounds__(kThreads) radix_upsweep_kernel(const uint32_t* __restrict__ keys,
                                                                 uint64_t n, int shift,
                                                                 uint32_t mask, uint64_t tstride,
                                                                 uint32_t* __restrict__ hist) {
    static_assert(kUpTiles == 8, "two 16-byte stores per digit");
    extern __shared__ uint32_t sh[];  // [kUpTiles][bins]
    const uint32_t bins = mask + 1;
    for (uint32_t d = threadIdx.x; d < kUpTiles * bins; d += kThreads) sh[d] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* wh = sh + wid * bins;
    const uint64_t base = (uint64_t(blockIdx.x) * kUpTiles + wid) * kTile;
    constexpr int R = 16;
    for (int r0 = 0; r0 < int(kTile / 32); r0 += R) {
        uint32_t k[R];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const uint64_t idx = base + uint64_t(r0 + q) * 32 + lane;
            k[q] = idx < n ? __ldcs(keys + idx) : 0u;
        }
#pragma unroll
        for (int q = 0; q < R; ++q)
            if (base + uint64_t(r0 + q) * 32 + lane < n) atomicAdd(wh + ((k[q] >> shift) & mask), 1u);
    }
    __syncthreads();
    for (uint32_t d = threadIdx.x; d < bins; d += kThreads) {
        uint4* dst = reinterpret_cast<uint4*>(hist + uint64_t(d) * tstride + uint64_t(blockIdx.x) * kUpTiles);
        dst[0] = make_uint4(sh[d], sh[bins + d], sh[2 * bins + d], sh[3 * bins + d]);
        dst[1] = make_uint4(sh[4 * bins + d], sh[5 * bins + d], sh[6 * bins + d], sh[7 * bins + d]);
    }
}

// Exclusive scan of one value per thread over the block (warp shuffles, one
// barrier); `s_warp` holds kWarps entries and must not be reused before the
// next barrier.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    uint32_t pre = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) pre += (w < wid) ? s_warp[w] : 0u;
    return pre + x - v;
}

// Stable scatter of one tile (4096 nonzeros in index order), staged through
// shared memory so the global writes are contiguous runs per digit:
//   A. warp w ranks its 512 consecutive items (16 rounds of 32, lane order =
//      index order): the lanes sharing a digit come from one ballot per digit
//      bit (unrolled: the digit width is a template parameter), the group's
//      lowest lane advances the warp's counter for that digit with one shared
//      atomic (u16 counters packed in pairs) and broadcasts the old count --
//      no block barrier, and the rounds' atomics pipeline (same-warp shared
//      atomics to one address stay in order).  Measured on cfg2 against this:
//      __match_any_sync (throughput-bound, +40 %), per-warp shared peer masks
//      built with atomicOr (a longer dependent chain per round, +12 %);
//   B. per digit, exclusive offsets over the warps and the tile's digit
//      starts (one block scan);
//   C. every item lands in the tile's digit-sorted order in shared memory;
//   D. consecutive threads write consecutive staged items: within a digit
//      they go to consecutive global positions.
// The order is the stable counting sort's (index order within a digit).
// FIRST: rows come from the CSR itself -- each row start inside the tile
// marks its position, an inclusive scan of the marks gives every item's row
// (empty rows included).
constexpr int kDownSmemFixed = 3 * kThreads * kItems * 4;  // staged keys, rows, vals

template <bool FIRST, bool VALS, int DB>
__global__ void __launch_bounds__(kThreads, 3) radix_downsweep_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ rows_in,
    const float* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ rows_out, float* __restrict__ vals_out, uint64_t n, int shift,
    int dbits, uint64_t tstride, const uint32_t* __restrict__ hist_scan,
    const uint64_t* __restrict__ rp, uint32_t m, const uint32_t* __restrict__ tile_row0) {
    constexpr int T = kThreads * kItems;  // 4096
    constexpr int WI = T / kWarps;        // 512 items per warp
    extern __shared__ __align__(16) uint32_t sh[];
    static_assert(DB >= 1 && DB <= kMaxDigitBits, "digit width");
    (void)dbits;
    constexpr uint32_t bins = 1u << DB;
    constexpr uint32_t mask = bins - 1;
    // bins per thread for the digit bookkeeping (1 when bins < kThreads)
    constexpr uint32_t bpt = bins >= uint32_t(kThreads) ? bins / kThreads : 1u;
    constexpr uint32_t cwords = bins / 2;
    uint32_t* skey = sh;                    // [T] (FIRST: first the row marks, then the rows)
    // staged (row, value) pairs as one 8-byte store / load per item (not in
    // the first pass: the extra registers spill there); else rows and values
    // apart
    constexpr bool PACK = VALS && !FIRST;
    uint2* srv = reinterpret_cast<uint2*>(sh + T);   // [T] PACK
    uint32_t* srow = sh + T;                          // [T] otherwise
    float* sval = reinterpret_cast<float*>(sh + 2 * T);
    uint32_t* smark = skey;
    uint32_t* sgoff = sh + 3 * T;           // [bins] global offset - tile digit start
    uint32_t* sdst = sgoff + bins;          // [bins] tile digit start
    uint32_t* wcnt = sdst + bins;           // [kWarps][bins / 2]: u16 counters in pairs
    uint16_t* wc16 = reinterpret_cast<uint16_t*>(wcnt);  // [kWarps][bins]
    __shared__ uint32_t s_warp[2][kWarps];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t base = uint64_t(blockIdx.x) * T;
    const uint32_t cnt = uint32_t(min(uint64_t(T), n - base));
    for (uint32_t d = threadIdx.x; d < kWarps * cwords; d += kThreads) wcnt[d] = 0;
    uint32_t r0 = 0;
    if (FIRST) {
        r0 = __ldg(tile_row0 + blockIdx.x);
        for (int i = threadIdx.x; i < T; i += kThreads) smark[i] = 0;
    }
    // every load of the tile in flight together: items, the tile's global
    // digit offsets, (FIRST) the row starts inside the tile
    uint32_t kk[kItems], rr[kItems];
    float vv[kItems];
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
        const uint32_t li = uint32_t(wid * WI + q * 32 + lane);
        const bool valid = li < cnt;
        const uint64_t idx = base + li;
        kk[q] = valid ? __ldcs(keys_in + idx) : 0u;
        rr[q] = valid && !FIRST ? __ldcs(rows_in + idx) : 0u;
        vv[q] = valid && VALS ? __ldcs(vals_in + idx) : 0.0f;
    }
    // the tile's global digit offsets go straight to shared memory (cp.async:
    // no registers held while they are in flight)
    for (uint32_t b = 0; b < bpt; ++b) {
        const uint32_t d = threadIdx.x * bpt + b;
        if (d < bins) {
            const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(sgoff + d));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst),
                         "l"(hist_scan + uint64_t(d) * tstride + blockIdx.x)
                         : "memory");
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (FIRST) {
        __syncthreads();  // marks zeroed
        // mark every row start strictly inside the tile (empty rows stack up)
        for (uint32_t r = r0 + 1 + threadIdx.x; r <= m; r += kThreads) {
            const uint64_t st = __ldg(rp + r);
            if (st >= base + cnt) break;
            atomicAdd(smark + (st - base), 1u);
        }
        __syncthreads();
        // inclusive scan of the marks: item i's row = r0 + marks(<= i)
        uint32_t loc[kItems], acc = 0;
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            acc += smark[threadIdx.x * kItems + q];
            loc[q] = acc;
        }
        const uint32_t pre = r0 + block_exclusive_scan(acc, s_warp[0]);
#pragma unroll
        for (int q = 0; q < kItems; ++q) smark[threadIdx.x * kItems + q] = pre + loc[q];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kItems; ++q) rr[q] = smark[wid * WI + q * 32 + lane];
    }
    __syncthreads();  // counters zeroed (and FIRST: the rows read before staging reuses skey)
    // A. warp-local stable ranks
    const unsigned lt = (1u << lane) - 1u;
    uint32_t* mycnt = wcnt + wid * cwords;
    uint32_t pk[kItems];  // digit << 16 | rank within the warp's digit
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
        const uint32_t li = uint32_t(wid * WI + q * 32 + lane);
        const bool valid = li < cnt;
        const uint32_t d = (kk[q] >> shift) & mask;
        unsigned peers = __ballot_sync(kFull, valid);
#pragma unroll
        for (int b = 0; b < DB; ++b) {
            const bool bit = (d >> b) & 1u;
            const unsigned bal = __ballot_sync(kFull, bit);
            peers &= bit ? bal : ~bal;
        }
        const int leader = valid ? __ffs(peers) - 1 : lane;
        const uint32_t hsh = (d & 1u) * 16u;
        uint32_t old = 0;
        if (valid && leader == lane) old = atomicAdd(mycnt + (d >> 1), uint32_t(__popc(peers)) << hsh);
        old = __shfl_sync(kFull, old, leader);
        pk[q] = valid ? (d << 16) | (((old >> hsh) & 0xffffu) + __popc(peers & lt)) : 0xffffffffu;
    }
    __syncthreads();
    // B. per digit: exclusive offsets over the warps, tile totals (parked in
    // sdst), block scan, then the tile's digit starts
    asm volatile("cp.async.wait_all;" ::: "memory");
    uint32_t run = 0;
    if constexpr (bpt >= 2) {
        // a thread's digits are whole counter words: both halves per access
        constexpr uint32_t wpt = bpt / 2;
#pragma unroll
        for (uint32_t b = 0; b < wpt; ++b) {
            const uint32_t wi = threadIdx.x * wpt + b;  // digits 2 wi, 2 wi + 1
            uint32_t tlo = 0, thi = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t c = wcnt[w * cwords + wi];
                wcnt[w * cwords + wi] = tlo | (thi << 16);
                tlo += c & 0xffffu;
                thi += c >> 16;
            }
            sdst[2 * wi] = tlo;
            sdst[2 * wi + 1] = thi;
            run += tlo + thi;
        }
    } else {
        const uint32_t d = threadIdx.x;
        if (d < bins) {
            uint32_t t = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t c = wc16[w * bins + d];
                wc16[w * bins + d] = uint16_t(t);
                t += c;
            }
            sdst[d] = t;
            run += t;
        }
    }
    uint32_t start = block_exclusive_scan(run, s_warp[1]);
    for (uint32_t b = 0; b < bpt; ++b) {
        const uint32_t d = threadIdx.x * bpt + b;
        if (d < bins) {
            const uint32_t t = sdst[d];
            sdst[d] = start;
            sgoff[d] -= start;
            start += t;
        }
    }
    __syncthreads();
    // C. stage in the tile's digit-sorted order
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
        if (pk[q] == 0xffffffffu) continue;
        const uint32_t d = pk[q] >> 16;
        const uint32_t slot = sdst[d] + wc16[wid * bins + d] + (pk[q] & 0xffffu);
        skey[slot] = kk[q];
        if (PACK) {
            srv[slot] = make_uint2(rr[q], __float_as_uint(vv[q]));
        } else {
            srow[slot] = rr[q];
            if (VALS) sval[slot] = vv[q];
        }
    }
    __syncthreads();
    // D. contiguous runs per digit to global memory
    for (uint32_t k = threadIdx.x; k < cnt; k += kThreads) {
        const uint32_t key = skey[k];
        const uint64_t dst = uint64_t(sgoff[(key >> shift) & mask]) + k;
        keys_out[dst] = key;
        if (PACK) {
            const uint2 rv = srv[k];
            rows_out[dst] = rv.x;
            vals_out[dst] = __uint_as_float(rv.y);
        } else {
            rows_out[dst] = srow[k];
            if (VALS) vals_out[dst] = sval[k];
        }
    }
}

template <bool FIRST, int DB>
sgnn_status launch_down_db(bool vals, const uint32_t* ki, const uint32_t* ri, const float* vi, uint32_t* ko,
                           uint32_t* ro, float* vo, uint64_t n, int shift, uint64_t tiles, uint64_t tstride,
                           const uint32_t* hs,
                           const uint64_t* rp, uint32_t m, const uint32_t* tr0, cudaStream_t s) {
    constexpr size_t bins = size_t(1) << DB;
    const size_t smem = kDownSmemFixed + 2 * 4 * bins + 4 * kWarps * (bins / 2);
    auto k = vals ? radix_downsweep_kernel<FIRST, true, DB> : radix_downsweep_kernel<FIRST, false, DB>;
    SGNN_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    SGNN_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    k<<<unsigned(tiles), kThreads, smem, s>>>(ki, ri, vi, ko, ro, vo, n, shift, DB, tstride, hs, rp, m, tr0);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

// the digit width is a template parameter: the ranking's ballots unroll
template <bool FIRST>
sgnn_status launch_down(bool vals, const uint32_t* ki, const uint32_t* ri, const float* vi, uint32_t* ko,
                        uint32_t* ro, float* vo, uint64_t n, int shift, int dbits, uint64_t tiles,
                        uint64_t tstride, const uint32_t* hs, const uint64_t* rp, uint32_t m, const uint32_t* tr0,
                        cudaStream_t s) {
#define SGNN_DOWN_CASE(D) \
    case D: return launch_down_db<FIRST, D>(vals, ki, ri, vi, ko, ro, vo, n, shift, tiles, tstride, hs, rp, m, tr0, s);
    switch (dbits) {
        SGNN_DOWN_CASE(1) SGNN_DOWN_CASE(2) SGNN_DOWN_CASE(3) SGNN_DOWN_CASE(4) SGNN_DOWN_CASE(5)
        SGNN_DOWN_CASE(6) SGNN_DOWN_CASE(7) SGNN_DOWN_CASE(8) SGNN_DOWN_CASE(9)
    }
#undef SGNN_DOWN_CASE
    return fail(SGNN_ERR_INTERNAL, "transpose: digit width out of range");
}

__global__ void row_degrees_kernel(const uint64_t* __restrict__ rp, uint32_t m,
                                   uint32_t* __restrict__ deg) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        deg[i] = uint32_t(__ldg(rp + i + 1) - __ldg(rp + i));
}

__global__ void mean_scale_kernel(const uint32_t* __restrict__ ci, const float* __restrict__ vin,
                                  const uint32_t* __restrict__ deg, uint64_t nnz,
                                  float* __restrict__ vout) {
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz;
         e += uint64_t(gridDim.x) * blockDim.x)
        vout[e] = __fdiv_rn(vin[e], float(__ldg(deg + __ldg(ci + e))));
}

// is_symmetric with half the searches: only the upper entries (i, j > i)
// binary-search their mirror (j, i) in row j (value must match); lower
// entries are only counted.  Every upper entry matched and #upper == #lower
// <=> the mirror map is a bijection of the off-diagonal entries <=> the
// reference's check (every entry's mirror exists with an equal value) holds.
// flag[0] = 0 on a mismatch; cnt[0] / cnt[1] accumulate #upper / #lower.
__global__ void __launch_bounds__(kThreads) symmetric_kernel(const uint64_t* __restrict__ rp,
                                                             const uint32_t* __restrict__ ci,
                                                             const float* __restrict__ v,
                                                             uint32_t m, uint64_t nnz,
                                                             int* __restrict__ flag,
                                                             unsigned long long* __restrict__ cnt) {
    __shared__ uint32_t s_rows[2];
    __shared__ int s_done;
    const uint64_t base = uint64_t(blockIdx.x) * kTile;
    if (threadIdx.x == 0) {
        // the answer is already "no" (sparse.hpp:179-192 stops at the first
        // mismatch too): tiles scheduled after it skip their searches
        s_done = *reinterpret_cast<volatile int*>(flag) == 0;
        uint32_t lo = 0, hi = 0;
        if (!s_done) tile_rows(rp, m, base, min(base + kTile, nnz) - 1, &lo, &hi);
        s_rows[0] = lo;
        s_rows[1] = hi + 1;
    }
    __syncthreads();
    if (s_done) return;
    bool ok = true;
    uint32_t up = 0, low = 0;
    for (int r = 0; r < kItems; ++r) {
        const uint64_t e = base + uint64_t(r) * kThreads + threadIdx.x;
        if (e >= nnz) break;
        const uint32_t i = find_row(rp, s_rows[0], s_rows[1], e);
        const uint32_t j = __ldg(ci + e);
        if (j < i) {
            ++low;
            continue;
        }
        if (j == i) continue;
        ++up;
        uint64_t lo = __ldg(rp + j), hi = __ldg(rp + j + 1);
        const uint64_t end = hi;
        while (lo < hi) {  // lower_bound of i in row j
            const uint64_t mid = lo + (hi - lo) / 2;
            if (__ldg(ci + mid) < i) lo = mid + 1;
            else hi = mid;
        }
        if (lo == end || __ldg(ci + lo) != i || __ldg(v + lo) != __ldg(v + e)) ok = false;
    }
    // block sums of the counts (warp reduce, one atomic per warp)
    for (int o = 16; o >= 1; o >>= 1) {
        up += __shfl_xor_sync(0xffffffffu, up, o);
        low += __shfl_xor_sync(0xffffffffu, low, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (up) atomicAdd(cnt, (unsigned long long)up);
        if (low) atomicAdd(cnt + 1, (unsigned long long)low);
    }
    if (__syncthreads_or(!ok) && threadIdx.x == 0) atomicExch(flag, 0);
}

}  // namespace

size_t transpose_workspace_bytes(const sgnn_csr* a) {
    const RadixPlan rp = radix_plan(a->n_cols, a->nnz);
    return carve(nullptr, a, rp).bytes;
}

sgnn_status run_transpose(const sgnn_csr* a, uint64_t* trp, uint32_t* tci, float* tv, void* ws,
                          size_t ws_bytes, cudaStream_t s) {
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    const RadixPlan plan = radix_plan(a->n_cols, a->nnz);
    if (a->nnz == 0) {  // every column empty
        SGNN_CUDA_TRY(cudaMemsetAsync(trp, 0, sizeof(uint64_t) * (size_t(a->n_cols) + 1), s));
        return SGNN_OK;
    }
    const size_t need = carve(nullptr, a, plan).bytes;
    void* own = nullptr;
    if (!ws) {
        SGNN_TRY(scratch_alloc(&own, need, s));
        ws = own;
    } else if (ws_bytes < need) {
        return fail(SGNN_ERR_CONFIG, "transpose: workspace too small (need " +
                                         std::to_string(need) + " bytes)");
    }
    Workspace w = carve(ws, a, plan);
    sgnn_status st = SGNN_OK;
    do {
        // the row of every tile's first nonzero (the first pass's row recovery)
        {
            const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(a->n_rows, 256), uint64_t(dp.sm_count) * 16);
            tile_row0_kernel<<<unsigned(std::max<uint64_t>(blocks, 1)), 256, 0, s>>>(a->row_ptr, a->n_rows,
                                                                                    w.tile_row0);
            if (cudaGetLastError() != cudaSuccess) {
                st = fail(SGNN_ERR_CUDA, "transpose: tile_row0 launch failed");
                break;
            }
        }
        // stable LSD radix passes (sparse.hpp:80-86 placement order)
        const bool vals = tv != nullptr;
        const uint32_t mask = plan.bins - 1;
        const uint32_t* keys_src = a->col_idx;
        const uint32_t* rows_src = nullptr;
        const float* vals_src = a->values;
        for (int p = 0; p < plan.passes && st == SGNN_OK; ++p) {
            const bool first = p == 0;
            // the last pass lands in (tci, tv); earlier passes alternate with set A
            const bool to_out = ((plan.passes - 1 - p) % 2) == 0;
            uint32_t* keys_dst = (p % 2 == 0) ? w.keys_a : w.keys_b;
            uint32_t* rows_dst = to_out ? tci : w.rows_a;
            float* vals_dst = to_out ? tv : w.vals_a;
            const int shift = p * plan.dbits;
            const size_t up_smem = sizeof(uint32_t) * plan.bins * kUpTiles;
            if (cudaFuncSetAttribute(radix_upsweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(up_smem)) != cudaSuccess) {
                st = fail(SGNN_ERR_CUDA, "transpose: upsweep attribute failed");
                break;
            }
            radix_upsweep_kernel<<<unsigned(plan.tstride / kUpTiles), kThreads, up_smem, s>>>(
                keys_src, a->nnz, shift, mask, plan.tstride, w.hist);
            if (cudaGetLastError() != cudaSuccess) {
                st = fail(SGNN_ERR_CUDA, "transpose: upsweep launch failed");
                break;
            }
            st = exclusive_scan_u32(w.hist, w.hist, uint64_t(plan.bins) * plan.tstride, s);
            if (st != SGNN_OK) break;
            if (first)
                st = launch_down<true>(vals, keys_src, rows_src, vals_src, keys_dst, rows_dst, vals_dst, a->nnz,
                                       shift, plan.dbits, plan.tiles, plan.tstride, w.hist, a->row_ptr, a->n_rows, w.tile_row0, s);
            else
                st = launch_down<false>(vals, keys_src, rows_src, vals_src, keys_dst, rows_dst, vals_dst, a->nnz,
                                        shift, plan.dbits, plan.tiles, plan.tstride, w.hist, a->row_ptr, a->n_rows, w.tile_row0, s);
            keys_src = keys_dst;
            rows_src = rows_dst;
            vals_src = vals_dst;
        }
        if (st != SGNN_OK) break;
        // t_row_ptr from the sorted keys (sparse.hpp:75-76's histogram + scan)
        if (cudaMemsetAsync(trp, 0xff, sizeof(uint64_t) * size_t(a->n_cols), s) != cudaSuccess) {
            st = fail(SGNN_ERR_CUDA, "transpose: memset failed");
            break;
        }
        const uint64_t blocks = ceil_div_u64(ceil_div_u64(a->nnz + 1, 4), 256);
        col_starts_kernel<<<unsigned(blocks), 256, 0, s>>>(keys_src, a->nnz, a->n_cols, trp);
        const uint64_t gblocks = std::min<uint64_t>(ceil_div_u64(a->n_cols, 256), uint64_t(dp.sm_count) * 16);
        if (a->n_cols) col_gaps_kernel<<<unsigned(gblocks), 256, 0, s>>>(keys_src, a->nnz, a->n_cols, trp);
        if (cudaGetLastError() != cudaSuccess) st = fail(SGNN_ERR_CUDA, "transpose: column-start launch failed");
    } while (false);
    if (own) scratch_free(own, s);
    return st;
}

sgnn_status run_row_degrees(const sgnn_csr* a, uint32_t* deg, cudaStream_t s) {
    if (a->n_rows == 0) return SGNN_OK;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(a->n_rows, 256), uint64_t(dp.sm_count) * 8);
    row_degrees_kernel<<<unsigned(blocks), 256, 0, s>>>(a->row_ptr, a->n_rows, deg);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

sgnn_status run_mean_scale(const uint32_t* col_idx, const float* vin, const uint32_t* deg,
                           uint64_t nnz, float* vout, cudaStream_t s) {
    if (nnz == 0) return SGNN_OK;
    DeviceProps dp;
    SGNN_TRY(device_props(&dp));
    const uint64_t blocks = std::min<uint64_t>(ceil_div_u64(nnz, 256), uint64_t(dp.sm_count) * 16);
    mean_scale_kernel<<<unsigned(blocks), 256, 0, s>>>(col_idx, vin, deg, nnz, vout);
    SGNN_LAUNCH_CHECK();
    return SGNN_OK;
}

sgnn_status run_is_symmetric(const sgnn_csr* a, int* out, cudaStream_t s) {
    *out = 0;
    if (a->n_rows != a->n_cols) return SGNN_OK;  // sparse.hpp:180
    if (a->nnz == 0) {
        *out = 1;
        return SGNN_OK;
    }
    // scratch: flag (int, padded to 8 bytes) | #upper | #lower
    unsigned long long* buf = nullptr;
    SGNN_TRY(scratch_alloc(reinterpret_cast<void**>(&buf), 3 * sizeof(unsigned long long), s));
    int* flag = reinterpret_cast<int*>(buf);
    const unsigned long long init[3] = {1ull, 0ull, 0ull};  // flag word = 1 (little endian)
    sgnn_status st = SGNN_OK;
    if (cudaMemcpyAsync(buf, init, sizeof(init), cudaMemcpyHostToDevice, s) != cudaSuccess)
        st = fail(SGNN_ERR_CUDA, "is_symmetric: memcpy failed");
    if (st == SGNN_OK) {
        symmetric_kernel<<<unsigned(ceil_div_u64(a->nnz, kTile)), kThreads, 0, s>>>(
            a->row_ptr, a->col_idx, a->values, a->n_rows, a->nnz, flag, buf + 1);
        if (cudaGetLastError() != cudaSuccess) st = fail(SGNN_ERR_CUDA, "is_symmetric: launch failed");
    }
    unsigned long long res[3] = {0, 0, 0};
    if (st == SGNN_OK &&
        (cudaMemcpyAsync(res, buf, sizeof(res), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
         cudaStreamSynchronize(s) != cudaSuccess))
        st = fail(SGNN_ERR_CUDA, "is_symmetric: readback failed");
    scratch_free(buf, s);
    if (st == SGNN_OK) *out = (int(res[0] & 0xffffffffu) != 0 && res[1] == res[2]) ? 1 : 0;
    return st;
}

}  // namespace sgnn
