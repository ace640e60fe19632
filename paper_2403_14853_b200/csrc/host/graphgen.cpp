// graphgen.cpp -- deterministic, multithreaded synthetic inputs (sgnn_host.h)
// and the host-side nnz-balanced row partitioner.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "../../../include/sgnn_host.h"

namespace {

inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

inline uint64_t counter_hash(uint64_t seed, uint64_t stream, uint64_t i) {
    return splitmix64(splitmix64(seed ^ splitmix64(stream * 0xd1342543de82ef95ull + 1)) + i);
}

inline double u01(uint64_t h) { return double(h >> 11) * 0x1.0p-53; }

int resolve(int threads) {
    if (threads > 0) return threads;
    unsigned hw = std::thread::hardware_concurrency();
    return hw ? int(hw) : 1;
}

template <class Fn>
void parallel_range(uint64_t n, int threads, Fn&& fn) {
    int t = resolve(threads);
    if (n < 65536 || t <= 1) {
        fn(uint64_t(0), n);
        return;
    }
    t = int(std::min<uint64_t>(uint64_t(t), n / 4096 + 1));
    std::vector<std::thread> ws;
    for (int c = 1; c < t; ++c)
        ws.emplace_back([&, c] { fn(n * c / t, n * (c + 1) / t); });
    fn(0, n / t);
    for (auto& w : ws) w.join();
}

// Parallel LSD radix sort of u64 keys over the low `bits` bits (8-bit digits).
void radix_sort(std::vector<uint64_t>& keys, int bits, int threads) {
    const uint64_t n = keys.size();
    if (n < 2) return;
    std::vector<uint64_t> tmp(n);
    int t = resolve(threads);
    t = int(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(t), n / 65536 + 1)));
    std::vector<uint64_t> hist(size_t(t) * 256);
    for (int shift = 0; shift < bits; shift += 8) {
        std::fill(hist.begin(), hist.end(), 0);
        auto count = [&](int c) {
            uint64_t* h = hist.data() + size_t(c) * 256;
            for (uint64_t i = n * c / t; i < n * (c + 1) / t; ++i) ++h[(keys[i] >> shift) & 255];
        };
        {
            std::vector<std::thread> ws;
            for (int c = 1; c < t; ++c) ws.emplace_back(count, c);
            count(0);
            for (auto& w : ws) w.join();
        }
        uint64_t run = 0;  // digit-major, then chunk: stable
        for (int d = 0; d < 256; ++d)
            for (int c = 0; c < t; ++c) {
                const uint64_t v = hist[size_t(c) * 256 + d];
                hist[size_t(c) * 256 + d] = run;
                run += v;
            }
        auto scatter = [&](int c) {
            uint64_t* h = hist.data() + size_t(c) * 256;
            for (uint64_t i = n * c / t; i < n * (c + 1) / t; ++i)
                tmp[h[(keys[i] >> shift) & 255]++] = keys[i];
        };
        {
            std::vector<std::thread> ws;
            for (int c = 1; c < t; ++c) ws.emplace_back(scatter, c);
            scatter(0);
            for (auto& w : ws) w.join();
        }
        keys.swap(tmp);
    }
}

struct RmatGraph {
    uint32_t n = 0;
    std::vector<uint64_t> rp;
    std::vector<uint32_t> ci;
};

}  // namespace

extern "C" {

void sgnn_host_fill_uniform(float* out, uint64_t n, double lo, double hi, uint64_t seed,
                            uint64_t stream, int threads) {
    parallel_range(n, threads, [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i)
            out[i] = float(lo + (hi - lo) * u01(counter_hash(seed, stream, i)));
    });
}

void sgnn_host_fill_normal(float* out, uint64_t n, double mean, double std, uint64_t seed,
                           uint64_t stream, int threads) {
    // Box-Muller on the pair (2i, 2i+1) of counter draws.
    parallel_range(n, threads, [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i) {
            const double u1 = u01(counter_hash(seed, stream, 2 * i));
            const double u2 = u01(counter_hash(seed, stream, 2 * i + 1));
            const double r = std::sqrt(-2.0 * std::log(1.0 - u1));
            out[i] = float(mean + std * r * std::cos(6.283185307179586476925286766559 * u2));
        }
    });
}

int sgnn_host_er(uint32_t n_rows, uint32_t n_cols, uint32_t deg, uint64_t seed, uint64_t* rp,
                 uint32_t* ci, int threads) {
    if (deg > n_cols) return 3;
    for (uint64_t i = 0; i <= n_rows; ++i) rp[i] = i * deg;
    parallel_range(n_rows, threads, [&](uint64_t b, uint64_t e) {
        std::vector<uint32_t> row(deg);
        for (uint64_t i = b; i < e; ++i) {
            uint64_t draw = 0;
            uint32_t have = 0;
            while (have < deg) {
                const uint64_t h = counter_hash(seed, i, draw++);
                // unbiased below(n_cols) by rejection, as rng.hpp:48-56
                const uint64_t bound = n_cols;
                const uint64_t limit = ~uint64_t(0) - (~uint64_t(0) % bound + 1) % bound;
                if (h > limit) continue;
                const uint32_t col = uint32_t(h % bound);
                bool dup = false;
                for (uint32_t q = 0; q < have; ++q) dup |= (row[q] == col);
                if (!dup) row[have++] = col;
            }
            std::sort(row.begin(), row.end());
            std::memcpy(ci + i * deg, row.data(), sizeof(uint32_t) * deg);
        }
    });
    return 0;
}

void* sgnn_host_rmat_build(uint32_t scale, uint64_t n_samples, double a, double b, double c,
                           uint64_t seed, int symmetrize, int self_loops, int threads) {
    if (scale == 0 || scale > 31) return nullptr;
    auto* g = new RmatGraph;
    const uint32_t n = 1u << scale;
    g->n = n;
    const uint64_t per = symmetrize ? 2 : 1;
    std::vector<uint64_t> keys(n_samples * per + (self_loops ? n : 0));
    // thresholds in 2^32 units for the quadrant choice
    const uint64_t ta = uint64_t(a * 4294967296.0);
    const uint64_t tb = uint64_t((a + b) * 4294967296.0);
    const uint64_t tc = uint64_t((a + b + c) * 4294967296.0);
    parallel_range(n_samples, threads, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t s = lo; s < hi; ++s) {
            uint64_t row = 0, col = 0, h = 0;
            for (uint32_t lvl = 0; lvl < scale; ++lvl) {
                if ((lvl & 1) == 0) h = counter_hash(seed, 0x524d4154ull, s * 16 + lvl / 2);
                const uint64_t u = (lvl & 1) ? (h >> 32) : (h & 0xffffffffull);
                const uint64_t rb = u >= tb;                       // quadrants c, d
                const uint64_t cb = (u >= ta && u < tb) || u >= tc;  // quadrants b, d
                row = (row << 1) | rb;
                col = (col << 1) | cb;
            }
            keys[s * per] = (row << scale) | col;
            if (symmetrize) keys[s * per + 1] = (col << scale) | row;
        }
    });
    if (self_loops)
        for (uint64_t i = 0; i < n; ++i) keys[n_samples * per + i] = (i << scale) | i;
    radix_sort(keys, 2 * int(scale), threads);
    // unique
    uint64_t m = 0;
    for (uint64_t i = 0; i < keys.size(); ++i)
        if (i == 0 || keys[i] != keys[i - 1]) keys[m++] = keys[i];
    keys.resize(m);
    g->rp.assign(uint64_t(n) + 1, 0);
    g->ci.resize(m);
    for (uint64_t i = 0; i < m; ++i) {
        ++g->rp[(keys[i] >> scale) + 1];
        g->ci[i] = uint32_t(keys[i] & (uint64_t(n) - 1));
    }
    for (uint32_t i = 0; i < n; ++i) g->rp[i + 1] += g->rp[i];
    return g;
}

uint64_t sgnn_host_rmat_nnz(void* h) { return static_cast<RmatGraph*>(h)->ci.size(); }

void sgnn_host_rmat_export(void* h, uint64_t* rp, uint32_t* ci) {
    auto* g = static_cast<RmatGraph*>(h);
    std::memcpy(rp, g->rp.data(), sizeof(uint64_t) * g->rp.size());
    std::memcpy(ci, g->ci.data(), sizeof(uint32_t) * g->ci.size());
}

void sgnn_host_rmat_free(void* h) { delete static_cast<RmatGraph*>(h); }

void sgnn_host_balanced_row_partition(const uint64_t* rp, uint32_t n_rows, int n_chunks,
                                      uint32_t* bounds) {
    // parallel.hpp:28-41: cumulative cost through row i is rp[i] + i.
    for (int c = 0; c <= n_chunks; ++c) bounds[c] = n_rows;
    bounds[0] = 0;
    const uint64_t total = rp[n_rows] + n_rows;
    uint32_t row = 0;
    for (int c = 1; c < n_chunks; ++c) {
        const uint64_t target = total * uint64_t(c) / uint64_t(n_chunks);
        while (row < n_rows && rp[row] + row < target) ++row;
        bounds[c] = row;
    }
}

void sgnn_host_weighted_row_partition(const uint64_t* rp, uint32_t n_rows, int n_chunks, uint32_t row_weight,
                                      uint32_t* bounds) {
    // cost(i) = rp[i] + w * i, monotone in i: bound c is the first row whose
    // cost reaches c/n_chunks of the total (w = 1: balanced_row_partition's
    // rule and result, parallel.hpp:28-41); binary search per bound.
    const uint64_t w = row_weight;
    auto cost = [&](uint32_t i) { return rp[i] + w * uint64_t(i); };
    for (int c = 0; c <= n_chunks; ++c) bounds[c] = n_rows;
    bounds[0] = 0;
    const uint64_t total = cost(n_rows);
    uint32_t lo_row = 0;
    for (int c = 1; c < n_chunks; ++c) {
        const uint64_t target = total * uint64_t(c) / uint64_t(n_chunks);
        uint32_t lo = lo_row, hi = n_rows;  // first i in [lo, n_rows] with cost(i) >= target
        while (lo < hi) {
            const uint32_t mid = lo + (hi - lo) / 2;
            if (cost(mid) < target) lo = mid + 1;
            else hi = mid;
        }
        bounds[c] = lo;
        lo_row = lo;
    }
}

uint64_t sgnn_host_partition_block(const uint64_t* rp, const uint32_t* ci, const float* v,
                                   const uint32_t* bounds, int n_parts, int part, uint32_t stride,
                                   uint64_t* out_rp, uint32_t* out_ci, float* out_v, int threads) {
    const uint32_t r0 = bounds[part], r1 = bounds[part + 1];
    const uint64_t e0 = rp[r0], e1 = rp[r1];
    for (uint32_t r = r0; r <= r1; ++r) out_rp[r - r0] = rp[r] - e0;
    parallel_range(e1 - e0, threads, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t e = lo; e < hi; ++e) {
            const uint32_t c = ci[e0 + e];
            // owner = last q with bounds[q] <= c (n_parts <= a few dozen: linear is fine)
            int q = 0;
            while (q + 1 < n_parts && bounds[q + 1] <= c) ++q;
            out_ci[e] = uint32_t(q) * stride + (c - bounds[q]);
            if (out_v) out_v[e] = v[e0 + e];
        }
    });
    return e1 - e0;
}

}  // extern "C"
