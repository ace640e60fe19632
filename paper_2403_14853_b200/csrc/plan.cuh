// plan.cuh -- the SpMM/FusedMM work decomposition ("plan").
//
// The reference balances CPU threads by contiguous row chunks of equal
// (nnz + rows) cost (parallel.hpp:28-41).  On the B200 the same cost model is
// applied at the granularity of a *worker* (a group of 4..32 lanes): worker w
// owns the cost interval [w*D, (w+1)*D) of the cumulative cost
// cost(r) = row_ptr[r] + r.  A boundary that falls inside a row is snapped to
// the nearer row boundary when the row is short (<= split_rows_over nonzeros),
// and down to a multiple of SGNN_SEGMENT nonzeros from the row start when the
// row is long, so hub rows are spread over many workers while every short row
// is computed by one worker in ascending order.  Segment partials of split
// rows go to a workspace and a fixup pass adds them left to right.
#pragma once

#include <atomic>

#include "common.cuh"

struct sgnn_plan_s {
    // identity of the matrix / width the plan was built for
    const uint64_t* row_ptr = nullptr;
    uint32_t n_rows = 0, n_cols = 0;
    uint64_t nnz = 0;
    uint32_t k = 0;
    sgnn_plan_params p{};
    bool vec = false;       // float4 path chosen (K % 4 == 0)
    uint32_t kt = 0;        // floats of K per pass
    uint64_t split_T = 0;   // rows with more nonzeros than this may be split

    uint32_t n_workers = 0;
    uint32_t n_slots = 0;   // segment partials of split rows (per pass)
    uint32_t n_fix = 0;     // split rows
    uint32_t max_deg = 0;   // longest row (clamped to u32)

    // device arrays (one allocation)
    void* mem = nullptr;
    uint32_t* wrow = nullptr;   // [n_workers+1]
    uint64_t* wnz = nullptr;    // [n_workers+1]
    uint32_t* wslot = nullptr;  // [n_workers+1] exclusive scan of per-worker slot counts
    uint32_t* fix_row = nullptr;   // [n_fix]
    uint32_t* fix_slot = nullptr;  // [n_fix] first slot of the row
    uint32_t* fix_long = nullptr;  // [n_long] split rows with > SGNN_FIXUP_LONG segments
    uint32_t n_long = 0;
    float* slots = nullptr;        // [n_slots * kt]
    void* fmem = nullptr;          // allocation holding fix_row/fix_slot/slots
    // dynamic worker schedule: [0] workers taken past the first round, [1]
    // warps exited; the last warp of a launch zeroes both (plan_counter)
    uint32_t* wctr = nullptr;
    mutable std::atomic<uintptr_t> ctr_owner{0};  // stream key (+1) owning wctr
};

namespace sgnn {

// The dynamic-schedule counter for a launch with `p` on stream `s`, or null
// (static grid-stride schedule).  Launches on one stream are ordered, so the
// counter belongs to the first ordinary stream that launches with the plan;
// other streams, the per-thread default stream and graph captures take the
// static schedule (same results: the schedule only decides which warp runs
// which worker).
uint32_t* plan_counter(const sgnn_plan_s* p, cudaStream_t s);

// Library defaults for (A, K) (used when params fields are 0).
void default_params(const sgnn_csr* a, uint32_t k, bool vec_ok, const DeviceProps& dp,
                    sgnn_plan_params* p);
// Validates/normalises params; fills plan->p, vec, kt, split_T.
sgnn_status resolve_params(const sgnn_csr* a, uint32_t k, bool vec_ok, const DeviceProps& dp,
                           const sgnn_plan_params* in, sgnn_plan_s* plan);
sgnn_status build_plan(const sgnn_csr* a, uint32_t k, const sgnn_plan_params* params, bool vec_ok,
                       sgnn_plan_s** out, cudaStream_t s);
void destroy_plan(sgnn_plan_s* p);
// Does this plan serve (a, k)?
bool plan_matches(const sgnn_plan_s* p, const sgnn_csr* a, uint32_t k);

}  // namespace sgnn
