// One-call multiply: symbolic phase, numeric phase and the norms of C, enqueued back to back on
// one stream with no host round trip (numeric.multiply, pkg/src/spamm/numeric.py:302-313, for the
// beta == 0 case).  Every count the later kernels need (product leaves, step records, super-tile
// nodes) stays in device memory; buffers are sized by capacities and an overflow is flagged in
// plan.counts[2] for the caller to check whenever it first synchronises.
#include <stdlib.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"

int spamm_plan_impl(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int32_t row0, int32_t row1,
                    const spamm_plan_buffers *out, void *ws, size_t ws_bytes, bool prezeroed,
                    const spamm_product_buffers *cgrid, uint32_t **clean_ptr, int *clean_words, int fine_weight,
                    void *stream);
size_t spamm_plan_zero_bytes(int64_t step_capacity, int64_t leaf_capacity);
int spamm_launch_interior(const double *leaf_sq, int depth, float *norm, float *norm_t, double *sq_levels,
                          unsigned int *ticket, cudaStream_t st);
int spamm_execute_impl(const spamm_tree_view *a, const spamm_tree_view *b, const spamm_plan_buffers *plan,
                       int64_t nsteps, int64_t nC, double tau, float alpha, int granularity, int exact,
                       float *c_values, float *c_values_t, double *c_leaf_sq, unsigned long long *counters,
                       const spamm_product_buffers *cgrid, uint32_t *clean_ptr, int clean_words, void *stream,
                       unsigned long long *gates = nullptr);

static int multiply_impl(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int granularity, int exact,
                         float alpha, int32_t row0, int32_t row1, const spamm_plan_buffers *plan, void *plan_ws,
                         size_t plan_ws_bytes, const spamm_product_buffers *c, const spamm_host_operands *host, void *stream)
{
    if (!a || !b || !plan || !c) return SPAMM_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    // Four kernels, no memset: plan count (which also empties C's leaf grids), plan emit (records, pieces,
    // counts), execute, interior norms; deep trees: root / expand / tiles / order in place of the first two.
    if (!plan_ws) return SPAMM_EWORKSPACE;
    // The planner needs a prefix of its workspace zero and leaves it zero; behind the prefix lie scratch lists.
    // How long the prefix is depends on the capacities: when they grow from one multiply to the next on the
    // same workspace, the part of the new prefix that was scratch before is cleared here (stream-ordered).
    {
        static std::mutex mu;
        static std::unordered_map<const void *, size_t> prefix;      // workspace -> zero prefix of its last multiply
        const size_t zb = spamm_plan_zero_bytes(plan->step_capacity, plan->leaf_capacity);
        if (zb > plan_ws_bytes) return SPAMM_EWORKSPACE;
        std::lock_guard<std::mutex> lock(mu);
        auto it = prefix.find(plan_ws);
        if (it != prefix.end() && zb > it->second &&
            cudaMemsetAsync(static_cast<char *>(plan_ws) + it->second, 0, zb - it->second, st) != cudaSuccess)
            return SPAMM_ECUDA;
        prefix[plan_ws] = zb;
    }
    static const int stop = getenv("SPAMM_PIPE_STOP") ? atoi(getenv("SPAMM_PIPE_STOP")) : 0;   // tuning aid: truncate
    uint32_t *clean_ptr = nullptr;      // planner state the numeric kernel returns to zero
    int clean_words = 0;
    int rc = spamm_plan_impl(a, b, tau, row0, row1, plan, plan_ws, plan_ws_bytes, true, c, stop == 2 ? nullptr : &clean_ptr,
                             stop == 2 ? nullptr : &clean_words, granularity == SPAMM_FINE4 ? 1 : 0, stream);
    if (rc != SPAMM_OK || stop == 2) return rc;
    if (host) {
        // operands whose leaf values are still in host memory: mark the leaves the plan reads and let the GPU
        // fetch their blocks (the left operand is read through values_t, the right one through values)
        const bool same = host->b_blocks == nullptr || (host->b_blocks == host->a_blocks && host->b_flags == host->a_flags);
        if (!host->a_blocks || !host->a_flags || (!same && !host->b_flags)) return SPAMM_EINVAL;
        unsigned char *fb = same ? host->a_flags : host->b_flags;
        if (cudaMemsetAsync(host->a_flags, 0, (size_t)host->a_nleaf, st) != cudaSuccess) return SPAMM_ECUDA;
        if (!same && cudaMemsetAsync(fb, 0, (size_t)host->b_nleaf, st) != cudaSuccess) return SPAMM_ECUDA;
        if (host->fetched && cudaMemsetAsync(host->fetched, 0, 16, st) != cudaSuccess) return SPAMM_ECUDA;
        rc = spamm_mark_touched(plan, host->a_flags, fb, stream);
        if (rc != SPAMM_OK) return rc;
        if (same) {
            rc = spamm_gather_blocks(host->a_blocks, host->a_flags, host->a_nleaf, 3, const_cast<float *>(a->values),
                                     const_cast<float *>(a->values_t), host->fetched, stream);
        } else {
            rc = spamm_gather_blocks(host->a_blocks, host->a_flags, host->a_nleaf, 2, nullptr, const_cast<float *>(a->values_t),
                                     host->fetched, stream);
            if (rc == SPAMM_OK)
                rc = spamm_gather_blocks(host->b_blocks, fb, host->b_nleaf, 1, const_cast<float *>(b->values), nullptr,
                                         host->fetched ? host->fetched + 1 : nullptr, stream);
        }
        if (rc != SPAMM_OK) return rc;
    }
    // executed micro products are counted in plan->counts[8..9]
    rc = spamm_execute_impl(a, b, plan, -1, -1, tau, alpha, granularity, exact, c->values, c->values_t, c->leaf_sq,
                            reinterpret_cast<unsigned long long *>(plan->counts + 8), c, clean_ptr, clean_words, stream);
    if (rc != SPAMM_OK || stop == 3) return rc;
    // interior norms of C: compute_norms, numeric.py:179 / core.py:331-345
    return spamm_launch_interior(c->leaf_sq_grid, c->depth, c->norm, c->norm_t, c->sq_levels,
                                 reinterpret_cast<unsigned int *>(plan->counts + 10), st);
}

extern "C" int spamm_multiply(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int granularity, int exact,
                              float alpha, int32_t row0, int32_t row1, const spamm_plan_buffers *plan, void *plan_ws,
                              size_t plan_ws_bytes, const spamm_product_buffers *c, void *stream)
{
    return multiply_impl(a, b, tau, granularity, exact, alpha, row0, row1, plan, plan_ws, plan_ws_bytes, c, nullptr, stream);
}

extern "C" int spamm_multiply_host(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int granularity, int exact,
                                   float alpha, int32_t row0, int32_t row1, const spamm_plan_buffers *plan, void *plan_ws,
                                   size_t plan_ws_bytes, const spamm_product_buffers *c, const spamm_host_operands *host,
                                   void *stream)
{
    if (!host) return SPAMM_EINVAL;
    return multiply_impl(a, b, tau, granularity, exact, alpha, row0, row1, plan, plan_ws, plan_ws_bytes, c, host, stream);
}

// ---- the same on ONE caller-provided allocation ------------------------------------------------
static inline int64_t arena_take(int64_t &o, int64_t bytes)
{
    const int64_t at = o;
    o = (o + bytes + 255) / 256 * 256;
    return at;
}

extern "C" int spamm_multiply_arena_layout(int depth, int c_depth, int64_t step_capacity, int64_t leaf_capacity,
                                           spamm_arena_layout *out)
{
    if (!out || depth < 0 || depth > 15 || c_depth < 0 || c_depth > 15 || step_capacity < 1 || leaf_capacity < 1)
        return SPAMM_EINVAL;
    const int64_t cells = int64_t(1) << (2 * c_depth);
    const int64_t total = spamm_level_offset(c_depth) + cells;
    int64_t o = 0;
    out->counts = arena_take(o, SPAMM_PLAN_COUNTS * 4);
    out->steps = arena_take(o, step_capacity * (int64_t)sizeof(spamm_step));
    out->c_keys = arena_take(o, leaf_capacity * 4);
    out->tile_off = arena_take(o, (leaf_capacity + 1) * 4);
    out->tile_order = arena_take(o, (2 * leaf_capacity + SPAMM_UNIT_EXTRA) * 4);   // units, then the chain flags
    out->chain = out->tile_order + (leaf_capacity + SPAMM_UNIT_EXTRA) * 4;
    out->plan_ws_bytes = (int64_t)spamm_plan_workspace_bytes(depth, step_capacity, leaf_capacity);   // not in the arena
    out->values = arena_take(o, leaf_capacity * SPAMM_REC_BYTES);
    out->values_t = arena_take(o, leaf_capacity * SPAMM_REC_BYTES);
    out->leaf_sq = arena_take(o, leaf_capacity * 8);
    out->slot = arena_take(o, cells * 4);
    out->slot_t = arena_take(o, cells * 4);
    out->norm = arena_take(o, total * 4);
    out->norm_t = arena_take(o, total * 4);
    out->leaf_sq_grid = arena_take(o, cells * 8);
    out->sq_levels = arena_take(o, total * 8);
    out->total = o;
    return SPAMM_OK;
}

static int multiply_arena_impl(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int granularity,
                               int exact, float alpha, int32_t row0, int32_t row1, int c_depth, int64_t step_capacity,
                               int64_t leaf_capacity, void *arena, size_t arena_bytes, void *plan_ws,
                               size_t plan_ws_bytes, const spamm_host_operands *host, void *stream)
{
    if (!a || !b || !arena || !plan_ws) return SPAMM_EINVAL;
    spamm_arena_layout l;
    int rc = spamm_multiply_arena_layout(a->depth, c_depth, step_capacity, leaf_capacity, &l);
    if (rc != SPAMM_OK) return rc;
    if ((int64_t)arena_bytes < l.total || (int64_t)plan_ws_bytes < l.plan_ws_bytes) return SPAMM_EWORKSPACE;
    char *p = reinterpret_cast<char *>(arena);
    spamm_plan_buffers plan;
    plan.steps = reinterpret_cast<spamm_step *>(p + l.steps);
    plan.c_keys = reinterpret_cast<uint32_t *>(p + l.c_keys);
    plan.tile_off = reinterpret_cast<int32_t *>(p + l.tile_off);
    plan.tile_order = reinterpret_cast<int32_t *>(p + l.tile_order);
    plan.chain = reinterpret_cast<int32_t *>(p + l.chain);
    plan.step_capacity = step_capacity;
    plan.leaf_capacity = leaf_capacity;
    plan.counts = reinterpret_cast<int32_t *>(p + l.counts);
    spamm_product_buffers c;
    c.values = reinterpret_cast<float *>(p + l.values);
    c.values_t = reinterpret_cast<float *>(p + l.values_t);
    c.leaf_sq = reinterpret_cast<double *>(p + l.leaf_sq);
    c.slot = reinterpret_cast<int32_t *>(p + l.slot);
    c.slot_t = reinterpret_cast<int32_t *>(p + l.slot_t);
    c.norm = reinterpret_cast<float *>(p + l.norm);
    c.norm_t = reinterpret_cast<float *>(p + l.norm_t);
    c.leaf_sq_grid = reinterpret_cast<double *>(p + l.leaf_sq_grid);
    c.sq_levels = reinterpret_cast<double *>(p + l.sq_levels);
    c.depth = c_depth;
    return multiply_impl(a, b, tau, granularity, exact, alpha, row0, row1, &plan, plan_ws, plan_ws_bytes, &c, host, stream);
}

extern "C" int spamm_multiply_arena(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int granularity,
                                    int exact, float alpha, int32_t row0, int32_t row1, int c_depth, int64_t step_capacity,
                                    int64_t leaf_capacity, void *arena, size_t arena_bytes, void *plan_ws,
                                    size_t plan_ws_bytes, void *stream)
{
    return multiply_arena_impl(a, b, tau, granularity, exact, alpha, row0, row1, c_depth, step_capacity, leaf_capacity, arena,
                               arena_bytes, plan_ws, plan_ws_bytes, nullptr, stream);
}

extern "C" int spamm_multiply_arena_host(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int granularity,
                                         int exact, float alpha, int32_t row0, int32_t row1, int c_depth,
                                         int64_t step_capacity, int64_t leaf_capacity, void *arena, size_t arena_bytes,
                                         void *plan_ws, size_t plan_ws_bytes, const spamm_host_operands *host, void *stream)
{
    if (!host) return SPAMM_EINVAL;
    return multiply_arena_impl(a, b, tau, granularity, exact, alpha, row0, row1, c_depth, step_capacity, leaf_capacity, arena,
                               arena_bytes, plan_ws, plan_ws_bytes, host, stream);
}
