// One-call multiply: symbolic phase, numeric phase and the norms of C, enqueued back to back on
// one stream with no host round trip (numeric.multiply, pkg/src/spamm/numeric.py:302-313, for the
// beta == 0 case).  Every count the later kernels need (product leaves, step records, super-tile
// nodes) stays in device memory; buffers are sized by capacities and an overflow is flagged in
// plan.counts[2] for the caller to check whenever it first synchronises.
#include "common.cuh"

int spamm_index_leaves_impl(const uint32_t *keys, const double *leaf_sq_packed, int64_t nleaf, const int32_t *nleaf_dev,
                            int depth, int32_t *slot, int32_t *slot_t, float *norm, float *norm_t, double *leaf_sq_grid,
                            cudaStream_t st);

extern "C" int spamm_multiply(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int granularity, int exact,
                              float alpha, int32_t row0, int32_t row1, const spamm_plan_buffers *plan, void *plan_ws,
                              size_t plan_ws_bytes, const spamm_product_buffers *c, unsigned long long *counters,
                              void *stream)
{
    if (!a || !b || !plan || !c || !counters) return SPAMM_EINVAL;
    int rc = spamm_plan(a, b, tau, row0, row1, plan, plan_ws, plan_ws_bytes, stream);
    if (rc != SPAMM_OK) return rc;
    rc = spamm_execute(a, b, plan, -1, -1, tau, alpha, granularity, exact, c->values, c->values_t, c->leaf_sq, counters,
                       stream);
    if (rc != SPAMM_OK) return rc;
    // C's tree: leaf grids from the packed product leaves (their count is plan.counts[0]), then the
    // interior norms -- compute_norms, numeric.py:179 / core.py:331-345
    rc = spamm_index_leaves_impl(plan->c_keys, c->leaf_sq, plan->leaf_capacity, plan->counts, c->depth, c->slot, c->slot_t,
                                 c->norm, c->norm_t, c->leaf_sq_grid, (cudaStream_t)stream);
    if (rc != SPAMM_OK) return rc;
    return spamm_build_interior(c->leaf_sq_grid, c->depth, c->norm, c->norm_t, c->sq_levels, 0, stream);
}
