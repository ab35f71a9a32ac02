/*
 * spamm_b200.h -- C ABI of the B200 SpAMM multiply path.
 *
 * The reference (`spamm` v0.1.0, pure Python) has no FFI layer; its boundary for
 * this path is the Python API `multiply / build_plan / execute_plan`
 * (pkg/src/spamm/numeric.py:302-313, symbolic.py:151-159, numeric.py:138-151)
 * on `QuadtreeMatrix` operands (core.py:146-405).  The Python package
 * `paper_1203_1692_b200` re-implements that API and calls the entry points below
 * through ctypes; INTEGRATION.md shows the stub a maintainer of the reference
 * would add.  Every function:
 *   - takes raw DEVICE pointers, sizes and a cudaStream_t (as void*),
 *   - is stream-ordered, never allocates and never synchronises (the env-gated tuning traces
 *     SPAMM_EX_TRACE / SPAMM_PLAN_TRACE do both; they are diagnostics, off by default),
 *   - returns 0 on success, a SPAMM_E* code otherwise (spamm_error_string()).
 * Counts that the host needs (leaves, tasks) are written to device memory; the
 * caller decides when to read them back.
 *
 * Sizes: n_b = 16 (core.py:21).  A tree of depth d has a leaf grid of side
 * L = 2^d.  Level t (0 = root .. d = leaves) is a 2^t x 2^t row-major grid that
 * starts at element spamm_level_offset(t) of a level buffer (levels packed root first,
 * each start rounded up to 4 elements).
 */
#ifndef SPAMM_B200_H
#define SPAMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPAMM_ABI_VERSION 2

enum {
    SPAMM_OK = 0,
    SPAMM_EINVAL = 1,      /* bad argument (-> ValueError on the Python side) */
    SPAMM_ECUDA = 2,       /* CUDA runtime error (-> RuntimeError)            */
    SPAMM_EWORKSPACE = 3   /* workspace too small                             */
};

enum { SPAMM_FINE4 = 0, SPAMM_COARSE16 = 1 };        /* numeric.py:26 GRANULARITIES   */
enum { SPAMM_ORDER_DENSE = 0, SPAMM_ORDER_REFRESH = 1 }; /* leaf sum order, see below */
enum { SPAMM_EXEC_FMA = 0, SPAMM_EXEC_EXACT = 1 };   /* EXACT: separate mul/add rounding */

/* Device view of one QuadtreeMatrix (core.py:146-167, :387-405).  All pointers
 * are device pointers owned by the caller.
 *   keys      [nleaf]       Morton key of each stored leaf, ascending (packed_leaves()[0])
 *   values    [nleaf][272]  row-major 16x16 leaf values (packed_leaves()[1]) followed by the
 *                           16 sub-block norms transposed, tail[q*4+r] = sub[r][q]
 *   values_t  [nleaf][272]  the leaf transposed (the A-operand staging layout) followed by
 *                           the sub-block norms row-major, tail[p*4+r]  (packed_leaves()[2])
 *   slot      [L*L]         leaf (i,j) -> index into the packed arrays, -1 = absent
 *   slot_t    [L*L]         transposed grid: (j,i) -> index
 *   norm      level buffer  node norms, -1 = absent node        (TreeNode.norm, core.py:138-143)
 *   norm_t    level buffer  every level's grid transposed
 *   sub       [L*L]         optional (may be NULL): per leaf the range of its 16 sub-block norms,
 *                           bf16(max) rounded up << 16 | bf16(min) rounded down, 0xFFFFFFFF = absent
 *                           or not finite (spamm_subrange_grids); lets the planner classify the
 *                           tasks whose 64 gated micro products (numeric.py:233-238) all pass or all fail
 *   sub_t     [L*L]         the same grid transposed
 */
typedef struct {
    int32_t m, n;           /* logical size */
    int32_t depth;          /* leaf level; grids have side 1 << depth */
    int32_t nleaf;          /* stored leaves (host copy) */
    const uint32_t *keys;
    const float *values;
    const float *values_t;
    const int32_t *slot;
    const int32_t *slot_t;
    const float *norm;
    const float *norm_t;
    const uint32_t *sub;
    const uint32_t *sub_t;
} spamm_tree_view;

int spamm_abi_version(void);
int64_t spamm_level_offset_of(int t);      /* t == 0 ? 0 : 4 + (4^t - 4)/3 */
const char *spamm_error_string(int code);
/* Number of kernels launched by this library since load (for bench.py's gpu_launches). */
int64_t spamm_launch_count(void);

/* ---- tree construction: QuadtreeMatrix.from_dense (core.py:213-266) -------- */

/* Leaf pass over a dense row-major m x n matrix (row stride ld, in floats):
 * per leaf of the 2^depth grid the 16 sub-block norms, the double square sum and
 * the leaf norm (-1 where the leaf is all zero or outside the matrix).
 * sub4_grid [L*L][16], leaf_sq [L*L], leaf_norm [L*L].  Replaces core.py:225-233. */
int spamm_leaf_norms_dense(const float *dense, int64_t m, int64_t n, int64_t ld, int depth,
                           float *sub4_grid, double *leaf_sq, float *leaf_norm, void *stream);

/* Stored leaves in ascending Morton order (core.py:235-237): slot/slot_t grids, keys,
 * and the leaf count in *nleaf_dev.  ws: spamm_scan_workspace_bytes(L*L) bytes. */
size_t spamm_scan_workspace_bytes(int64_t n);
int spamm_assign_slots(const float *leaf_norm, int depth, int32_t *slot, int32_t *slot_t,
                       uint32_t *keys, int32_t *nleaf_dev, void *ws, size_t ws_bytes, void *stream);

/* Copy the stored leaves out of the dense matrix (core.py:239-248): values, values_t records.
 * nleaf is the host copy of *nleaf_dev. */
int spamm_pack_leaves(const float *dense, int64_t m, int64_t n, int64_t ld, int depth,
                      const uint32_t *keys, int64_t nleaf, const float *sub4_grid,
                      float *values, float *values_t, void *stream);

/* Interior norms (_build_interior, core.py:252-266): fills levels 0..depth-1 of norm / norm_t
 * and sq_levels from the leaf level.  leaf_sq is the L*L grid of double square sums; the leaf
 * level of `norm` must be in place (-1 = absent); when write_leaf_transpose != 0 the leaf level
 * of norm_t is written from it as well. */
int spamm_build_interior(const double *leaf_sq, int depth, float *norm, float *norm_t,
                         double *sq_levels, int write_leaf_transpose, void *stream);

/* ---- trees given as packed leaves: put_leaf + compute_norms (core.py:315-345) */

/* Leaf norms of packed leaves, in the order compute_norms uses (core.py:108-116): fills the
 * sub-norm tails of the `values` records, the whole `values_t` records and leaf_sq [nleaf]. */
int spamm_leaf_norms_packed(float *values, int64_t nleaf, float *values_t, double *leaf_sq,
                            void *stream);

/* The same from plain leaf blocks: `blocks` holds nleaf row-major 16x16 blocks (256 floats each, the
 * value array of the reference's packed_leaves(), core.py:387-405); writes the whole `values` and
 * `values_t` records and leaf_sq [nleaf].  All pointers are device pointers. */
int spamm_leaves_from_blocks(const float *blocks, int64_t nleaf, float *values, float *values_t,
                             double *leaf_sq, void *stream);

/* QuadtreeMatrix.sparsify (core.py:347-383) on packed leaves: zeroes every 4x4 sub-block with
 * 0 < sub-norm < eps in both record layouts, refreshes the norms of the leaves it touched
 * (compute_norms order) and sets leaf_sq of the untouched ones to float64(norm)^2, the value the
 * reference feeds to the interior sums.  *dropped += zeroed sub-blocks.  Leaves left with
 * leaf_sq == 0 are to be removed by the caller before re-indexing. */
int spamm_sparsify_leaves(float *values, float *values_t, double *leaf_sq, int64_t nleaf, float eps,
                          unsigned long long *dropped, void *stream);

/* values_t records from values records whose sub-norm tails are already filled (leaves received
 * from another GPU keep the norms their owner computed): transposition only. */
int spamm_transpose_records(const float *values, int64_t nleaf, float *values_t, void *stream);

/* Scatter packed leaves (keys, leaf_sq; a key of 0xFFFFFFFF marks an unused slot and is skipped,
 * as in a shard gathered from several GPUs) into the grids of a depth-`depth` tree:
 * slot, slot_t, the leaf level of norm/norm_t and the double leaf_sq grid (all L*L). */
int spamm_index_leaves(const uint32_t *keys, const double *leaf_sq_packed, int64_t nleaf, int depth,
                       int32_t *slot, int32_t *slot_t, float *norm, float *norm_t,
                       double *leaf_sq_grid, void *stream);

/* Sub-norm range grids of a tree (see spamm_tree_view.sub): from the sub-norm tails of the `values`
 * records through the slot grid at `depth`. */
int spamm_subrange_grids(const float *values, const int32_t *slot, int depth, uint32_t *sub,
                         uint32_t *sub_t, void *stream);

/* QuadtreeMatrix.to_dense (core.py:268-276): out is m x n, row stride ld, fully written. */
int spamm_to_dense(const spamm_tree_view *t, float *out, int64_t ld, void *stream);

/* ---- symbolic phase: build_plan (symbolic.py:92-159) --------------------------- */

/* The compacted task list.  Leaves are grouped in aligned 4x4 blocks (16 consecutive Morton
 * keys, contiguous in the packed arrays).  For every super-tile (I,J) of product leaves and,
 * in ascending order, every block index K with at least one surviving task, the plan holds
 * one 64-byte step record: the block product C[I,J] += A[I,K] B[K,J] restricted to its live
 * leaf tasks.  Bit pos = morton4(di,dj) of live[kk] stands for the task
 * (i,k,j) = (4I+di, 4K+kk, 4J+dj); tasks of one product leaf therefore appear in ascending k,
 * the only order the numeric phase depends on (numeric.py:203-217).  The records of a
 * super-tile are contiguous, super-tiles ascend in Morton order.  Leaf (r,c) of a block sits
 * at packed index first + popcount(present16 & ((1 << morton4(r,c)) - 1)). */
#define STEP_FIRST (1u << 16)   /* first record of its super-tile */
#define STEP_LAST (1u << 17)    /* last record of its super-tile  */
/* Work units of the numeric phase (tile_order).  A unit is a run [b, e) of consecutive step
 * records, stored as four ints (b, tb, ts, e): tb = end of the super-tile record b lies in (b
 * itself when b starts a tile), ts = start of the tile record e - 1 lies in (e itself when e
 * ends one).  The numeric kernel runs two teams of warps per SM; the planner cuts the record stream into counts[12] pieces of equal weight (live tasks plus a constant
 * per record), a whole number of rounds of one piece per team: units [0, counts[12]).  A piece may
 * begin and end inside a super-tile; the kernel then runs the head of the tile it begins at its
 * end first, its whole tiles next and the rest of the tile it starts in last, so that a piece never
 * waits long for the piece before it.  Only a plan with fewer than three records per team gets a
 * second region: its last quarter is cut into short segments of single tiles, five ranges of
 * counts[16..20] units at unit index counts[12] + x * counts[21], handed out after the pieces.  The
 * accumulators of a tile pass from one unit to the next through C's own value records; chain[]
 * holds, per product leaf, the record index up to which the sums there are complete, which keeps
 * the ascending-k summation order.  Word 15 of a step record = records of its tile | position of
 * the record in the tile << 16. */
#define SPAMM_UNIT_EXTRA 8192   /* room in tile_order beyond one unit per super-tile */
typedef struct {
    uint32_t kblock;       /* K: contraction block index, k = 4K + kk                      */
    uint32_t flags;        /* STEP_FIRST, STEP_LAST                                        */
    uint32_t c_base;       /* packed index of the super-tile's first product leaf          */
    uint32_t tile;         /* Morton index of the super-tile (product leaf key >> 4)       */
    uint32_t a_first;      /* packed index of the first stored leaf of block A[I,K]        */
    uint32_t a_present;    /* its stored leaves, bit morton4(di,kk)                        */
    uint32_t b_first;      /* packed index of the first stored leaf of block B[K,J]        */
    uint32_t b_present;    /* its stored leaves, bit morton4(kk,dj)                        */
    uint32_t live[4];      /* bits 0..15: live tasks of k = 4K + kk, bit morton4(di,dj);
                              bits 16..31: those of them whose 64 gated micro products all
                              pass (fine4, numeric.py:233-238), known from the sub-norm ranges */
    uint32_t present;      /* product leaves of the super-tile (same bit numbering)        */
    uint32_t dead[2];      /* live tasks of which NO gated micro product passes: kk = 0, 1
                              in the halves of dead[0], kk = 2, 3 in dead[1]; a task in
                              neither set is gated per micro product by the numeric kernel
                              (all zero when the operands carry no sub-norm ranges)         */
    uint32_t tile_pos;     /* records of this super-tile | position of this record in it << 16 */
} spamm_step;

/* counts[]: [0] product leaves nC, [1] super-tiles with at least one task,
 * [2] overflow flag, [3] largest intermediate list, [4] step records, [5] unit slots used in
 * tile_order, [6..7] tasks T as one uint64, [8..9] executed 4x4x4 products as one uint64
 * (spamm_multiply only), [10] scratch, [11] all super-tile nodes (tile_off has one more entry),
 * [12] pieces, [16..20] units in the five ranges of short segments and [21] the stride between
 * the ranges (see "work units" above), [13..14] the numeric kernel's hand-out and exit counters
 * when it is launched by spamm_execute (zero between launches), [15] set by the numeric kernel if a
 * wait for a chained unit ever gives up (a scheduling bug, never in a correct run): results invalid */
#define SPAMM_PLAN_COUNTS 32
typedef struct {
    spamm_step *steps;       /* [step_capacity]                                   */
    uint32_t *c_keys;        /* [leaf_capacity] product leaf keys, ascending      */
    int32_t *tile_off;       /* [leaf_capacity + 1] first step of each super-tile node */
    int32_t *tile_order;     /* [leaf_capacity + SPAMM_UNIT_EXTRA] work units, four words each, 16-byte aligned */
    int32_t *chain;          /* [leaf_capacity] hand-over state per product leaf (numeric phase scratch, zero between launches) */
    int64_t step_capacity;
    int64_t leaf_capacity;
    int32_t *counts;         /* [SPAMM_PLAN_COUNTS]                               */
} spamm_plan_buffers;

size_t spamm_plan_workspace_bytes(int depth, int64_t step_capacity, int64_t leaf_capacity);

/* Task set { (i,k,j) : both leaves stored, double(normA) * double(normB) >= tau }
 * (symbolic.py:118-125), produced by a top-down walk of the two norm pyramids.  Both views
 * must be indexed at the same depth (the caller re-indexes a shallower tree); [row0,row1)
 * limits the product to those rows of leaves (row blocks of the multi-GPU split).  When
 * counts[2] is set a capacity was too small and the buffers are incomplete. */
int spamm_plan(const spamm_tree_view *a, const spamm_tree_view *b, double tau,
               int32_t row0, int32_t row1, const spamm_plan_buffers *out,
               void *ws, size_t ws_bytes, void *stream);

/* Surviving tasks per row of product leaves, row_tasks [1 << depth] (zeroed by the call): the
 * quantity the multi-GPU split balances when it hands row blocks of C to the ranks. */
int spamm_plan_row_counts(const spamm_plan_buffers *plan, int depth, int32_t *row_tasks, void *stream);

/* ---- numeric phase: execute_plan (numeric.py:138-284) ------------------------- */

/* Runs every task of the plan: C leaf = alpha32 * sum_k gate(A_ik B_kj), accumulated in
 * ascending k in FP32 -- fused multiply-add, or separately rounded multiply and add when
 * exact != 0 (bit-identical to numeric.py:252-259).  With SPAMM_FINE4 each 4x4x4 micro product
 * (p,q,r) runs iff double(subA[p][r]) * double(subB[r][q]) >= tau (numeric.py:232-238), with
 * SPAMM_COARSE16 all 64 run.  Outputs for product leaf x (plan order): the 272-float records
 * c_values[x] / c_values_t[x] (values + sub-norms, see spamm_tree_view) and c_leaf_sq[x], the
 * norms in compute_norms order (core.py:108-116).  counters[0] += executed micro products.
 * nsteps and nC are the host copies of counts[4] and counts[0]. */
int spamm_execute(const spamm_tree_view *a, const spamm_tree_view *b,
                  const spamm_plan_buffers *plan, int64_t nsteps, int64_t nC,
                  double tau, float alpha, int granularity, int exact,
                  float *c_values, float *c_values_t, double *c_leaf_sq,
                  unsigned long long *counters, void *stream);

/* spamm_execute (fine4, fused multiply-add, alpha = 1) that also reports the gate the kernel itself
 * evaluated: gates[record * 64 + kk * 16 + morton4(di,dj)] receives bit r*16 + p*4 + q for every
 * 4x4x4 micro product (p,q,r) of that task that ran (numeric.py:233-238).  gates holds 64 words per
 * step record and must be zero when the call is enqueued.  Evidence for the parity tests. */
int spamm_execute_gates(const spamm_tree_view *a, const spamm_tree_view *b,
                        const spamm_plan_buffers *plan, int64_t nsteps, int64_t nC, double tau,
                        float *c_values, float *c_values_t, double *c_leaf_sq,
                        unsigned long long *counters, unsigned long long *gates, void *stream);

/* Leaf set of C for beta != 0: the union of the accumulator's stored leaves (slot_old, an L*L
 * grid) and the produced leaves (prod_keys, ascending), in ascending Morton order.  For output
 * leaf x: out_keys[x], and the packed index of the leaf on either side (idx_old / idx_prod, -1
 * when absent).  slot_prod_scratch is an L*L int32 scratch grid; ws as for spamm_assign_slots. */
int spamm_union_leaves(const int32_t *slot_old, const uint32_t *prod_keys, int64_t nprod, int depth,
                       int32_t *slot_prod_scratch, uint32_t *out_keys, int32_t *idx_old,
                       int32_t *idx_prod, int32_t *nout_dev, void *ws, size_t ws_bytes, void *stream);

/* ---- operands whose leaf values stay in host memory ----------------------------------
 * The reference's trees live on the host (core.py:146-405).  For one product only the leaves that
 * occur in a surviving task are needed on the device -- 28 % of config 2's at tau = 1e-8.  With the
 * keys, leaf norms and sub-block norms on the device (a few MB) the symbolic phase runs first; these
 * three calls then bring in exactly the values the numeric phase will read, fetched by the GPU from
 * pinned (device-readable) host memory. */

/* Sub-norm tails of the leaf records from the reference's sub-norm array subs [nleaf][4][4]
 * (core.py:387-405; device pointer): values (tail transposed) and / or values_t (tail row-major). */
int spamm_subnorm_tails(const float *subs, int64_t nleaf, float *values, float *values_t, void *stream);

/* flags_a[x] = 1 / flags_b[x] = 1 for every packed leaf x of the left / right operand that a live
 * task of the plan reads.  The arrays (one byte per leaf) must be zero on entry and may be the same
 * array when both operands are one tree. */
int spamm_mark_touched(const spamm_plan_buffers *plan, unsigned char *flags_a, unsigned char *flags_b,
                       void *stream);

/* For every flagged leaf: its row-major 16x16 block blocks[leaf*256 ..] -- pinned host memory the
 * device can read, or device memory -- into the record of `values` (want & 1) and / or transposed
 * into that of `values_t` (want & 2).  *copied (optional, device) += leaves fetched. */
int spamm_gather_blocks(const float *blocks, const unsigned char *flags, int64_t nleaf, int want,
                        float *values, float *values_t, unsigned long long *copied, void *stream);

/* ---- one call: multiply (numeric.py:302-313), beta == 0 ---------------------------- */

/* Storage of the product tree, sized by the plan's leaf_capacity (packed arrays) and by the
 * depth of C (grids and level buffers, see spamm_tree_view). */
typedef struct {
    float *values;           /* [leaf_capacity][272] */
    float *values_t;         /* [leaf_capacity][272] */
    double *leaf_sq;         /* [leaf_capacity]      */
    int32_t *slot;           /* [L*L] */
    int32_t *slot_t;         /* [L*L] */
    float *norm;             /* level buffer */
    float *norm_t;           /* level buffer */
    double *leaf_sq_grid;    /* [L*L] */
    double *sq_levels;       /* level buffer (scratch) */
    int32_t depth;
} spamm_product_buffers;

/* build_plan + execute_plan + compute_norms on C, enqueued back to back on `stream` with no
 * host synchronisation: C = alpha32 * sum of the surviving leaf products.  The product leaves
 * are plan->c_keys[0 .. counts[0]) with their records in c->values / c->values_t; the number of
 * executed micro products (ExecCounters.products4) is left in counts[8..9] (set afresh by every call).  The caller
 * reads plan->counts when it next synchronises; counts[2] != 0 means a capacity was too small
 * (nothing was computed) and the call must be repeated with larger buffers.
 * plan_ws (spamm_plan_workspace_bytes() bytes) must be ALL ZERO when it is first used: clear it once
 * after allocating it, then reuse it for every multiply on the same stream (one workspace per
 * stream).  The planner keeps the prefix it relies on zero from one multiply to the next, so the
 * four kernels of a multiply run without any memset; only when the capacities GROW between two
 * multiplies on the same workspace does the call clear the part of the longer prefix that was
 * scratch before (one small stream-ordered memset). */
int spamm_multiply(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int granularity,
                   int exact, float alpha, int32_t row0, int32_t row1,
                   const spamm_plan_buffers *plan, void *plan_ws, size_t plan_ws_bytes,
                   const spamm_product_buffers *c, void *stream);

/* The same on ONE caller-provided device allocation: spamm_multiply_arena_layout() gives the byte
 * offset of every buffer of the plan and of the product (fields named as in spamm_plan_buffers /
 * spamm_product_buffers) and the total size; spamm_multiply_arena() carves `arena` that way and
 * runs spamm_multiply.  One allocation and one call per product on the host side; the planner's
 * workspace (plan_ws_bytes of the layout, zero-initialised, see spamm_multiply) is shared by all
 * products of a stream and therefore not part of the arena. */
typedef struct {
    int64_t counts, steps, c_keys, tile_off, tile_order, chain, plan_ws_bytes;   /* plan_ws_bytes: size of the separate workspace */
    int64_t values, values_t, leaf_sq, slot, slot_t, norm, norm_t, leaf_sq_grid, sq_levels;
    int64_t total;
} spamm_arena_layout;
int spamm_multiply_arena_layout(int depth, int c_depth, int64_t step_capacity, int64_t leaf_capacity,
                                spamm_arena_layout *out);

/* The one-call multiply for operands whose leaf VALUES are still in host memory (see "operands whose
 * leaf values stay in host memory" above): between the symbolic and the numeric phase the leaves
 * the plan reads are marked and their blocks fetched by the GPU -- the left operand's into
 * a->values_t, the right one's into b->values; one tree as both operands (b_blocks NULL or the same
 * pointers): into both of its layouts.  a_blocks / b_blocks: [nleaf][256] floats in pinned,
 * device-readable host memory (or device memory); a_flags / b_flags: [nleaf] bytes of device
 * scratch; fetched (optional, device): [2] counts of leaves fetched (left, right).  Still no host
 * synchronisation. */
typedef struct {
    const float *a_blocks;
    int64_t a_nleaf;
    unsigned char *a_flags;
    const float *b_blocks;
    int64_t b_nleaf;
    unsigned char *b_flags;
    unsigned long long *fetched;
} spamm_host_operands;
int spamm_multiply_host(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int granularity,
                        int exact, float alpha, int32_t row0, int32_t row1,
                        const spamm_plan_buffers *plan, void *plan_ws, size_t plan_ws_bytes,
                        const spamm_product_buffers *c, const spamm_host_operands *host, void *stream);
int spamm_multiply_arena_host(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int granularity,
                              int exact, float alpha, int32_t row0, int32_t row1, int c_depth,
                              int64_t step_capacity, int64_t leaf_capacity, void *arena, size_t arena_bytes,
                              void *plan_ws, size_t plan_ws_bytes, const spamm_host_operands *host,
                              void *stream);
int spamm_multiply_arena(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int granularity,
                         int exact, float alpha, int32_t row0, int32_t row1, int c_depth,
                         int64_t step_capacity, int64_t leaf_capacity, void *arena, size_t arena_bytes,
                         void *plan_ws, size_t plan_ws_bytes, void *stream);

/* _compose with beta != 0 (numeric.py:276-284): out leaf x = (alpha32 * prod[ip]) + (old[io] * beta32)
 * with ip / io = -1 when that side has no leaf; the alpha == 1 / beta == 1 special cases keep
 * the reference's exact expressions. */
int spamm_compose(const float *prod_values, const float *old_values,
                  const int32_t *idx_prod, const int32_t *idx_old, int64_t nout,
                  float alpha, float beta, int alpha_is_one, int beta_is_one,
                  float *out_values, void *stream);

/* ---- multi-GPU: the exchange step of the row-block split (no counterpart in the reference) ---- */

/* Every rank holds the stored leaves of its block of leaf rows; C's rows are split like A's and every
 * product leaf has one owner, so the only exchange is bringing B's leaves to the rank.  This is the
 * all-gather form: each rank contributes `cap` slots (its leaves first, unused slots carry the key
 * 0xFFFFFFFF) of keys, 272-float records and leaf square sums; rank r's part lands at slot r * cap of
 * the outputs, on which spamm_index_leaves + spamm_build_interior then build the tree of B, and
 * spamm_multiply with the rank's rows of A (or row0, row1) yields the rank's rows of C.  nccl_comm is
 * the caller's ncclComm_t; NCCL is looked up in the running process, not linked. */
int spamm_exchange_allgather(void *nccl_comm, const uint32_t *keys, const float *records,
                             const double *leaf_sq, int64_t cap, uint32_t *out_keys, float *out_records,
                             double *out_leaf_sq, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SPAMM_B200_H */
