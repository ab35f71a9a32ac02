// Symbolic phase on the device: the pruned recursion flattened into a compacted task list.
//
// Replaces symbolic.build_plan / convolve (pkg/src/spamm/symbolic.py:92-159).  The task set is
//   { (i,k,j) : leaves A_ik and B_kj stored,  double(|A_ik|) * double(|B_kj|) >= tau }
// (symbolic.py:118-125).  Because every parent norm bounds its children's (norms are correctly
// rounded square roots of FP64 sums of non-negative terms, core.py:252-266), a node product below
// tau can be dropped at any level without losing a leaf task -- the argument that makes
// reference.recursive_spamm (reference.py:72-129) equal to the flat plan.
//
// One level is the list of product nodes (i,j) that still have candidates, in ascending Morton
// order, each with its ascending list of contraction indices k (CSR).  Going one level down,
// node (i,j) with list {k} yields children (2i+di, 2j+dj) with candidates {2k, 2k+1}; order is
// preserved by construction.  Survivors are counted with warp ballots and placed with a
// decoupled look-back prefix sum; nothing returns to the host between levels.
//
// The walk stops two levels above the leaves: a node there is a 4x4 super-tile of product
// leaves, the unit of work of the numeric kernel.  The last kernel tests the leaf norms of every
// block product (I,K,J) directly (four k per block) and emits, per super-tile and in ascending K, one 64-byte STEP record
//   (K, 4 x 16 live bits = the tasks (4I+di, 4K+kk, 4J+dj) that survive, where the two leaf blocks sit)
// so the compacted task list comes out already in the order and grouping the numeric phase
// consumes: ascending k per product leaf (numeric.py:203-217), leaves in Morton order.
// For n <= 8192 the walk starts densely at the super-tile level (one kernel, no coarser levels).
// A last kernel cuts the record stream into pieces of equal weight for the persistent CTAs of the
// numeric kernel (a static partition: no hand-out counter, no uneven finish), empties C's leaf grids,
// publishes the counts and returns the workspace to all-zero, so a sequence of plans on one stream
// needs no memset.
#include <stddef.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "plan_format.cuh"

#define PLAN_WARPS 8
#define PLAN_THREADS (PLAN_WARPS * 32)
#define PLAN_MAX_LEVELS 16

struct LevelBuf {
    uint32_t *node;   // Morton index of each active product node
    int32_t *off;     // CSR offsets into ks (one more entry than nodes)
    uint32_t *ks;     // contraction indices
};

#define PLAN_DENSE_MAX_LEVEL 7   // up to 128 x 128 super-tiles (n <= 8192) the walk starts densely at the tile level

// Lives at the start of the workspace.  The workspace prefix (this struct and the look-back states
// behind it) must be zero when a plan starts; the last kernel of a plan leaves it zero again, so
// one workspace serves a sequence of plans on a stream without memsets.
struct PlanShared {
    int32_t res[SPAMM_PLAN_COUNTS];           // the plan counts while they are being accumulated
    unsigned int order_ticket;
    unsigned int tile_counter[PLAN_MAX_LEVELS + 1];
    int32_t counts[PLAN_MAX_LEVELS + 1][2];   // (nodes, candidates) per level
    unsigned int exec_ticket[2];              // the numeric kernel's pieces drawn / teams finished when it runs
                                              // inside spamm_multiply: zero between launches
};

// ---- start level: dense enumeration by one block ---------------------------------------
// side = 2^level <= 32, so at most 1024 product nodes (one thread each) with at most 32 candidates.
#define ROOT_THREADS 1024
#define ROOT_MAX_LEVEL 5
__global__ void __launch_bounds__(ROOT_THREADS) plan_root_kernel(const float *__restrict__ norm_a,
                                                                 const float *__restrict__ norm_bt, int level, int shift,
                                                                 int row0, int row1, double tau, LevelBuf out,
                                                                 int32_t *counts_out, int64_t cap_nodes, int64_t cap_tasks,
                                                                 int32_t *overflow)
{
    pdl_enter();
    __shared__ uint32_t s_cnt[ROOT_THREADS], s_act[ROOT_THREADS];
    __shared__ uint32_t s_wc[ROOT_THREADS / 32], s_wa[ROOT_THREADS / 32];
    const int S = 1 << level;
    const int c = threadIdx.x;
    uint32_t i = 0, j = 0, live = 0;
    if (c < S * S) {
        morton_decode((uint32_t)c, i, j);
        const bool row_ok = ((int)((i + 1) << shift) > row0) && ((int)(i << shift) < row1);
        if (row_ok)
            for (int k = 0; k < S; ++k)
                if (norm_test(norm_a[i * S + k], norm_bt[j * S + k], tau)) live |= 1u << k;
    }
    const uint32_t cnt = __popc(live), act = cnt > 0;
    // block exclusive scan of (cnt, act): warp shuffles, then the 32 warp totals by warp 0
    uint32_t ic = cnt, ia = act;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t vc = __shfl_up_sync(FULL_MASK, ic, d), va = __shfl_up_sync(FULL_MASK, ia, d);
        if (lane_id() >= (uint32_t)d) { ic += vc; ia += va; }
    }
    if (lane_id() == 31) { s_wc[c >> 5] = ic; s_wa[c >> 5] = ia; }
    __syncthreads();
    __shared__ uint32_t s_tot[2];
    if (c < 32) {
        const uint32_t vc0 = s_wc[c], va0 = s_wa[c];
        uint32_t wc = vc0, wa = va0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t xc = __shfl_up_sync(FULL_MASK, wc, d), xa = __shfl_up_sync(FULL_MASK, wa, d);
            if (c >= d) { wc += xc; wa += xa; }
        }
        s_wc[c] = wc - vc0;
        s_wa[c] = wa - va0;
        if (c == 31) { s_tot[0] = wc; s_tot[1] = wa; }
    }
    __syncthreads();
    const uint32_t tc = s_tot[0], ta = s_tot[1];
    s_cnt[c] = s_wc[c >> 5] + ic - cnt;
    s_act[c] = s_wa[c >> 5] + ia - act;
    if (c == 0) {
        counts_out[0] = (int32_t)ta;
        counts_out[1] = (int32_t)tc;
        if ((int64_t)ta > cap_nodes || (int64_t)tc > cap_tasks) *overflow = 1;
        else out.off[ta] = (int32_t)tc;
    }
    if (cnt == 0) return;
    const uint32_t an = s_act[c];
    uint32_t kb = s_cnt[c];
    if ((int64_t)an >= cap_nodes || (int64_t)kb + cnt > cap_tasks) return;
    out.node[an] = (uint32_t)c;
    out.off[an] = (int32_t)kb;
    for (int k = 0; k < S; ++k)
        if (live >> k & 1) out.ks[kb++] = (uint32_t)k;
}

// ---- one level down ------------------------------------------------------------------------
struct ExpandArgs {
    const float *norm_a;     // child level grid of A, row-major (i,k)
    const float *norm_bt;    // child level grid of B transposed (j,k)
    int S;                   // side of the child level
    int shift;               // leaf rows per child node = 1 << shift
    int row0, row1;          // product leaf rows kept
    double tau;
    LevelBuf in, out;
    const int32_t *counts_in;
    int32_t *counts_out;
    int64_t cap_nodes, cap_tasks;
    int32_t *overflow;
    int32_t *max_list;
    unsigned int *tile_counter;
    volatile unsigned long long *tile_state;
};

// pass bits of one parent candidate k: bit (c*2 + dk), c = di*2 + dj
__device__ __forceinline__ uint32_t child_tests(const ExpandArgs &a, uint32_t pi, uint32_t pj, uint32_t k, uint32_t rowmask)
{
    const float2 a0 = __ldg(reinterpret_cast<const float2 *>(a.norm_a + (int64_t)(2 * pi) * a.S + 2 * k));
    const float2 a1 = __ldg(reinterpret_cast<const float2 *>(a.norm_a + (int64_t)(2 * pi + 1) * a.S + 2 * k));
    const float2 b0 = __ldg(reinterpret_cast<const float2 *>(a.norm_bt + (int64_t)(2 * pj) * a.S + 2 * k));
    const float2 b1 = __ldg(reinterpret_cast<const float2 *>(a.norm_bt + (int64_t)(2 * pj + 1) * a.S + 2 * k));
    uint32_t bits = 0;
    bits |= (uint32_t)norm_test(a0.x, b0.x, a.tau) << 0;   // c=0 (di0,dj0) dk0
    bits |= (uint32_t)norm_test(a0.y, b0.y, a.tau) << 1;
    bits |= (uint32_t)norm_test(a0.x, b1.x, a.tau) << 2;   // c=1 (di0,dj1)
    bits |= (uint32_t)norm_test(a0.y, b1.y, a.tau) << 3;
    bits |= (uint32_t)norm_test(a1.x, b0.x, a.tau) << 4;   // c=2 (di1,dj0)
    bits |= (uint32_t)norm_test(a1.y, b0.y, a.tau) << 5;
    bits |= (uint32_t)norm_test(a1.x, b1.x, a.tau) << 6;   // c=3 (di1,dj1)
    bits |= (uint32_t)norm_test(a1.y, b1.y, a.tau) << 7;
    return bits & rowmask;
}

__global__ void __launch_bounds__(PLAN_THREADS) plan_expand_kernel(ExpandArgs a)
{
    pdl_enter();
    __shared__ int s_tile;
    __shared__ uint32_t s_wtasks[PLAN_WARPS], s_wact[PLAN_WARPS];
    __shared__ uint32_t s_base_lo, s_base_hi;
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const int n_nodes = *a.overflow ? 0 : a.counts_in[0];   // after an overflow the lists above are incomplete
    const int ntiles = (n_nodes + PLAN_WARPS - 1) / PLAN_WARPS;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_tile = (int)atomicAdd(a.tile_counter, 1u);
        __syncthreads();
        const int tile = s_tile;
        if (tile >= ntiles) return;
        const int pidx = tile * PLAN_WARPS + warp;
        const bool valid = pidx < n_nodes;
        uint32_t pm = 0, pi = 0, pj = 0, rowmask = 0;
        int s = 0, e = 0;
        if (valid) {
            pm = a.in.node[pidx];
            morton_decode(pm, pi, pj);
            s = a.in.off[pidx];
            e = a.in.off[pidx + 1];
            const bool r0 = ((int)((2 * pi + 1) << a.shift) > a.row0) && ((int)((2 * pi) << a.shift) < a.row1);
            const bool r1 = ((int)((2 * pi + 2) << a.shift) > a.row0) && ((int)((2 * pi + 1) << a.shift) < a.row1);
            rowmask = (r0 ? 0x0Fu : 0u) | (r1 ? 0xF0u : 0u);
        }
        // phase 1: count survivors per child
        uint32_t cnt[4] = {0, 0, 0, 0};
        for (int b = s; b < e; b += 32) {
            const int t = b + (int)lane;
            uint32_t bits = 0;
            if (t < e) bits = child_tests(a, pi, pj, a.in.ks[t], rowmask);
#pragma unroll
            for (int c = 0; c < 4; ++c) cnt[c] += __popc((bits >> (2 * c)) & 3u);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) cnt[c] = __reduce_add_sync(FULL_MASK, cnt[c]);
        const uint32_t wtasks = cnt[0] + cnt[1] + cnt[2] + cnt[3];
        const uint32_t wact = (cnt[0] > 0) + (cnt[1] > 0) + (cnt[2] > 0) + (cnt[3] > 0);
        if (lane == 0) { s_wtasks[warp] = wtasks; s_wact[warp] = wact; }
        __syncthreads();
        // phase 2: block scan + look-back
        if (warp == 0) {
            uint32_t vt = lane < PLAN_WARPS ? s_wtasks[lane] : 0u, va = lane < PLAN_WARPS ? s_wact[lane] : 0u;
            uint32_t it = vt, ia = va;          // inclusive scan over the block's warps
#pragma unroll
            for (int d = 1; d < PLAN_WARPS; d <<= 1) {
                const uint32_t xt = __shfl_up_sync(FULL_MASK, it, d), xa = __shfl_up_sync(FULL_MASK, ia, d);
                if (lane >= (uint32_t)d) { it += xt; ia += xa; }
            }
            const uint32_t rt = __shfl_sync(FULL_MASK, it, PLAN_WARPS - 1), ra = __shfl_sync(FULL_MASK, ia, PLAN_WARPS - 1);
            if (lane < PLAN_WARPS) { s_wtasks[lane] = it - vt; s_wact[lane] = ia - va; }
            uint32_t ex_lo, ex_hi;
            lb_exclusive_warp(a.tile_state, tile, rt, ra, ex_lo, ex_hi);
            if (lane == 0) {
                s_base_lo = ex_lo;
                s_base_hi = ex_hi;
            }
            if (lane == 0 && tile == ntiles - 1) {
                const int64_t tot_t = (int64_t)ex_lo + rt, tot_a = (int64_t)ex_hi + ra;
                a.counts_out[0] = (int32_t)tot_a;
                a.counts_out[1] = (int32_t)tot_t;
                atomicMax(a.max_list, (int32_t)tot_t);
                if (tot_a > a.cap_nodes || tot_t > a.cap_tasks) *a.overflow = 1;
                else a.out.off[tot_a] = (int32_t)tot_t;
            }
        }
        __syncthreads();
        if (!valid || wtasks == 0) continue;
        // phase 3: place nodes and candidates in order
        int64_t kb = (int64_t)s_base_lo + s_wtasks[warp];
        int64_t nb = (int64_t)s_base_hi + s_wact[warp];
        if (nb + wact > a.cap_nodes || kb + wtasks > a.cap_tasks) {
            if (lane == 0) *a.overflow = 1;
            continue;
        }
        int64_t base[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            base[c] = kb;
            if (cnt[c] > 0) {
                if (lane == 0) {
                    a.out.node[nb] = 4u * pm + (uint32_t)c;
                    a.out.off[nb] = (int32_t)kb;
                }
                ++nb;
            }
            kb += cnt[c];
        }
        const uint32_t lt = lanemask_lt();
        for (int b = s; b < e; b += 32) {
            const int t = b + (int)lane;
            uint32_t bits = 0, k = 0;
            if (t < e) {
                k = a.in.ks[t];
                bits = child_tests(a, pi, pj, k, rowmask);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t p0 = (bits >> (2 * c)) & 1u, p1 = (bits >> (2 * c + 1)) & 1u;
                const uint32_t b0 = __ballot_sync(FULL_MASK, p0), b1 = __ballot_sync(FULL_MASK, p1);
                if ((b0 | b1) == 0) continue;
                int64_t pos = base[c] + __popc(b0 & lt) + __popc(b1 & lt);
                if (p0) a.out.ks[pos++] = 2 * k;
                if (p1) a.out.ks[pos] = 2 * k + 1;
                base[c] += __popc(b0) + __popc(b1);
            }
        }
    }
}

// ---- last stage: super-tile nodes -> step records --------------------------------------------
__device__ __forceinline__ unsigned long long plan_timer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct TileArgs {
    unsigned long long *trace;   // tuning aid (SPAMM_PLAN_TRACE): per block 6 timestamps
    unsigned long long *tile_wprefix;   // tasks in the super-tile nodes before each node (one extra entry: all)
    volatile unsigned long long *tile_state_w;   // look-back states of that prefix
    int all_resident;            // block b may take tile b: the grid has a block per tile
    const float *norm_a;      // leaf level grid of A, row-major (i,k)
    const float *norm_bt;     // leaf level grid of B transposed (j,k)
    const int32_t *slot_a;    // leaf slots of A (i,k)
    const int32_t *slot_bt;   // leaf slots of B transposed (j,k)
    const uint32_t *sub_a;    // sub-norm ranges of A's leaves (i,k), see spamm_tree_view.sub; NULL: no classification
    const uint32_t *sub_bt;   // the same for B, transposed (j,k)
    int fine_weight;          // balance the numeric kernel's pieces for fine4 gating: dead tasks weigh nothing
    const float *norm_a_t;    // super-tile level grids (dense start only)
    const float *norm_bt_t;
    int St;                   // side of the super-tile level
    int L;                    // leaf grid side
    int sub;                  // leaves per block side: 4 (2 or 1 for depth 1 or 0)
    int row0, row1;
    double tau;
    LevelBuf in;
    const int32_t *counts_in;
    spamm_step *steps;
    uint32_t *c_keys;
    int32_t *tile_off;
    int64_t cap_steps, cap_leaves;
    int32_t *counts;          // plan counts, see spamm_b200.h (accumulated in the workspace)
    int32_t *out_counts;      // the caller's plan counts
    // cleared here, while the first loads of the walk are in flight: the numeric kernel's per-leaf hand-over
    // flags and (optional) C's leaf grids, which its epilogue fills
    int32_t *chain;
    int64_t chain_words;
    int64_t cells;
    int32_t *c_slot, *c_slot_t;
    float *c_norm, *c_norm_t;
    double *c_leaf_sq_grid;
    unsigned int *tile_counter;
    volatile unsigned long long *tile_state;
};

// One lane looks at one k = sub*K + kk of block product (I,K,J): the 16 leaf tests, and which
// leaves of the A column / B row at this k are stored.
struct LaneTests {
    uint32_t live;       // bit morton4(di,dj): task (sub*I+di, k, sub*J+dj) survives
    uint32_t a_here;     // bit di: leaf A(sub*I+di, k) stored
    uint32_t b_here;     // bit dj: leaf B(k, sub*J+dj) stored
    uint32_t full;       // live tasks whose 64 gated micro products all pass (fine4, numeric.py:233-238)
    uint32_t dead;       // live tasks of which none passes
};

// leaf norms of A(sub*I+d, k) and B(k, sub*J+d), -1 = absent
struct LaneNorms { float na[4], nb[4]; };

__device__ __forceinline__ LaneNorms tile_norms(const TileArgs &a, uint32_t I, uint32_t J, uint32_t k, bool valid)
{
    LaneNorms n;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        n.na[d] = -1.0f;
        n.nb[d] = -1.0f;
        if (valid && d < a.sub) {
            n.na[d] = __ldg(a.norm_a + (int64_t)(a.sub * I + d) * a.L + k);
            n.nb[d] = __ldg(a.norm_bt + (int64_t)(a.sub * J + d) * a.L + k);
        }
    }
    return n;
}

// WITH_SUB: also classify the live tasks from the sub-norm ranges of their leaves (loaded here, only by
// lanes that have a live task; not prefetched -- the registers are better spent on the norms)
// sub-norm range words of the leaves A(sub*I+d, k) and B(k, sub*J+d) (spamm_tree_view.sub)
struct SubWords { uint32_t sa[4], sb[4]; };
__device__ __forceinline__ SubWords tile_subs(const TileArgs &a, uint32_t I, uint32_t J, uint32_t k, bool valid)
{
    SubWords w;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        w.sa[d] = w.sb[d] = 0xFFFFFFFFu;
        if (valid && a.sub_a && d < a.sub) {
            w.sa[d] = __ldg(a.sub_a + (int64_t)(a.sub * I + d) * a.L + k);
            w.sb[d] = __ldg(a.sub_bt + (int64_t)(a.sub * J + d) * a.L + k);
        }
    }
    return w;
}

template <bool WITH_SUB>
__device__ __forceinline__ LaneTests tile_tests(const TileArgs &a, const LaneNorms &n, uint32_t rowok, uint32_t I = 0,
                                                uint32_t J = 0, uint32_t k = 0, const SubWords *pre = nullptr)
{
    LaneTests t{0u, 0u, 0u, 0u, 0u};
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        t.a_here |= (n.na[d] >= 0.0f) ? (1u << d) : 0u;
        t.b_here |= (n.nb[d] >= 0.0f) ? (1u << d) : 0u;
    }
#pragma unroll
    for (int di = 0; di < 4; ++di)
#pragma unroll
        for (int dj = 0; dj < 4; ++dj)
            if ((rowok >> di & 1u) && norm_test(n.na[di], n.nb[dj], a.tau)) t.live |= 1u << step_pos(di, dj);
    if (WITH_SUB && a.sub_a && t.live) {
        uint32_t sa[4], sb[4];
        if (pre) {
#pragma unroll
            for (int d = 0; d < 4; ++d) { sa[d] = pre->sa[d]; sb[d] = pre->sb[d]; }
        } else {
            const SubWords w = tile_subs(a, I, J, k, true);
#pragma unroll
            for (int d = 0; d < 4; ++d) { sa[d] = w.sa[d]; sb[d] = w.sb[d]; }
        }
#pragma unroll
        for (int di = 0; di < 4; ++di)
#pragma unroll
            for (int dj = 0; dj < 4; ++dj)
                if (t.live >> step_pos(di, dj) & 1u) {
                    // lower bounds of the smallest, upper bounds of the largest sub-norm of either leaf
                    // (NaN for a leaf that cannot be classified: every comparison is then false)
                    const float mna = __uint_as_float(sa[di] << 16), mxa = __uint_as_float(sa[di] & 0xFFFF0000u);
                    const float mnb = __uint_as_float(sb[dj] << 16), mxb = __uint_as_float(sb[dj] & 0xFFFF0000u);
                    if (norm_test(mna, mnb, a.tau)) t.full |= 1u << step_pos(di, dj);
                    else if (mxa >= 0.0f && mxb >= 0.0f && __dmul_rn((double)mxa, (double)mxb) < a.tau)
                        t.dead |= 1u << step_pos(di, dj);
                }
    }
    return t;
}

// DENSE: there is no list from a coarser level; every super-tile node of the 2^tl x 2^tl grid
// (tl <= PLAN_DENSE_MAX_LEVEL) builds its candidate list itself from the level-tl norms, into shared memory.
// TW: super-tile nodes (= warps) per block.  32 keeps the look-back chains of a large product short; a small
// dense start uses 8, so that the blocks on the band -- the only ones with work -- spread over all SMs.
template <bool DENSE, int TW>
__global__ void __launch_bounds__(TW * 32, 2048 / (TW * 32) / 2) plan_tiles_kernel(TileArgs a)
{
    constexpr int TILE_WARPS = TW;
    pdl_enter();
    __shared__ int s_tile;
    __shared__ uint32_t s_wsteps[TILE_WARPS], s_wleaves[TILE_WARPS], s_wtasks[TILE_WARPS];
    __shared__ uint32_t s_base_lo, s_base_hi;
    __shared__ unsigned long long s_base_w;
    __shared__ uint32_t s_ks[DENSE ? TILE_WARPS : 1][DENSE ? (1 << PLAN_DENSE_MAX_LEVEL) : 1];
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const int n_nodes = DENSE ? (a.St * a.St) : (a.counts[2] ? 0 : a.counts_in[0]);
    const int ntiles = (n_nodes + TILE_WARPS - 1) / TILE_WARPS;
    const int sub = a.sub, per = 32 / sub;       // lanes per block product, block products per warp pass
    const uint32_t kk = lane % sub;              // my k inside the block
    const uint32_t grp = (lane / sub) * sub;     // first lane of my group
    unsigned long long tasks_total = 0;
    uint32_t tiles_total = 0;            // super-tiles with at least one record
    if (blockIdx.x == 0 && threadIdx.x < 8) a.out_counts[16 + threadIdx.x] = 0;     // accumulated by plan_order_kernel
    {
        const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gsz = (int64_t)gridDim.x * blockDim.x;
        for (int64_t x = gtid; x < a.chain_words; x += gsz) a.chain[x] = 0;
        if (a.c_slot) {
            for (int64_t x = gtid; x < a.cells; x += gsz) {
                a.c_slot[x] = -1;
                a.c_slot_t[x] = -1;
                a.c_norm[x] = -1.0f;
                a.c_norm_t[x] = -1.0f;
                a.c_leaf_sq_grid[x] = 0.0;
            }
        }
    }
    if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 6] = plan_timer();
    // dense start with no more tiles than blocks: block b takes tile b, no hand-out counter
    const bool fixed_tiles = DENSE && a.all_resident && ntiles <= (int)gridDim.x;
    for (int round = 0;; ++round) {
        __syncthreads();
        if (!fixed_tiles && threadIdx.x == 0) s_tile = (int)atomicAdd(a.tile_counter, 1u);
        __syncthreads();
        const int tile = fixed_tiles ? (round == 0 ? (int)blockIdx.x : ntiles) : s_tile;
        if (tile >= ntiles) break;
        if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 6 + 1] = plan_timer();
        const int pidx = tile * TILE_WARPS + warp;
        const bool valid = pidx < n_nodes;
        uint32_t pm = 0, I = 0, J = 0, rowok = 0;
        int s = 0, e = 0;
        const uint32_t *ks = DENSE ? s_ks[warp] : a.in.ks;
        if (valid) {
            pm = DENSE ? (uint32_t)pidx : a.in.node[pidx];
            morton_decode(pm, I, J);
            for (int d = 0; d < sub; ++d) {
                const int row = (int)(sub * I + d);
                if (row >= a.row0 && row < a.row1) rowok |= 1u << d;
            }
            if (DENSE) {
                // candidates K of this node: the level-tl test (symbolic.py:118-125 one level up)
                if (rowok) {
                    for (int k0 = 0; k0 < a.St; k0 += 32) {
                        const int K = k0 + (int)lane;
                        const bool pass = K < a.St && norm_test(__ldg(a.norm_a_t + (int64_t)I * a.St + K),
                                                                __ldg(a.norm_bt_t + (int64_t)J * a.St + K), a.tau);
                        const uint32_t bal = __ballot_sync(FULL_MASK, pass);
                        if (pass) s_ks[warp][e + __popc(bal & lanemask_lt())] = (uint32_t)K;
                        e += __popc(bal);
                    }
                }
                __syncwarp();
            } else {
                s = a.in.off[pidx];
                e = a.in.off[pidx + 1];
            }
        }
        if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 6 + 2] = plan_timer();
        // phase 1: count step records and product leaves of this super-tile
        uint32_t nsteps = 0, present = 0, ntasks = 0, nheavy = 0;
        // the norms of the next pass are fetched before the tests of the current one
        LaneNorms nrm = tile_norms(a, I, J, (s + (int)lane / sub < e) ? sub * ks[s + (int)lane / sub] + kk : 0u,
                                          s + (int)lane / sub < e);
        for (int b = s; b < e; b += per) {
            const int t = b + (int)lane / sub, t2 = t + per;
            const LaneNorms nxt = tile_norms(a, I, J, t2 < e ? sub * ks[t2] + kk : 0u, t2 < e);
            uint32_t live = 0, heavy = 0;
            if (t < e) {
                const LaneTests tt = tile_tests<false>(a, nrm, rowok);
                live = heavy = tt.live;
            }
            nrm = nxt;
            const uint32_t bal = __ballot_sync(FULL_MASK, live != 0);
            // one record per group of `sub` lanes with any live task
            uint32_t groups = bal;
            if (sub >= 2) groups |= groups >> 1;
            if (sub >= 4) groups |= groups >> 2;
            groups &= (sub == 4 ? 0x11111111u : sub == 2 ? 0x55555555u : 0xFFFFFFFFu);
            nsteps += __popc(groups);
            present |= live;
            ntasks += __popc(live);
            nheavy += __popc(heavy);
        }
        present = __reduce_or_sync(FULL_MASK, present);
        ntasks = __reduce_add_sync(FULL_MASK, ntasks);
        nheavy = __reduce_add_sync(FULL_MASK, nheavy);
        const uint32_t nleaves = __popc(present);
        if (lane == 0) {
            s_wsteps[warp] = nsteps; s_wleaves[warp] = nleaves; s_wtasks[warp] = nheavy; tasks_total += ntasks;
            tiles_total += nsteps > 0 ? 1u : 0u;
        }
        __syncthreads();
        if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 6 + 3] = plan_timer();
        // phase 2: block scan + look-back over (records, product leaves)
        if (warp == 0) {
            uint32_t vs = lane < TILE_WARPS ? s_wsteps[lane] : 0u, vl = lane < TILE_WARPS ? s_wleaves[lane] : 0u;
            uint32_t vt = lane < TILE_WARPS ? s_wtasks[lane] : 0u;
            uint32_t is = vs, il = vl, it = vt;          // inclusive scan over the block's warps
#pragma unroll
            for (int d = 1; d < TILE_WARPS; d <<= 1) {
                const uint32_t xs = __shfl_up_sync(FULL_MASK, is, d), xl = __shfl_up_sync(FULL_MASK, il, d);
                const uint32_t xt = __shfl_up_sync(FULL_MASK, it, d);
                if (lane >= (uint32_t)d) { is += xs; il += xl; it += xt; }
            }
            const uint32_t rs = __shfl_sync(FULL_MASK, is, TILE_WARPS - 1), rl = __shfl_sync(FULL_MASK, il, TILE_WARPS - 1);
            const uint32_t rt = __shfl_sync(FULL_MASK, it, TILE_WARPS - 1);
            if (lane < TILE_WARPS) { s_wsteps[lane] = is - vs; s_wleaves[lane] = il - vl; s_wtasks[lane] = it - vt; }
            // both aggregates are published before either look-back waits
            if (lane == 0) lb64_publish(a.tile_state_w, tile, (unsigned long long)rt);
            uint32_t ex_lo, ex_hi;
            unsigned long long ex_w;
            if (fixed_tiles && ntiles <= PLAN_ALL_EXCLUSIVE_MAX) {
                all_exclusive_warp(a.tile_state, tile, rs, rl, ex_lo, ex_hi);
                ex_w = all64_exclusive_warp(a.tile_state_w, tile);
            } else {
                lb_exclusive_warp(a.tile_state, tile, rs, rl, ex_lo, ex_hi);
                ex_w = lb64_exclusive_warp(a.tile_state_w, tile, (unsigned long long)rt);
            }
            if (lane == 0) {
                s_base_lo = ex_lo;
                s_base_hi = ex_hi;
                s_base_w = ex_w;
            }
            if (lane == 0 && tile == ntiles - 1) {
                const int64_t tot_s = (int64_t)ex_lo + rs, tot_l = (int64_t)ex_hi + rl;
                a.counts[0] = (int32_t)tot_l;
                a.counts[4] = (int32_t)tot_s;
                a.counts[11] = n_nodes;
                a.tile_off[n_nodes] = (int32_t)tot_s;
                a.tile_wprefix[n_nodes] = ex_w + rt;
                if (tot_s > a.cap_steps || tot_l > a.cap_leaves) a.counts[2] = 1;
            }
        }
        __syncthreads();
        if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 6 + 4] = plan_timer();
        if (valid && lane == 0) {
            a.tile_off[pidx] = (int32_t)(s_base_lo + s_wsteps[warp]);
            a.tile_wprefix[pidx] = s_base_w + s_wtasks[warp];
        }
        if (!valid || nsteps == 0) continue;
        // phase 3: product leaf keys and step records, in ascending K
        int64_t sb = (int64_t)s_base_lo + s_wsteps[warp];
        const int64_t cb = (int64_t)s_base_hi + s_wleaves[warp];
        if (sb + nsteps > a.cap_steps || cb + nleaves > a.cap_leaves) {
            if (lane == 0) a.counts[2] = 1;
            continue;
        }
        if (lane < 16 && (present >> lane & 1u))
            a.c_keys[cb + __popc(present & ((1u << lane) - 1u))] = pm * (uint32_t)(sub * sub) + lane;
        const int64_t s_first = sb, s_last = sb + nsteps - 1;
        const uint32_t lt = lanemask_lt();
        const uint32_t lead_mask = (sub == 4 ? 0x11111111u : sub == 2 ? 0x55555555u : 0xFFFFFFFFu);
        nrm = tile_norms(a, I, J, (s + (int)lane / sub < e) ? sub * ks[s + (int)lane / sub] + kk : 0u, s + (int)lane / sub < e);
        for (int b = s; b < e; b += per) {
            const int t = b + (int)lane / sub, t2 = t + per;
            const LaneNorms nxt = tile_norms(a, I, J, t2 < e ? sub * ks[t2] + kk : 0u, t2 < e);
            LaneTests lt4{0u, 0u, 0u, 0u, 0u};
            uint32_t K = 0;
            if (t < e) {
                K = ks[t];
                lt4 = tile_tests<true>(a, nrm, rowok, I, J, (uint32_t)sub * K + kk);
            }
            nrm = nxt;
            // gather the group's four lanes: live per kk, stored leaves of both blocks
            uint32_t live4[4] = {0, 0, 0, 0}, dead4[4] = {0, 0, 0, 0}, a_present = 0, b_present = 0, any = 0;
            // first stored leaf of each block in Morton order and the lane that knows its slot
            int a_best = 16, b_best = 16;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int src = (int)grp + (x < sub ? x : 0);
                const uint32_t lv = __shfl_sync(FULL_MASK, lt4.live | (lt4.full << 16), src);
                const uint32_t dd = __shfl_sync(FULL_MASK, lt4.dead, src);
                const uint32_t ah = __shfl_sync(FULL_MASK, lt4.a_here, src);
                const uint32_t bh = __shfl_sync(FULL_MASK, lt4.b_here, src);
                if (x < sub) {
                    live4[x] = lv;
                    dead4[x] = dd;
                    any |= lv & 0xFFFFu;
#pragma unroll
                    for (int d = 0; d < 4; ++d) {
                        if (ah >> d & 1u) { a_present |= 1u << step_pos(d, x); }     // A leaf (di=d, kk=x)
                        if (bh >> d & 1u) { b_present |= 1u << step_pos(x, d); }     // B leaf (kk=x, dj=d)
                    }
                }
            }
            if (a_present) a_best = __ffs(a_present) - 1;
            if (b_present) b_best = __ffs(b_present) - 1;
            const uint32_t bal = __ballot_sync(FULL_MASK, any != 0 && lane == grp);
            if (any != 0 && lane == grp) {
                const int64_t x = sb + __popc(bal & lt);
                uint32_t flags = 0;
                if (x == s_first) flags |= STEP_FIRST;
                if (x == s_last) flags |= STEP_LAST;
                const uint32_t a_first = (uint32_t)__ldg(
                    a.slot_a + (int64_t)(sub * I + step_pos_di(a_best)) * a.L + (sub * K + step_pos_dj(a_best)));
                const uint32_t b_first = (uint32_t)__ldg(
                    a.slot_bt + (int64_t)(sub * J + step_pos_dj(b_best)) * a.L + (sub * K + step_pos_di(b_best)));
                uint4 *rec = reinterpret_cast<uint4 *>(a.steps + x);
                rec[0] = make_uint4(K, flags, (uint32_t)cb, pm);
                rec[1] = make_uint4(a_first, a_present, b_first, b_present);
                rec[2] = make_uint4(live4[0], live4[1], live4[2], live4[3]);
                // last word: records of this tile | position of this record in it << 16 (tiles have at
                // most L/4 <= 8192 records), from which the numeric kernel finds the tile's ends
                rec[3] = make_uint4(present, dead4[0] | (dead4[1] << 16), dead4[2] | (dead4[3] << 16),
                                    nsteps | ((uint32_t)(x - s_first) << 16));
            }
            sb += __popc(bal & lead_mask);
        }
    }
    if (lane == 0 && tasks_total) atomicAdd(reinterpret_cast<unsigned long long *>(a.counts + 6), tasks_total);
    if (lane == 0 && tiles_total) atomicAdd(a.counts + 1, (int32_t)tiles_total);
    __syncthreads();
    if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 6 + 5] = plan_timer();
}

// Work units of the numeric kernel, claimed by its teams from one counter in the order given here.
// A unit is a run [b, e) of consecutive step records (two ints in plan.tile_order).  Where a run
// begins or ends inside a super-tile, the tile's accumulators pass from team to team through C's
// value records; the numeric kernel works out from the records themselves (tile length and position,
// last word of spamm_step) which part of a unit is the head of a tile that the next unit finishes
// (run FIRST), which are whole tiles, and which is the tail of a tile another unit began (run LAST).
// The records (tile after tile, in Morton order) form two regions.
//   Region A, the bulk: P pieces of equal weight (live tasks + rec_weight per record), one per team
//   (or a few rounds of them for a large product, so that the teams work on neighbouring super-tiles
//   at any time and share operand blocks in L2).  This is McNaughton's wrap-around rule for
//   preemptive scheduling, with the split tile's two parts at opposite ends of the two teams' time
//   lines so that the ascending-k order of a tile's records is kept.  One warp looks at one tile and
//   places the cuts that fall into it: cut g is the first record boundary at which the weight prefix
//   reaches g W_A / P.
//   Region B, the last tiles (about a quarter of the work, at least 1.25 tiles per team): no model of
//   a team's speed is exact, so the teams do not finish their pieces together; the tiles of B are cut
//   into a long first segment and up to two short ones, handed out in LAYERS -- all first segments,
//   then all second ones, then all third ones -- so that a segment's predecessor was claimed a
//   whole layer earlier and is finished when its successor starts.  Five ranges of unit slots, range x
//   at P + x * stride with counts[16 + x] slots in use (counts[21] = stride): the first segments of the
//   tiles with three, with two segments and the whole tiles (longest first), the second segments, the
//   third segments; the numeric kernel maps its claim numbers onto the slots in use.
#define ORDER_MAX_B_NODES 4096      // region B: at most this many super-tile nodes
#define ORDER_MAX_SEGS 3
struct OrderArgs {
    const int32_t *tile_off;
    const unsigned long long *tile_wprefix;
    const spamm_step *steps;
    int defer_clean;              // the caller's next kernel clears PlanShared (spamm_multiply)
    int32_t *counts;              // the caller's plan counts: written here
    PlanShared *shared;
    uint32_t *ws_tail;            // workspace prefix behind PlanShared (look-back states), left zero
    int64_t ws_tail_words;
    int32_t *units;               // plan.tile_order: 2 ints per unit
    int64_t unit_capacity;
    int num_teams, piece_records, rec_weight;
    int tail_records;             // region B: records per short segment (0: no region B)
    int tail_percent;             // region B: its share of the work (at least 1.25 tiles per team anyway)
};

__global__ void __launch_bounds__(256) plan_order_kernel(OrderArgs a)
{
    const int32_t *__restrict__ tile_off = a.tile_off;
    int32_t *counts = a.shared->res;
    __shared__ bool s_last;
    pdl_enter();
    // the planner's look-back states are done with and go back to zero
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gsz = (int64_t)gridDim.x * blockDim.x;
    for (int64_t x = gtid; x < a.ws_tail_words; x += gsz) a.ws_tail[x] = 0u;
    const int t = threadIdx.x;
    const uint32_t lane = lane_id();
    const int n_nodes = counts[2] ? 0 : counts[11];
    const long long R = counts[2] ? 0 : counts[4];
    const unsigned long long T = a.tile_wprefix[counts[11]];
    const unsigned long long RW = (unsigned long long)a.rec_weight;
    const unsigned long long W = T + RW * (unsigned long long)R;
    // ---- region B: where it begins (every block finds the same answer)
    __shared__ int s_lo, s_hi;
    const int n_tiles = counts[2] ? 0 : counts[1];
    auto wnode = [&](int i) -> unsigned long long { return a.tile_wprefix[i] + RW * (unsigned long long)tile_off[i]; };
    int idxB = n_nodes;
    // measured (B200): with a piece of several tiles per team the static split alone finishes within a few
    // per cent; the layered tail is worth its hand-overs only when a team's share is shorter than a tile
    const int tail_records = a.tail_records >= 0 ? a.tail_records : (R < 3ll * a.num_teams ? 3 : 0);
    // room in the plan: region B (only plans that use it) may take all unit slots but one round of pieces,
    // five slots per node
    const int64_t b_room = tail_records > 0 ? (a.unit_capacity - a.num_teams) / 5 : 0;
    const int max_b_nodes = (int)(b_room < 0 ? 0 : (b_room < ORDER_MAX_B_NODES ? b_room : ORDER_MAX_B_NODES));
    if (tail_records > 0 && n_tiles > 0 && R > 0 && max_b_nodes > 0) {
        // (64-bit products: a plan's weight stays far below 2^48 -- at most 2^31 records of at most 96 -- and
        // the factors here below 2^15)
        unsigned long long wB = W * (unsigned long long)a.tail_percent / 100ull;
        const unsigned long long wmin = W * (unsigned long long)(a.num_teams + a.num_teams / 4) / (unsigned long long)n_tiles;
        if (wB < wmin) wB = wmin;
        const unsigned long long targetA = wB >= W ? 0ull : W - wB;
        // largest node index whose weight prefix is <= targetA: 256-ary search over the monotone prefix
        int lo = n_nodes > max_b_nodes ? n_nodes - max_b_nodes : 0, hi = n_nodes;   // answer in [lo, hi]
        if (wnode(lo) > targetA) hi = lo;                                           // region B is capped: starts at lo
        while (hi - lo > 1) {
            const long long span = hi - lo;
            const int probe = lo + (int)((span * (t + 1)) / 257);
            const bool le = probe > lo && probe < hi && wnode(probe) <= targetA;
            __syncthreads();
            if (t == 0) { s_lo = lo; s_hi = hi; }
            __syncthreads();
            if (probe > lo && probe < hi) {
                if (le) atomicMax(&s_lo, probe);
                else atomicMin(&s_hi, probe);
            }
            __syncthreads();
            lo = s_lo; hi = s_hi;
            if (span <= 257) break;             // every interior point was probed
        }
        idxB = lo;
    }
    const long long RA = idxB < n_nodes ? tile_off[idxB] : R;        // records of region A
    const unsigned long long WA = idxB < n_nodes ? wnode(idxB) : W;
    // ---- region A: pieces, one per team, or several rounds of them when the product is large
    long long rounds = RA / ((long long)a.num_teams * a.piece_records);
    if (rounds < 1) rounds = 1;
    if (rounds > 64) rounds = 64;
    const int64_t cap_a = a.unit_capacity - 5ll * max_b_nodes;
    if (rounds * a.num_teams > cap_a) rounds = cap_a / a.num_teams;
    const long long P = RA > 0 ? (rounds >= 1 ? rounds * a.num_teams : cap_a) : 0;
    int32_t *__restrict__ uw = a.units;
    // weight prefix at which cut g is placed (at least 1, so that every cut falls into some tile)
    auto target_of = [&](long long g) -> unsigned long long {
        const unsigned long long x = (unsigned long long)g * WA / (unsigned long long)P;
        return x < 1ull ? 1ull : x;
    };
    // a unit is (b, tb, ts, e): records [b, e); tb = end of the tile record b lies in (= b when b starts a
    // tile), ts = start of the tile record e - 1 lies in (= e when e ends a tile).  The numeric kernel runs
    // the head [max(ts, min(tb, e)), e) first, the whole tiles in between next and the tail [b, min(tb, e)) last.
    if (gtid == 0 && P > 0) {
        uw[0] = 0;                              // piece 0 begins at record 0, at a tile start
        uw[1] = 0;
        uw[4 * (P - 1) + 2] = (int32_t)RA;      // the last piece ends with region A, at a tile end
        uw[4 * (P - 1) + 3] = (int32_t)RA;
    }
    // one warp per tile: the records' weights in parallel, a warp scan, every lane places the cuts that
    // fall behind its record (cut g = boundary after the first record at which the prefix reaches target(g))
    const int64_t gwarp = gtid >> 5, nwarps = gsz >> 5;
    for (int64_t idx = gwarp; idx < idxB && P > 1; idx += nwarps) {
        const int ts = tile_off[idx], te = tile_off[idx + 1];
        if (te == ts) continue;
        const unsigned long long w0 = a.tile_wprefix[idx] + RW * (unsigned long long)ts;
        const unsigned long long w1 = a.tile_wprefix[idx + 1] + RW * (unsigned long long)te;
        long long g0 = (long long)(w0 * (unsigned long long)P / WA);
        if (g0 < 1) g0 = 1;
        while (g0 < P && target_of(g0) <= w0) ++g0;          // first cut behind w0
        if (g0 >= P || target_of(g0) > w1) continue;         // no cut in this tile
        unsigned long long run = w0;
        for (int base = ts; base < te; base += 32) {
            const int r = base + (int)lane;
            unsigned long long wr = 0;
            if (r < te) {
                const uint4 live = *(reinterpret_cast<const uint4 *>(a.steps + r) + 2);
                wr = RW + __popc(live.x & 0xFFFFu) + __popc(live.y & 0xFFFFu) + __popc(live.z & 0xFFFFu) + __popc(live.w & 0xFFFFu);
            }
            unsigned long long inc = wr;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long y = __shfl_up_sync(FULL_MASK, inc, d);
                if (lane >= (uint32_t)d) inc += y;
            }
            const unsigned long long hi_w = run + inc, lo_w = hi_w - wr;      // prefix after / before my record
            if (r < te && wr > 0) {
                long long g = (long long)(lo_w * (unsigned long long)P / WA);
                if (g < 1) g = 1;
                while (g < P && target_of(g) <= lo_w) ++g;
                for (; g < P && target_of(g) <= hi_w; ++g) {
                    const int c = r + 1;               // the cut: in (ts, te]
                    uw[4 * g] = c;                            // b of piece g
                    uw[4 * g + 1] = te;                       // its tile ends at te (c == te: b starts the next tile)
                    uw[4 * (g - 1) + 2] = c == te ? c : ts;   // piece g - 1 ends in this tile
                    uw[4 * (g - 1) + 3] = c;                  // e of piece g - 1
                }
            }
            run += __shfl_sync(FULL_MASK, inc, 31);
        }
    }
    // ---- region B: layered segments; every warp takes 32 nodes at a time, slots by one atomic per warp and range.
    // Five ranges of unit slots, each nB long, handed out in this order: first segments of the tiles with 3,
    // with 2 segments, whole tiles (longest first inside the first layer), then second, then third segments.
    const int nB = n_nodes - idxB;                   // range stride
    if (nB > 0) {
        const int sl = tail_records > 0 ? tail_records : 1;
        // segments of a tile of ns records: ns <= sl: 1; ns <= 2 sl: 2 (ns - sl, sl); else 3 (ns - 2 sl, sl, sl)
        for (int64_t base = idxB + gwarp * 32; base < n_nodes; base += nwarps * 32) {
            const int64_t idx = base + lane;
            int ts = 0, te = 0;
            if (idx < n_nodes) { ts = tile_off[idx]; te = tile_off[idx + 1]; }
            const int ns = te - ts;
            const int nseg = ns <= 0 ? 0 : (ns <= sl ? 1 : (ns <= 2 * sl ? 2 : 3));
            int sb = ts;
#pragma unroll
            for (int x = 0; x < 5; ++x) {
                // range x: segment index l of the tiles with the given number of segments
                const int l = x < 3 ? 0 : x - 2;
                const bool in = x < 3 ? nseg == 3 - x : nseg > l;
                const uint32_t m = __ballot_sync(FULL_MASK, in);
                if (m == 0) continue;
                int slot0 = 0;
                if (lane == (uint32_t)(__ffs(m) - 1)) slot0 = atomicAdd(&a.counts[16 + x], __popc(m));
                slot0 = __shfl_sync(FULL_MASK, slot0, __ffs(m) - 1);
                if (in) {
                    const int se = l + 1 == nseg ? te : (l == 0 ? te - (nseg - 1) * sl : sb + sl);
                    int32_t *u = uw + 4 * (P + (long long)x * nB + slot0 + __popc(m & lanemask_lt()));
                    *reinterpret_cast<int4 *>(u) = make_int4(sb, sb == ts ? sb : te, se == te ? se : ts, se);
                    sb = se;
                }
            }
        }
    }
    if (a.defer_clean) {
        // the numeric kernel that follows returns the shared planner state to zero (its first block,
        // once this kernel has completed); the counts are final already, block 0 publishes them (the
        // layer counts [16..18] are accumulated in place by all blocks)
        if (blockIdx.x == 0 && t < 16) {
            int32_t v = 0;
            if (t == 0 || t == 1 || t == 2 || t == 3 || t == 4 || t == 6 || t == 7 || t == 11) v = counts[t];
            if (t == 5) v = (int32_t)(P + 5ll * nB);     // unit slots; [16..20] say how many of region B's are in use
            if (t == 12) v = (int32_t)P;
            a.counts[t] = v;
        }
        if (blockIdx.x == 0 && t == 0) a.counts[21] = nB;
        return;
    }
    // the last block publishes the counts and leaves the shared planner state zero for the next plan
    __threadfence();
    __syncthreads();
    if (t == 0) s_last = atomicAdd(&a.shared->order_ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (t < 16) {
        int32_t v = 0;
        if (t == 0 || t == 1 || t == 2 || t == 3 || t == 4 || t == 6 || t == 7 || t == 11) v = counts[t];
        if (t == 5) v = (int32_t)(P + 5ll * nB);
        if (t == 12) v = (int32_t)P;
        a.counts[t] = v;
    }
    if (t == 0) a.counts[21] = nB;
    __syncthreads();
    uint32_t *sh = reinterpret_cast<uint32_t *>(a.shared);
    for (int x = t; x < (int)(sizeof(PlanShared) / 4); x += blockDim.x) sh[x] = 0u;
}

// ---- small dense products (n <= 4096): count, then emit and cut ----------------------------------
// Two kernels instead of plan_tiles + plan_order.  Only the super-tiles on the band have work, and with
// one node per warp and 32 warps per block they sit in a quarter of the blocks; here a block has 8
// nodes, so the band spreads over all SMs, and nobody polls: plan_count_kernel leaves one aggregate
// per block, plan_emit_kernel (after it, programmatic dependent launch) sums the aggregates of its
// predecessors, writes the records and -- the totals being known to every block -- places the cuts of
// the numeric kernel's pieces while the records' live words are still in registers.
#define SMALL_WARPS 8
#define SMALL_MAX_TILES 512          // 64 x 64 super-tile nodes / 8
struct SmallArgs {
    TileArgs t;
    unsigned long long *node_info;   // per node, between the kernels: records | present << 8 | tasks << 24 (= tile_wprefix)
    unsigned long long *agg_a;       // per block: records | product leaves << 32
    unsigned long long *agg_b;       // per block: tasks | super-tiles with records << 32
    // grids of more than 512 blocks (n = 8192): the same sums per group of `group` consecutive blocks, made by
    // the last block of a group to finish (tickets: zero between launches); plan_emit_kernel sums the groups
    int group;
    unsigned long long *grp_a, *grp_b;
    unsigned int *grp_ticket;
    int32_t *units;
    int64_t unit_capacity;
    int num_teams, piece_records, rec_weight, tail_records, tail_percent;
    int dbg;                         // tuning aid (SPAMM_PLAN_DEBUG, with SPAMM_PIPE_STOP=2 only): 1 = place no cuts, 2 = no classification
};

__device__ __forceinline__ void small_clear(const TileArgs &a)
{
    if (blockIdx.x == 0 && threadIdx.x < 8) a.out_counts[16 + threadIdx.x] = 0;     // accumulated by plan_emit_kernel
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gsz = (int64_t)gridDim.x * blockDim.x;
    for (int64_t x = gtid; x < a.chain_words; x += gsz) a.chain[x] = 0;
    if (a.c_slot) {
        for (int64_t x = gtid; x < a.cells; x += gsz) {
            a.c_slot[x] = -1;
            a.c_slot_t[x] = -1;
            a.c_norm[x] = -1.0f;
            a.c_norm_t[x] = -1.0f;
            a.c_leaf_sq_grid[x] = 0.0;
        }
    }
}

// candidates K of node (I,J): the level-tl test (symbolic.py:118-125 one level up); returns their number
__device__ __forceinline__ int small_candidates(const TileArgs &a, uint32_t I, uint32_t J, uint32_t rowok, uint32_t *ks)
{
    const uint32_t lane = lane_id();
    int e = 0;
    if (rowok) {
        for (int k0 = 0; k0 < a.St; k0 += 32) {
            const int K = k0 + (int)lane;
            const bool pass = K < a.St && norm_test(__ldg(a.norm_a_t + (int64_t)I * a.St + K),
                                                    __ldg(a.norm_bt_t + (int64_t)J * a.St + K), a.tau);
            const uint32_t bal = __ballot_sync(FULL_MASK, pass);
            if (pass) ks[e + __popc(bal & lanemask_lt())] = (uint32_t)K;
            e += __popc(bal);
        }
    }
    __syncwarp();
    return e;
}

__global__ void __launch_bounds__(SMALL_WARPS * 32, 4) plan_count_kernel(SmallArgs sa)
{
    const TileArgs &a = sa.t;
    pdl_enter();
    if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 6] = plan_timer();
    __shared__ uint32_t s_ks[SMALL_WARPS][1 << PLAN_DENSE_MAX_LEVEL];
    __shared__ uint32_t s_steps[SMALL_WARPS], s_leaves[SMALL_WARPS], s_tasks[SMALL_WARPS];
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const int n_nodes = a.St * a.St;
    const int sub = a.sub, per = 32 / sub;
    const uint32_t kk = lane % sub;
    small_clear(a);
    const int pidx = (int)blockIdx.x * SMALL_WARPS + warp;
    uint32_t nsteps = 0, present = 0, ntasks = 0;
    if (pidx < n_nodes) {
        uint32_t I, J, rowok = 0;
        morton_decode((uint32_t)pidx, I, J);
        for (int d = 0; d < sub; ++d) {
            const int row = (int)(sub * I + d);
            if (row >= a.row0 && row < a.row1) rowok |= 1u << d;
        }
        const uint32_t *ks = s_ks[warp];
        const int e = small_candidates(a, I, J, rowok, s_ks[warp]);
        LaneNorms nrm = tile_norms(a, I, J, ((int)lane / sub < e) ? sub * ks[(int)lane / sub] + kk : 0u, (int)lane / sub < e);
        for (int b = 0; b < e; b += per) {
            const int t = b + (int)lane / sub, t2 = t + per;
            const LaneNorms nxt = tile_norms(a, I, J, t2 < e ? sub * ks[t2] + kk : 0u, t2 < e);
            uint32_t live = 0;
            if (t < e) live = tile_tests<false>(a, nrm, rowok).live;
            nrm = nxt;
            uint32_t groups = __ballot_sync(FULL_MASK, live != 0);
            if (sub >= 2) groups |= groups >> 1;
            if (sub >= 4) groups |= groups >> 2;
            groups &= (sub == 4 ? 0x11111111u : sub == 2 ? 0x55555555u : 0xFFFFFFFFu);
            nsteps += __popc(groups);
            present |= live;
            ntasks += __popc(live);
        }
        present = __reduce_or_sync(FULL_MASK, present);
        ntasks = __reduce_add_sync(FULL_MASK, ntasks);
        if (lane == 0)
            sa.node_info[pidx] = (unsigned long long)nsteps | ((unsigned long long)present << 8) | ((unsigned long long)ntasks << 24);
    }
    if (lane == 0) { s_steps[warp] = nsteps; s_leaves[warp] = __popc(present); s_tasks[warp] = ntasks; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long st = 0, lv = 0, tk = 0, ne = 0;
        for (int w = 0; w < SMALL_WARPS; ++w) { st += s_steps[w]; lv += s_leaves[w]; tk += s_tasks[w]; ne += s_steps[w] ? 1u : 0u; }
        sa.agg_a[blockIdx.x] = st | (lv << 32);
        sa.agg_b[blockIdx.x] = tk | (ne << 32);
        if (sa.group > 1) {
            const int g = (int)blockIdx.x / sa.group, first = g * sa.group;
            const int members = min(sa.group, (int)gridDim.x - first);
            __threadfence();
            if (atomicAdd(sa.grp_ticket + g, 1u) == (unsigned int)(members - 1)) {
                __threadfence();
                unsigned long long ga = 0, gb = 0;
                for (int j = 0; j < members; ++j) { ga += __ldcg(sa.agg_a + first + j); gb += __ldcg(sa.agg_b + first + j); }
                sa.grp_a[g] = ga;
                sa.grp_b[g] = gb;
                sa.grp_ticket[g] = 0u;
            }
        }
        if (a.trace) a.trace[blockIdx.x * 6 + 1] = plan_timer();
    }
}

__global__ void __launch_bounds__(SMALL_WARPS * 32, 4) plan_emit_kernel(SmallArgs sa)
{
    const TileArgs &a = sa.t;
    __shared__ uint32_t s_ks[SMALL_WARPS][1 << PLAN_DENSE_MAX_LEVEL];
    __shared__ unsigned long long s_a[SMALL_MAX_TILES], s_b[SMALL_MAX_TILES];     // exclusive prefixes of the block aggregates
    __shared__ unsigned long long s_wa[SMALL_WARPS], s_wb[SMALL_WARPS], s_tot[2];
    __shared__ int s_bB;
    const int warp = threadIdx.x >> 5, t = threadIdx.x;
    const uint32_t lane = lane_id();
    const int n_nodes = a.St * a.St;
    // the prefix sums below run over the blocks themselves, or over groups of blocks when there are more than 512
    const int gsz = sa.group, ntiles = ((int)gridDim.x + gsz - 1) / gsz;
    const unsigned long long *agg_a = gsz > 1 ? sa.grp_a : sa.agg_a, *agg_b = gsz > 1 ? sa.grp_b : sa.agg_b;
    const int sub = a.sub, per = 32 / sub;
    const uint32_t kk = lane % sub, grp = (lane / sub) * sub;
    const int pidx = (int)blockIdx.x * SMALL_WARPS + warp;
    const bool valid = pidx < n_nodes;
    uint32_t I = 0, J = 0, rowok = 0;
    if (valid) {
        morton_decode((uint32_t)pidx, I, J);
        for (int d = 0; d < sub; ++d) {
            const int row = (int)(sub * I + d);
            if (row >= a.row0 && row < a.row1) rowok |= 1u << d;
        }
    }
    // the candidate lists again (level-tl norms: independent of the preceding kernel)
    const uint32_t *ks = s_ks[warp];
    const int e = valid ? small_candidates(a, I, J, rowok, s_ks[warp]) : 0;
    if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 6 + 2] = plan_timer();
    pdl_enter();
    if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 6 + 3] = plan_timer();
    // ---- every block: prefix sums over ALL block aggregates (at most 512: two per thread)
    {
        unsigned long long va[2], vb[2];
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            const int i = 2 * t + x;
            va[x] = i < ntiles ? __ldcg(agg_a + i) : 0ull;
            vb[x] = i < ntiles ? __ldcg(agg_b + i) : 0ull;
        }
        unsigned long long ia = va[0] + va[1], ib = vb[0] + vb[1];       // inclusive scan of the pair sums
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long xa = __shfl_up_sync(FULL_MASK, ia, d), xb = __shfl_up_sync(FULL_MASK, ib, d);
            if (lane >= (uint32_t)d) { ia += xa; ib += xb; }
        }
        if (lane == 31) { s_wa[warp] = ia; s_wb[warp] = ib; }
        __syncthreads();
        unsigned long long oa = 0, ob = 0;
        for (int w = 0; w < warp; ++w) { oa += s_wa[w]; ob += s_wb[w]; }
        const unsigned long long ea = oa + ia - (va[0] + va[1]), eb = ob + ib - (vb[0] + vb[1]);     // exclusive, first of the pair
        if (2 * t < SMALL_MAX_TILES) { s_a[2 * t] = ea; s_b[2 * t] = eb; }
        if (2 * t + 1 < SMALL_MAX_TILES) { s_a[2 * t + 1] = ea + va[0]; s_b[2 * t + 1] = eb + vb[0]; }
        if (t == SMALL_WARPS * 32 - 1) { s_tot[0] = oa + ia; s_tot[1] = ob + ib; }
        if (t == 0) s_bB = -1;
        __syncthreads();
    }
    if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 6 + 4] = plan_timer();
    const long long R = (long long)(s_tot[0] & 0xFFFFFFFFull), LC = (long long)(s_tot[0] >> 32);
    const unsigned long long T = s_tot[1] & 0xFFFFFFFFull;
    const int n_tiles = (int)(s_tot[1] >> 32);                   // super-tiles with at least one record
    const bool overflow = R > a.cap_steps || LC > a.cap_leaves;
    const unsigned long long RW = (unsigned long long)sa.rec_weight;
    const unsigned long long W = T + RW * (unsigned long long)R;
    auto wblock = [&](int i) -> unsigned long long { return (s_b[i] & 0xFFFFFFFFull) + RW * (s_a[i] & 0xFFFFFFFFull); };
    // ---- region B (plan_order_kernel's rule, at block granularity): where it begins
    int bB = ntiles;
    // (a grid in groups is a large product: no layered tail there)
    const int tail_records = gsz > 1 ? 0 : (sa.tail_records >= 0 ? sa.tail_records : (R < 3ll * sa.num_teams ? 3 : 0));
    // room in the plan: region B (only plans that use it) may take all unit slots but one round of pieces
    const int64_t b_room = tail_records > 0 ? (sa.unit_capacity - sa.num_teams) / 5 : 0;
    const int max_b_nodes = (int)(b_room < 0 ? 0 : (b_room < ORDER_MAX_B_NODES ? b_room : ORDER_MAX_B_NODES));
    if (tail_records > 0 && n_tiles > 0 && R > 0 && max_b_nodes >= SMALL_WARPS && !overflow) {
        unsigned long long wB = W * (unsigned long long)sa.tail_percent / 100ull;
        const unsigned long long wmin = W * (unsigned long long)(sa.num_teams + sa.num_teams / 4) / (unsigned long long)n_tiles;
        if (wB < wmin) wB = wmin;
        const unsigned long long targetA = wB >= W ? 0ull : W - wB;
        const int lo = ntiles > max_b_nodes / SMALL_WARPS ? ntiles - max_b_nodes / SMALL_WARPS : 0;       // region B is capped
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            const int i = 2 * t + x;
            if (i < ntiles && (i == lo || (i > lo && wblock(i) <= targetA))) atomicMax(&s_bB, i);
        }
        __syncthreads();
        bB = s_bB;
    }
    const long long RA = bB < ntiles ? (long long)(s_a[bB] & 0xFFFFFFFFull) : R;
    const unsigned long long WA = bB < ntiles ? wblock(bB) : W;
    const int idxB = bB < ntiles ? bB * SMALL_WARPS : n_nodes;
    const int nB = n_nodes - idxB;
    // ---- region A: pieces, one per team, or several rounds of them when the product is large
    long long rounds = RA / ((long long)sa.num_teams * sa.piece_records);
    if (rounds < 1) rounds = 1;
    if (rounds > 64) rounds = 64;
    const int64_t cap_a = sa.unit_capacity - 5ll * max_b_nodes;
    if (rounds * sa.num_teams > cap_a) rounds = cap_a / sa.num_teams;
    const long long P = (RA > 0 && !overflow) ? (rounds >= 1 ? rounds * sa.num_teams : cap_a) : 0;
    int32_t *__restrict__ uw = sa.units;
    // the same function of g in every thread (all that matters); products stay below 2^53
    const double wa_over_p = (double)WA / (double)(P > 0 ? P : 1), p_over_wa = (double)P / (double)(WA > 0 ? WA : 1);
    auto target_of = [&](long long g) -> unsigned long long {
        const unsigned long long x = (unsigned long long)((double)g * wa_over_p);
        return x < 1ull ? 1ull : x;
    };
    auto piece_of = [&](unsigned long long w) -> long long { const long long g = (long long)((double)w * p_over_wa) - 1; return g < 1 ? 1 : g; };
    if (blockIdx.x == 0) {
        // the plan's counts (spamm_b200.h); [16..20] are accumulated below by the blocks of region B
        if (t < 16) {
            int32_t v = 0;
            if (t == 0) v = (int32_t)LC;
            if (t == 1) v = n_tiles;
            if (t == 2) v = overflow ? 1 : 0;
            if (t == 4) v = (int32_t)R;
            if (t == 5) v = (int32_t)(P + 5ll * nB);
            if (t == 6) v = (int32_t)(T & 0xFFFFFFFFull);
            if (t == 7) v = (int32_t)(T >> 32);
            if (t == 11) v = n_nodes;
            if (t == 12) v = (int32_t)P;
            a.out_counts[t] = v;
        }
        if (t == 16) a.out_counts[21] = nB;
        if (t == 17) { a.tile_off[n_nodes] = (int32_t)R; sa.node_info[n_nodes] = T; }
        if (t == 18 && P > 0) {
            uw[0] = 0;                              // piece 0 begins at record 0, at a tile start
            uw[1] = 0;
            uw[4 * (P - 1) + 2] = (int32_t)RA;      // the last piece ends with region A, at a tile end
            uw[4 * (P - 1) + 3] = (int32_t)RA;
        }
    }
    // ---- my node: what plan_count_kernel found, and where its records and leaves go
    unsigned long long info = valid ? __ldcg(sa.node_info + pidx) : 0ull;
    __syncthreads();                                 // every warp has its node's word before any is overwritten
    const uint32_t nsteps = (uint32_t)(info & 0xFFu), present = (uint32_t)((info >> 8) & 0xFFFFu);
    const uint32_t ntasks = (uint32_t)(info >> 24), nleaves = __popc(present);
    if (lane == 0) { s_wa[warp] = nsteps | ((unsigned long long)nleaves << 32); s_wb[warp] = ntasks; }
    __syncthreads();
    unsigned long long oa = s_a[blockIdx.x / gsz], ob = s_b[blockIdx.x / gsz] & 0xFFFFFFFFull;
    for (int j = (int)(blockIdx.x / gsz) * gsz; j < (int)blockIdx.x; ++j) {        // the blocks of my group before me
        oa += __ldcg(sa.agg_a + j);
        ob += __ldcg(sa.agg_b + j) & 0xFFFFFFFFull;
    }
    for (int w = 0; w < warp; ++w) { oa += s_wa[w]; ob += s_wb[w]; }
    int64_t sb = (int64_t)(oa & 0xFFFFFFFFull);
    const int64_t cb = (int64_t)(oa >> 32);
    if (valid && lane == 0) {
        a.tile_off[pidx] = (int32_t)sb;
        sa.node_info[pidx] = ob;                     // tasks before this node (tile_wprefix)
    }
    if (!valid || nsteps == 0 || overflow) {
        if (a.trace && lane == 0) atomicMax(a.trace + blockIdx.x * 6 + 5, plan_timer());
        return;
    }
    const int ts = (int)sb, te = (int)sb + (int)nsteps;
    // ---- region B: layered segments of this node (lane 0), slots by one atomic per range
    if (pidx >= idxB) {
        if (lane == 0) {
            const int sl = tail_records > 0 ? tail_records : 1;
            const int ns = te - ts;
            const int nseg = ns <= sl ? 1 : (ns <= 2 * sl ? 2 : 3);
            int sbeg = ts;
#pragma unroll
            for (int x = 0; x < 5; ++x) {
                const int l = x < 3 ? 0 : x - 2;
                const bool in = x < 3 ? nseg == 3 - x : nseg > l;
                if (!in) continue;
                const int slot = atomicAdd(&a.out_counts[16 + x], 1);
                const int se = l + 1 == nseg ? te : (l == 0 ? te - (nseg - 1) * sl : sbeg + sl);
                *reinterpret_cast<int4 *>(uw + 4 * (P + (long long)x * nB + slot)) =
                    make_int4(sbeg, sbeg == ts ? sbeg : te, se == te ? se : ts, se);
                sbeg = se;
            }
        }
    }
    // does a cut of region A fall into this tile?  (cut g sits behind the first record at which the weight
    // prefix reaches target(g))
    const unsigned long long w0 = ob + RW * (unsigned long long)ts;
    const unsigned long long w1 = w0 + ntasks + RW * (unsigned long long)nsteps;
    bool cuts = false;
    if (pidx < idxB && P > 1 && !(sa.dbg & 1)) {
        long long g0 = piece_of(w0);
        while (g0 < P && target_of(g0) <= w0) ++g0;
        cuts = g0 < P && target_of(g0) <= w1;
    }
    // ---- product leaf keys and step records, in ascending K (plan_tiles_kernel's phase 3)
    if (lane < 16 && (present >> lane & 1u))
        a.c_keys[cb + __popc(present & ((1u << lane) - 1u))] = (uint32_t)pidx * (uint32_t)(sub * sub) + lane;
    const int64_t s_first = sb, s_last = sb + nsteps - 1;
    const uint32_t lt = lanemask_lt();
    const uint32_t lead_mask = (sub == 4 ? 0x11111111u : sub == 2 ? 0x55555555u : 0xFFFFFFFFu);
    unsigned long long run = w0;
    LaneNorms nrm = tile_norms(a, I, J, ((int)lane / sub < e) ? sub * ks[(int)lane / sub] + kk : 0u, (int)lane / sub < e);
    for (int b = 0; b < e; b += per) {
        const int tt = b + (int)lane / sub, t2 = tt + per;
        const LaneNorms nxt = tile_norms(a, I, J, t2 < e ? sub * ks[t2] + kk : 0u, t2 < e);
        LaneTests lt4{0u, 0u, 0u, 0u, 0u};
        uint32_t K = 0;
        if (tt < e) {
            K = ks[tt];
            lt4 = tile_tests<true>(a, nrm, rowok, I, J, (uint32_t)sub * K + kk);
        }
        nrm = nxt;
        uint32_t live4[4] = {0, 0, 0, 0}, dead4[4] = {0, 0, 0, 0}, a_present = 0, b_present = 0, any = 0;
        int a_best = 16, b_best = 16;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const int src = (int)grp + (x < sub ? x : 0);
            const uint32_t lv = __shfl_sync(FULL_MASK, lt4.live | (lt4.full << 16), src);
            const uint32_t dd = __shfl_sync(FULL_MASK, lt4.dead, src);
            const uint32_t ah = __shfl_sync(FULL_MASK, lt4.a_here, src);
            const uint32_t bh = __shfl_sync(FULL_MASK, lt4.b_here, src);
            if (x < sub) {
                live4[x] = lv;
                dead4[x] = dd;
                any |= lv & 0xFFFFu;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    if (ah >> d & 1u) { a_present |= 1u << step_pos(d, x); }
                    if (bh >> d & 1u) { b_present |= 1u << step_pos(x, d); }
                }
            }
        }
        if (a_present) a_best = __ffs(a_present) - 1;
        if (b_present) b_best = __ffs(b_present) - 1;
        const bool writer = any != 0 && lane == grp;
        const uint32_t bal = __ballot_sync(FULL_MASK, writer);
        const int64_t x = sb + __popc(bal & lt);
        if (writer) {
            uint32_t flags = 0;
            if (x == s_first) flags |= STEP_FIRST;
            if (x == s_last) flags |= STEP_LAST;
            const uint32_t a_first = (uint32_t)__ldg(
                a.slot_a + (int64_t)(sub * I + step_pos_di(a_best)) * a.L + (sub * K + step_pos_dj(a_best)));
            const uint32_t b_first = (uint32_t)__ldg(
                a.slot_bt + (int64_t)(sub * J + step_pos_dj(b_best)) * a.L + (sub * K + step_pos_di(b_best)));
            uint4 *rec = reinterpret_cast<uint4 *>(a.steps + x);
            rec[0] = make_uint4(K, flags, (uint32_t)cb, (uint32_t)pidx);
            rec[1] = make_uint4(a_first, a_present, b_first, b_present);
            rec[2] = make_uint4(live4[0], live4[1], live4[2], live4[3]);
            rec[3] = make_uint4(present, dead4[0] | (dead4[1] << 16), dead4[2] | (dead4[3] << 16),
                                nsteps | ((uint32_t)(x - s_first) << 16));
        }
        if (cuts) {
            // weight prefix behind every record of this pass, in record order (the writers, ascending lanes)
            const unsigned long long wr = writer ? RW + __popc(live4[0] & 0xFFFFu) + __popc(live4[1] & 0xFFFFu) +
                                                       __popc(live4[2] & 0xFFFFu) + __popc(live4[3] & 0xFFFFu) : 0ull;
            unsigned long long inc = wr;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long y = __shfl_up_sync(FULL_MASK, inc, d);
                if (lane >= (uint32_t)d) inc += y;
            }
            const unsigned long long hi_w = run + inc, lo_w = hi_w - wr;
            if (writer) {
                long long g = piece_of(lo_w);
                while (g < P && target_of(g) <= lo_w) ++g;
                for (; g < P && target_of(g) <= hi_w; ++g) {
                    const int c = (int)x + 1;                 // the cut: in (ts, te]
                    uw[4 * g] = c;
                    uw[4 * g + 1] = te;
                    uw[4 * (g - 1) + 2] = c == te ? c : ts;
                    uw[4 * (g - 1) + 3] = c;
                }
            }
            run += __shfl_sync(FULL_MASK, inc, 31);
        }
        sb += __popc(bal & lead_mask);
    }
    if (a.trace && lane == 0) atomicMax(a.trace + blockIdx.x * 6 + 5, plan_timer());
}

// ---- host side ---------------------------------------------------------------------------------
int spamm_execute_piece_base();     // pieces per round = teams of the numeric kernel (execute.cu)

static int plan_env(const char *name, int dflt, int lo, int hi)
{
    int v = dflt;
    if (const char *e = getenv(name)) v = atoi(e);
    return v < lo ? lo : (v > hi ? hi : v);
}
static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct PlanWorkspace {
    PlanShared *shared;
    unsigned long long *tile_state[PLAN_MAX_LEVELS + 1];   // per parent level
    unsigned long long *tile_state_w;                      // second look-back of the last stage (task prefix)
    unsigned long long *tile_wprefix;                      // tasks before each super-tile node
    LevelBuf buf[2];
    size_t zero_bytes;                // prefix of the workspace that must be cleared per plan
    size_t total;
};

static PlanWorkspace carve(void *ws, int64_t list_cap, int64_t node_cap)
{
    PlanWorkspace w;
    char *p = reinterpret_cast<char *>(ws);
    size_t o = 0;
    w.shared = reinterpret_cast<PlanShared *>(p + o);
    o = align_up(o + sizeof(PlanShared), 256);
    for (int lvl = 0; lvl <= PLAN_MAX_LEVELS; ++lvl) {   // a level has at most min(4^lvl, node_cap) nodes
        int64_t nodes = (lvl < 15) ? (int64_t(1) << (2 * lvl)) : node_cap;
        if (nodes > node_cap) nodes = node_cap;
        w.tile_state[lvl] = reinterpret_cast<unsigned long long *>(p + o);
        o = align_up(o + sizeof(unsigned long long) * (size_t)((nodes + PLAN_WARPS - 1) / PLAN_WARPS + 1), 256);
    }
    w.tile_state_w = reinterpret_cast<unsigned long long *>(p + o);
    o = align_up(o + sizeof(unsigned long long) * (size_t)((node_cap + PLAN_WARPS - 1) / PLAN_WARPS + 1), 256);
    w.zero_bytes = o;
    w.tile_wprefix = reinterpret_cast<unsigned long long *>(p + o);
    o = align_up(o + sizeof(unsigned long long) * (size_t)(node_cap + 2), 256);
    for (int x = 0; x < 2; ++x) {
        w.buf[x].node = reinterpret_cast<uint32_t *>(p + o);
        o = align_up(o + 4 * (size_t)(node_cap + 1), 256);
        w.buf[x].off = reinterpret_cast<int32_t *>(p + o);
        o = align_up(o + 4 * (size_t)(node_cap + 2), 256);
        w.buf[x].ks = reinterpret_cast<uint32_t *>(p + o);
        o = align_up(o + 4 * (size_t)(list_cap + 1), 256);
    }
    w.total = o;
    return w;
}

// Surviving tasks per row of product leaves: what the multi-GPU split balances (rows of C are
// handed to ranks in contiguous blocks of about equal task count).
__global__ void plan_row_counts_kernel(const spamm_step *__restrict__ steps, const int32_t *__restrict__ counts,
                                       int sub_shift, int32_t *__restrict__ row_tasks)
{
    const int nsteps = counts[2] ? 0 : counts[4];
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nsteps; s += gridDim.x * blockDim.x) {
        const uint4 head = *reinterpret_cast<const uint4 *>(steps + s);
        const uint4 live = *(reinterpret_cast<const uint4 *>(steps + s) + 2);
        uint32_t ti, tj;
        morton_decode(head.w, ti, tj);
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const uint32_t m = step_rowmask(d);
            const int c = __popc(live.x & m) + __popc(live.y & m) + __popc(live.z & m) + __popc(live.w & m);
            if (c) atomicAdd(&row_tasks[(ti << sub_shift) + d], c);
        }
    }
}

extern "C" int spamm_plan_row_counts(const spamm_plan_buffers *plan, int depth, int32_t *row_tasks, void *stream)
{
    if (!plan || !row_tasks || depth < 0 || depth > 15) return SPAMM_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(row_tasks, 0, sizeof(int32_t) << depth, st) != cudaSuccess) return SPAMM_ECUDA;
    plan_row_counts_kernel<<<SPAMM_NUM_SMS * 4, 256, 0, st>>>(plan->steps, plan->counts, depth >= 2 ? 2 : depth, row_tasks);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

extern "C" size_t spamm_plan_workspace_bytes(int depth, int64_t step_capacity, int64_t leaf_capacity)
{
    (void)depth;
    return carve(nullptr, step_capacity, leaf_capacity).total;
}

// bytes at the start of the workspace that must be zero when the planner starts
size_t spamm_plan_zero_bytes(int64_t step_capacity, int64_t leaf_capacity)
{
    return carve(nullptr, step_capacity, leaf_capacity).zero_bytes;
}

// prezeroed: the caller has already cleared that region and out->counts on the stream
int spamm_plan_impl(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int32_t row0, int32_t row1,
                    const spamm_plan_buffers *out, void *ws, size_t ws_bytes, bool prezeroed,
                    const spamm_product_buffers *cgrid, uint32_t **clean_ptr, int *clean_words, int fine_weight,
                    void *stream)
{
    if (!a || !b || !out || !ws) return SPAMM_EINVAL;
    if (!(tau >= 0.0)) return SPAMM_EINVAL;                       // NaN or negative (symbolic.py:99-100)
    if (a->depth != b->depth || a->depth < 0 || a->depth > 15) return SPAMM_EINVAL;
    if (out->step_capacity < 1 || out->leaf_capacity < 1 || out->step_capacity >= (int64_t(1) << 31) - 64) return SPAMM_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    PlanWorkspace w = carve(ws, out->step_capacity, out->leaf_capacity);
    if (ws_bytes < w.total) return SPAMM_EWORKSPACE;
    if (!prezeroed && cudaMemsetAsync(ws, 0, w.zero_bytes, st) != cudaSuccess) return SPAMM_ECUDA;

    const int depth = a->depth;
    const int tl = depth >= 2 ? depth - 2 : 0;          // super-tile level
    const int l0 = tl < ROOT_MAX_LEVEL ? tl : ROOT_MAX_LEVEL;   // start level
    int32_t *res = w.shared->res;       // accumulated here, copied to out->counts by the last kernel
    int32_t *overflow = res + 2, *max_list = res + 3;
    int cur = 0;
    const bool dense = tl <= PLAN_DENSE_MAX_LEVEL && out->leaf_capacity >= (int64_t(1) << (2 * tl));
    const int grid = SPAMM_NUM_SMS * 4;
    if (!dense) {
    if (spamm_launch_pdl(plan_root_kernel, dim3(1), dim3(ROOT_THREADS), 0, st, a->norm + spamm_level_offset(l0),
                         b->norm_t + spamm_level_offset(l0), l0, depth - l0, row0, row1, tau, w.buf[cur],
                         w.shared->counts[l0], out->leaf_capacity, out->step_capacity, overflow) != cudaSuccess)
        return SPAMM_ECUDA;
    SPAMM_CHECK_LAUNCH();
    for (int lvl = l0; lvl < tl; ++lvl) {
        ExpandArgs x;
        x.norm_a = a->norm + spamm_level_offset(lvl + 1);
        x.norm_bt = b->norm_t + spamm_level_offset(lvl + 1);
        x.S = 1 << (lvl + 1);
        x.shift = depth - (lvl + 1);
        x.row0 = row0; x.row1 = row1; x.tau = tau;
        x.in = w.buf[cur];
        x.out = w.buf[cur ^ 1];
        x.counts_in = w.shared->counts[lvl];
        x.counts_out = w.shared->counts[lvl + 1];
        x.cap_nodes = out->leaf_capacity; x.cap_tasks = out->step_capacity;
        x.overflow = overflow; x.max_list = max_list;
        x.tile_counter = &w.shared->tile_counter[lvl];
        x.tile_state = w.tile_state[lvl];
        if (spamm_launch_pdl(plan_expand_kernel, dim3(grid), dim3(PLAN_THREADS), 0, st, x) != cudaSuccess) return SPAMM_ECUDA;
        SPAMM_CHECK_LAUNCH();
        cur ^= 1;
    }
    }
    TileArgs t;
    t.trace = nullptr;
    static const char *trace_path = getenv("SPAMM_PLAN_TRACE");      // tuning aid: allocates and synchronises
    // a small dense start (n <= 4096): blocks of 8 nodes, count + emit kernels; else two 1024-thread blocks
    // per SM that draw tiles of 32 nodes from a counter
    static const bool small_off = getenv("SPAMM_PLAN_SMALL") && atoi(getenv("SPAMM_PLAN_SMALL")) == 0;    // tuning aid
    const bool small = dense && !small_off;      // dense: tl <= PLAN_DENSE_MAX_LEVEL = 7, at most 2048 blocks of 8 nodes
    const int tgrid = small ? ((1 << (2 * tl)) + SMALL_WARPS - 1) / SMALL_WARPS : (dense && tl <= 6) ? SPAMM_NUM_SMS : SPAMM_NUM_SMS * 2;
    if (trace_path && cudaMalloc(&t.trace, 8 * 6 * tgrid) == cudaSuccess) cudaMemsetAsync(t.trace, 0, 8 * 6 * tgrid, st);
    t.norm_a_t = a->norm + spamm_level_offset(tl);
    t.norm_bt_t = b->norm_t + spamm_level_offset(tl);
    t.St = 1 << tl;
    t.norm_a = a->norm + spamm_level_offset(depth);
    t.norm_bt = b->norm_t + spamm_level_offset(depth);
    t.slot_a = a->slot;
    t.slot_bt = b->slot_t;
    t.sub_a = (a->sub && b->sub_t) ? a->sub : nullptr;
    t.sub_bt = (a->sub && b->sub_t) ? b->sub_t : nullptr;
    // the pieces are balanced by live tasks whatever the gating; a product that is known to run with coarse16
    // gating (spamm_multiply) skips the classification of its tasks -- a plan without it is still valid for
    // fine4, every task is then gated by the numeric kernel itself
    t.fine_weight = 0;
    if (!fine_weight) t.sub_a = t.sub_bt = nullptr;
    t.L = 1 << depth;
    t.sub = 1 << (depth - tl);
    t.row0 = row0; t.row1 = row1; t.tau = tau;
    t.in = w.buf[cur];
    t.counts_in = w.shared->counts[tl];
    t.steps = out->steps;
    t.c_keys = out->c_keys;
    {
        static int sms = -1;
        if (sms < 0) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        }
        t.all_resident = sms >= tgrid ? 1 : 0;      // 1024 threads x 64 registers: one block per SM
    }
    t.tile_off = out->tile_off;
    t.tile_wprefix = w.tile_wprefix;
    t.tile_state_w = w.tile_state_w;
    t.cap_steps = out->step_capacity; t.cap_leaves = out->leaf_capacity;
    t.counts = res;
    t.out_counts = out->counts;
    t.chain = out->chain;
    t.chain_words = out->leaf_capacity;
    t.cells = 0;
    t.c_slot = t.c_slot_t = nullptr; t.c_norm = t.c_norm_t = nullptr; t.c_leaf_sq_grid = nullptr;
    if (cgrid) {
        const int64_t off = spamm_level_offset(cgrid->depth);
        t.cells = int64_t(1) << (2 * cgrid->depth);
        t.c_slot = cgrid->slot; t.c_slot_t = cgrid->slot_t;
        t.c_norm = cgrid->norm + off; t.c_norm_t = cgrid->norm_t + off;
        t.c_leaf_sq_grid = cgrid->leaf_sq_grid;
    }
    t.tile_counter = &w.shared->tile_counter[PLAN_MAX_LEVELS];
    t.tile_state = w.tile_state[PLAN_MAX_LEVELS];
    // tuning aids: records per piece from which a product is cut into several rounds of pieces,
    // and the weight of a record (in tasks) in the balance
    static const int piece_records = plan_env("SPAMM_PIECE_RECORDS", 192, 1, 1 << 20);
    static const int rec_weight = plan_env("SPAMM_REC_WEIGHT", 32, 1, 256);
    // region B (the layered tail) pays only when the pieces would otherwise be shorter than a super-tile
    // (SPAMM_TAIL_RECORDS = -1: decide by the size of the plan; 0: never; n: always, n records per short segment)
    static const int tail_records = plan_env("SPAMM_TAIL_RECORDS", -1, -1, 64);
    static const int tail_percent = plan_env("SPAMM_TAIL_PERCENT", 25, 0, 100);
    auto dump_trace = [&]() {          // tuning aid (SPAMM_PLAN_TRACE): six time stamps per block
        if (!t.trace) return;
        unsigned long long *h = (unsigned long long *)malloc(8 * 6 * tgrid);
        cudaStreamSynchronize(st);
        cudaMemcpy(h, t.trace, 8 * 6 * tgrid, cudaMemcpyDeviceToHost);
        if (FILE *f = fopen(trace_path, "w")) {
            for (int x = 0; x < tgrid; ++x)
                fprintf(f, "%d %llu %llu %llu %llu %llu %llu\n", x, h[6 * x], h[6 * x + 1], h[6 * x + 2], h[6 * x + 3],
                        h[6 * x + 4], h[6 * x + 5]);
            fclose(f);
        }
        free(h);
        cudaFree(t.trace);
    };
    if (small) {
        // count, then emit + cut: two kernels, no look-back, no separate ordering kernel (see plan_count_kernel)
        SmallArgs sa;
        sa.t = t;
        sa.node_info = w.tile_wprefix;
        sa.agg_a = reinterpret_cast<unsigned long long *>(w.buf[0].node);      // level lists: unused by a dense start
        sa.agg_b = reinterpret_cast<unsigned long long *>(w.buf[1].node);
        sa.group = tgrid > SMALL_MAX_TILES ? (tgrid + SMALL_MAX_TILES - 1) / SMALL_MAX_TILES : 1;
        sa.grp_a = sa.agg_a + tgrid;
        sa.grp_b = sa.agg_b + tgrid;
        // tickets in the part of the workspace that is zero between plans (a look-back array of the other path)
        sa.grp_ticket = reinterpret_cast<unsigned int *>(w.tile_state[PLAN_MAX_LEVELS]);
        sa.units = out->tile_order;
        sa.unit_capacity = spamm_unit_capacity(out->leaf_capacity);
        sa.num_teams = spamm_execute_piece_base(); sa.piece_records = piece_records; sa.rec_weight = rec_weight;
        sa.tail_records = tail_records;
        sa.tail_percent = tail_percent;
        static const int small_dbg = plan_env("SPAMM_PLAN_DEBUG", 0, 0, 3);
        sa.dbg = small_dbg;
        if (small_dbg & 2) sa.t.sub_a = sa.t.sub_bt = nullptr;
        if (spamm_launch_pdl(plan_count_kernel, dim3(tgrid), dim3(SMALL_WARPS * 32), 0, st, sa) != cudaSuccess) return SPAMM_ECUDA;
        SPAMM_CHECK_LAUNCH();
        if (spamm_launch_pdl(plan_emit_kernel, dim3(tgrid), dim3(SMALL_WARPS * 32), 0, st, sa) != cudaSuccess) return SPAMM_ECUDA;
        SPAMM_CHECK_LAUNCH();
        dump_trace();
        if (clean_words) {
            *clean_ptr = reinterpret_cast<uint32_t *>(w.shared);
            *clean_words = cgrid != nullptr ? (int)(offsetof(PlanShared, exec_ticket) / 4) : 0;
        }
        return SPAMM_OK;
    }
    if (spamm_launch_pdl(dense ? plan_tiles_kernel<true, 32> : plan_tiles_kernel<false, 32>,
                         dim3(tgrid), dim3(32 * 32), 0, st, t) != cudaSuccess)
        return SPAMM_ECUDA;
    SPAMM_CHECK_LAUNCH();
    dump_trace();
    OrderArgs oa;
    oa.defer_clean = (cgrid != nullptr && clean_words) ? 1 : 0;
    if (clean_words) {
        *clean_ptr = reinterpret_cast<uint32_t *>(w.shared);
        // everything before exec_ticket: the numeric kernel's teams draw their first piece from it before
        // they wait for this kernel, and the last team to finish leaves it zero
        *clean_words = oa.defer_clean ? (int)(offsetof(PlanShared, exec_ticket) / 4) : 0;
    }
    oa.tile_off = out->tile_off;
    oa.tile_wprefix = w.tile_wprefix;
    oa.steps = out->steps;
    oa.counts = out->counts;
    oa.shared = w.shared;
    {
        const size_t head = align_up(sizeof(PlanShared), 256);
        oa.ws_tail = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(ws) + head);
        oa.ws_tail_words = (int64_t)((w.zero_bytes - head) / 4);
    }
    oa.units = out->tile_order;
    oa.unit_capacity = spamm_unit_capacity(out->leaf_capacity);
    oa.num_teams = spamm_execute_piece_base(); oa.piece_records = piece_records; oa.rec_weight = rec_weight;
    oa.tail_records = tail_records;
    oa.tail_percent = tail_percent;
    if (spamm_launch_pdl(plan_order_kernel, dim3(SPAMM_NUM_SMS), dim3(256), 0, st, oa) != cudaSuccess) return SPAMM_ECUDA;
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

extern "C" int spamm_plan(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int32_t row0, int32_t row1,
                          const spamm_plan_buffers *out, void *ws, size_t ws_bytes, void *stream)
{
    // balanced for the default granularity (fine4, numeric.py:36)
    return spamm_plan_impl(a, b, tau, row0, row1, out, ws, ws_bytes, false, nullptr, nullptr, nullptr, 1, stream);
}
