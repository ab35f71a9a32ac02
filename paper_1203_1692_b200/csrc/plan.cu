// Symbolic phase on the device: the pruned recursion flattened into a compacted task list.
//
// Replaces symbolic.build_plan / convolve (pkg/src/spamm/symbolic.py:92-159).  The task set is
//   { (i,k,j) : leaves A_ik and B_kj stored,  double(|A_ik|) * double(|B_kj|) >= tau }
// (symbolic.py:118-125).  Because every parent norm bounds its children's (norms are the
// correctly rounded square roots of FP64 sums of non-negative terms, core.py:252-266), a
// node product below tau can be dropped at any level without losing a leaf task -- the same
// argument that makes reference.recursive_spamm (reference.py:72-129) equal to the flat plan.
//
// Layout of one level: the product nodes (i,j) that still have candidates, in ascending
// Morton order, each with its ascending list of contraction indices k (CSR).  Going one level
// down, node (i,j) with list {k} yields children (2i+di, 2j+dj) with candidates {2k, 2k+1};
// order is preserved by construction, so the leaf level comes out sorted by product leaf
// (Morton) and ascending k -- the accumulation order the numeric phase needs
// (numeric.py:203-217) -- without any sort.  Survivors are counted with warp ballots and
// placed with a decoupled look-back prefix sum; nothing returns to the host between levels.
#include "common.cuh"

#define PLAN_WARPS 8
#define PLAN_THREADS (PLAN_WARPS * 32)
#define PLAN_MAX_LEVELS 16

struct LevelBuf {
    uint32_t *node;   // Morton index of each active product node
    int32_t *off;     // CSR offsets into ks (one more entry than nodes)
    uint32_t *ks;     // contraction indices
};

struct PlanShared {      // lives at the start of the workspace, zeroed once per plan
    unsigned int tile_counter[PLAN_MAX_LEVELS];
    int32_t counts[PLAN_MAX_LEVELS + 1][2];   // (nodes, candidates) per level
};

struct LeafOut {
    const int32_t *slot_a;     // A grid, row-major (i,k)
    const int32_t *slot_bt;    // B grid transposed (j,k)
    const float *sub_a;
    const float *sub_b;
    uint32_t *task_a, *task_b;
    uint64_t *task_mask;
    int L;
};

// fine4 gate of one task (numeric.py:232-238): bit r*16 + p*4 + q.
__device__ __forceinline__ uint64_t fine_mask(const float *__restrict__ sa, const float *__restrict__ sb, double tau)
{
    float a[16], b[16];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
        float4 va = __ldg(reinterpret_cast<const float4 *>(sa) + x);
        float4 vb = __ldg(reinterpret_cast<const float4 *>(sb) + x);
        a[4 * x] = va.x; a[4 * x + 1] = va.y; a[4 * x + 2] = va.z; a[4 * x + 3] = va.w;
        b[4 * x] = vb.x; b[4 * x + 1] = vb.y; b[4 * x + 2] = vb.z; b[4 * x + 3] = vb.w;
    }
    uint64_t m = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (__dmul_rn((double)a[p * 4 + r], (double)b[r * 4 + q]) >= tau) m |= 1ull << (r * 16 + p * 4 + q);
    return m;
}

template <bool FINE>
__device__ __forceinline__ void emit_leaf_task(const LeafOut &lo, int64_t pos, uint32_t i, uint32_t k, uint32_t j,
                                               double tau)
{
    const int32_t sa = lo.slot_a[(int64_t)i * lo.L + k];
    const int32_t sb = lo.slot_bt[(int64_t)j * lo.L + k];
    lo.task_a[pos] = (uint32_t)sa;
    lo.task_b[pos] = (uint32_t)sb;
    lo.task_mask[pos] = FINE ? fine_mask(lo.sub_a + (int64_t)sa * 16, lo.sub_b + (int64_t)sb * 16, tau) : ~0ull;
}

// ---- start level: dense enumeration by one block ---------------------------------------
// side = 2^level <= 16, so at most 256 product nodes with at most 16 candidates each.
template <bool LEAF, bool FINE>
__global__ void __launch_bounds__(256) plan_root_kernel(const float *__restrict__ norm_a, const float *__restrict__ norm_bt,
                                                        int level, int shift, int row0, int row1, double tau, LevelBuf out,
                                                        int32_t *counts_out, int64_t cap_nodes, int64_t cap_tasks,
                                                        int32_t *overflow, LeafOut lo)
{
    __shared__ uint32_t s_cnt[256], s_act[256];
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
    const uint32_t cnt = __popc(live);
    s_cnt[c] = cnt;
    s_act[c] = cnt > 0;
    __syncthreads();
    if (c == 0) {   // tiny serial exclusive scan
        uint32_t rc = 0, ra = 0;
        for (int x = 0; x < 256; ++x) {
            uint32_t tc = s_cnt[x], ta = s_act[x];
            s_cnt[x] = rc; s_act[x] = ra;
            rc += tc; ra += ta;
        }
        counts_out[0] = (int32_t)ra;
        counts_out[1] = (int32_t)rc;
        if ((int64_t)ra > cap_nodes || (int64_t)rc > cap_tasks) *overflow = 1;
        else out.off[ra] = (int32_t)rc;
    }
    __syncthreads();
    if (cnt == 0) return;
    const uint32_t an = s_act[c];
    uint32_t kb = s_cnt[c];
    if ((int64_t)an >= cap_nodes || (int64_t)kb + cnt > cap_tasks) return;
    out.node[an] = (uint32_t)c;
    out.off[an] = (int32_t)kb;
    for (int k = 0; k < S; ++k)
        if (live >> k & 1) {
            out.ks[kb] = (uint32_t)k;
            if (LEAF) emit_leaf_task<FINE>(lo, kb, i, (uint32_t)k, j, tau);
            ++kb;
        }
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
    LeafOut lo;
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

template <bool LEAF, bool FINE>
__global__ void __launch_bounds__(PLAN_THREADS) plan_expand_kernel(ExpandArgs a)
{
    __shared__ int s_tile;
    __shared__ uint32_t s_wtasks[PLAN_WARPS], s_wact[PLAN_WARPS];
    __shared__ uint32_t s_base_lo, s_base_hi;
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const int n_nodes = a.counts_in[0];
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
            // children rows 2pi, 2pi+1 against the kept leaf-row range
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
        if (threadIdx.x == 0) {
            uint32_t rt = 0, ra = 0;
            for (int w = 0; w < PLAN_WARPS; ++w) {
                uint32_t vt = s_wtasks[w], va = s_wact[w];
                s_wtasks[w] = rt; s_wact[w] = ra;
                rt += vt; ra += va;
            }
            uint32_t ex_lo, ex_hi;
            lb_exclusive(a.tile_state, tile, rt, ra, ex_lo, ex_hi);
            s_base_lo = ex_lo;
            s_base_hi = ex_hi;
            if (tile == ntiles - 1) {
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
        if (nb + wact > a.cap_nodes || kb + wtasks > a.cap_tasks) {   // flagged by the last tile too
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
                const uint32_t ci = 2 * pi + (c >> 1), cj = 2 * pj + (c & 1);
                if (p0) {
                    a.out.ks[pos] = 2 * k;
                    if (LEAF) emit_leaf_task<FINE>(a.lo, pos, ci, 2 * k, cj, a.tau);
                    ++pos;
                }
                if (p1) {
                    a.out.ks[pos] = 2 * k + 1;
                    if (LEAF) emit_leaf_task<FINE>(a.lo, pos, ci, 2 * k + 1, cj, a.tau);
                }
                base[c] += __popc(b0) + __popc(b1);
            }
        }
    }
}

// ---- host side ---------------------------------------------------------------------------------
static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct PlanWorkspace {
    PlanShared *shared;
    unsigned long long *tile_state[PLAN_MAX_LEVELS];   // per parent level
    LevelBuf buf[2];
    size_t zero_bytes;                // prefix of the workspace that must be cleared per plan
    size_t total;
};

static PlanWorkspace carve(void *ws, int64_t task_cap, int64_t leaf_cap)
{
    PlanWorkspace w;
    char *p = reinterpret_cast<char *>(ws);
    size_t o = 0;
    w.shared = reinterpret_cast<PlanShared *>(p + o);
    o = align_up(o + sizeof(PlanShared), 256);
    for (int lvl = 0; lvl < PLAN_MAX_LEVELS; ++lvl) {   // a level has at most min(4^lvl, leaf_cap) nodes
        int64_t nodes = (lvl < 15) ? (int64_t(1) << (2 * lvl)) : leaf_cap;
        if (nodes > leaf_cap) nodes = leaf_cap;
        w.tile_state[lvl] = reinterpret_cast<unsigned long long *>(p + o);
        o = align_up(o + sizeof(unsigned long long) * (size_t)((nodes + PLAN_WARPS - 1) / PLAN_WARPS + 1), 256);
    }
    w.zero_bytes = o;
    for (int x = 0; x < 2; ++x) {
        w.buf[x].node = reinterpret_cast<uint32_t *>(p + o);
        o = align_up(o + 4 * (size_t)(leaf_cap + 1), 256);
        w.buf[x].off = reinterpret_cast<int32_t *>(p + o);
        o = align_up(o + 4 * (size_t)(leaf_cap + 2), 256);
        w.buf[x].ks = reinterpret_cast<uint32_t *>(p + o);
        o = align_up(o + 4 * (size_t)(task_cap + 1), 256);
    }
    w.total = o;
    return w;
}

extern "C" size_t spamm_plan_workspace_bytes(int depth, int64_t task_capacity, int64_t leaf_capacity)
{
    (void)depth;
    return carve(nullptr, task_capacity, leaf_capacity).total;
}

template <bool FINE>
static int run_plan(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int32_t row0, int32_t row1,
                    const spamm_plan_buffers *out, const PlanWorkspace &w, cudaStream_t st)
{
    const int depth = a->depth;
    const int L = 1 << depth;
    LeafOut lo{a->slot, b->slot_t, a->sub4, b->sub4, out->task_a, out->task_b, out->task_mask, L};
    LevelBuf final_buf{out->c_keys, out->c_off, out->task_k};
    int32_t *overflow = out->counts + 2, *max_list = out->counts + 3;
    const int l0 = depth == 0 ? 0 : (depth - 1 < 4 ? depth - 1 : 4);
    int cur = 0;
    {
        const float *na = a->norm + spamm_level_offset(l0), *nbt = b->norm_t + spamm_level_offset(l0);
        if (depth == 0) {
            plan_root_kernel<true, FINE><<<1, 256, 0, st>>>(na, nbt, 0, 0, row0, row1, tau, final_buf, out->counts,
                                                           out->leaf_capacity, out->task_capacity, overflow, lo);
            SPAMM_CHECK_LAUNCH();
            return SPAMM_OK;
        }
        plan_root_kernel<false, FINE><<<1, 256, 0, st>>>(na, nbt, l0, depth - l0, row0, row1, tau, w.buf[cur],
                                                        w.shared->counts[l0], out->leaf_capacity, out->task_capacity,
                                                        overflow, lo);
        SPAMM_CHECK_LAUNCH();
    }
    for (int lvl = l0; lvl < depth; ++lvl) {
        const bool last = (lvl + 1 == depth);
        ExpandArgs x;
        x.norm_a = a->norm + spamm_level_offset(lvl + 1);
        x.norm_bt = b->norm_t + spamm_level_offset(lvl + 1);
        x.S = 1 << (lvl + 1);
        x.shift = depth - (lvl + 1);
        x.row0 = row0; x.row1 = row1; x.tau = tau;
        x.in = w.buf[cur];
        x.out = last ? final_buf : w.buf[cur ^ 1];
        x.counts_in = w.shared->counts[lvl];
        x.counts_out = last ? out->counts : w.shared->counts[lvl + 1];
        x.cap_nodes = out->leaf_capacity; x.cap_tasks = out->task_capacity;
        x.overflow = overflow; x.max_list = max_list;
        x.tile_counter = &w.shared->tile_counter[lvl];
        x.tile_state = w.tile_state[lvl];
        x.lo = lo;
        const int grid = SPAMM_NUM_SMS * 4;
        if (last) plan_expand_kernel<true, FINE><<<grid, PLAN_THREADS, 0, st>>>(x);
        else plan_expand_kernel<false, FINE><<<grid, PLAN_THREADS, 0, st>>>(x);
        SPAMM_CHECK_LAUNCH();
        cur ^= 1;
    }
    return SPAMM_OK;
}

extern "C" int spamm_plan(const spamm_tree_view *a, const spamm_tree_view *b, double tau, int granularity, int32_t row0,
                          int32_t row1, const spamm_plan_buffers *out, void *ws, size_t ws_bytes, void *stream)
{
    if (!a || !b || !out || !ws) return SPAMM_EINVAL;
    if (!(tau >= 0.0)) return SPAMM_EINVAL;                       // NaN or negative (symbolic.py:99-100)
    if (a->depth != b->depth || a->depth < 0 || a->depth > 15) return SPAMM_EINVAL;
    if (granularity != SPAMM_FINE4 && granularity != SPAMM_COARSE16) return SPAMM_EINVAL;
    if (out->task_capacity < 1 || out->leaf_capacity < 1 || out->task_capacity >= (int64_t(1) << 31) - 64) return SPAMM_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    PlanWorkspace w = carve(ws, out->task_capacity, out->leaf_capacity);
    if (ws_bytes < w.total) return SPAMM_EWORKSPACE;
    if (cudaMemsetAsync(ws, 0, w.zero_bytes, st) != cudaSuccess) return SPAMM_ECUDA;
    if (cudaMemsetAsync(out->counts, 0, 4 * sizeof(int32_t), st) != cudaSuccess) return SPAMM_ECUDA;
    return granularity == SPAMM_FINE4 ? run_plan<true>(a, b, tau, row0, row1, out, w, st)
                                      : run_plan<false>(a, b, tau, row0, row1, out, w, st);
}
