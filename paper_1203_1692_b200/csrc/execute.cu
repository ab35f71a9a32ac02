// Numeric phase on the device: the leaf-block products of a plan.
//
// Replaces numeric.execute_plan / _run_batched / _compose (pkg/src/spamm/numeric.py:138-284):
// for every product leaf, its tasks are accumulated in ascending k; inside a task the 4x4x4
// micro products run for r = 0..3, kk ascending, and micro product (p,q,r) is skipped when
// double(subA[p][r]) * double(subB[r][q]) < tau (fine4, numeric.py:232-259).  One thread owns one
// 4x4 sub-block (p,q) of one product leaf for the whole super-tile, so every C element has a
// single owner and a fixed summation order: results are identical run to run and, in EXACT mode
// (separately rounded multiply and add), bit-identical to the reference.
//
// Work unit: a super-tile of 4x4 product leaves, described by the plan's step records, one per
// contraction block K: C[I,J] += A[I,K] B[K,J] on 4x4 blocks of leaves, with 4 x 16 live-task
// bits.  The stored leaves of a block are contiguous in the packed arrays (Morton order), so the
// producer warp stages each block with ONE bulk copy (TMA 1-D, cp.async.bulk, SASS UBLKCP; up to
// 17 KB: 16 leaf records of 1088 B holding values and sub-block norms) into a ring of
// shared-memory stages guarded by mbarriers.  Eight consumer warps (two product leaves each)
// gate and multiply from shared memory; with fine4 a tenth warp first classifies the tasks of each
// stage (all 64 micro products run / none / undecided).  The persistent CTAs (two per SM) claim work
// units from an atomic counter: whole super-tiles, or -- when the product has few of them -- chained
// segments of a super-tile's records whose accumulators pass from CTA to CTA through C's value
// records (plan_format.cuh, spamm_b200.h).  Launched with programmatic dependent launch.
// Tuning aids: SPAMM_EX_STAGES, SPAMM_EX_CTAS, SPAMM_EX_DEBUG, SPAMM_EX_TRACE (per-CTA time stamps).
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "plan_format.cuh"

#define EX_MAX_STAGES 6
#define EX_CONSUMERS 8
#define EX_THREADS (32 * (EX_CONSUMERS + 1))          // coarse16: consumers + producer
#define EX_THREADS_FINE (32 * (EX_CONSUMERS + 2))     // fine4: + the classifier warp
#define EX_EXIT (1u << 31)
#define EX_CHAIN_IN (1u << 30)    // first step of a later segment: accumulators come from C's records
#define EX_CHAIN_OUT (1u << 29)   // last step of a segment that is not the tile's last: hand them on
#define EX_PREFETCH 4
#define EX_BLOCK_BYTES (16 * SPAMM_REC_BYTES)     // one 4x4 block of leaf records

struct __align__(16) StageDesc {
    uint32_t live[4];      // live tasks per kk (one 16-byte read)
    uint32_t flags;        // STEP_FIRST | STEP_LAST | EX_EXIT | EX_CHAIN_*
    uint32_t c_base;
    uint32_t present;      // product leaves of the super-tile
    uint32_t a_present;    // stored leaves of the staged A block, bit morton4(di,kk)
    uint32_t b_present;    // stored leaves of the staged B block, bit morton4(kk,dj)
    uint32_t tile;         // Morton index of the super-tile
    uint32_t seg;          // segment of the tile this step belongs to
    uint32_t pad;
    // fine4, written by the classifier warp: tasks whose 64 micro products all run / none runs,
    // bit morton4(di,dj) + 16 * (kk & 1) of word kk >> 1
    uint32_t full[2];
    uint32_t dead[2];
};

struct ExecArgs {
    const float *a_values_t;
    const float *b_values;
    const spamm_step *steps;
    const int32_t *tile_off;     // step offset of every super-tile node, one extra entry
    const int32_t *tile_order;   // work units (node | segment << 24) in hand-out order
    const int32_t *counts;       // plan counts (device): [5] = number of units, [12] = records per segment
    int32_t *chain;              // finished segments per product leaf (zeroed before the launch)
    unsigned int *tile_counter;
    double tau;
    float alpha;
    int alpha_is_one;
    float *c_values, *c_values_t;
    double *c_leaf_sq;
    unsigned long long *counters;
    // optional: the leaf-level grids of C (spamm_product_buffers); the epilogue then indexes the
    // product leaves itself (slot, norm and square sum of leaf (i,j)), replacing spamm_index_leaves
    int32_t *c_slot, *c_slot_t;
    float *c_norm, *c_norm_t;
    double *c_sq_grid;
    int c_L;                     // side of C's leaf grid
    int sub2;                    // leaves per super-tile (16; 4 or 1 for tiny trees)
    int nstages;                 // depth of the shared-memory ring
    int static_first;            // every CTA of the grid is resident: CTA b may take unit b without asking
    int32_t *error_flag;         // plan counts[15]: set when a hand-over wait gives up (never in a correct run)
    uint32_t *clean_ptr;         // the planner's shared state, returned to zero here on behalf of the planner
    int clean_words;             // (spamm_multiply; 0 otherwise)
    int dbg;                     // tuning aid (SPAMM_EX_DEBUG): 1 = no copies, 2 = no math
    unsigned long long *trace;   // tuning aid (SPAMM_EX_TRACE): per CTA start / first data / end / units
};

__device__ __forceinline__ unsigned long long global_timer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double ex_row_sq(float4 v)
{
    double x = v.x, y = v.y, z = v.z, w = v.w;
    double r = __dmul_rn(x, x);
    r = __fma_rn(y, y, r);
    r = __fma_rn(z, z, r);
    r = __fma_rn(w, w, r);
    return r;
}

// Two C elements of one column (rows 2h, 2h+1) advance together: packed FP32 (sm_100 FFMA2 with a
// broadcast scalar operand) halves the issue slots the multiply-accumulates take.  EXACT rounds the
// product and the sum separately (numeric.py:252-259) with scalar FMUL + FADD.
template <bool EXACT>
__device__ __forceinline__ void mac2(float2 &acc, float2 a, float b)
{
    if (EXACT) {   // scalar: nvcc 12.9 contracts __fmul2_rn + __fadd2_rn into one FFMA2
        acc.x = __fadd_rn(acc.x, __fmul_rn(a.x, b));
        acc.y = __fadd_rn(acc.y, __fmul_rn(a.y, b));
    } else {
        acc = __ffma2_rn(a, make_float2(b, b), acc);
    }
}

template <bool EXACT, bool FINE>
#ifndef EX_MIN_BLOCKS
#define EX_MIN_BLOCKS 2
#endif
__global__ void __launch_bounds__(EX_THREADS_FINE, EX_MIN_BLOCKS) execute_kernel(ExecArgs g)
{
    // dynamic shared memory: nstages x (A block + B block), then descriptors and barriers
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nstages = g.nstages;
    unsigned char *sA = smem_raw;
    unsigned char *sB = smem_raw + (size_t)nstages * EX_BLOCK_BYTES;
    StageDesc *desc = reinterpret_cast<StageDesc *>(smem_raw + (size_t)nstages * 2 * EX_BLOCK_BYTES);
    uint64_t *full_bar = reinterpret_cast<uint64_t *>(desc + EX_MAX_STAGES);
    uint64_t *empty_bar = full_bar + EX_MAX_STAGES;
    uint64_t *ready_bar = empty_bar + EX_MAX_STAGES;      // fine4: the stage's tasks are classified

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    pdl_enter();
    if (blockIdx.x == 0)
        for (int x = threadIdx.x; x < g.clean_words; x += blockDim.x) g.clean_ptr[x] = 0u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nstages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], EX_CONSUMERS);
            mbar_init(&ready_bar[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    int stage = 0;
    uint32_t phase = 0;
    if (g.trace && threadIdx.x == 0) g.trace[blockIdx.x * 4] = global_timer();

    if (warp == EX_CONSUMERS) {
        // ============ producer: stream step records, stage leaf blocks with bulk copies ============
        // the first unit is read together with the counts (tile_order always has room for one entry per CTA)
        uint32_t unit_pre = (uint32_t)__ldg(g.tile_order + blockIdx.x);
        const int ntiles = g.counts[2] ? 0 : g.counts[5];      // an overflowed plan is incomplete: do nothing
        const int seg_len = g.counts[12];
        const bool claim_late = ntiles < 16 * (int)gridDim.x;
        const uint32_t *words = reinterpret_cast<const uint32_t *>(g.steps);
        int tile = 0, units_done = 0;
        // With the whole grid resident the first unit needs no hand-out: CTA b takes unit b, the counter
        // hands out the rest.  (Otherwise a unit could wait for a predecessor owned by a CTA that has
        // not started yet, so every unit is claimed.)
        tile = (int)blockIdx.x;
        if (!g.static_first) {
            if (lane == 0) tile = (int)atomicAdd(g.tile_counter, 1u);
            tile = __shfl_sync(FULL_MASK, tile, 0);
        }
        const int claim_base = g.static_first ? (int)gridDim.x : 0;
        while (tile < ntiles) {
            ++units_done;
            const uint32_t unit = unit_pre;
            const int node = seg_len ? (int)(unit & ((1u << UNIT_NODE_BITS) - 1u)) : (int)unit;
            const int seg = seg_len ? (int)((unit >> UNIT_NODE_BITS) & 63u) : 0;
            int beg = g.tile_off[node], end = g.tile_off[node + 1];
            bool chain_in = false, chain_out = false;
            if (seg_len) {      // this unit is one segment of the tile
                const int ns = end - beg, nseg = (int)(unit >> 26);
                end = beg + unit_begin(ns, nseg, seg + 1);
                beg = beg + unit_begin(ns, nseg, seg);
                chain_in = seg > 0;
                chain_out = seg + 1 < nseg;
            }
            // With few units per CTA the next unit is claimed late, two records before the
            // end of this one: its latency still hides behind the staged records, and a CTA never sits
            // on a whole unit it has not started while others run dry.  With many whole tiles it is
            // claimed right away.
            int next_tile = 0;
            if (lane == 0 && !claim_late) next_tile = (int)atomicAdd(g.tile_counter, 1u) + claim_base;
            // lane l < 16 holds word l of a record (struct spamm_step)
            uint32_t w[EX_PREFETCH];
#pragma unroll
            for (int x = 0; x < EX_PREFETCH; ++x)
                w[x] = (lane < 16 && beg + x < end) ? __ldg(words + (size_t)(beg + x) * 16 + lane) : 0u;
            for (int r = beg; r < end; ++r) {
                if (lane == 0 && claim_late && (r + 2 == end || (r == beg && r + 2 > end)))
                    next_tile = (int)atomicAdd(g.tile_counter, 1u) + claim_base;
                const uint32_t cur = w[0];
#pragma unroll
                for (int x = 0; x + 1 < EX_PREFETCH; ++x) w[x] = w[x + 1];
                w[EX_PREFETCH - 1] =
                    (lane < 16 && r + EX_PREFETCH < end) ? __ldg(words + (size_t)(r + EX_PREFETCH) * 16 + lane) : 0u;
                const uint32_t na = __popc(__shfl_sync(FULL_MASK, cur, 5));
                const uint32_t nb = __popc(__shfl_sync(FULL_MASK, cur, 7));
                mbar_wait(&empty_bar[stage], phase ^ 1u);
                uint32_t *d = reinterpret_cast<uint32_t *>(&desc[stage]);
                if (lane == 1)                                   // flags
                    d[4] = cur | (chain_in && r == beg ? EX_CHAIN_IN : 0u) | (chain_out && r + 1 == end ? EX_CHAIN_OUT : 0u);
                if (lane == 13) d[10] = (uint32_t)seg;
                if (lane == 2) d[5] = cur;                       // c_base
                if (lane == 12) d[6] = cur;                      // present
                if (lane == 3) d[9] = cur;                       // tile
                if (lane == 5) d[7] = cur;                       // a_present
                if (lane == 7) d[8] = cur;                       // b_present
                if (lane >= 8 && lane < 12) d[lane - 8] = cur;   // live[kk]
                __syncwarp();
                const bool copy = !(g.dbg & 1);
                if (lane == 0) mbar_arrive_expect_tx(&full_bar[stage], copy ? (na + nb) * SPAMM_REC_BYTES : 0u);
                __syncwarp();
                if (copy && lane == 4)
                    bulk_copy_g2s(sA + (size_t)stage * EX_BLOCK_BYTES, g.a_values_t + (size_t)cur * SPAMM_REC,
                                  na * SPAMM_REC_BYTES, &full_bar[stage]);
                if (copy && lane == 6)
                    bulk_copy_g2s(sB + (size_t)stage * EX_BLOCK_BYTES, g.b_values + (size_t)cur * SPAMM_REC,
                                  nb * SPAMM_REC_BYTES, &full_bar[stage]);
                if (++stage == nstages) { stage = 0; phase ^= 1u; }
            }
            tile = __shfl_sync(FULL_MASK, next_tile, 0);
            if (tile < ntiles) unit_pre = (uint32_t)g.tile_order[tile];
        }
        mbar_wait(&empty_bar[stage], phase ^ 1u);
        if (lane == 0) {
            desc[stage].flags = EX_EXIT;
            mbar_arrive(&full_bar[stage]);
            if (g.trace) g.trace[blockIdx.x * 4 + 3] = (unsigned long long)units_done;
            // the last CTA to run out of units leaves both counters at zero for the next launch
            if (atomicAdd(g.tile_counter + 1, 1u) == gridDim.x - 1) {
                g.tile_counter[0] = 0u;
                g.tile_counter[1] = 0u;
            }
        }
        return;
    }

    if (FINE && warp == EX_CONSUMERS + 1) {
        // ============ classifier warp (fine4) ============
        // Most tasks away from the band edge run all 64 micro products, and some run none.  Both
        // cases follow from the extreme sub-block norms of the two leaves: min(subA) * min(subB) >= tau
        // means every product passes the gate, max(subA) * max(subB) < tau means none does (products
        // of non-negative floats are exact in double and monotone).  Lane l finds the extremes of
        // staged leaf l (A block: lanes 0..15, B block: 16..31); consumers then skip the per-lane
        // gate arithmetic for classified tasks.  A NaN sub-norm leaves the task unclassified.
        for (;;) {
            mbar_wait(&full_bar[stage], phase);
            StageDesc &ds = desc[stage];
            if (ds.flags & EX_EXIT) {
                if (lane == 0) mbar_arrive(&ready_bar[stage]);
                break;
            }
            const uint32_t a_present = ds.a_present, b_present = ds.b_present;
            const uint32_t mine_present = lane < 16 ? a_present : b_present;
            const float *blk = reinterpret_cast<const float *>((lane < 16 ? sA : sB) + (size_t)stage * EX_BLOCK_BYTES);
            float mn = 0.0f, mx = 0.0f;
            bool bad = true;
            if ((lane & 15u) < (uint32_t)__popc(mine_present) && !(g.dbg & 1)) {
                const float4 *tl = reinterpret_cast<const float4 *>(blk + (lane & 15u) * SPAMM_REC + 256);
                const float4 t0 = tl[0], t1 = tl[1], t2 = tl[2], t3 = tl[3];
                mn = fminf(fminf(fminf(t0.x, t0.y), fminf(t0.z, t0.w)), fminf(fminf(t1.x, t1.y), fminf(t1.z, t1.w)));
                mn = fminf(mn, fminf(fminf(fminf(t2.x, t2.y), fminf(t2.z, t2.w)), fminf(fminf(t3.x, t3.y), fminf(t3.z, t3.w))));
                mx = fmaxf(fmaxf(fmaxf(t0.x, t0.y), fmaxf(t0.z, t0.w)), fmaxf(fmaxf(t1.x, t1.y), fmaxf(t1.z, t1.w)));
                mx = fmaxf(mx, fmaxf(fmaxf(fmaxf(t2.x, t2.y), fmaxf(t2.z, t2.w)), fmaxf(fmaxf(t3.x, t3.y), fmaxf(t3.z, t3.w))));
                const float sum = ((t0.x + t0.y) + (t0.z + t0.w)) + ((t1.x + t1.y) + (t1.z + t1.w)) +
                                  ((t2.x + t2.y) + (t2.z + t2.w)) + ((t3.x + t3.y) + (t3.z + t3.w));
                bad = !(sum == sum) || !(sum - sum == 0.0f);      // a NaN or an infinity among the 16 norms
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int kk = 2 * h + (int)(lane >> 4), pos = (int)(lane & 15u);
                const int gi = step_pos_di(pos), gj = step_pos_dj(pos);
                const int ia = __popc(a_present & ((1u << step_pos(gi, kk)) - 1u));
                const int ib = 16 + __popc(b_present & ((1u << step_pos(kk, gj)) - 1u));
                const float mna = __shfl_sync(FULL_MASK, mn, ia), mnb = __shfl_sync(FULL_MASK, mn, ib);
                const float mxa = __shfl_sync(FULL_MASK, mx, ia), mxb = __shfl_sync(FULL_MASK, mx, ib);
                const int bad_a = __shfl_sync(FULL_MASK, (int)bad, ia), bad_b = __shfl_sync(FULL_MASK, (int)bad, ib);
                const bool unk = (bad_a | bad_b) != 0;       // both shuffles unconditionally: all lanes take part
                const bool full = !unk && __dmul_rn((double)mna, (double)mnb) >= g.tau;
                const bool dead = !unk && __dmul_rn((double)mxa, (double)mxb) < g.tau;
                const uint32_t fb = __ballot_sync(FULL_MASK, full), db = __ballot_sync(FULL_MASK, dead);
                if (lane == 0) {
                    ds.full[h] = fb;
                    ds.dead[h] = db;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&ready_bar[stage]);
            if (++stage == nstages) { stage = 0; phase ^= 1u; }
        }
        return;
    }

    // ======================================= consumers =======================================
    // lane = p1 q1 half p0 q0 (bits 4..0).  A 128-bit shared load is served one quarter-warp at a
    // time and quarters only share a wavefront when their banks are disjoint (measured with ncu):
    // with (p1,q1) selecting the quarter, the A fragment (address by p) and the B fragment (address
    // by half,q) each take 2 wavefronts instead of 2 and 4.
    const int half = (lane >> 2) & 1;
    const int p = ((lane >> 4) & 1) << 1 | ((lane >> 1) & 1), q = ((lane >> 3) & 1) << 1 | (lane & 1);
    const int t16 = p * 4 + q;
    const int mypos = 2 * warp + half;
    const int di = step_pos_di(mypos), dj = step_pos_dj(mypos);
    uint32_t executed = 0;
    float2 acc2[2][4];     // acc2[h][j] = C sub-block elements (2h, j) and (2h+1, j)
    bool traced = false;
    for (;;) {
        mbar_wait(FINE ? &ready_bar[stage] : &full_bar[stage], phase);
        const StageDesc &ds = desc[stage];
        const uint32_t flags = ds.flags;
        if (g.trace && threadIdx.x == 0 && !traced) {
            g.trace[blockIdx.x * 4 + 1] = global_timer();
            traced = true;
        }
        if (flags & EX_EXIT) break;
        if (flags & STEP_FIRST) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc2[h][j] = make_float2(0.0f, 0.0f);
        } else if (flags & EX_CHAIN_IN) {
            // continue a tile another CTA started: wait for its segment, then take the partial sums
            // from C's value record (written below under EX_CHAIN_OUT); L1 is bypassed
            const uint32_t present_in = ds.present;
            if ((present_in >> mypos) & 1u) {
                const int64_t cs = (int64_t)ds.c_base + __popc(present_in & ((1u << mypos) - 1u));
                const int want = (int)ds.seg;
                // the predecessor was handed out earlier to a running CTA; the bound only turns a
                // scheduling bug into an error flag instead of a hang
                for (unsigned spins = 0; ld_acquire_gpu(g.chain + cs) < want; ++spins) {
                    __nanosleep(40);
                    if (spins > (1u << 25)) {
                        if (g.error_flag) *g.error_flag = 1;
                        break;
                    }
                }
                // thread t16 keeps its 16 partial sums in registers order at floats [16 t16, 16 t16 + 16)
                const float4 *cv = reinterpret_cast<const float4 *>(g.c_values + cs * SPAMM_REC + 16 * t16);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float4 u = __ldcg(cv + 2 * h), v = __ldcg(cv + 2 * h + 1);
                    acc2[h][0] = make_float2(u.x, u.y);
                    acc2[h][1] = make_float2(u.z, u.w);
                    acc2[h][2] = make_float2(v.x, v.y);
                    acc2[h][3] = make_float2(v.z, v.w);
                }
            }
        }
        const uint32_t a_present = ds.a_present, b_present = ds.b_present;
        const float *Ablk = reinterpret_cast<const float *>(sA + (size_t)stage * EX_BLOCK_BYTES);
        const float *Bblk = reinterpret_cast<const float *>(sB + (size_t)stage * EX_BLOCK_BYTES);
        const uint4 live4 = *reinterpret_cast<const uint4 *>(ds.live);
        uint32_t cls_full[2] = {0u, 0u}, cls_dead[2] = {0u, 0u};
        if (FINE) {
            cls_full[0] = ds.full[0]; cls_full[1] = ds.full[1];
            cls_dead[0] = ds.dead[0]; cls_dead[1] = ds.dead[1];
        }
#pragma unroll     // all four k unrolled: +4-5 % (their addresses become constants), measured
        for (int kk = 0; kk < 4; ++kk) {
            const uint32_t live = kk == 0 ? live4.x : kk == 1 ? live4.y : kk == 2 ? live4.z : live4.w;
            if (!((live >> (2 * warp)) & 3u) || (g.dbg & 2)) continue;
            const bool mine = (live >> mypos) & 1u;
            // leaf (r,c) of a block sits at index popc(present & below(morton4(r,c)))
            const float *As = Ablk + __popc(a_present & ((1u << step_pos(di, kk)) - 1u)) * SPAMM_REC;
            const float *Bs = Bblk + __popc(b_present & ((1u << step_pos(kk, dj)) - 1u)) * SPAMM_REC;
            uint32_t on = 0;       // bit r: micro product (p,q,r) of my task runs
            if (FINE) {
                const uint32_t cbit = 1u << (mypos + 16 * (kk & 1));
                if (mine && (cls_full[kk >> 1] & cbit)) {
                    on = 15u;
                } else if (mine && !(cls_dead[kk >> 1] & cbit)) {
                    const float4 sa = *reinterpret_cast<const float4 *>(As + 256 + 4 * p);   // subA[p][0..3]
                    const float4 sb = *reinterpret_cast<const float4 *>(Bs + 256 + 4 * q);   // subB[0..3][q]
                    on |= (__dmul_rn((double)sa.x, (double)sb.x) >= g.tau) ? 1u : 0u;
                    on |= (__dmul_rn((double)sa.y, (double)sb.y) >= g.tau) ? 2u : 0u;
                    on |= (__dmul_rn((double)sa.z, (double)sb.z) >= g.tau) ? 4u : 0u;
                    on |= (__dmul_rn((double)sa.w, (double)sb.w) >= g.tau) ? 8u : 0u;
                }
                executed += __popc(on);
            } else {
                on = mine ? 15u : 0u;
            }
            // Fast path (the common case away from the band edge): every lane runs all four r or
            // none, so the 16 k of the task form one branch-free block and the compiler overlaps the
            // shared-memory reads of r+1 with the multiplies of r.
            if (__all_sync(FULL_MASK, on == 15u || on == 0u)) {
                if (on) {
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        float4 a[4], b[4];
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            a[x] = *reinterpret_cast<const float4 *>(As + (4 * r + x) * 16 + 4 * p);
                            b[x] = *reinterpret_cast<const float4 *>(Bs + (4 * r + x) * 16 + 4 * q);
                        }
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            const float2 a01 = make_float2(a[x].x, a[x].y), a23 = make_float2(a[x].z, a[x].w);
                            const float bv[4] = {b[x].x, b[x].y, b[x].z, b[x].w};
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                mac2<EXACT>(acc2[0][j], a01, bv[j]);
                                mac2<EXACT>(acc2[1][j], a23, bv[j]);
                            }
                        }
                    }
                }
                continue;
            }
#pragma unroll 1
            for (int r = 0; r < 4; ++r) {
                const bool go = (on >> r) & 1u;
                if (!__any_sync(FULL_MASK, go)) continue;
                if (go) {
                    float4 a[4], b[4];
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        a[x] = *reinterpret_cast<const float4 *>(As + (4 * r + x) * 16 + 4 * p);
                        b[x] = *reinterpret_cast<const float4 *>(Bs + (4 * r + x) * 16 + 4 * q);
                    }
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const float2 a01 = make_float2(a[x].x, a[x].y), a23 = make_float2(a[x].z, a[x].w);
                        const float bv[4] = {b[x].x, b[x].y, b[x].z, b[x].w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            mac2<EXACT>(acc2[0][j], a01, bv[j]);
                            mac2<EXACT>(acc2[1][j], a23, bv[j]);
                        }
                    }
                }
            }
        }
        uint32_t c_base = 0, present = 0, tile_id = 0, seg_done = 0;
        if (flags & (STEP_LAST | EX_CHAIN_OUT)) {
            c_base = ds.c_base;
            tile_id = ds.tile;
            present = ds.present;
            seg_done = ds.seg + 1u;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[stage]);
        if (++stage == nstages) { stage = 0; phase ^= 1u; }
        if (flags & EX_CHAIN_OUT) {
            // hand the partial sums to the CTA that runs the next segment of this tile
            if ((present >> mypos) & 1u) {
                const int64_t cs = (int64_t)c_base + __popc(present & ((1u << mypos) - 1u));
                float4 *cv = reinterpret_cast<float4 *>(g.c_values + cs * SPAMM_REC + 16 * t16);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    __stcg(cv + 2 * h, make_float4(acc2[h][0].x, acc2[h][0].y, acc2[h][1].x, acc2[h][1].y));
                    __stcg(cv + 2 * h + 1, make_float4(acc2[h][2].x, acc2[h][2].y, acc2[h][3].x, acc2[h][3].y));
                }
            }
            __syncwarp();      // the 16 lanes' stores happen before the release below
            if (t16 == 0 && ((present >> mypos) & 1u)) {
                const int64_t cs = (int64_t)c_base + __popc(present & ((1u << mypos) - 1u));
                st_release_gpu(g.chain + cs, (int)seg_done);
            }
            continue;
        }
        if (!(flags & STEP_LAST)) continue;

        // epilogue of the super-tile: alpha scaling (numeric.py:273-275), both leaf layouts with
        // their sub-norm tails, leaf square sum in compute_norms order (core.py:108-116)
        const bool exists = (present >> mypos) & 1u;
        const int64_t cslot = (int64_t)c_base + __popc(present & ((1u << mypos) - 1u));
        float acc[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            acc[0][j] = acc2[0][j].x; acc[1][j] = acc2[0][j].y;
            acc[2][j] = acc2[1][j].x; acc[3][j] = acc2[1][j].y;
        }
        float4 rows[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (!g.alpha_is_one) {
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fmul_rn(g.alpha, acc[i][j]);
            }
            rows[i] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        }
        double S = ex_row_sq(rows[0]);
        S = __dadd_rn(S, ex_row_sq(rows[1]));
        S = __dadd_rn(S, ex_row_sq(rows[2]));
        S = __dadd_rn(S, ex_row_sq(rows[3]));
        // numpy's pairwise order over the 16 sub-sums S[p*4+q]: index bits 3,0,1,2 = lane bits p1,q0,q1,p0
        double tot = __dadd_rn(S, __shfl_xor_sync(FULL_MASK, S, 16));
        tot = __dadd_rn(tot, __shfl_xor_sync(FULL_MASK, tot, 1));
        tot = __dadd_rn(tot, __shfl_xor_sync(FULL_MASK, tot, 8));
        tot = __dadd_rn(tot, __shfl_xor_sync(FULL_MASK, tot, 2));
        if (exists) {
            float *cv = g.c_values + cslot * SPAMM_REC;
            float *ct = g.c_values_t + cslot * SPAMM_REC;
#pragma unroll
            for (int i = 0; i < 4; ++i) *reinterpret_cast<float4 *>(cv + (4 * p + i) * 16 + 4 * q) = rows[i];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                *reinterpret_cast<float4 *>(ct + (4 * q + j) * 16 + 4 * p) =
                    make_float4(acc[0][j], acc[1][j], acc[2][j], acc[3][j]);
            const float sn = (float)sqrt(S);
            cv[256 + q * 4 + p] = sn;
            ct[256 + t16] = sn;
            if (t16 == 0) {
                if (seg_done > 1u) g.chain[cslot] = 0;      // last reader of the flag: leave it clear
                g.c_leaf_sq[cslot] = tot;
                if (g.c_slot) {
                    uint32_t ci, cj;
                    morton_decode(tile_id * (uint32_t)g.sub2 + (uint32_t)mypos, ci, cj);
                    const float nv = (float)sqrt(tot);
                    g.c_slot[(int64_t)ci * g.c_L + cj] = (int32_t)cslot;
                    g.c_slot_t[(int64_t)cj * g.c_L + ci] = (int32_t)cslot;
                    g.c_norm[(int64_t)ci * g.c_L + cj] = nv;
                    g.c_norm_t[(int64_t)cj * g.c_L + ci] = nv;
                    g.c_sq_grid[(int64_t)ci * g.c_L + cj] = tot;
                }
            }
        }
    }
    if (g.trace && threadIdx.x == 0) g.trace[blockIdx.x * 4 + 2] = global_timer();
    if (FINE) {
        executed = __reduce_add_sync(FULL_MASK, executed);
        if (lane == 0 && executed) atomicAdd(g.counters, (unsigned long long)executed);
    }
}

struct ExecTuning { int stages, ctas_per_sm, dbg; };
static ExecTuning exec_tuning();
int spamm_execute_grid()
{
    static const ExecTuning tune = exec_tuning();
    return SPAMM_NUM_SMS * tune.ctas_per_sm;
}
static ExecTuning exec_tuning()
{
    ExecTuning t{3, 2, 0};
    if (const char *e = getenv("SPAMM_EX_STAGES")) t.stages = atoi(e);
    if (const char *e = getenv("SPAMM_EX_CTAS")) t.ctas_per_sm = atoi(e);
    if (const char *e = getenv("SPAMM_EX_DEBUG")) t.dbg = atoi(e);
    if (t.stages < 2) t.stages = 2;
    if (t.stages > EX_MAX_STAGES) t.stages = EX_MAX_STAGES;
    if (t.ctas_per_sm < 1) t.ctas_per_sm = 1;
    return t;
}

int spamm_execute_impl(const spamm_tree_view *a, const spamm_tree_view *b, const spamm_plan_buffers *plan,
                       int64_t nsteps, int64_t nC, double tau, float alpha, int granularity, int exact,
                       float *c_values, float *c_values_t, double *c_leaf_sq, unsigned long long *counters,
                       const spamm_product_buffers *cgrid, uint32_t *clean_ptr, int clean_words, void *stream)
{
    if (!a || !b || !plan || nsteps < -1 || nC < -1) return SPAMM_EINVAL;
    if (granularity != SPAMM_FINE4 && granularity != SPAMM_COARSE16) return SPAMM_EINVAL;
    if (nC == 0 || nsteps == 0) return SPAMM_OK;          // pass -1 when the counts are still on the device
    cudaStream_t st = (cudaStream_t)stream;
    ExecArgs g;
    g.a_values_t = a->values_t;
    g.b_values = b->values;
    g.steps = plan->steps;
    g.tile_off = plan->tile_off;
    g.tile_order = plan->tile_order;
    g.counts = plan->counts;
    g.tile_counter = reinterpret_cast<unsigned int *>(plan->counts + 13);   // [13] hand-out, [14] exited CTAs
    g.chain = plan->chain;
    g.error_flag = plan->counts + 15;
    g.clean_ptr = clean_ptr;
    g.clean_words = clean_words;
    g.tau = tau;
    g.alpha = alpha;
    g.alpha_is_one = (alpha == 1.0f);
    g.c_values = c_values;
    g.c_values_t = c_values_t;
    g.c_leaf_sq = c_leaf_sq;
    g.counters = counters;
    g.c_slot = g.c_slot_t = nullptr;
    g.c_norm = g.c_norm_t = nullptr;
    g.c_sq_grid = nullptr;
    g.c_L = 0;
    {
        const int sub = a->depth >= 2 ? 4 : (1 << a->depth);
        g.sub2 = sub * sub;
    }
    if (cgrid) {
        const int64_t off = spamm_level_offset(cgrid->depth);
        g.c_slot = cgrid->slot;
        g.c_slot_t = cgrid->slot_t;
        g.c_norm = cgrid->norm + off;
        g.c_norm_t = cgrid->norm_t + off;
        g.c_sq_grid = cgrid->leaf_sq_grid;
        g.c_L = 1 << cgrid->depth;
    }
    // counts[13..14] and the chain flags are zero here: spamm_plan clears them and every launch of
    // the kernel leaves them clear again
    static const ExecTuning tune = exec_tuning();
    g.nstages = tune.stages;
    g.dbg = tune.dbg;
    const int grid = SPAMM_NUM_SMS * tune.ctas_per_sm;
    const size_t smem = (size_t)tune.stages * 2 * EX_BLOCK_BYTES + EX_MAX_STAGES * (sizeof(StageDesc) + 24);
    const bool fine = granularity == SPAMM_FINE4;
    void (*kern)(ExecArgs) = exact ? (fine ? execute_kernel<true, true> : execute_kernel<true, false>)
                                   : (fine ? execute_kernel<false, true> : execute_kernel<false, false>);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return SPAMM_ECUDA;
    g.trace = nullptr;
    static const char *trace_path = getenv("SPAMM_EX_TRACE");     // tuning aid: allocates and synchronises
    if (trace_path && cudaMalloc(&g.trace, sizeof(unsigned long long) * 4 * grid) != cudaSuccess) g.trace = nullptr;
    if (g.trace) cudaMemsetAsync(g.trace, 0, sizeof(unsigned long long) * 4 * grid, st);
    {
        // is the whole persistent grid resident at once on this device?
        static int resident[4] = {-1, -1, -1, -1};
        const int which = (exact ? 2 : 0) + (fine ? 1 : 0);
        if (resident[which] < 0) {
            int dev = 0, sms = 0, per_sm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, fine ? EX_THREADS_FINE : EX_THREADS, smem);
            resident[which] = (long long)per_sm * sms >= grid ? 1 : 0;
        }
        g.static_first = resident[which];
    }
    if (spamm_launch_pdl(kern, dim3(grid), dim3(fine ? EX_THREADS_FINE : EX_THREADS), smem, st, g) != cudaSuccess)
        return SPAMM_ECUDA;
    SPAMM_CHECK_LAUNCH();
    if (g.trace) {
        unsigned long long *h = (unsigned long long *)malloc(sizeof(unsigned long long) * 4 * grid);
        cudaStreamSynchronize(st);
        cudaMemcpy(h, g.trace, sizeof(unsigned long long) * 4 * grid, cudaMemcpyDeviceToHost);
        if (FILE *f = fopen(trace_path, "w")) {
            for (int x = 0; x < grid; ++x)
                fprintf(f, "%d %llu %llu %llu %llu\n", x, h[4 * x], h[4 * x + 1], h[4 * x + 2], h[4 * x + 3]);
            fclose(f);
        }
        free(h);
        cudaFree(g.trace);
    }
    return SPAMM_OK;
}

extern "C" int spamm_execute(const spamm_tree_view *a, const spamm_tree_view *b, const spamm_plan_buffers *plan,
                             int64_t nsteps, int64_t nC, double tau, float alpha, int granularity, int exact,
                             float *c_values, float *c_values_t, double *c_leaf_sq, unsigned long long *counters,
                             void *stream)
{
    return spamm_execute_impl(a, b, plan, nsteps, nC, tau, alpha, granularity, exact, c_values, c_values_t, c_leaf_sq,
                              counters, nullptr, nullptr, 0, stream);
}

// ---- beta != 0: union of the old and the produced leaf sets, then _compose ----------------------
#include "scan.cuh"

struct UnionScanOp {
    const int32_t *slot_old, *slot_prod;   // L*L grids, -1 = absent
    uint32_t *keys;
    int32_t *idx_old, *idx_prod;
    int L;
    __device__ __forceinline__ int flag(int64_t e) const
    {
        uint32_t i, j;
        morton_decode((uint32_t)e, i, j);
        const int64_t x = (int64_t)i * L + j;
        return (slot_old[x] >= 0 || slot_prod[x] >= 0) ? 1 : 0;
    }
    __device__ __forceinline__ void emit(int64_t e, int flag, int32_t idx) const
    {
        if (!flag) return;
        uint32_t i, j;
        morton_decode((uint32_t)e, i, j);
        const int64_t x = (int64_t)i * L + j;
        keys[idx] = (uint32_t)e;
        idx_old[idx] = slot_old[x];
        idx_prod[idx] = slot_prod[x];
    }
};

__global__ void fill_i32_kernel(int32_t *p, int64_t n, int32_t v)
{
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) p[x] = v;
}
__global__ void scatter_slots_kernel(const uint32_t *__restrict__ keys, int64_t n, int L, int32_t *slot)
{
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    uint32_t i, j;
    morton_decode(keys[s], i, j);
    slot[(int64_t)i * L + j] = (int32_t)s;
}

extern "C" int spamm_union_leaves(const int32_t *slot_old, const uint32_t *prod_keys, int64_t nprod, int depth,
                                  int32_t *slot_prod_scratch, uint32_t *out_keys, int32_t *idx_old, int32_t *idx_prod,
                                  int32_t *nout_dev, void *ws, size_t ws_bytes, void *stream)
{
    if (depth < 0 || depth > 15 || nprod < 0) return SPAMM_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int L = 1 << depth;
    const int64_t cells = (int64_t)L * L;
    int blocks = (int)((cells + 255) / 256);
    if (blocks > SPAMM_NUM_SMS * 16) blocks = SPAMM_NUM_SMS * 16;
    fill_i32_kernel<<<blocks, 256, 0, st>>>(slot_prod_scratch, cells, -1);
    SPAMM_CHECK_LAUNCH();
    if (nprod > 0) {
        scatter_slots_kernel<<<(unsigned)((nprod + 255) / 256), 256, 0, st>>>(prod_keys, nprod, L, slot_prod_scratch);
        SPAMM_CHECK_LAUNCH();
    }
    UnionScanOp op{slot_old, slot_prod_scratch, out_keys, idx_old, idx_prod, L};
    return scan_flags(op, cells, nout_dev, ws, ws_bytes, st);
}

// out = (alpha32 * prod) + (old * beta32), the reference's expressions (numeric.py:276-284);
// operates on the 256 values of each 272-float leaf record
__global__ void __launch_bounds__(256) compose_kernel(const float *__restrict__ prod, const float *__restrict__ old,
                                                      const int32_t *__restrict__ idx_prod,
                                                      const int32_t *__restrict__ idx_old, float alpha, float beta,
                                                      int alpha_is_one, int beta_is_one, float *__restrict__ out)
{
    const int64_t x = blockIdx.x;
    const int32_t ip = idx_prod[x], io = idx_old[x];
    float v;
    if (io < 0) {
        const float pv = prod[(int64_t)ip * SPAMM_REC + threadIdx.x];
        v = alpha_is_one ? pv : __fmul_rn(alpha, pv);
    } else {
        const float ov = old[(int64_t)io * SPAMM_REC + threadIdx.x];
        v = beta_is_one ? ov : __fmul_rn(ov, beta);
        if (ip >= 0) {
            const float pv = prod[(int64_t)ip * SPAMM_REC + threadIdx.x];
            v = __fadd_rn(alpha_is_one ? pv : __fmul_rn(alpha, pv), v);
        }
    }
    out[x * SPAMM_REC + threadIdx.x] = v;
}

extern "C" int spamm_compose(const float *prod_values, const float *old_values, const int32_t *idx_prod,
                             const int32_t *idx_old, int64_t nout, float alpha, float beta, int alpha_is_one,
                             int beta_is_one, float *out_values, void *stream)
{
    if (nout == 0) return SPAMM_OK;
    if (nout < 0 || !out_values) return SPAMM_EINVAL;
    compose_kernel<<<(unsigned)nout, 256, 0, (cudaStream_t)stream>>>(prod_values, old_values, idx_prod, idx_old, alpha, beta,
                                                                    alpha_is_one, beta_is_one, out_values);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}
