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
// gate and multiply from shared memory; with fine4 the planner has already classified most tasks from
// the sub-norm ranges of their leaves (all 64 micro products run / none / undecided, spamm_step.live
// and .dead), so only band-edge tasks pay for per-lane gate arithmetic.  The persistent CTAs (two per SM) run a
// STATIC partition of the record stream that the planner cut into pieces of equal weight (plan.cu,
// plan_order_kernel); a piece is whole super-tiles plus at most one head and one tail segment of a
// tile shared with the neighbouring piece, whose accumulators pass from team to team through C's
// value records (spamm_b200.h).  One CTA per SM holds TWO TEAMS, each a producer warp, a ring and
// eight consumer warps; team t owns the warps with (warp & 1) == t, i.e. two of the SM's four warp
// schedulers to itself.  (Two co-resident CTAs share every scheduler and the hardware favours one of
// them about 2:1 -- measured -- so equal pieces would not finish together; teams on disjoint schedulers
// have identical resources.)  A team draws its pieces from one counter in stream order: the first
// round is in effect a static assignment, a large product continues dynamically.
// Launched with programmatic dependent launch.
// Tuning aids: SPAMM_EX_STAGES, SPAMM_EX_CTAS, SPAMM_EX_DEBUG, SPAMM_EX_TRACE (per-CTA time stamps).
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "plan_format.cuh"

#define EX_MAX_STAGES 6
#define EX_CONSUMERS 8
#ifndef EX_TEAMS
#define EX_TEAMS 2                                        // teams per CTA; 1 = two independent CTAs per SM instead
#endif
#define EX_THREADS (32 * EX_TEAMS * (EX_CONSUMERS + 1))   // per team: consumers + producer
#define EX_CTAS_PER_SM (EX_TEAMS == 1 ? 2 : 1)
#define EX_EXIT (1u << 31)
#define EX_CHAIN_IN (1u << 30)    // first step of a later segment: accumulators come from C's records
#define EX_CHAIN_OUT (1u << 29)   // last step of a segment that is not the tile's last: hand them on
#define EX_PREFETCH 4
#define EX_BLOCK_BYTES (16 * SPAMM_REC_BYTES)     // one 4x4 block of leaf records
#define EX_TRACE2_RECORDS 96
#ifndef EX_KK_UNROLL
#define EX_KK_UNROLL 4
#endif
#ifndef EX_FINE_ROLLED
#define EX_FINE_ROLLED 1    // fine4: a rolled loop that skips the r no lane of the warp runs
#endif
#define EX_ZERO_BYTES 256      // per team: zeros read in place of gated-off operand sub-blocks

// A stage's descriptor: the step record as it is in the plan (one store per lane of the producer), the
// shared-memory addresses of the staged leaves, and what the producer adds (run flags, record index).
struct __align__(16) StageDesc {
    spamm_step rec;        // kblock, flags, c_base, tile, a_first, a_present, b_first, b_present, live[4], present, dead[2], len|pos
    // shared-memory addresses (32-bit, shared window) of the staged leaves, written by the producer so that
    // the consumers do no index arithmetic: a_leaf[di][kk] = leaf A(di, kk), b_leaf[dj][kk] = leaf B(kk, dj)
    uint32_t a_leaf[4][4];
    uint32_t b_leaf[4][4];
    uint32_t flags;        // rec.flags | EX_EXIT | EX_CHAIN_*
    uint32_t index;        // index of the record in the plan
    uint32_t pad[2];
};

struct ExecArgs {
    const float *a_values_t;
    const float *b_values;
    const spamm_step *steps;
    const int32_t *pieces;       // plan.tile_order: the work units (b, e), see plan_order_kernel
    const int32_t *counts;       // plan counts (device): [12] pieces of region A, [16..21] ranges of region B
    int32_t *chain;              // per product leaf: the record up to which its partial sums are handed on (0 = none)
    unsigned int *ticket;        // [0] pieces drawn, [1] teams that ran out of work; zero between launches
    int ticket_early;            // the tickets are not touched by the preceding kernel: draw before waiting for it
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
    uint32_t producer_nap_ns;    // pause between the producer's polls for a free stage (SPAMM_EX_NAP, ns)
    uint32_t leaf_copy_below;    // copy leaf by leaf when under this many 128ths of a record's leaves are touched (SPAMM_EX_LEAFCOPY)
    int32_t *error_flag;         // plan counts[15]: set when a hand-over wait gives up (never in a correct run)
    uint32_t *clean_ptr;         // the planner's shared state, returned to zero here on behalf of the planner
    int clean_words;             // (spamm_multiply; 0 otherwise)
    unsigned long long *gates;   // optional (spamm_execute_gates): the 64 gate bits of every task as evaluated HERE
    int dbg;                     // tuning aid (SPAMM_EX_DEBUG): 1 = no copies, 2 = no math
    unsigned long long *trace;   // tuning aid (SPAMM_EX_TRACE): per CTA start / first data / end / units
    long long *trace2;           // tuning aid (SPAMM_EX_TRACE2): SM clock of every warp of team 0 of CTA 0 at the
                                 // points of its first EX_TRACE2_RECORDS records (consumers: wait begin, data
                                 // ready, math done; producer: stage free, copies issued)
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

// generic pointer to a 32-bit shared-window address
__device__ __forceinline__ const float *shared_ptr(uint32_t addr)
{
    return reinterpret_cast<const float *>(__cvta_shared_to_generic((size_t)addr));
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

// DBG: the instantiation with the tuning aids (time stamps, gate evidence, SPAMM_EX_DEBUG switches); the
// product path runs the one without them, which keeps their state out of the hot loop's registers.
template <bool EXACT, bool FINE, bool DBG>
__global__ void __launch_bounds__(EX_THREADS, EX_CTAS_PER_SM) execute_kernel(ExecArgs g)
{
    // dynamic shared memory, per team: nstages x (A block + B block), descriptors, barriers
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nstages = g.nstages;
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    // Teams on disjoint warp schedulers: warp w runs on scheduler w % 4, so the even warps (team 0)
    // have schedulers 0 and 2 to themselves and the odd warps (team 1) schedulers 1 and 3.
    const int team = EX_TEAMS == 1 ? 0 : (warp & 1);
    const int vwarp = EX_TEAMS == 1 ? warp : (warp >> 1);          // 0 .. 7 consumers, 8 = the team's producer
    const size_t team_bytes = (size_t)nstages * 2 * EX_BLOCK_BYTES + EX_MAX_STAGES * (sizeof(StageDesc) + 16) + EX_ZERO_BYTES;
    static_assert(sizeof(StageDesc) == 208 && sizeof(spamm_step) == 64, "StageDesc layout");
    static_assert((EX_MAX_STAGES * (sizeof(StageDesc) + 16) + EX_ZERO_BYTES) % 16 == 0 && EX_BLOCK_BYTES % 128 == 0,
                  "the second team's buffers must stay aligned for the bulk copies");
    unsigned char *tbase = smem_raw + (size_t)team * team_bytes;
    unsigned char *sA = tbase;
    unsigned char *sB = tbase + (size_t)nstages * EX_BLOCK_BYTES;
    StageDesc *desc = reinterpret_cast<StageDesc *>(tbase + (size_t)nstages * 2 * EX_BLOCK_BYTES);
    uint64_t *full_bar = reinterpret_cast<uint64_t *>(desc + EX_MAX_STAGES);
    uint64_t *empty_bar = full_bar + EX_MAX_STAGES;
    // zeros that stand in for the operand sub-blocks of a gated-off micro product (fine4)
    const float *zeros = reinterpret_cast<const float *>(empty_bar + EX_MAX_STAGES);

    // everything that does not depend on the preceding kernel comes before the wait for it
    if (vwarp == EX_CONSUMERS && lane == 0) {
        for (int s = 0; s < nstages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], EX_CONSUMERS);
        }
        fence_barrier_init();
    }
    if (vwarp == EX_CONSUMERS) {
        float *z = const_cast<float *>(zeros);
        for (int x = (int)lane; x < EX_ZERO_BYTES / 4; x += 32) z[x] = 0.0f;
    }
    // First piece: pieces are drawn from one counter, in stream order.  A team only ever waits for
    // partial sums of the piece before one of its own, which was drawn earlier by a team that is
    // running and begins with the segment in question: no assumption about residency or dispatch order.
    int piece = 0;
    if (vwarp == EX_CONSUMERS && g.ticket_early) {
        if (lane == 0) piece = (int)atomicAdd(g.ticket, 1u);
        piece = __shfl_sync(FULL_MASK, piece, 0);
    }
    pdl_enter();
    if (blockIdx.x == 0)
        for (int x = threadIdx.x; x < g.clean_words; x += blockDim.x) g.clean_ptr[x] = 0u;
    __syncthreads();
    int stage = 0;
    uint32_t phase = 0;
    const int trace_slot = (int)blockIdx.x * EX_TEAMS + team;
    if (DBG && g.trace && vwarp == 0 && lane == 0) g.trace[trace_slot * 4] = global_timer();

    if (vwarp == EX_CONSUMERS) {
        // ============ producer: stream step records, stage leaf blocks with bulk copies ============
        // the plan's counts are requested before the ticket so that the two round trips overlap
        const int c_over = g.counts[2], c_pieces = g.counts[12], stride = g.counts[21];
        int nr[5];
#pragma unroll
        for (int x = 0; x < 5; ++x) nr[x] = g.counts[16 + x];
        if (!g.ticket_early) {
            if (lane == 0) piece = (int)atomicAdd(g.ticket, 1u);
            piece = __shfl_sync(FULL_MASK, piece, 0);
        }
        const bool plan_ok = c_over == 0;                       // an overflowed plan is incomplete: do nothing
        // unit slots: region A's pieces [0, P), then region B's five ranges, range x at P + x * stride with nr[x] in use
        const int P = plan_ok ? c_pieces : 0;
#pragma unroll
        for (int x = 0; x < 5; ++x) nr[x] = plan_ok ? nr[x] : 0;
        const int first_piece = piece;
        const uint32_t *words = reinterpret_cast<const uint32_t *>(g.steps);
        const int4 *units = reinterpret_cast<const int4 *>(g.pieces);
        auto slot_of = [&](int t) -> int {          // claim number -> unit slot, -1 = no work left
            if (t < P) return t;
            t -= P;
#pragma unroll
            for (int x = 0; x < 5; ++x) {
                if (t < nr[x]) return P + x * stride + t;
                t -= nr[x];
            }
            return -1;
        };
        // Cursor over the records of my units.  A unit [b, e) is run as: the head segment [me, e) of a tile
        // that the next unit finishes, the whole tiles [mb, me), the tail segment [b, mb) of a tile another
        // unit began; the planner stores with b and e where b's tile ends and where the tile of e - 1 starts.
        // The next unit is claimed in two steps while the last records of the current one are fetched
        // (counter, unit), so that neither latency is exposed.
        int run = 2, r = 0, rend = 0, rbeg = 0, left = 0, units_done = 0;
        int ub = 0, umb = 0, ume = 0, ue = 0;
        int cstate = 1, tk = piece;               // 0: nothing claimed, 1: counter drawn, 3: unit loaded, 4: no work left
        int4 nu = make_int4(0, 0, 0, 0);
        bool more = true;
        auto claim_step = [&]() {
            if (cstate == 0) {
                if (lane == 0) tk = (int)atomicAdd(g.ticket, 1u);
                cstate = 1;
            } else if (cstate == 1) {
                const int slot = slot_of(__shfl_sync(FULL_MASK, tk, 0));
                if (slot < 0) cstate = 4;
                else { nu = __ldg(units + slot); cstate = 3; }
            }
        };
        // fetch: the next record of the cursor -> (word of lane l < 16, meta); meta = rec | first << 30 | last << 31, ~0 = none
        auto fetch = [&](uint32_t &wd, uint32_t &meta) {
            if (left > 3 && r + 1 < rend) {        // the common case: well inside a run, nothing to claim yet
                wd = lane < 16 ? __ldg(words + (size_t)r * 16 + lane) : 0u;
                meta = (uint32_t)r | (r == rbeg ? (1u << 30) : 0u);
                ++r;
                --left;
                return;
            }
            for (;;) {
                if (!more) { wd = 0u; meta = 0xFFFFFFFFu; return; }
                if (cstate < 3 && left <= 2 - cstate) claim_step();
                if (r < rend) break;
                ++run;
                if (run == 3) {
                    while (cstate < 3) claim_step();
                    if (cstate == 4) { more = false; continue; }
                    ub = nu.x; ue = nu.w;
                    umb = ue > ub ? min(nu.y, ue) : ub;
                    ume = ue > ub ? max(nu.z, umb) : ue;
                    left = ue - ub;
                    cstate = 0;
                    run = 0;
                    ++units_done;
                }
                if (run == 0) { r = ume; rend = ue; }
                else if (run == 1) { r = umb; rend = ume; }
                else { r = ub; rend = umb; }
                rbeg = r;
            }
            wd = lane < 16 ? __ldg(words + (size_t)r * 16 + lane) : 0u;
            meta = (uint32_t)r | (r == rbeg ? (1u << 30) : 0u) | (r + 1 == rend ? (1u << 31) : 0u);
            ++r;
            --left;
        };
        uint32_t w[EX_PREFETCH], m[EX_PREFETCH];
        int prec = 0;
#pragma unroll
        for (int x = 0; x < EX_PREFETCH; ++x) fetch(w[x], m[x]);
        while (m[0] != 0xFFFFFFFFu) {
            const uint32_t cur = w[0], meta = m[0];
#pragma unroll
            for (int x = 0; x + 1 < EX_PREFETCH; ++x) { w[x] = w[x + 1]; m[x] = m[x + 1]; }
            fetch(w[EX_PREFETCH - 1], m[EX_PREFETCH - 1]);
            const uint32_t ap = __shfl_sync(FULL_MASK, cur, 5), bp = __shfl_sync(FULL_MASK, cur, 7);   // a_present, b_present
            const bool t2p = DBG && g.trace2 && blockIdx.x == 0 && team == 0 && prec < EX_TRACE2_RECORDS && lane == 0;
            if (t2p) g.trace2[(prec * 9 + 8) * 4 + 0] = clock64();
            mbar_wait_relaxed(&empty_bar[stage], phase ^ 1u, g.producer_nap_ns);
            if (t2p) g.trace2[(prec * 9 + 8) * 4 + 1] = clock64();
            uint32_t *d = reinterpret_cast<uint32_t *>(&desc[stage]);
            if (lane < 16) d[lane] = cur;                    // the record itself
            if (lane == 1) {                                 // flags: a run that starts or ends inside a tile is chained
                uint32_t f = cur;
                if ((meta >> 30 & 1u) && !(cur & STEP_FIRST)) f |= EX_CHAIN_IN;
                if ((meta >> 31 & 1u) && !(cur & STEP_LAST)) f |= EX_CHAIN_OUT;
                d[48] = f;
                d[49] = meta & 0x3FFFFFFFu;                  // record index
            }
            // leaf (r,c) of a block sits at index popc(present & below(morton4(r,c))); lane l < 16 is leaf
            // A(x, kk), lane l >= 16 leaf B(kk, x)
            const int x = (int)(lane & 15u) >> 2, kk = (int)(lane & 3u);
            const uint32_t idx = lane < 16 ? __popc(ap & ((1u << step_pos(x, kk)) - 1u))
                                           : __popc(bp & ((1u << step_pos(kk, x)) - 1u));
            unsigned char *dst = (lane < 16 ? sA : sB) + (size_t)stage * EX_BLOCK_BYTES + (size_t)idx * SPAMM_REC_BYTES;
            d[16 + lane] = smem_u32(dst);
            // a leaf is touched when one of the tasks of its row (A) or column (B) of the super-tile runs at kk
            uint32_t lv = __shfl_sync(FULL_MASK, cur, 8 + kk) & 0xFFFFu;
            if (FINE) lv &= ~(__shfl_sync(FULL_MASK, cur, 13 + (kk >> 1)) >> ((kk & 1) * 16));
            const uint32_t sel = lane < 16 ? 0x0033u << (((x >> 1) << 3) | ((x & 1) << 1)) : 0x0505u << (((x >> 1) << 2) | (x & 1));
            const bool touched = (lv & sel) != 0u;
            const uint32_t ntouched = __popc(__ballot_sync(FULL_MASK, touched));
            const uint32_t a_first = __shfl_sync(FULL_MASK, cur, 4), b_first = __shfl_sync(FULL_MASK, cur, 6);
            const bool copy = !(DBG && (g.dbg & 1));
            const uint32_t na = __popc(ap), nb = __popc(bp);
            // two copies of the whole blocks when most of their leaves are touched, else one copy per touched leaf
            const bool per_leaf = ntouched * 128u < (na + nb) * g.leaf_copy_below;
            if (lane == 0) mbar_arrive_expect_tx(&full_bar[stage], copy ? (per_leaf ? ntouched : na + nb) * SPAMM_REC_BYTES : 0u);
            __syncwarp();
            if (copy && per_leaf) {
                if (touched)
                    bulk_copy_g2s(dst, (lane < 16 ? g.a_values_t + (size_t)a_first * SPAMM_REC : g.b_values + (size_t)b_first * SPAMM_REC) +
                                           (size_t)idx * SPAMM_REC, SPAMM_REC_BYTES, &full_bar[stage]);
            } else if (copy) {
                if (lane == 4)
                    bulk_copy_g2s(sA + (size_t)stage * EX_BLOCK_BYTES, g.a_values_t + (size_t)cur * SPAMM_REC,
                                  na * SPAMM_REC_BYTES, &full_bar[stage]);
                if (lane == 6)
                    bulk_copy_g2s(sB + (size_t)stage * EX_BLOCK_BYTES, g.b_values + (size_t)cur * SPAMM_REC,
                                  nb * SPAMM_REC_BYTES, &full_bar[stage]);
            }
            if (t2p) g.trace2[(prec * 9 + 8) * 4 + 2] = clock64();
            ++prec;
            if (++stage == nstages) { stage = 0; phase ^= 1u; }
        }
        mbar_wait_relaxed(&empty_bar[stage], phase ^ 1u, g.producer_nap_ns);
        if (lane == 0) {
            desc[stage].flags = EX_EXIT;
            mbar_arrive(&full_bar[stage]);
            if (DBG && g.trace) g.trace[trace_slot * 4 + 3] = (unsigned long long)units_done | ((unsigned long long)first_piece << 32);
            // the last team to run out of work leaves both counters at zero for the next launch
            if (atomicAdd(g.ticket + 1, 1u) == gridDim.x * EX_TEAMS - 1) {
                g.ticket[0] = 0u;
                g.ticket[1] = 0u;
            }
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
    const int mypos = 2 * vwarp + half;
    const int di = step_pos_di(mypos), dj = step_pos_dj(mypos);
    uint32_t executed = 0;
    float2 acc2[2][4];     // acc2[h][j] = C sub-block elements (2h, j) and (2h+1, j)
    bool traced = false;
    bool chained = false;  // the sums of the current tile came (partly) from another CTA
    int crec = 0;
    for (;;) {
        const bool t2c = DBG && g.trace2 && blockIdx.x == 0 && team == 0 && crec < EX_TRACE2_RECORDS && lane == 0;
        if (t2c) g.trace2[(crec * 9 + vwarp) * 4 + 0] = clock64();
        mbar_wait(&full_bar[stage], phase);
        if (t2c) g.trace2[(crec * 9 + vwarp) * 4 + 1] = clock64();
        const StageDesc &ds = desc[stage];
        const uint32_t flags = ds.flags;
        if (DBG && g.trace && vwarp == 0 && lane == 0 && !traced) {
            g.trace[trace_slot * 4 + 1] = global_timer();
            traced = true;
        }
        if (flags & EX_EXIT) break;
        if (flags & STEP_FIRST) {
            chained = false;
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc2[h][j] = make_float2(0.0f, 0.0f);
        } else if (flags & EX_CHAIN_IN) {
            chained = true;
            // continue a tile another CTA started: wait for its segment, then take the partial sums
            // from C's value record (written below under EX_CHAIN_OUT); L1 is bypassed
            const uint32_t present_in = ds.rec.present;
            if ((present_in >> mypos) & 1u) {
                const int64_t cs = (int64_t)ds.rec.c_base + __popc(present_in & ((1u << mypos) - 1u));
                const int want = (int)ds.index;    // the records before this one are in the partial sums
                // the predecessor belongs to a CTA that started earlier and runs it first; the bound
                // only turns a scheduling bug into an error flag instead of a hang
                for (unsigned spins = 0; ld_acquire_gpu(g.chain + cs) != want; ++spins) {
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
        // where my A leaves (row di) and B leaves (column dj) of the four k sit in shared memory
        const uint4 a_at = *reinterpret_cast<const uint4 *>(ds.a_leaf[di]);
        const uint4 b_at = *reinterpret_cast<const uint4 *>(ds.b_leaf[dj]);
        const uint4 live4 = *reinterpret_cast<const uint4 *>(ds.rec.live);
        uint32_t dead01 = 0u, dead23 = 0u;
        if (FINE) {
            dead01 = ds.rec.dead[0];
            dead23 = ds.rec.dead[1];
        }
        constexpr int kk_unroll = EX_KK_UNROLL;
#pragma unroll kk_unroll     // all four k unrolled: +4-5 % (their addresses become constants), measured
        for (int kk = 0; kk < 4; ++kk) {
            const uint32_t lw = kk == 0 ? live4.x : kk == 1 ? live4.y : kk == 2 ? live4.z : live4.w;
            // fine4: a task the planner found dead runs no micro product (and counts none)
            const uint32_t dead = FINE && !(DBG && (g.dbg & 8)) ? ((kk < 2 ? dead01 : dead23) >> (16 * (kk & 1))) : 0u;
            const uint32_t live = lw & 0xFFFFu & ~dead;
            if (!((live >> (2 * vwarp)) & 3u) || (DBG && (g.dbg & 2))) continue;
            const bool mine = (live >> mypos) & 1u;
            const float *As = shared_ptr(kk == 0 ? a_at.x : kk == 1 ? a_at.y : kk == 2 ? a_at.z : a_at.w);
            const float *Bs = shared_ptr(kk == 0 ? b_at.x : kk == 1 ? b_at.y : kk == 2 ? b_at.z : b_at.w);
            uint32_t on = 0;       // bit r: micro product (p,q,r) of my task runs
            if (FINE) {
                if (mine && (((lw >> (16 + mypos)) & 1u) || (DBG && (g.dbg & 4)))) {
                    on = 15u;
                } else if (mine) {
                    const float4 sa = *reinterpret_cast<const float4 *>(As + 256 + 4 * p);   // subA[p][0..3]
                    const float4 sb = *reinterpret_cast<const float4 *>(Bs + 256 + 4 * q);   // subB[0..3][q]
                    on |= (__dmul_rn((double)sa.x, (double)sb.x) >= g.tau) ? 1u : 0u;
                    on |= (__dmul_rn((double)sa.y, (double)sb.y) >= g.tau) ? 2u : 0u;
                    on |= (__dmul_rn((double)sa.z, (double)sb.z) >= g.tau) ? 4u : 0u;
                    on |= (__dmul_rn((double)sa.w, (double)sb.w) >= g.tau) ? 8u : 0u;
                }
                executed += __popc(on);
                if (DBG && g.gates && ((lw >> mypos) & 1u)) {
                    // evidence for the tests: bit r*16 + p*4 + q of the task's word (numeric.py:233-238)
                    unsigned long long bits = 0ull;
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if ((on >> r) & 1u) bits |= 1ull << (r * 16 + t16);
                    if (bits) atomicOr(g.gates + ((size_t)ds.index * 64 + kk * 16 + mypos), bits);
                }
            } else {
                on = mine ? 15u : 0u;
            }
            // One multiply-accumulate block per r: 4 k of the leaf product.  A lane whose micro product
            // (p,q,r) is gated off reads zeros in place of both operand sub-blocks, so the warp stays
            // converged and the sums it keeps are unchanged (x + 0*0 = x; only a -0 would become +0).
            auto micro = [&](const float *ar, const float *br) {
                float4 a[4], b[4];
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    a[x] = *reinterpret_cast<const float4 *>(ar + x * 16);
                    b[x] = *reinterpret_cast<const float4 *>(br + x * 16);
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
            };
            if (!FINE) {
                // every lane runs all four r or none: one branch-free block, the compiler overlaps the
                // shared-memory reads of r+1 with the multiplies of r
                if (on) {
#pragma unroll
                    for (int r = 0; r < 4; ++r) micro(As + 64 * r + 4 * p, Bs + 64 * r + 4 * q);
                }
                continue;
            }
            const uint32_t onany = __reduce_or_sync(FULL_MASK, on);      // r that some lane of the warp runs
            if (onany == 15u || !EX_FINE_ROLLED) {
                if (!EX_FINE_ROLLED && !onany) continue;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const bool go = (on >> r) & 1u;
                    micro(go ? As + 64 * r + 4 * p : zeros, go ? Bs + 64 * r + 4 * q : zeros);
                }
                continue;
            }
#pragma unroll 1
            for (int r = 0; r < 4; ++r) {
                if (!((onany >> r) & 1u)) continue;
                const bool go = (on >> r) & 1u;
                micro(go ? As + 64 * r + 4 * p : zeros, go ? Bs + 64 * r + 4 * q : zeros);
            }
        }
        uint32_t c_base = 0, present = 0, tile_id = 0, seg_done = 0;
        if (flags & (STEP_LAST | EX_CHAIN_OUT)) {
            c_base = ds.rec.c_base;
            tile_id = ds.rec.tile;
            present = ds.rec.present;
            seg_done = ds.index + 1u;
        }
        __syncwarp();
        if (t2c) g.trace2[(crec * 9 + vwarp) * 4 + 2] = clock64();
        ++crec;
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
                if (chained) g.chain[cslot] = 0;            // last reader of the flag: leave it clear
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
    if (DBG && g.trace && vwarp == 0 && lane == 0) g.trace[trace_slot * 4 + 2] = global_timer();
    if (FINE) {
        executed = __reduce_add_sync(FULL_MASK, executed);
        if (lane == 0 && executed) atomicAdd(g.counters, (unsigned long long)executed);
    }
}

struct ExecTuning { int stages, ctas_per_sm, dbg, nap, leaf_copy; };
static ExecTuning exec_tuning();
int spamm_execute_grid()
{
    static const ExecTuning tune = exec_tuning();
    return SPAMM_NUM_SMS * tune.ctas_per_sm;
}
// teams that draw pieces at the start of the kernel: the planner cuts one round of that many pieces
int spamm_execute_piece_base() { return spamm_execute_grid() * EX_TEAMS; }
static ExecTuning exec_tuning()
{
    ExecTuning t{3, EX_CTAS_PER_SM, 0, 256, 96};
    if (const char *e = getenv("SPAMM_EX_STAGES")) t.stages = atoi(e);
    if (const char *e = getenv("SPAMM_EX_CTAS")) t.ctas_per_sm = atoi(e);
    if (const char *e = getenv("SPAMM_EX_DEBUG")) t.dbg = atoi(e);
    if (const char *e = getenv("SPAMM_EX_NAP")) t.nap = atoi(e);
    if (const char *e = getenv("SPAMM_EX_LEAFCOPY")) t.leaf_copy = atoi(e);
    if (t.nap < 0) t.nap = 0;
    if (t.leaf_copy < 0) t.leaf_copy = 0;
    if (t.stages < 2) t.stages = 2;
    if (t.stages > EX_MAX_STAGES) t.stages = EX_MAX_STAGES;
    if (t.ctas_per_sm < 1) t.ctas_per_sm = 1;
    return t;
}

int spamm_execute_impl(const spamm_tree_view *a, const spamm_tree_view *b, const spamm_plan_buffers *plan,
                       int64_t nsteps, int64_t nC, double tau, float alpha, int granularity, int exact,
                       float *c_values, float *c_values_t, double *c_leaf_sq, unsigned long long *counters,
                       const spamm_product_buffers *cgrid, uint32_t *clean_ptr, int clean_words, void *stream,
                       unsigned long long *gates = nullptr)
{
    if (!a || !b || !plan || nsteps < -1 || nC < -1) return SPAMM_EINVAL;
    if (granularity != SPAMM_FINE4 && granularity != SPAMM_COARSE16) return SPAMM_EINVAL;
    if (nC == 0 || nsteps == 0) return SPAMM_OK;          // pass -1 when the counts are still on the device
    cudaStream_t st = (cudaStream_t)stream;
    ExecArgs g;
    g.a_values_t = a->values_t;
    g.b_values = b->values;
    g.steps = plan->steps;
    g.pieces = plan->tile_order;
    g.counts = plan->counts;
    // pieces drawn and teams finished: in the planner's workspace when the call comes from spamm_multiply
    // (untouched by the preceding kernel, so the first piece can be drawn early), else plan counts [13..14]
    g.ticket = clean_ptr ? clean_ptr + clean_words : reinterpret_cast<unsigned int *>(plan->counts + 13);
    g.ticket_early = clean_ptr ? 1 : 0;
    g.chain = plan->chain;
    g.error_flag = plan->counts + 15;
    g.clean_ptr = clean_ptr;
    g.clean_words = clean_words;
    g.gates = gates;
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
    g.producer_nap_ns = (uint32_t)tune.nap;
    g.leaf_copy_below = (uint32_t)tune.leaf_copy;
    g.dbg = tune.dbg;
    const int grid = SPAMM_NUM_SMS * tune.ctas_per_sm;
    const size_t smem = EX_TEAMS * ((size_t)tune.stages * 2 * EX_BLOCK_BYTES + EX_MAX_STAGES * (sizeof(StageDesc) + 16) + EX_ZERO_BYTES);
    const bool fine = granularity == SPAMM_FINE4;
    static const char *trace2_path = getenv("SPAMM_EX_TRACE2");   // tuning aids: allocate and synchronise
    static const char *trace_path = getenv("SPAMM_EX_TRACE");
    const bool dbg = !exact && (gates || trace_path || trace2_path || tune.dbg);
    void (*kern)(ExecArgs) = exact ? (fine ? execute_kernel<true, true, false> : execute_kernel<true, false, false>)
                             : dbg ? (fine ? execute_kernel<false, true, true> : execute_kernel<false, false, true>)
                                   : (fine ? execute_kernel<false, true, false> : execute_kernel<false, false, false>);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return SPAMM_ECUDA;
    g.trace = nullptr;
    g.trace2 = nullptr;
    const size_t trace2_words = (size_t)EX_TRACE2_RECORDS * 9 * 4;
    if (trace2_path && cudaMalloc(&g.trace2, 8 * trace2_words) == cudaSuccess) cudaMemsetAsync(g.trace2, 0, 8 * trace2_words, st);
    const int nslots = grid * EX_TEAMS;
    if (trace_path && cudaMalloc(&g.trace, sizeof(unsigned long long) * 4 * nslots) != cudaSuccess) g.trace = nullptr;
    if (g.trace) cudaMemsetAsync(g.trace, 0, sizeof(unsigned long long) * 4 * nslots, st);
    if (spamm_launch_pdl(kern, dim3(grid), dim3(EX_THREADS), smem, st, g) != cudaSuccess)
        return SPAMM_ECUDA;
    SPAMM_CHECK_LAUNCH();
    if (g.trace2) {
        long long *h = (long long *)malloc(8 * trace2_words);
        cudaStreamSynchronize(st);
        cudaMemcpy(h, g.trace2, 8 * trace2_words, cudaMemcpyDeviceToHost);
        if (FILE *f = fopen(trace2_path, "w")) {
            for (size_t x = 0; x < trace2_words; x += 4) fprintf(f, "%zu %zu %lld %lld %lld\n", x / 36, (x / 4) % 9, h[x], h[x + 1], h[x + 2]);
            fclose(f);
        }
        free(h);
        cudaFree(g.trace2);
    }
    if (g.trace) {
        unsigned long long *h = (unsigned long long *)malloc(sizeof(unsigned long long) * 4 * nslots);
        cudaStreamSynchronize(st);
        cudaMemcpy(h, g.trace, sizeof(unsigned long long) * 4 * nslots, cudaMemcpyDeviceToHost);
        if (FILE *f = fopen(trace_path, "w")) {
            for (int x = 0; x < nslots; ++x)
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

// The same run, additionally reporting the gate the kernel evaluated: gates[(record * 64) + kk * 16 +
// morton4(di,dj)] |= the 64 bits (r*16 + p*4 + q) of that task's micro products that ran.  `gates`
// holds 64 words per step record and must be zero when the call is enqueued.  Test evidence for the
// device-side gate (numeric.py:233-238); not used by the product path.
extern "C" int spamm_execute_gates(const spamm_tree_view *a, const spamm_tree_view *b, const spamm_plan_buffers *plan,
                                   int64_t nsteps, int64_t nC, double tau, float *c_values, float *c_values_t,
                                   double *c_leaf_sq, unsigned long long *counters, unsigned long long *gates, void *stream)
{
    if (!gates) return SPAMM_EINVAL;
    return spamm_execute_impl(a, b, plan, nsteps, nC, tau, 1.0f, SPAMM_FINE4, 0, c_values, c_values_t, c_leaf_sq, counters,
                              nullptr, nullptr, 0, stream, gates);
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
