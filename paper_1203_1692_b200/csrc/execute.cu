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
// STATIC partition of the record stream that the planner cut into pieces of equal weight, one per SM
// (plan.cu, plan_order_kernel); a piece is whole super-tiles plus at most one head and one tail
// segment of a tile shared with the neighbouring piece, whose accumulators pass from CTA to CTA
// through C's value records (spamm_b200.h).  The CTAs resident on one SM find each other through
// %smid and share the SM's piece tile by tile (a compare-and-swap cursor per piece): two CTAs on an SM
// do not advance equally, SMs do, so all SMs finish together without a global hand-out counter.
// Launched with programmatic dependent launch.
// Tuning aids: SPAMM_EX_STAGES, SPAMM_EX_CTAS, SPAMM_EX_DEBUG, SPAMM_EX_TRACE (per-CTA time stamps).
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "plan_format.cuh"

#define EX_MAX_STAGES 6
#define EX_CONSUMERS 8
#define EX_THREADS (32 * (EX_CONSUMERS + 1))          // consumers + producer
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
    uint32_t rec;          // index of the record in the plan
    uint32_t pad;
    uint32_t dead[2];      // fine4: live tasks none of whose micro products runs (spamm_step.dead)
    uint32_t pad2[2];
};

struct ExecArgs {
    const float *a_values_t;
    const float *b_values;
    const spamm_step *steps;
    const int32_t *pieces;       // plan.tile_order: (b, mb, me, e) per piece, see plan_order_kernel
    int32_t *cursor;             // per piece: how far its jobs (head segment, tiles, tail segment) are handed out
    const int32_t *counts;       // plan counts (device): [5] = number of pieces
    int32_t *chain;              // per product leaf: the record up to which its partial sums are handed on (0 = none)
    unsigned int *xs;            // ExecShared: piece tickets, exited CTAs, per-SM tables; zero between launches
    int xs_early;                // xs is not touched by the preceding kernel: the SM's CTAs pair up before waiting for it
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
    int32_t *error_flag;         // plan counts[15]: set when a hand-over wait gives up (never in a correct run)
    uint32_t *clean_ptr;         // the planner's shared state, returned to zero here on behalf of the planner
    int clean_words;             // (spamm_multiply; 0 otherwise)
    unsigned long long *gates;   // optional (spamm_execute_gates): the 64 gate bits of every task as evaluated HERE
    int dbg;                     // tuning aid (SPAMM_EX_DEBUG): 1 = no copies, 2 = no math
    unsigned long long *trace;   // tuning aid (SPAMM_EX_TRACE): per CTA start / first data / end / units
};

// ExecShared (uint32 words): [0] piece tickets drawn, [1] CTAs that have run out of work,
// [2 .. 258) CTAs arrived per SM, [258 .. 514) the piece (+ 1) the CTAs of an SM currently share
#define XS_TICKET 0
#define XS_EXITED 1
#define XS_ARRIVE 2
#define XS_PIECE 258
#define XS_WORDS 514
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int *p)
{
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int *p, unsigned int v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

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
__global__ void __launch_bounds__(EX_THREADS, EX_MIN_BLOCKS) execute_kernel(ExecArgs g)
{
    // dynamic shared memory: nstages x (A block + B block), then descriptors and barriers
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nstages = g.nstages;
    unsigned char *sA = smem_raw;
    unsigned char *sB = smem_raw + (size_t)nstages * EX_BLOCK_BYTES;
    StageDesc *desc = reinterpret_cast<StageDesc *>(smem_raw + (size_t)nstages * 2 * EX_BLOCK_BYTES);
    uint64_t *full_bar = reinterpret_cast<uint64_t *>(desc + EX_MAX_STAGES);
    uint64_t *empty_bar = full_bar + EX_MAX_STAGES;

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    // everything that does not depend on the preceding kernel comes before the wait for it
    if (threadIdx.x == 0) {
        for (int s = 0; s < nstages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], EX_CONSUMERS);
        }
        fence_barrier_init();
    }
    // The CTAs of one SM share a piece.  The first to arrive on an SM draws a piece ticket and
    // publishes it in the SM's table entry; the others read it there.  Tickets are drawn in order, and
    // whoever draws a piece starts with its head segment, so the CTA that later waits for that head
    // (the tail of the next piece, run last) waits for a running CTA: no assumption about residency.
    uint32_t smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    smid &= 255u;
    int piece = 0;
    auto pair_up = [&]() {
        if (lane == 0) {
            if (atomicAdd(g.xs + XS_ARRIVE + smid, 1u) == 0u) {
                piece = (int)atomicAdd(g.xs + XS_TICKET, 1u);
                st_release_u32(g.xs + XS_PIECE + smid, (unsigned int)piece + 1u);
            } else {
                unsigned int v;
                while ((v = ld_acquire_u32(g.xs + XS_PIECE + smid)) == 0u) __nanosleep(64);
                piece = (int)v - 1;
            }
        }
        piece = __shfl_sync(FULL_MASK, piece, 0);
    };
    if (warp == EX_CONSUMERS && g.xs_early) pair_up();
    pdl_enter();
    if (blockIdx.x == 0)
        for (int x = threadIdx.x; x < g.clean_words; x += blockDim.x) g.clean_ptr[x] = 0u;
    __syncthreads();
    int stage = 0;
    uint32_t phase = 0;
    if (g.trace && threadIdx.x == 0) g.trace[blockIdx.x * 4] = global_timer();

    if (warp == EX_CONSUMERS) {
        // ============ producer: stream step records, stage leaf blocks with bulk copies ============
        if (!g.xs_early) pair_up();
        const int npieces = g.counts[2] ? 0 : g.counts[5];      // an overflowed plan is incomplete: do nothing
        const uint32_t *words = reinterpret_cast<const uint32_t *>(g.steps);
        const int4 *pieces = reinterpret_cast<const int4 *>(g.pieces);
        int4 pd = make_int4(0, 0, 0, 0);
        if (piece < npieces) pd = __ldg(pieces + piece);
        // Jobs of a piece, in hand-out order: the head segment [me, e), the whole tiles of [mb, me) one by
        // one, the tail segment [b, mb).  The cursor counts handed-out records in that order.  claim():
        // the next job of the SM's piece -- or of the piece the SM moves on to -- as records [jb, je).
        int jb = 0, je = 0, units_done = 0;
        auto claim = [&]() -> bool {
            for (;;) {
                if (piece >= npieces) return false;
                int got = 0;
                if (lane == 0) {
                    const int h = pd.w - pd.z, t = pd.z - pd.y, tl = pd.y - pd.x, total = h + t + tl;
                    for (;;) {
                        const int v = ld_acquire_gpu(g.cursor + piece);
                        if (v >= total) { got = 0; break; }
                        int nv;
                        if (v < h) { nv = h; jb = pd.z; je = pd.w; }
                        else if (v < h + t) {
                            const int r0 = pd.y + (v - h);
                            int len = (int)__ldg(words + (size_t)r0 * 16 + 15);      // records of this tile
                            if (len < 1) len = 1;
                            if (r0 + len > pd.z) len = pd.z - r0;
                            nv = v + len; jb = r0; je = r0 + len;
                        } else { nv = total; jb = pd.x; je = pd.y; }
                        if (atomicCAS(g.cursor + piece, v, nv) == v) { got = 1; break; }
                    }
                }
                got = __shfl_sync(FULL_MASK, got, 0);
                if (got) {
                    jb = __shfl_sync(FULL_MASK, jb, 0);
                    je = __shfl_sync(FULL_MASK, je, 0);
                    return true;
                }
                // the piece is handed out: join the piece the SM's other CTAs moved on to, or draw the next
                if (lane == 0) {
                    const unsigned int cur = ld_acquire_u32(g.xs + XS_PIECE + smid);
                    if (cur != (unsigned int)piece + 1u) {
                        piece = (int)cur - 1;
                    } else {
                        const int np = (int)atomicAdd(g.xs + XS_TICKET, 1u);
                        atomicCAS(g.xs + XS_PIECE + smid, (unsigned int)piece + 1u, (unsigned int)np + 1u);
                        piece = np;      // mine in any case; if the entry had moved meanwhile, I rejoin it afterwards
                    }
                }
                piece = __shfl_sync(FULL_MASK, piece, 0);
                if (piece < npieces) pd = __ldg(pieces + piece);
            }
        };
        // cursor over the records of my jobs.  The next job is claimed two records before the cursor
        // leaves the current one: the claim's latency hides behind the staged records, and no CTA sits
        // on a job it has not started while its neighbour runs dry.
        int r = 0, rend = 0, rbeg = 0, nb = 0, ne = 0;
        bool have_next = false, dry = false, more = true;
        // fetch: the next record of the cursor -> (word of lane l < 16, meta); meta = rec | first << 30 | last << 31, ~0 = none
        auto fetch = [&](uint32_t &wd, uint32_t &meta) {
            for (;;) {
                if (!more) { wd = 0u; meta = 0xFFFFFFFFu; return; }
                if (!have_next && !dry && rend - r <= 2) {
                    have_next = claim();
                    dry = !have_next;
                    nb = jb; ne = je;
                }
                if (r < rend) break;
                if (!have_next) { more = false; continue; }
                r = rbeg = nb; rend = ne;
                have_next = false;
                ++units_done;
            }
            wd = lane < 16 ? __ldg(words + (size_t)r * 16 + lane) : 0u;
            meta = (uint32_t)r | (r == rbeg ? (1u << 30) : 0u) | (r + 1 == rend ? (1u << 31) : 0u);
            ++r;
        };
        uint32_t w[EX_PREFETCH], m[EX_PREFETCH];
#pragma unroll
        for (int x = 0; x < EX_PREFETCH; ++x) fetch(w[x], m[x]);
        while (m[0] != 0xFFFFFFFFu) {
            const uint32_t cur = w[0], meta = m[0];
#pragma unroll
            for (int x = 0; x + 1 < EX_PREFETCH; ++x) { w[x] = w[x + 1]; m[x] = m[x + 1]; }
            fetch(w[EX_PREFETCH - 1], m[EX_PREFETCH - 1]);
            const uint32_t na = __popc(__shfl_sync(FULL_MASK, cur, 5));
            const uint32_t nb = __popc(__shfl_sync(FULL_MASK, cur, 7));
            mbar_wait(&empty_bar[stage], phase ^ 1u);
            uint32_t *d = reinterpret_cast<uint32_t *>(&desc[stage]);
            if (lane == 1) {                                 // flags: a run that starts or ends inside a tile is chained
                uint32_t f = cur;
                if ((meta >> 30 & 1u) && !(cur & STEP_FIRST)) f |= EX_CHAIN_IN;
                if ((meta >> 31 & 1u) && !(cur & STEP_LAST)) f |= EX_CHAIN_OUT;
                d[4] = f;
            }
            if (lane == 15) d[10] = meta & 0x3FFFFFFFu;      // record index
            if (lane == 13 || lane == 14) d[lane - 1] = cur; // dead[0..1]
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
        mbar_wait(&empty_bar[stage], phase ^ 1u);
        if (lane == 0) {
            desc[stage].flags = EX_EXIT;
            mbar_arrive(&full_bar[stage]);
            if (g.trace) g.trace[blockIdx.x * 4 + 3] = (unsigned long long)units_done;
        }
        // the last CTA to run out of work leaves the shared state and the cursors at zero for the next launch
        int last = 0;
        if (lane == 0) last = atomicAdd(g.xs + XS_EXITED, 1u) == gridDim.x - 1 ? 1 : 0;
        if (__shfl_sync(FULL_MASK, last, 0)) {
            for (int x = (int)lane; x < npieces; x += 32) g.cursor[x] = 0;
            for (int x = (int)lane; x < XS_WORDS; x += 32) g.xs[x] = 0u;
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
    bool chained = false;  // the sums of the current tile came (partly) from another CTA
    for (;;) {
        mbar_wait(&full_bar[stage], phase);
        const StageDesc &ds = desc[stage];
        const uint32_t flags = ds.flags;
        if (g.trace && threadIdx.x == 0 && !traced) {
            g.trace[blockIdx.x * 4 + 1] = global_timer();
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
            const uint32_t present_in = ds.present;
            if ((present_in >> mypos) & 1u) {
                const int64_t cs = (int64_t)ds.c_base + __popc(present_in & ((1u << mypos) - 1u));
                const int want = (int)ds.rec;      // the records before this one are in the partial sums
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
        const uint32_t a_present = ds.a_present, b_present = ds.b_present;
        const float *Ablk = reinterpret_cast<const float *>(sA + (size_t)stage * EX_BLOCK_BYTES);
        const float *Bblk = reinterpret_cast<const float *>(sB + (size_t)stage * EX_BLOCK_BYTES);
        const uint4 live4 = *reinterpret_cast<const uint4 *>(ds.live);
        uint32_t dead01 = 0u, dead23 = 0u;
        if (FINE) {
            dead01 = ds.dead[0];
            dead23 = ds.dead[1];
        }
#pragma unroll     // all four k unrolled: +4-5 % (their addresses become constants), measured
        for (int kk = 0; kk < 4; ++kk) {
            const uint32_t lw = kk == 0 ? live4.x : kk == 1 ? live4.y : kk == 2 ? live4.z : live4.w;
            // fine4: a task the planner found dead runs no micro product (and counts none)
            const uint32_t dead = FINE ? ((kk < 2 ? dead01 : dead23) >> (16 * (kk & 1))) : 0u;
            const uint32_t live = lw & 0xFFFFu & ~dead;
            if (!((live >> (2 * warp)) & 3u) || (g.dbg & 2)) continue;
            const bool mine = (live >> mypos) & 1u;
            // leaf (r,c) of a block sits at index popc(present & below(morton4(r,c)))
            const float *As = Ablk + __popc(a_present & ((1u << step_pos(di, kk)) - 1u)) * SPAMM_REC;
            const float *Bs = Bblk + __popc(b_present & ((1u << step_pos(kk, dj)) - 1u)) * SPAMM_REC;
            uint32_t on = 0;       // bit r: micro product (p,q,r) of my task runs
            if (FINE) {
                if (mine && ((lw >> (16 + mypos)) & 1u)) {
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
                if (g.gates && ((lw >> mypos) & 1u)) {
                    // evidence for the tests: bit r*16 + p*4 + q of the task's word (numeric.py:233-238)
                    unsigned long long bits = 0ull;
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if ((on >> r) & 1u) bits |= 1ull << (r * 16 + t16);
                    if (bits) atomicOr(g.gates + ((size_t)ds.rec * 64 + kk * 16 + mypos), bits);
                }
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
            seg_done = ds.rec + 1u;
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
int spamm_execute_piece_base() { return SPAMM_NUM_SMS; }
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
    const int64_t piece_cap = spamm_piece_capacity(plan->leaf_capacity);
    g.cursor = plan->tile_order + 4 * piece_cap;
    g.counts = plan->counts;
    // the kernel's shared state: in the planner's workspace when the call comes from spamm_multiply
    // (untouched by the preceding kernel, so the CTAs of an SM can pair up early), else behind the
    // plan's cursors
    g.xs = clean_ptr ? clean_ptr + clean_words : reinterpret_cast<unsigned int *>(plan->tile_order + 5 * piece_cap);
    g.xs_early = clean_ptr ? 1 : 0;
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
    g.dbg = tune.dbg;
    const int grid = SPAMM_NUM_SMS * tune.ctas_per_sm;
    const size_t smem = (size_t)tune.stages * 2 * EX_BLOCK_BYTES + EX_MAX_STAGES * (sizeof(StageDesc) + 16);
    const bool fine = granularity == SPAMM_FINE4;
    void (*kern)(ExecArgs) = exact ? (fine ? execute_kernel<true, true> : execute_kernel<true, false>)
                                   : (fine ? execute_kernel<false, true> : execute_kernel<false, false>);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return SPAMM_ECUDA;
    g.trace = nullptr;
    static const char *trace_path = getenv("SPAMM_EX_TRACE");     // tuning aid: allocates and synchronises
    if (trace_path && cudaMalloc(&g.trace, sizeof(unsigned long long) * 4 * grid) != cudaSuccess) g.trace = nullptr;
    if (g.trace) cudaMemsetAsync(g.trace, 0, sizeof(unsigned long long) * 4 * grid, st);
    if (spamm_launch_pdl(kern, dim3(grid), dim3(EX_THREADS), smem, st, g) != cudaSuccess)
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
