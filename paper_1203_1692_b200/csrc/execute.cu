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
// Work unit: a super-tile of 4x4 product leaves, described by the plan's step records (one per
// k with a live task).  Per CTA, one producer warp streams the records (prefetched four ahead)
// and for each stages the needed A leaves (transposed copies) and B leaves -- 1088-byte records
// holding the values and the 4x4 sub-block norms -- with bulk copies (TMA 1-D, cp.async.bulk,
// SASS UBLKCP) into a ring of shared-memory stages guarded by mbarriers; eight consumer warps
// (two product leaves each) gate and multiply from shared memory.  Super-tiles are handed out
// through an atomic counter.
#include "common.cuh"
#include "plan_format.cuh"

#define EX_STAGES 4
#define EX_CONSUMERS 8
#define EX_THREADS (32 * (EX_CONSUMERS + 1))
#define EX_EXIT (1u << 31)
#define EX_PREFETCH 4

struct __align__(16) StageDesc {
    uint32_t flags;      // live bits | STEP_FIRST | STEP_LAST | EX_EXIT
    uint32_t c_base;
    uint32_t present;
    uint32_t pad;
};

struct ExecArgs {
    const float *a_values_t;
    const float *b_values;
    const spamm_step *steps;
    const int32_t *tile_off;     // step offset of every super-tile node, one extra entry
    const int32_t *counts;       // plan counts (device): [5] = number of super-tile nodes
    unsigned int *tile_counter;
    double tau;
    float alpha;
    int alpha_is_one;
    float *c_values, *c_values_t;
    double *c_leaf_sq;
    unsigned long long *counters;
};

__device__ __forceinline__ double ex_row_sq(float4 v)
{
    double x = v.x, y = v.y, z = v.z, w = v.w;
    double r = __dmul_rn(x, x);
    r = __fma_rn(y, y, r);
    r = __fma_rn(z, z, r);
    r = __fma_rn(w, w, r);
    return r;
}

template <bool EXACT>
__device__ __forceinline__ void mac(float &acc, float a, float b)
{
    if (EXACT) acc = __fadd_rn(acc, __fmul_rn(a, b));   // numeric.py:252-259: two roundings
    else acc = fmaf(a, b, acc);
}

template <bool EXACT, bool FINE>
__global__ void __launch_bounds__(EX_THREADS, 2) execute_kernel(ExecArgs g)
{
    __shared__ __align__(128) float sA[EX_STAGES][4][SPAMM_REC];
    __shared__ __align__(128) float sB[EX_STAGES][4][SPAMM_REC];
    __shared__ StageDesc desc[EX_STAGES];
    __shared__ __align__(8) uint64_t full_bar[EX_STAGES], empty_bar[EX_STAGES];

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    if (threadIdx.x == 0) {
        for (int s = 0; s < EX_STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], EX_CONSUMERS);
        }
        fence_barrier_init();
    }
    __syncthreads();
    int stage = 0;
    uint32_t phase = 0;

    if (warp == EX_CONSUMERS) {
        // ============ producer: stream step records, stage leaves with bulk copies ============
        const int ntiles = g.counts[5];
        const uint32_t *words = reinterpret_cast<const uint32_t *>(g.steps);
        int tile = 0;
        if (lane == 0) tile = (int)atomicAdd(g.tile_counter, 1u);
        tile = __shfl_sync(FULL_MASK, tile, 0);
        while (tile < ntiles) {
            const int beg = g.tile_off[tile], end = g.tile_off[tile + 1];
            int next_tile = 0;
            if (lane == 0) next_tile = (int)atomicAdd(g.tile_counter, 1u);   // its latency hides behind this tile
            // lane l < 16 holds word l of a record: 0 k, 1 flags, 2 c_base, 3 tile, 4-7 a_slot, 8-11 b_slot, 12 present
            uint32_t w[EX_PREFETCH];
#pragma unroll
            for (int x = 0; x < EX_PREFETCH; ++x)
                w[x] = (lane < 16 && beg + x < end) ? __ldg(words + (size_t)(beg + x) * 16 + lane) : 0u;
            for (int r = beg; r < end; ++r) {
                const uint32_t cur = w[0];
#pragma unroll
                for (int x = 0; x + 1 < EX_PREFETCH; ++x) w[x] = w[x + 1];
                w[EX_PREFETCH - 1] =
                    (lane < 16 && r + EX_PREFETCH < end) ? __ldg(words + (size_t)(r + EX_PREFETCH) * 16 + lane) : 0u;
                const uint32_t flags = __shfl_sync(FULL_MASK, cur, 1);
                const uint32_t live = flags & SPAMM_STEP_LIVE;
                mbar_wait(&empty_bar[stage], phase ^ 1u);
                if (lane == 1) desc[stage].flags = cur;
                if (lane == 2) desc[stage].c_base = cur;
                if (lane == 12) desc[stage].present = cur;
                uint32_t need = 0;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    need += (live & step_rowmask(d)) ? 1u : 0u;
                    need += (live & step_colmask(d)) ? 1u : 0u;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_expect_tx(&full_bar[stage], need * SPAMM_REC_BYTES);
                __syncwarp();
                if (lane >= 4 && lane < 8) {
                    const int d = lane - 4;
                    if (live & step_rowmask(d))
                        bulk_copy_g2s(&sA[stage][d][0], g.a_values_t + (size_t)cur * SPAMM_REC, SPAMM_REC_BYTES,
                                      &full_bar[stage]);
                } else if (lane >= 8 && lane < 12) {
                    const int d = lane - 8;
                    if (live & step_colmask(d))
                        bulk_copy_g2s(&sB[stage][d][0], g.b_values + (size_t)cur * SPAMM_REC, SPAMM_REC_BYTES,
                                      &full_bar[stage]);
                }
                if (++stage == EX_STAGES) { stage = 0; phase ^= 1u; }
            }
            tile = __shfl_sync(FULL_MASK, next_tile, 0);
        }
        mbar_wait(&empty_bar[stage], phase ^ 1u);
        if (lane == 0) {
            desc[stage].flags = EX_EXIT;
            mbar_arrive(&full_bar[stage]);
        }
        return;
    }

    // ======================================= consumers =======================================
    const int half = lane >> 4, t16 = lane & 15, p = t16 >> 2, q = t16 & 3;
    const int mypos = 2 * warp + half;
    const int di = step_pos_di(mypos), dj = step_pos_dj(mypos);
    uint32_t executed = 0;
    float acc[4][4];
    for (;;) {
        mbar_wait(&full_bar[stage], phase);
        const uint32_t flags = desc[stage].flags;
        if (flags & EX_EXIT) break;
        if (flags & STEP_FIRST) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
        }
        const uint32_t live = flags & SPAMM_STEP_LIVE;
        if ((live >> (2 * warp)) & 3u) {
            const bool mine = (live >> mypos) & 1u;
            const float *As = &sA[stage][di][0];
            const float *Bs = &sB[stage][dj][0];
            uint32_t on = 0;       // bit r: micro product (p,q,r) of my task runs
            if (FINE) {
                const float4 sa = *reinterpret_cast<const float4 *>(As + 256 + 4 * p);   // subA[p][0..3]
                const float4 sb = *reinterpret_cast<const float4 *>(Bs + 256 + 4 * q);   // subB[0..3][q]
                if (mine) {
                    on |= (__dmul_rn((double)sa.x, (double)sb.x) >= g.tau) ? 1u : 0u;
                    on |= (__dmul_rn((double)sa.y, (double)sb.y) >= g.tau) ? 2u : 0u;
                    on |= (__dmul_rn((double)sa.z, (double)sb.z) >= g.tau) ? 4u : 0u;
                    on |= (__dmul_rn((double)sa.w, (double)sb.w) >= g.tau) ? 8u : 0u;
                }
                executed += __popc(on);
            } else {
                on = mine ? 15u : 0u;
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const bool go = (on >> r) & 1u;
                if (!__any_sync(FULL_MASK, go)) continue;
                float4 a[4], b[4];
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    a[kk] = *reinterpret_cast<const float4 *>(As + (4 * r + kk) * 16 + 4 * p);
                    b[kk] = *reinterpret_cast<const float4 *>(Bs + (4 * r + kk) * 16 + 4 * q);
                }
                if (go) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const float av[4] = {a[kk].x, a[kk].y, a[kk].z, a[kk].w};
                        const float bv[4] = {b[kk].x, b[kk].y, b[kk].z, b[kk].w};
#pragma unroll
                        for (int i = 0; i < 4; ++i)
#pragma unroll
                            for (int j = 0; j < 4; ++j) mac<EXACT>(acc[i][j], av[i], bv[j]);
                    }
                }
            }
        }
        uint32_t c_base = 0, present = 0;
        if (flags & STEP_LAST) {
            c_base = desc[stage].c_base;
            present = desc[stage].present;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[stage]);
        if (++stage == EX_STAGES) { stage = 0; phase ^= 1u; }
        if (!(flags & STEP_LAST)) continue;

        // epilogue of the super-tile: alpha scaling (numeric.py:273-275), both leaf layouts with
        // their sub-norm tails, leaf square sum in compute_norms order (core.py:108-116)
        const bool exists = (present >> mypos) & 1u;
        const int64_t cslot = (int64_t)c_base + __popc(present & ((1u << mypos) - 1u));
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
        double tot = __dadd_rn(S, __shfl_xor_sync(FULL_MASK, S, 8));
        tot = __dadd_rn(tot, __shfl_xor_sync(FULL_MASK, tot, 1));
        tot = __dadd_rn(tot, __shfl_xor_sync(FULL_MASK, tot, 2));
        tot = __dadd_rn(tot, __shfl_xor_sync(FULL_MASK, tot, 4));
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
            if (t16 == 0) g.c_leaf_sq[cslot] = tot;
        }
    }
    if (FINE) {
        executed = __reduce_add_sync(FULL_MASK, executed);
        if (lane == 0 && executed) atomicAdd(g.counters, (unsigned long long)executed);
    }
}

extern "C" int spamm_execute(const spamm_tree_view *a, const spamm_tree_view *b, const spamm_plan_buffers *plan,
                             int64_t nsteps, int64_t nC, double tau, float alpha, int granularity, int exact,
                             float *c_values, float *c_values_t, double *c_leaf_sq, unsigned long long *counters,
                             void *stream)
{
    if (!a || !b || !plan || nsteps < 0 || nC < 0) return SPAMM_EINVAL;
    if (granularity != SPAMM_FINE4 && granularity != SPAMM_COARSE16) return SPAMM_EINVAL;
    if (nC == 0 || nsteps == 0) return SPAMM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    ExecArgs g;
    g.a_values_t = a->values_t;
    g.b_values = b->values;
    g.steps = plan->steps;
    g.tile_off = plan->tile_off;
    g.counts = plan->counts;
    g.tile_counter = reinterpret_cast<unsigned int *>(plan->counts + 1);
    g.tau = tau;
    g.alpha = alpha;
    g.alpha_is_one = (alpha == 1.0f);
    g.c_values = c_values;
    g.c_values_t = c_values_t;
    g.c_leaf_sq = c_leaf_sq;
    g.counters = counters;
    if (cudaMemsetAsync(plan->counts + 1, 0, sizeof(int32_t), st) != cudaSuccess) return SPAMM_ECUDA;
    const int grid = SPAMM_NUM_SMS * 2;
    const bool fine = granularity == SPAMM_FINE4;
    if (exact) {
        if (fine) execute_kernel<true, true><<<grid, EX_THREADS, 0, st>>>(g);
        else execute_kernel<true, false><<<grid, EX_THREADS, 0, st>>>(g);
    } else {
        if (fine) execute_kernel<false, true><<<grid, EX_THREADS, 0, st>>>(g);
        else execute_kernel<false, false><<<grid, EX_THREADS, 0, st>>>(g);
    }
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
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
