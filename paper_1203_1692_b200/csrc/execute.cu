// Numeric phase on the device: the leaf-block products of a plan.
//
// Replaces numeric.execute_plan / _run_batched / _compose (pkg/src/spamm/numeric.py:138-284):
// for every product leaf, its tasks are accumulated in ascending k; inside a task the 4x4x4
// micro products run for r = 0..3, kk ascending, and a micro product (p,q,r) is skipped when its
// fine4 bit is clear (numeric.py:232-259).  One thread owns one 4x4 sub-block (p,q) of one
// product leaf for the whole tile, so each C element has a single owner and a fixed order:
// results are identical run to run and, in EXACT mode (separately rounded multiply and add),
// bit-identical to the reference.
//
// Work unit: a super-tile of 4x4 product leaves (16 consecutive Morton keys).  A producer warp
// merges the (up to 16) ascending k-lists of the tile, and for every k that has at least one
// live task stages the needed A leaves (transposed copies) and B leaves with 1 KB bulk copies
// (TMA 1-D, cp.async.bulk -> SASS UBLKCP) into a ring of shared-memory stages guarded by
// mbarriers; eight consumer warps (two product leaves each) do the FP32 math from shared memory.
#include "common.cuh"
#include "scan.cuh"

#define EX_STAGES 4
#define EX_CONSUMERS 8
#define EX_THREADS (32 * (EX_CONSUMERS + 1))
#define EX_B_STRIDE 272          // floats between B leaves in a stage: odd leaves land 64 B off -> no bank clash
#define EX_END_OF_TILE 1u

struct __align__(16) StepDesc {
    unsigned long long mask[16];   // fine4 bits of the task at tile position pos (0 when not live)
    uint32_t live;                 // bit pos set when the task (pos, k) exists
    uint32_t flags;
};

struct ExecArgs {
    const float *a_values_t;
    const float *b_values;
    const uint32_t *c_keys;
    const int32_t *c_off;
    const uint32_t *task_k, *task_a, *task_b;
    const unsigned long long *task_mask;
    const int32_t *tile_first;
    const int32_t *ntiles;
    int64_t nC;
    float alpha;
    int alpha_is_one;
    float *c_values, *c_values_t, *c_sub4;
    double *c_leaf_sq;
    unsigned long long *counters;
};

// position inside the super-tile -> leaf coordinates (row bit above column bit)
__device__ __forceinline__ int pos_di(int pos) { return ((pos >> 3) & 1) << 1 | ((pos >> 1) & 1); }
__device__ __forceinline__ int pos_dj(int pos) { return ((pos >> 2) & 1) << 1 | (pos & 1); }

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

template <bool EXACT>
__global__ void __launch_bounds__(EX_THREADS, 2) execute_kernel(ExecArgs g)
{
    __shared__ __align__(128) float sA[EX_STAGES][4][SPAMM_LEAF];
    __shared__ __align__(128) float sB[EX_STAGES][4 * EX_B_STRIDE];
    __shared__ StepDesc desc[EX_STAGES];
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
    const int ntiles = *g.ntiles;
    int stage = 0;
    uint32_t phase = 0;

    if (warp == EX_CONSUMERS) {
        // ===================== producer: k-way merge + bulk copies =====================
        unsigned long long products = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int t0 = g.tile_first[tile];
            const int t1 = (tile + 1 < ntiles) ? g.tile_first[tile + 1] : (int)g.nC;
            const int cnt = t1 - t0;
            int pos = 0, cur = 0, end = 0;
            if ((int)lane < cnt) {
                pos = g.c_keys[t0 + lane] & 15u;
                cur = g.c_off[t0 + lane];
                end = g.c_off[t0 + lane + 1];
            }
            const int di = pos_di(pos), dj = pos_dj(pos);
            uint32_t curk = (cur < end) ? g.task_k[cur] : 0xFFFFFFFFu;
            for (;;) {
                const uint32_t kmin = __reduce_min_sync(FULL_MASK, curk);
                mbar_wait(&empty_bar[stage], phase ^ 1u);
                if (kmin == 0xFFFFFFFFu) {
                    if (lane == 0) {
                        desc[stage].live = 0;
                        desc[stage].flags = EX_END_OF_TILE;
                        mbar_arrive(&full_bar[stage]);
                    }
                    __syncwarp();
                    if (++stage == EX_STAGES) { stage = 0; phase ^= 1u; }
                    break;
                }
                const bool mine = (curk == kmin);
                uint32_t a_s = 0, b_s = 0;
                unsigned long long m = 0;
                if (mine) {
                    a_s = g.task_a[cur];
                    b_s = g.task_b[cur];
                    m = g.task_mask[cur];
                    products += __popcll(m);
                }
                if ((int)lane < cnt) desc[stage].mask[pos] = m;
                const uint32_t live = __reduce_or_sync(FULL_MASK, mine ? (1u << pos) : 0u);
                const uint32_t amask = __reduce_or_sync(FULL_MASK, mine ? (1u << di) : 0u);
                const uint32_t bmask = __reduce_or_sync(FULL_MASK, mine ? (1u << dj) : 0u);
                if (lane == 0) {
                    desc[stage].live = live;
                    desc[stage].flags = 0;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_expect_tx(&full_bar[stage], 1024u * (__popc(amask) + __popc(bmask)));
                __syncwarp();
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const uint32_t ba = __ballot_sync(FULL_MASK, mine && di == d);
                    if (ba && lane == (uint32_t)(__ffs(ba) - 1))
                        bulk_copy_g2s(&sA[stage][d][0], g.a_values_t + (size_t)a_s * SPAMM_LEAF, 1024u, &full_bar[stage]);
                    const uint32_t bb = __ballot_sync(FULL_MASK, mine && dj == d);
                    if (bb && lane == (uint32_t)(__ffs(bb) - 1))
                        bulk_copy_g2s(&sB[stage][d * EX_B_STRIDE], g.b_values + (size_t)b_s * SPAMM_LEAF, 1024u,
                                      &full_bar[stage]);
                }
                if (mine) {
                    ++cur;
                    curk = (cur < end) ? g.task_k[cur] : 0xFFFFFFFFu;
                }
                if (++stage == EX_STAGES) { stage = 0; phase ^= 1u; }
            }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) products += __shfl_xor_sync(FULL_MASK, products, d);
        if (lane == 0 && products) atomicAdd(g.counters, products);
        return;
    }

    // ============================== consumers ==============================
    const int half = lane >> 4, t16 = lane & 15, p = t16 >> 2, q = t16 & 3;
    const int mypos = 2 * warp + half;
    const int di = pos_di(mypos), dj = pos_dj(mypos);
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int t0 = g.tile_first[tile];
        const int t1 = (tile + 1 < ntiles) ? g.tile_first[tile + 1] : (int)g.nC;
        const int cnt = t1 - t0;
        uint32_t present = 0;
        if ((int)lane < cnt) present = 1u << (g.c_keys[t0 + lane] & 15u);
        present = __reduce_or_sync(FULL_MASK, present);
        const bool exists = (present >> mypos) & 1u;
        const int64_t cslot = (int64_t)t0 + __popc(present & ((1u << mypos) - 1u));

        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

        for (;;) {
            mbar_wait(&full_bar[stage], phase);
            const uint32_t live = desc[stage].live;
            const uint32_t flags = desc[stage].flags;
            if (!(flags & EX_END_OF_TILE) && ((live >> (2 * warp)) & 3u)) {
                const unsigned long long m = ((live >> mypos) & 1u) ? desc[stage].mask[mypos] : 0ull;
                const float *As = &sA[stage][di][4 * p];
                const float *Bs = &sB[stage][dj * EX_B_STRIDE + 4 * q];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const bool on = (m >> (r * 16 + t16)) & 1ull;
                    if (!__any_sync(FULL_MASK, on)) continue;
                    float4 a[4], b[4];
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        a[kk] = *reinterpret_cast<const float4 *>(As + (4 * r + kk) * 16);
                        b[kk] = *reinterpret_cast<const float4 *>(Bs + (4 * r + kk) * 16);
                    }
                    if (on) {
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
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[stage]);
            if (++stage == EX_STAGES) { stage = 0; phase ^= 1u; }
            if (flags & EX_END_OF_TILE) break;
        }

        // epilogue: alpha scaling (numeric.py:273-275), both leaf layouts, norms in
        // compute_norms order (core.py:108-116)
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
            float *cv = g.c_values + cslot * SPAMM_LEAF;
            float *ct = g.c_values_t + cslot * SPAMM_LEAF;
#pragma unroll
            for (int i = 0; i < 4; ++i) *reinterpret_cast<float4 *>(cv + (4 * p + i) * 16 + 4 * q) = rows[i];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                *reinterpret_cast<float4 *>(ct + (4 * q + j) * 16 + 4 * p) =
                    make_float4(acc[0][j], acc[1][j], acc[2][j], acc[3][j]);
            g.c_sub4[cslot * 16 + t16] = (float)sqrt(S);
            if (t16 == 0) g.c_leaf_sq[cslot] = tot;
        }
    }
}

// super-tile starts: product leaves whose key >> 4 differs from their predecessor's
struct TileScanOp {
    const uint32_t *keys;
    int32_t *tile_first;
    __device__ __forceinline__ int flag(int64_t e) const { return (e == 0) || ((keys[e] >> 4) != (keys[e - 1] >> 4)); }
    __device__ __forceinline__ void emit(int64_t e, int flag, int32_t idx) const
    {
        if (flag) tile_first[idx] = (int32_t)e;
    }
};

static inline size_t ex_align(size_t x) { return (x + 255) / 256 * 256; }

extern "C" size_t spamm_execute_workspace_bytes(int64_t nC)
{
    return ex_align(scan_workspace_bytes(nC)) + ex_align(4 * (size_t)(nC + 1)) + 256;
}

extern "C" int spamm_execute(const spamm_tree_view *a, const spamm_tree_view *b, const spamm_plan_buffers *plan, int64_t T,
                             int64_t nC, float alpha, int granularity, int exact, float *c_values, float *c_values_t,
                             float *c_sub4, double *c_leaf_sq, unsigned long long *counters, void *ws, size_t ws_bytes,
                             void *stream)
{
    (void)granularity;
    if (!a || !b || !plan || T < 0 || nC < 0) return SPAMM_EINVAL;
    if (nC == 0 || T == 0) return SPAMM_OK;
    if (!ws || ws_bytes < spamm_execute_workspace_bytes(nC)) return SPAMM_EWORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    char *w = reinterpret_cast<char *>(ws);
    void *scan_ws = w;
    const size_t scan_bytes = ex_align(scan_workspace_bytes(nC));
    int32_t *tile_first = reinterpret_cast<int32_t *>(w + scan_bytes);
    int32_t *ntiles = reinterpret_cast<int32_t *>(w + scan_bytes + ex_align(4 * (size_t)(nC + 1)));
    TileScanOp op{plan->c_keys, tile_first};
    int rc = scan_flags(op, nC, ntiles, scan_ws, scan_bytes, st);
    if (rc != SPAMM_OK) return rc;
    ExecArgs g;
    g.a_values_t = a->values_t;
    g.b_values = b->values;
    g.c_keys = plan->c_keys;
    g.c_off = plan->c_off;
    g.task_k = plan->task_k;
    g.task_a = plan->task_a;
    g.task_b = plan->task_b;
    g.task_mask = reinterpret_cast<const unsigned long long *>(plan->task_mask);
    g.tile_first = tile_first;
    g.ntiles = ntiles;
    g.nC = nC;
    g.alpha = alpha;
    g.alpha_is_one = (alpha == 1.0f);
    g.c_values = c_values;
    g.c_values_t = c_values_t;
    g.c_sub4 = c_sub4;
    g.c_leaf_sq = c_leaf_sq;
    g.counters = counters;
    int64_t max_tiles = (nC + 0) < 1 ? 1 : nC;
    int grid = SPAMM_NUM_SMS * 2;
    if ((int64_t)grid > max_tiles) grid = (int)max_tiles;
    if (exact) execute_kernel<true><<<grid, EX_THREADS, 0, st>>>(g);
    else execute_kernel<false><<<grid, EX_THREADS, 0, st>>>(g);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

// ---- beta != 0: union of the old and the produced leaf sets, then _compose ----------------------
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

// out = (alpha32 * prod) + (old * beta32), the reference's expressions (numeric.py:276-284)
__global__ void __launch_bounds__(256) compose_kernel(const float *__restrict__ prod, const float *__restrict__ old,
                                                      const int32_t *__restrict__ idx_prod,
                                                      const int32_t *__restrict__ idx_old, float alpha, float beta,
                                                      int alpha_is_one, int beta_is_one, float *__restrict__ out)
{
    const int64_t x = blockIdx.x;
    const int32_t ip = idx_prod[x], io = idx_old[x];
    float v;
    if (io < 0) {
        const float pv = prod[(int64_t)ip * SPAMM_LEAF + threadIdx.x];
        v = alpha_is_one ? pv : __fmul_rn(alpha, pv);
    } else {
        const float ov = old[(int64_t)io * SPAMM_LEAF + threadIdx.x];
        v = beta_is_one ? ov : __fmul_rn(ov, beta);
        if (ip >= 0) {
            const float pv = prod[(int64_t)ip * SPAMM_LEAF + threadIdx.x];
            v = __fadd_rn(alpha_is_one ? pv : __fmul_rn(alpha, pv), v);
        }
    }
    out[x * SPAMM_LEAF + threadIdx.x] = v;
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
