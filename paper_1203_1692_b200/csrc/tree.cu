// Tree construction kernels: the Frobenius-norm pyramid and the packed leaf store.
//
// Replaces QuadtreeMatrix.from_dense / compute_norms / packed_leaves / to_dense of the
// reference (pkg/src/spamm/core.py:213-276, :331-345, :387-405).  All square sums are
// accumulated in FP64 in the exact order numpy uses for the reference expressions (see
// oracle/spamm_oracle.c for the probe), so every float32 norm is bit-identical.
#include "common.cuh"
#include "scan.cuh"
#include "plan_format.cuh"

// ---------------------------------------------------------------------------------
// Sum of squares of a 4x4 sub-block held as four float4 rows (core.py:113-114, :230-232):
//   r_i = ((x_i0^2 + x_i1^2) + x_i2^2) + x_i3^2,   S = ((r_0 + r_1) + r_2) + r_3.
// x*x is exact in double for a float x, so fma(x, x, acc) rounds once like numpy's add.
__device__ __forceinline__ double row_sq(float4 v)
{
    double x = v.x, y = v.y, z = v.z, w = v.w;
    double r = __dmul_rn(x, x);
    r = __fma_rn(y, y, r);
    r = __fma_rn(z, z, r);
    r = __fma_rn(w, w, r);
    return r;
}
__device__ __forceinline__ double sub_block_sq(float4 r0, float4 r1, float4 r2, float4 r3)
{
    double s = row_sq(r0);
    s = __dadd_rn(s, row_sq(r1));
    s = __dadd_rn(s, row_sq(r2));
    s = __dadd_rn(s, row_sq(r3));
    return s;
}

__device__ __forceinline__ float4 load_row4(const float *dense, int64_t m, int64_t n, int64_t ld, int64_t row,
                                            int64_t col, bool vec_ok)
{
    if (row >= m || col >= n) return make_float4(0.f, 0.f, 0.f, 0.f);
    const float *p = dense + row * ld + col;
    if (vec_ok && col + 3 < n) return __ldg(reinterpret_cast<const float4 *>(p));
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    v.x = __ldg(p);
    if (col + 1 < n) v.y = __ldg(p + 1);
    if (col + 2 < n) v.z = __ldg(p + 2);
    if (col + 3 < n) v.w = __ldg(p + 3);
    return v;
}

// K1a. One thread per column of 4x4 sub-blocks inside a 16-row strip: a warp reads 512
// contiguous bytes per matrix row.  Four neighbouring lanes hold the 4 sub-blocks (q) of a
// leaf row p; lane q == 0 folds them in the order of core.py:233
//   R_p = ((S_p0 + S_p1) + S_p2) + S_p3,  total = ((R_0 + R_1) + R_2) + R_3.
__global__ void __launch_bounds__(256) leaf_norms_dense_kernel(const float *__restrict__ dense, int64_t m, int64_t n,
                                                               int64_t ld, int L, float *__restrict__ sub4_grid,
                                                               double *__restrict__ leaf_sq, float *__restrict__ leaf_norm,
                                                               bool vec_ok)
{
    const int leaf_row = blockIdx.y;
    const int sc = blockIdx.x * 256 + threadIdx.x;   // sub-block column in the padded grid
    const int leaf_col = sc >> 2, q = sc & 3;
    const bool in_grid = leaf_col < L;
    double total = 0.0;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int64_t row = (int64_t)leaf_row * 16 + p * 4, col = (int64_t)sc * 4;
        double S = 0.0;
        if (in_grid) {
            float4 r0 = load_row4(dense, m, n, ld, row + 0, col, vec_ok);
            float4 r1 = load_row4(dense, m, n, ld, row + 1, col, vec_ok);
            float4 r2 = load_row4(dense, m, n, ld, row + 2, col, vec_ok);
            float4 r3 = load_row4(dense, m, n, ld, row + 3, col, vec_ok);
            S = sub_block_sq(r0, r1, r2, r3);
            sub4_grid[((int64_t)leaf_row * L + leaf_col) * 16 + p * 4 + q] = (float)sqrt(S);
        }
        double s1 = __shfl_down_sync(FULL_MASK, S, 1);
        double s2 = __shfl_down_sync(FULL_MASK, S, 2);
        double s3 = __shfl_down_sync(FULL_MASK, S, 3);
        double R = __dadd_rn(__dadd_rn(__dadd_rn(S, s1), s2), s3);
        total = __dadd_rn(total, R);
    }
    if (in_grid && q == 0) {
        const int64_t leaf = (int64_t)leaf_row * L + leaf_col;
        leaf_sq[leaf] = total;
        leaf_norm[leaf] = (total != 0.0) ? (float)sqrt(total) : -1.0f;
    }
}

extern "C" int spamm_leaf_norms_dense(const float *dense, int64_t m, int64_t n, int64_t ld, int depth,
                                      float *sub4_grid, double *leaf_sq, float *leaf_norm, void *stream)
{
    if (!dense || m < 1 || n < 1 || ld < n || depth < 0 || depth > 15) return SPAMM_EINVAL;
    const int L = 1 << depth;
    if ((int64_t)L * 16 < m || (int64_t)L * 16 < n) return SPAMM_EINVAL;
    const bool vec_ok = (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(dense) & 15) == 0);
    dim3 grid((4 * L + 255) / 256, L);
    leaf_norms_dense_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(dense, m, n, ld, L, sub4_grid, leaf_sq, leaf_norm,
                                                                     vec_ok);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

// K1b. Stored leaves in ascending Morton order: exclusive scan of the presence flags
// walked along the Z curve (core.py:235-237).
struct SlotScanOp {
    const float *leaf_norm;
    int32_t *slot, *slot_t;
    uint32_t *keys;
    int L;
    __device__ __forceinline__ int flag(int64_t e) const
    {
        uint32_t i, j;
        morton_decode((uint32_t)e, i, j);
        return leaf_norm[(int64_t)i * L + j] >= 0.0f ? 1 : 0;
    }
    __device__ __forceinline__ void emit(int64_t e, int flag, int32_t idx) const
    {
        uint32_t i, j;
        morton_decode((uint32_t)e, i, j);
        slot[(int64_t)i * L + j] = flag ? idx : -1;
        slot_t[(int64_t)j * L + i] = flag ? idx : -1;
        if (flag) keys[idx] = (uint32_t)e;
    }
};

extern "C" size_t spamm_scan_workspace_bytes(int64_t n) { return scan_workspace_bytes(n); }

extern "C" int spamm_assign_slots(const float *leaf_norm, int depth, int32_t *slot, int32_t *slot_t, uint32_t *keys,
                                  int32_t *nleaf_dev, void *ws, size_t ws_bytes, void *stream)
{
    if (depth < 0 || depth > 15) return SPAMM_EINVAL;
    const int L = 1 << depth;
    SlotScanOp op{leaf_norm, slot, slot_t, keys, L};
    return scan_flags(op, (int64_t)L * L, nleaf_dev, ws, ws_bytes, (cudaStream_t)stream);
}

// K1c. One warp per stored leaf (8 per block, grid-stride).  A stored leaf is a 272-float record: 256
// values followed by its 16 sub-block norms, so one bulk copy stages both.  `values` holds the leaf
// row-major with the sub-norms transposed (tail[q*4+r] = sub4[r][q], what a B operand reads);
// `values_t` holds the transposed leaf with the sub-norms row-major (what an A operand reads).
// VEC: the dense rows can be read 16 bytes at a time (base and row stride aligned).
template <bool VEC>
__global__ void __launch_bounds__(256) pack_leaves_kernel(const float *__restrict__ dense, int64_t m, int64_t n, int64_t ld,
                                                          int L, const uint32_t *__restrict__ keys, int64_t nleaf,
                                                          const float *__restrict__ sub4_grid, float *__restrict__ values,
                                                          float *__restrict__ values_t)
{
    __shared__ float tile[8][16][17];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float(*t)[17] = tile[warp];
    for (int64_t s = (int64_t)blockIdx.x * 8 + warp; s < nleaf; s += (int64_t)gridDim.x * 8) {
        uint32_t bi, bj;
        morton_decode(keys[s], bi, bj);
        float4 *dst = reinterpret_cast<float4 *>(values + s * SPAMM_REC);
        float4 *dst_t = reinterpret_cast<float4 *>(values_t + s * SPAMM_REC);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = lane + 32 * h, r = e >> 2, c = (e & 3) * 4;
            const int64_t gi = (int64_t)bi * 16 + r, gj = (int64_t)bj * 16 + c;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (gi < m) {
                const float *src = dense + gi * ld + gj;
                if (VEC && gj + 3 < n) {
                    v = __ldg(reinterpret_cast<const float4 *>(src));
                } else {
                    if (gj < n) v.x = __ldg(src);
                    if (gj + 1 < n) v.y = __ldg(src + 1);
                    if (gj + 2 < n) v.z = __ldg(src + 2);
                    if (gj + 3 < n) v.w = __ldg(src + 3);
                }
            }
            dst[e] = v;
            t[r][c] = v.x; t[r][c + 1] = v.y; t[r][c + 2] = v.z; t[r][c + 3] = v.w;
        }
        float sn = 0.0f;
        if (lane < 16) sn = sub4_grid[((int64_t)bi * L + bj) * 16 + lane];      // lane = p*4+q
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = lane + 32 * h, r = e >> 2, c = (e & 3) * 4;
            dst_t[e] = make_float4(t[c][r], t[c + 1][r], t[c + 2][r], t[c + 3][r]);
        }
        if (lane < 16) {
            values_t[s * SPAMM_REC + 256 + lane] = sn;
            values[s * SPAMM_REC + 256 + (lane & 3) * 4 + (lane >> 2)] = sn;
        }
        __syncwarp();
    }
}

extern "C" int spamm_pack_leaves(const float *dense, int64_t m, int64_t n, int64_t ld, int depth,
                                 const uint32_t *keys, int64_t nleaf, const float *sub4_grid, float *values,
                                 float *values_t, void *stream)
{
    if (nleaf == 0) return SPAMM_OK;
    if (!dense || nleaf < 0 || depth < 0 || depth > 15) return SPAMM_EINVAL;
    int64_t blocks = (nleaf + 7) / 8;
    if (blocks > SPAMM_NUM_SMS * 16) blocks = SPAMM_NUM_SMS * 16;
    const bool vec = (reinterpret_cast<uintptr_t>(dense) % 16 == 0) && (ld % 4 == 0);
    if (vec)
        pack_leaves_kernel<true><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dense, m, n, ld, 1 << depth, keys, nleaf,
                                                                                    sub4_grid, values, values_t);
    else
        pack_leaves_kernel<false><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dense, m, n, ld, 1 << depth, keys, nleaf,
                                                                                     sub4_grid, values, values_t);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

// K1d. Interior levels (_build_interior, core.py:252-266).  np.add.reduceat over the stored
// children in Morton order evaluates  x_first + ((x_second + x_third) + x_fourth).
struct NodeSum {
    double first, rest;
    int seen;
    __device__ __forceinline__ void add(bool present, double sq)
    {
        if (!present) return;
        if (seen == 0) first = sq;
        else if (seen == 1) rest = sq;
        else rest = __dadd_rn(rest, sq);
        ++seen;
    }
    __device__ __forceinline__ double total() const { return seen == 1 ? first : __dadd_rn(first, rest); }
};

// One block folds a 32x32 region of child level `tc` (block coordinates bx, by) through up to five
// levels: the first from global memory, the rest from shared memory.
__device__ __forceinline__ void interior_fold(const double *__restrict__ child_sq, float *__restrict__ norm,
                                              float *__restrict__ norm_t, double *__restrict__ sq_levels, int tc, int bx,
                                              int by, double (*s_sq)[16][16], unsigned char (*s_pr)[16][16])
{
    const int Sc = 1 << tc;
    const int64_t off_c = spamm_level_offset(tc);
    const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
    // level tc-1: parent (pi, pj) from four children in global memory
    {
        const int Sp = Sc >> 1;
        const int pi = by * 16 + ty, pj = bx * 16 + tx;
        bool present = false;
        double sq = 0.0;
        if (pi < Sp && pj < Sp) {
            NodeSum acc{0.0, 0.0, 0};
#pragma unroll
            for (int qd = 0; qd < 4; ++qd) {
                const int64_t ci = 2 * pi + (qd >> 1), cj = 2 * pj + (qd & 1);
                // both loads in flight together (the square sum of an absent child is simply not used)
                const float nv = norm[off_c + ci * Sc + cj];
                const double sv = child_sq[ci * Sc + cj];
                acc.add(nv >= 0.0f, sv);
            }
            present = acc.seen > 0;
            sq = present ? acc.total() : 0.0;
            const int64_t off_p = spamm_level_offset(tc - 1);
            const float nv = present ? (float)sqrt(sq) : -1.0f;
            norm[off_p + (int64_t)pi * Sp + pj] = nv;
            norm_t[off_p + (int64_t)pj * Sp + pi] = nv;
            sq_levels[off_p + (int64_t)pi * Sp + pj] = sq;
        }
        s_sq[0][ty][tx] = sq;
        s_pr[0][ty][tx] = present;
    }
    int cur = 0;
    int side = 16;                      // side of the level held in shared memory
    for (int t = tc - 2; t >= 0 && side > 1; --t) {
        __syncthreads();
        const int pside = side >> 1;
        const int Sp = 1 << t;
        if (ty < pside && tx < pside) {
            const int pi = by * pside + ty, pj = bx * pside + tx;
            bool present = false;
            double sq = 0.0;
            if (pi < Sp && pj < Sp) {
                NodeSum acc{0.0, 0.0, 0};
#pragma unroll
                for (int qd = 0; qd < 4; ++qd) {
                    const int ci = 2 * ty + (qd >> 1), cj = 2 * tx + (qd & 1);
                    acc.add(s_pr[cur][ci][cj], s_sq[cur][ci][cj]);
                }
                present = acc.seen > 0;
                sq = present ? acc.total() : 0.0;
                const int64_t off_p = spamm_level_offset(t);
                const float nv = present ? (float)sqrt(sq) : -1.0f;
                norm[off_p + (int64_t)pi * Sp + pj] = nv;
                norm_t[off_p + (int64_t)pj * Sp + pi] = nv;
                sq_levels[off_p + (int64_t)pi * Sp + pj] = sq;
            }
            s_sq[cur ^ 1][ty][tx] = sq;
            s_pr[cur ^ 1][ty][tx] = present;
        }
        cur ^= 1;
        side = pside;
    }
}

// ticket (optional, zero on entry): the last block to finish also folds the remaining levels,
// which then fit one block (tc - 5 <= 5); it leaves the ticket at zero again.
__global__ void __launch_bounds__(256) interior_kernel(const double *__restrict__ child_sq, float *__restrict__ norm,
                                                       float *__restrict__ norm_t, double *__restrict__ sq_levels, int tc,
                                                       unsigned int *ticket)
{
    __shared__ double s_sq[2][16][16];
    __shared__ unsigned char s_pr[2][16][16];
    __shared__ bool s_last;
    pdl_enter();
    interior_fold(child_sq, norm, norm_t, sq_levels, tc, blockIdx.x, blockIdx.y, s_sq, s_pr);
    if (!ticket || tc <= 5) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int n = gridDim.x * gridDim.y;
        s_last = atomicAdd(ticket, 1u) == n - 1;
        if (s_last) *ticket = 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int t2 = tc - 5; t2 > 0; t2 -= 5) {
        __syncthreads();
        interior_fold(sq_levels + spamm_level_offset(t2), norm, norm_t, sq_levels, t2, 0, 0, s_sq, s_pr);
    }
}

__global__ void transpose_level_kernel(const float *__restrict__ src, float *__restrict__ dst, int S)
{
    __shared__ float tile[32][33];
    int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 32 + threadIdx.y;
    for (int r = 0; r < 32; r += 8)
        if (x < S && y + r < S) tile[threadIdx.y + r][threadIdx.x] = src[(int64_t)(y + r) * S + x];
    __syncthreads();
    x = blockIdx.y * 32 + threadIdx.x;
    y = blockIdx.x * 32 + threadIdx.y;
    for (int r = 0; r < 32; r += 8)
        if (x < S && y + r < S) dst[(int64_t)(y + r) * S + x] = tile[threadIdx.x][threadIdx.y + r];
}

int spamm_launch_interior(const double *leaf_sq, int depth, float *norm, float *norm_t, double *sq_levels,
                          unsigned int *ticket, cudaStream_t st)
{
    int tc = depth;
    const double *child = leaf_sq;
    while (tc > 0) {
        const int Sp = 1 << (tc - 1);
        const int g = (Sp + 15) / 16;
        const bool fuse = ticket && tc > 5 && tc - 5 <= 5;      // the rest fits one block
        if (spamm_launch_pdl(interior_kernel, dim3(g, g), dim3(256), 0, st, child, norm, norm_t, sq_levels, tc,
                             fuse ? ticket : (unsigned int *)nullptr) != cudaSuccess)
            return SPAMM_ECUDA;
        SPAMM_CHECK_LAUNCH();
        if (fuse) break;
        tc = (tc - 5 > 0) ? tc - 5 : 0;
        child = sq_levels + spamm_level_offset(tc);
    }
    return SPAMM_OK;
}

extern "C" int spamm_build_interior(const double *leaf_sq, int depth, float *norm, float *norm_t, double *sq_levels,
                                    int write_leaf_transpose, void *stream)
{
    if (depth < 0 || depth > 15 || !norm || !norm_t) return SPAMM_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (write_leaf_transpose) {
        const int L = 1 << depth;
        const int64_t off = spamm_level_offset(depth);
        dim3 tb(32, 8), tg((L + 31) / 32, (L + 31) / 32);
        transpose_level_kernel<<<tg, tb, 0, st>>>(norm + off, norm_t + off, L);
        SPAMM_CHECK_LAUNCH();
    }
    return spamm_launch_interior(leaf_sq, depth, norm, norm_t, sq_levels, nullptr, st);
}

// Packed leaves -> norms in compute_norms order (core.py:108-116): sub-block sums as above,
// leaf total = numpy pairwise sum of the 16 sub-sums: r_j = S_j + S_{j+8}, then
// ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)) -- an xor-butterfly over lane bits 3,0,1,2.
__device__ __forceinline__ double leaf_total_refresh(double S)
{
    double r = __dadd_rn(S, __shfl_xor_sync(FULL_MASK, S, 8));
    r = __dadd_rn(r, __shfl_xor_sync(FULL_MASK, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(FULL_MASK, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(FULL_MASK, r, 4));
    return r;
}

// src == nullptr: the values sit in the records already; else src holds plain 16x16 blocks (256 floats per
// leaf, the reference's packed_leaves() value array, `core.py:387-405`) and the record's value part is written too
__global__ void __launch_bounds__(256) leaf_norms_packed_kernel(const float *__restrict__ src, float *__restrict__ values,
                                                                int64_t nleaf, float *__restrict__ values_t,
                                                                double *__restrict__ leaf_sq)
{
    const int64_t leaf = (int64_t)blockIdx.x * 16 + (threadIdx.x >> 4);
    const int t = threadIdx.x & 15, p = t >> 2, q = t & 3;
    const bool ok = leaf < nleaf;
    const float *in = src ? src + leaf * 256 : values + leaf * SPAMM_REC;
    float4 r[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
        r[i] = ok ? *reinterpret_cast<const float4 *>(in + (4 * p + i) * 16 + 4 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
    const double S = sub_block_sq(r[0], r[1], r[2], r[3]);
    const double total = leaf_total_refresh(S);
    if (!ok) return;
    const float sn = (float)sqrt(S);
    if (src) {
#pragma unroll
        for (int i = 0; i < 4; ++i) *reinterpret_cast<float4 *>(values + leaf * SPAMM_REC + (4 * p + i) * 16 + 4 * q) = r[i];
    }
    values[leaf * SPAMM_REC + 256 + q * 4 + p] = sn;
    if (t == 0) leaf_sq[leaf] = total;
    float *vt = values_t + leaf * SPAMM_REC;
    vt[256 + t] = sn;
    *reinterpret_cast<float4 *>(vt + (4 * q + 0) * 16 + 4 * p) = make_float4(r[0].x, r[1].x, r[2].x, r[3].x);
    *reinterpret_cast<float4 *>(vt + (4 * q + 1) * 16 + 4 * p) = make_float4(r[0].y, r[1].y, r[2].y, r[3].y);
    *reinterpret_cast<float4 *>(vt + (4 * q + 2) * 16 + 4 * p) = make_float4(r[0].z, r[1].z, r[2].z, r[3].z);
    *reinterpret_cast<float4 *>(vt + (4 * q + 3) * 16 + 4 * p) = make_float4(r[0].w, r[1].w, r[2].w, r[3].w);
}

extern "C" int spamm_leaf_norms_packed(float *values, int64_t nleaf, float *values_t, double *leaf_sq, void *stream)
{
    if (nleaf == 0) return SPAMM_OK;
    if (!values || !values_t || nleaf < 0) return SPAMM_EINVAL;
    leaf_norms_packed_kernel<<<(unsigned)((nleaf + 15) / 16), 256, 0, (cudaStream_t)stream>>>(nullptr, values, nleaf,
                                                                                            values_t, leaf_sq);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

extern "C" int spamm_leaves_from_blocks(const float *blocks, int64_t nleaf, float *values, float *values_t,
                                        double *leaf_sq, void *stream)
{
    if (nleaf == 0) return SPAMM_OK;
    if (!blocks || !values || !values_t || !leaf_sq || nleaf < 0) return SPAMM_EINVAL;
    leaf_norms_packed_kernel<<<(unsigned)((nleaf + 15) / 16), 256, 0, (cudaStream_t)stream>>>(blocks, values, nleaf,
                                                                                            values_t, leaf_sq);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

// ---- operands that stay on the host: only the leaves a product touches cross PCIe ----------------
// A tree whose leaf VALUES are still in (pinned, device-readable) host memory: keys, leaf norms and sub-block
// norms are on the device, so the symbolic phase can run; the numeric phase then needs the values of the
// leaves that occur in a surviving task and of no others.  (1) the sub-norm tails of the records, from the
// reference's sub-norm array (core.py:387-405, [leaf][p][q]); (2) which leaves a plan touches; (3) their
// values, read by the GPU straight from host memory into both record layouts.
__global__ void __launch_bounds__(256) subnorm_tails_kernel(const float *__restrict__ subs, int64_t nleaf,
                                                            float *__restrict__ values, float *__restrict__ values_t)
{
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= nleaf * 16) return;
    const int64_t leaf = x >> 4;
    const int p = (int)(x & 15) >> 2, q = (int)x & 3;
    const float v = subs[x];                                 // sub[p][q]
    if (values) values[leaf * SPAMM_REC + 256 + q * 4 + p] = v;
    if (values_t) values_t[leaf * SPAMM_REC + 256 + p * 4 + q] = v;
}

extern "C" int spamm_subnorm_tails(const float *subs, int64_t nleaf, float *values, float *values_t, void *stream)
{
    if (nleaf == 0) return SPAMM_OK;
    if (!subs || nleaf < 0 || (!values && !values_t)) return SPAMM_EINVAL;
    subnorm_tails_kernel<<<(unsigned)((nleaf * 16 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(subs, nleaf, values, values_t);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

// flags_a[x] / flags_b[x] = 1 for every packed leaf x of the left / right operand that a live task of the plan
// reads (the arrays must be zero on entry; they may be the same array when both operands are one tree)
__global__ void __launch_bounds__(256) mark_touched_kernel(const spamm_step *__restrict__ steps, const int32_t *__restrict__ counts,
                                                           unsigned char *__restrict__ flags_a, unsigned char *__restrict__ flags_b)
{
    const int nsteps = counts[2] ? 0 : counts[4];
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nsteps; s += gridDim.x * blockDim.x) {
        const spamm_step r = steps[s];
        uint32_t ta = 0, tb = 0;                             // touched leaves of the A block / the B block (bit morton4)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const uint32_t live = r.live[kk] & 0xFFFFu;
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                if (live & step_rowmask(d)) ta |= 1u << step_pos(d, kk);      // A leaf (di = d, kk)
                if (live & step_colmask(d)) tb |= 1u << step_pos(kk, d);      // B leaf (kk, dj = d)
            }
        }
        for (uint32_t m = ta & r.a_present; m; m &= m - 1) {
            const int pos = __ffs(m) - 1;
            flags_a[(int64_t)r.a_first + __popc(r.a_present & ((1u << pos) - 1u))] = 1;
        }
        for (uint32_t m = tb & r.b_present; m; m &= m - 1) {
            const int pos = __ffs(m) - 1;
            flags_b[(int64_t)r.b_first + __popc(r.b_present & ((1u << pos) - 1u))] = 1;
        }
    }
}

extern "C" int spamm_mark_touched(const spamm_plan_buffers *plan, unsigned char *flags_a, unsigned char *flags_b, void *stream)
{
    if (!plan || !flags_a || !flags_b) return SPAMM_EINVAL;
    mark_touched_kernel<<<SPAMM_NUM_SMS * 4, 256, 0, (cudaStream_t)stream>>>(plan->steps, plan->counts, flags_a, flags_b);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

// One warp per flagged leaf: its 16x16 block from (device-readable) host memory into the row-major record
// (want & 1) and / or the transposed one (want & 2); `copied` counts the leaves fetched.
__global__ void __launch_bounds__(256) gather_blocks_kernel(const float *__restrict__ blocks, const unsigned char *__restrict__ flags,
                                                            int64_t nleaf, int want, float *__restrict__ values,
                                                            float *__restrict__ values_t, unsigned long long *copied)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    unsigned long long mine = 0;
    for (int64_t leaf = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); leaf < nleaf; leaf += warps) {
        if (!flags[leaf]) continue;
        ++mine;
        const float4 *src = reinterpret_cast<const float4 *>(blocks + leaf * 256);
        const float4 v0 = src[lane], v1 = src[lane + 32];        // elements 4*lane .. and 128 + 4*lane ..
        if (want & 1) {
            float4 *dst = reinterpret_cast<float4 *>(values + leaf * SPAMM_REC);
            dst[lane] = v0;
            dst[lane + 32] = v1;
        }
        if (want & 2) {
            float *dt = values_t + leaf * SPAMM_REC;
            const int r0 = lane >> 2, c0 = (lane & 3) * 4;       // v0 = row r0, columns c0..c0+3; v1 = row r0 + 8
            dt[(c0 + 0) * 16 + r0] = v0.x; dt[(c0 + 1) * 16 + r0] = v0.y; dt[(c0 + 2) * 16 + r0] = v0.z; dt[(c0 + 3) * 16 + r0] = v0.w;
            dt[(c0 + 0) * 16 + r0 + 8] = v1.x; dt[(c0 + 1) * 16 + r0 + 8] = v1.y; dt[(c0 + 2) * 16 + r0 + 8] = v1.z; dt[(c0 + 3) * 16 + r0 + 8] = v1.w;
        }
    }
    if (copied && lane == 0 && mine) atomicAdd(copied, mine);
}

extern "C" int spamm_gather_blocks(const float *blocks, const unsigned char *flags, int64_t nleaf, int want, float *values,
                                   float *values_t, unsigned long long *copied, void *stream)
{
    if (nleaf == 0) return SPAMM_OK;
    if (!blocks || !flags || nleaf < 0 || !(want & 3) || ((want & 1) && !values) || ((want & 2) && !values_t)) return SPAMM_EINVAL;
    gather_blocks_kernel<<<SPAMM_NUM_SMS * 8, 256, 0, (cudaStream_t)stream>>>(blocks, flags, nleaf, want, values, values_t, copied);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

// QuadtreeMatrix.sparsify (core.py:347-383): zero every 4x4 sub-block with 0 < sub-norm < eps.  A
// leaf that lost a sub-block gets its norms refreshed in compute_norms order; an untouched leaf
// keeps its norms and contributes float64(norm)^2 to the interior sums, as the reference does.
// 16 threads per leaf, thread (p,q) owns one sub-block.  dropped += number of zeroed sub-blocks.
__global__ void __launch_bounds__(256) sparsify_kernel(float *__restrict__ values, float *__restrict__ values_t,
                                                       double *__restrict__ leaf_sq, int64_t nleaf, float eps,
                                                       unsigned long long *dropped)
{
    const int64_t leaf = (int64_t)blockIdx.x * 16 + (threadIdx.x >> 4);
    const int t = threadIdx.x & 15, p = t >> 2, q = t & 3;
    const bool ok = leaf < nleaf;
    const float sn = ok ? values[leaf * SPAMM_REC + 256 + q * 4 + p] : 0.0f;
    const bool drop = ok && sn > 0.0f && sn < eps;
    const uint32_t bal = __ballot_sync(FULL_MASK, drop);
    const uint32_t mine = (bal >> (threadIdx.x & 16)) & 0xFFFFu;      // my leaf's 16 lanes
    float4 r[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
        r[i] = (ok && !drop) ? *reinterpret_cast<const float4 *>(values + leaf * SPAMM_REC + (4 * p + i) * 16 + 4 * q)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
    const double S = sub_block_sq(r[0], r[1], r[2], r[3]);
    const double total = leaf_total_refresh(S);
    if (!ok) return;
    if (!mine) {
        if (t == 0) {
            const double nv = (double)(float)sqrt(leaf_sq[leaf]);
            leaf_sq[leaf] = nv * nv;
        }
        return;
    }
    if (drop) {
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        float *v = values + leaf * SPAMM_REC, *vt = values_t + leaf * SPAMM_REC;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            *reinterpret_cast<float4 *>(v + (4 * p + i) * 16 + 4 * q) = z;
            *reinterpret_cast<float4 *>(vt + (4 * q + i) * 16 + 4 * p) = z;
        }
        v[256 + q * 4 + p] = 0.0f;
        vt[256 + t] = 0.0f;
    }
    if (t == 0) {
        leaf_sq[leaf] = total;
        atomicAdd(dropped, (unsigned long long)__popc(mine));
    }
}

extern "C" int spamm_sparsify_leaves(float *values, float *values_t, double *leaf_sq, int64_t nleaf, float eps,
                                     unsigned long long *dropped, void *stream)
{
    if (nleaf == 0) return SPAMM_OK;
    if (!values || !values_t || !leaf_sq || !dropped || nleaf < 0 || !(eps >= 0.0f)) return SPAMM_EINVAL;
    sparsify_kernel<<<(unsigned)((nleaf + 15) / 16), 256, 0, (cudaStream_t)stream>>>(values, values_t, leaf_sq, nleaf, eps,
                                                                                   dropped);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

// values -> values_t for leaves whose norms are already in the record tails (e.g. leaves that
// arrived from another GPU): transposes the 16x16 values and the 4x4 sub-norm tail, nothing else.
__global__ void __launch_bounds__(256) transpose_records_kernel(const float *__restrict__ values,
                                                                float *__restrict__ values_t, int64_t nleaf)
{
    // one warp per leaf and pass, 16-byte loads and stores, transposition through shared memory
    __shared__ float tile[8][16][17];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float(*t)[17] = tile[warp];
    for (int64_t s = (int64_t)blockIdx.x * 8 + warp; s < nleaf; s += (int64_t)gridDim.x * 8) {
        const float4 *src = reinterpret_cast<const float4 *>(values + s * SPAMM_REC);
        float4 *dst = reinterpret_cast<float4 *>(values_t + s * SPAMM_REC);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = lane + 32 * h, r = e >> 2, c = (e & 3) * 4;
            const float4 v = src[e];
            t[r][c] = v.x; t[r][c + 1] = v.y; t[r][c + 2] = v.z; t[r][c + 3] = v.w;
        }
        float tail = 0.0f;
        if (lane < 16) tail = values[s * SPAMM_REC + 256 + lane];
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = lane + 32 * h, r = e >> 2, c = (e & 3) * 4;
            dst[e] = make_float4(t[c][r], t[c + 1][r], t[c + 2][r], t[c + 3][r]);
        }
        // values tail is [q*4+p], values_t tail is [p*4+q]
        if (lane < 16) values_t[s * SPAMM_REC + 256 + (lane & 3) * 4 + (lane >> 2)] = tail;
        __syncwarp();
    }
}

extern "C" int spamm_transpose_records(const float *values, int64_t nleaf, float *values_t, void *stream)
{
    if (nleaf == 0) return SPAMM_OK;
    if (!values || !values_t || nleaf < 0) return SPAMM_EINVAL;
    int64_t blocks = (nleaf + 7) / 8;
    if (blocks > SPAMM_NUM_SMS * 16) blocks = SPAMM_NUM_SMS * 16;
    transpose_records_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(values, values_t, nleaf);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

// ---- sub-norm ranges (fine4 task classification in the planner) --------------------------------------
// Per cell of the leaf grid one word: bf16(max sub-norm) rounded up in the high half, bf16(min
// sub-norm) rounded down in the low half; 0xFFFFFFFF (two NaNs) for an absent leaf or one with a
// non-finite sub-norm.  With these bounds the planner can tell for most tasks, without reading the
// leaves, that all 64 gated micro products pass (min * min >= tau) or none does (max * max < tau):
// products of non-negative floats are monotone in both factors (numeric.py:233-238 is the exact rule).
__global__ void __launch_bounds__(256) subrange_kernel(const float *__restrict__ values,
                                                       const int32_t *__restrict__ slot, int L,
                                                       uint32_t *__restrict__ sub, uint32_t *__restrict__ sub_t)
{
    const int64_t cells = (int64_t)L * L;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < cells; x += (int64_t)gridDim.x * blockDim.x) {
        const int32_t s = slot[x];
        uint32_t word = 0xFFFFFFFFu;
        if (s >= 0) {
            const float4 *tl = reinterpret_cast<const float4 *>(values + (int64_t)s * SPAMM_REC + 256);
            const float4 t0 = tl[0], t1 = tl[1], t2 = tl[2], t3 = tl[3];
            float mn = fminf(fminf(fminf(t0.x, t0.y), fminf(t0.z, t0.w)), fminf(fminf(t1.x, t1.y), fminf(t1.z, t1.w)));
            mn = fminf(mn, fminf(fminf(fminf(t2.x, t2.y), fminf(t2.z, t2.w)), fminf(fminf(t3.x, t3.y), fminf(t3.z, t3.w))));
            float mx = fmaxf(fmaxf(fmaxf(t0.x, t0.y), fmaxf(t0.z, t0.w)), fmaxf(fmaxf(t1.x, t1.y), fmaxf(t1.z, t1.w)));
            mx = fmaxf(mx, fmaxf(fmaxf(fmaxf(t2.x, t2.y), fmaxf(t2.z, t2.w)), fmaxf(fmaxf(t3.x, t3.y), fmaxf(t3.z, t3.w))));
            const float sum = ((t0.x + t0.y) + (t0.z + t0.w)) + ((t1.x + t1.y) + (t1.z + t1.w)) +
                              ((t2.x + t2.y) + (t2.z + t2.w)) + ((t3.x + t3.y) + (t3.z + t3.w));
            const bool ok = (sum - sum == 0.0f) && mn >= 0.0f;      // no NaN, no infinity, nothing negative
            if (ok) {
                const uint32_t lo = __float_as_uint(mn) >> 16;                       // towards zero
                const uint32_t hi = (__float_as_uint(mx) + 0xFFFFu) >> 16;           // away from zero
                word = (hi << 16) | lo;
            }
        }
        sub[x] = word;
        const int64_t i = x / L, j = x - i * L;
        sub_t[j * L + i] = word;
    }
}

extern "C" int spamm_subrange_grids(const float *values, const int32_t *slot, int depth, uint32_t *sub, uint32_t *sub_t,
                                    void *stream)
{
    if (!slot || !sub || !sub_t || depth < 0 || depth > 15) return SPAMM_EINVAL;
    const int L = 1 << depth;
    int64_t blocks = ((int64_t)L * L + 255) / 256;
    if (blocks > SPAMM_NUM_SMS * 16) blocks = SPAMM_NUM_SMS * 16;
    subrange_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(values, slot, L, sub, sub_t);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}

// Grids of a tree given by packed leaves: clear, then scatter.
__global__ void clear_grids_kernel(int64_t cells, int32_t *slot, int32_t *slot_t, float *norm, float *norm_t,
                                   double *leaf_sq_grid)
{
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < cells; x += (int64_t)gridDim.x * blockDim.x) {
        slot[x] = -1;
        slot_t[x] = -1;
        norm[x] = -1.0f;
        norm_t[x] = -1.0f;
        leaf_sq_grid[x] = 0.0;
    }
}
// nleaf_dev (optional): the leaf count still lives on the device; nleaf is then only its upper bound
__global__ void scatter_leaves_kernel(const uint32_t *__restrict__ keys, const double *__restrict__ leaf_sq_packed,
                                      int64_t nleaf, const int32_t *__restrict__ nleaf_dev, int L, int32_t *slot,
                                      int32_t *slot_t, float *norm, float *norm_t, double *leaf_sq_grid)
{
    if (nleaf_dev && (int64_t)*nleaf_dev < nleaf) nleaf = *nleaf_dev;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nleaf; s += (int64_t)gridDim.x * blockDim.x) {
        uint32_t i, j;
        if (keys[s] == 0xFFFFFFFFu) continue;     // unused slot of a gathered shard
        morton_decode(keys[s], i, j);
        const double sq = leaf_sq_packed[s];
        const float nv = (float)sqrt(sq);       // a stored leaf keeps norm 0 when it is all zero (core.py:336-339)
        slot[(int64_t)i * L + j] = (int32_t)s;
        slot_t[(int64_t)j * L + i] = (int32_t)s;
        norm[(int64_t)i * L + j] = nv;
        norm_t[(int64_t)j * L + i] = nv;
        leaf_sq_grid[(int64_t)i * L + j] = sq;
    }
}

int spamm_index_leaves_impl(const uint32_t *keys, const double *leaf_sq_packed, int64_t nleaf, const int32_t *nleaf_dev,
                            int depth, int32_t *slot, int32_t *slot_t, float *norm, float *norm_t, double *leaf_sq_grid,
                            cudaStream_t st)
{
    if (depth < 0 || depth > 15 || nleaf < 0) return SPAMM_EINVAL;
    const int L = 1 << depth;
    const int64_t cells = (int64_t)L * L;
    const int64_t off = spamm_level_offset(depth);
    int blocks = (int)((cells + 255) / 256);
    if (blocks > SPAMM_NUM_SMS * 16) blocks = SPAMM_NUM_SMS * 16;
    clear_grids_kernel<<<blocks, 256, 0, st>>>(cells, slot, slot_t, norm + off, norm_t + off, leaf_sq_grid);
    SPAMM_CHECK_LAUNCH();
    if (nleaf > 0) {
        int sb = (int)((nleaf + 255) / 256);
        if (sb > SPAMM_NUM_SMS * 8) sb = SPAMM_NUM_SMS * 8;
        scatter_leaves_kernel<<<sb, 256, 0, st>>>(keys, leaf_sq_packed, nleaf, nleaf_dev, L, slot, slot_t, norm + off,
                                                  norm_t + off, leaf_sq_grid);
        SPAMM_CHECK_LAUNCH();
    }
    return SPAMM_OK;
}

extern "C" int spamm_index_leaves(const uint32_t *keys, const double *leaf_sq_packed, int64_t nleaf, int depth,
                                  int32_t *slot, int32_t *slot_t, float *norm, float *norm_t, double *leaf_sq_grid,
                                  void *stream)
{
    return spamm_index_leaves_impl(keys, leaf_sq_packed, nleaf, nullptr, depth, slot, slot_t, norm, norm_t, leaf_sq_grid,
                                   (cudaStream_t)stream);
}

// QuadtreeMatrix.to_dense (core.py:268-276): one block per 16x16 block of the output.
__global__ void __launch_bounds__(256) to_dense_kernel(const int32_t *__restrict__ slot, const float *__restrict__ values,
                                                       int L, int64_t m, int64_t n, float *__restrict__ out, int64_t ld)
{
    const int bi = blockIdx.y, bj = blockIdx.x;
    const int r = threadIdx.x >> 4, c = threadIdx.x & 15;
    const int64_t gi = (int64_t)bi * 16 + r, gj = (int64_t)bj * 16 + c;
    if (gi >= m || gj >= n) return;
    const int32_t s = slot[(int64_t)bi * L + bj];
    out[gi * ld + gj] = s >= 0 ? values[(int64_t)s * SPAMM_REC + threadIdx.x] : 0.0f;
}

extern "C" int spamm_to_dense(const spamm_tree_view *t, float *out, int64_t ld, void *stream)
{
    if (!t || !out || ld < t->n) return SPAMM_EINVAL;
    dim3 grid((t->n + 15) / 16, (t->m + 15) / 16);
    to_dense_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(t->slot, t->values, 1 << t->depth, t->m, t->n, out, ld);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}
