// Single-pass exclusive scan of 0/1 flags with decoupled look-back ("ballot + prefix sum"
// compaction).  Used wherever a list has to be compacted in a fixed order: stored leaves
// along the Z curve (tree.cu) and super-tile starts (execute.cu).
//
// Op must provide   int  flag(int64_t e) const;           // 0 or 1
//                   void emit(int64_t e, int flag, int32_t exclusive_prefix) const;
#pragma once

#include "common.cuh"

#define SCAN_THREADS 256
#define SCAN_ITEMS 8
#define SCAN_TILE (SCAN_THREADS * SCAN_ITEMS)

static inline size_t scan_workspace_bytes(int64_t n)
{
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    return (size_t)(16 + 8 * (tiles > 0 ? tiles : 1));
}

template <class Op>
__global__ void __launch_bounds__(SCAN_THREADS) scan_flags_kernel(Op op, int64_t n, int ntiles, int32_t *total_out,
                                                                  unsigned int *tile_counter,
                                                                  volatile unsigned long long *tile_state)
{
    __shared__ int s_tile;
    __shared__ uint32_t s_warp[SCAN_THREADS / 32];
    __shared__ uint32_t s_base;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_tile = (int)atomicAdd(tile_counter, 1u);
        __syncthreads();
        const int tile = s_tile;
        if (tile >= ntiles) return;
        const int64_t e0 = (int64_t)tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
        uint32_t bits = 0, cnt = 0;
#pragma unroll
        for (int x = 0; x < SCAN_ITEMS; ++x) {
            const int f = (e0 + x < n) ? op.flag(e0 + x) : 0;
            bits |= (uint32_t)f << x;
            cnt += f;
        }
        // warp inclusive scan of per-thread counts
        uint32_t inc = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t v = __shfl_up_sync(FULL_MASK, inc, d);
            if (lane_id() >= (uint32_t)d) inc += v;
        }
        if (lane_id() == 31) s_warp[threadIdx.x >> 5] = inc;
        __syncthreads();
        if (threadIdx.x < 32) {
            const uint32_t l = threadIdx.x;
            const uint32_t v = l < SCAN_THREADS / 32 ? s_warp[l] : 0u;
            uint32_t iv = v;                    // inclusive scan over the block's warps
#pragma unroll
            for (int d = 1; d < SCAN_THREADS / 32; d <<= 1) {
                const uint32_t x = __shfl_up_sync(FULL_MASK, iv, d);
                if (l >= (uint32_t)d) iv += x;
            }
            const uint32_t run = __shfl_sync(FULL_MASK, iv, SCAN_THREADS / 32 - 1);
            if (l < SCAN_THREADS / 32) s_warp[l] = iv - v;
            uint32_t ex, dummy;
            lb_exclusive_warp(tile_state, tile, run, 0u, ex, dummy);
            if (l == 0) {
                s_base = ex;
                if (tile == ntiles - 1) *total_out = (int32_t)(ex + run);
            }
        }
        __syncthreads();
        uint32_t pos = s_base + s_warp[threadIdx.x >> 5] + (inc - cnt);
#pragma unroll
        for (int x = 0; x < SCAN_ITEMS; ++x) {
            if (e0 + x < n) {
                const int f = (bits >> x) & 1;
                op.emit(e0 + x, f, (int32_t)pos);
                pos += f;
            }
        }
    }
}

template <class Op>
static int scan_flags(const Op &op, int64_t n, int32_t *total_dev, void *ws, size_t ws_bytes, cudaStream_t st)
{
    if (n < 0 || n > (int64_t(1) << 31) - 1) return SPAMM_EINVAL;
    const size_t need = scan_workspace_bytes(n);
    if (!ws || ws_bytes < need) return SPAMM_EWORKSPACE;
    if (cudaMemsetAsync(ws, 0, need, st) != cudaSuccess) return SPAMM_ECUDA;
    if (cudaMemsetAsync(total_dev, 0, sizeof(int32_t), st) != cudaSuccess) return SPAMM_ECUDA;
    if (n == 0) return SPAMM_OK;
    const int ntiles = (int)((n + SCAN_TILE - 1) / SCAN_TILE);
    int blocks = ntiles < SPAMM_NUM_SMS * 4 ? ntiles : SPAMM_NUM_SMS * 4;
    unsigned int *counter = reinterpret_cast<unsigned int *>(ws);
    volatile unsigned long long *state = reinterpret_cast<volatile unsigned long long *>(reinterpret_cast<char *>(ws) + 16);
    scan_flags_kernel<Op><<<blocks, SCAN_THREADS, 0, st>>>(op, n, ntiles, total_dev, counter, state);
    SPAMM_CHECK_LAUNCH();
    return SPAMM_OK;
}
