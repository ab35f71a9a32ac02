// Device helpers for the step records of a plan (struct spamm_step, include/spamm_b200.h).
#pragma once

#include "common.cuh"

// position of leaf (di, dj) inside its 4x4 super-tile = low four bits of its Morton key
__host__ __device__ __forceinline__ int step_pos(int di, int dj)
{
    return ((di >> 1) << 3) | ((dj >> 1) << 2) | ((di & 1) << 1) | (dj & 1);
}
__host__ __device__ __forceinline__ int step_pos_di(int pos) { return ((pos >> 3) & 1) << 1 | ((pos >> 1) & 1); }
__host__ __device__ __forceinline__ int step_pos_dj(int pos) { return ((pos >> 2) & 1) << 1 | (pos & 1); }
// Work units (spamm_b200.h).  When the planner cuts tiles (counts[12] = seg_len != 0) a unit is
// node | segment << 20 | segments << 26, otherwise just the node.
#define UNIT_NODE_BITS 20
#define UNIT_MAX_SEGMENTS 63
#define UNIT_SIZE_CLAMP 127      // tiles are ranked by (min(records, 127), how full the records are)
// size class of a super-tile for the longest-first hand-out: records first, then eighths of fill
// (live tasks per record slot), 0 for a tile without records; 1024 classes
__host__ __device__ __forceinline__ int tile_size_class(int nsteps, int ntasks)
{
    if (nsteps <= 0) return 0;
    const int st = nsteps < UNIT_SIZE_CLAMP ? nsteps : UNIT_SIZE_CLAMP;
    int fill = (int)(((long long)ntasks * 8 - 1) / (64ll * nsteps));
    fill = fill < 0 ? 0 : (fill > 7 ? 7 : fill);
    return st * 8 + fill;
}
__host__ __device__ __forceinline__ uint32_t unit_pack(int node, int seg, int nseg)
{
    return (uint32_t)node | ((uint32_t)seg << UNIT_NODE_BITS) | ((uint32_t)nseg << 26);
}
__host__ __device__ __forceinline__ int unit_segments(int ns, int seg_len)
{
    if (seg_len <= 0) return 1;
    const int c = ns < UNIT_SIZE_CLAMP ? ns : UNIT_SIZE_CLAMP;
    const int n = (c + seg_len - 1) / seg_len;
    return n < UNIT_MAX_SEGMENTS ? (n > 0 ? n : 1) : UNIT_MAX_SEGMENTS;
}
// first record (relative to the tile) of segment s of nseg
__host__ __device__ __forceinline__ int unit_begin(int ns, int nseg, int s)
{
    return (int)(((long long)s * ns) / nseg);
}
// positions that share leaf row di / leaf column dj
__host__ __device__ __forceinline__ uint32_t step_rowmask(int di)
{
    return di == 0 ? 0x0033u : di == 1 ? 0x00CCu : di == 2 ? 0x3300u : 0xCC00u;
}
__host__ __device__ __forceinline__ uint32_t step_colmask(int dj)
{
    return dj == 0 ? 0x0505u : dj == 1 ? 0x0A0Au : dj == 2 ? 0x5050u : 0xA0A0u;
}

// plan.tile_order holds 4 ints per work unit (b, end of b's tile, start of the tile of e - 1, e), see plan_order_kernel
__host__ __device__ __forceinline__ int64_t spamm_unit_capacity(int64_t leaf_capacity)
{
    return (leaf_capacity + SPAMM_UNIT_EXTRA) / 4;
}
