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
// positions that share leaf row di / leaf column dj
__host__ __device__ __forceinline__ uint32_t step_rowmask(int di)
{
    return di == 0 ? 0x0033u : di == 1 ? 0x00CCu : di == 2 ? 0x3300u : 0xCC00u;
}
__host__ __device__ __forceinline__ uint32_t step_colmask(int dj)
{
    return dj == 0 ? 0x0505u : dj == 1 ? 0x0A0Au : dj == 2 ? 0x5050u : 0xA0A0u;
}
