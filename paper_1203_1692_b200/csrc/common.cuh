// Shared device/host helpers for the SpAMM B200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/spamm_b200.h"

#define SPAMM_NB 16
#define SPAMM_LEAF 256
#define SPAMM_REC 272              // floats per stored leaf: 256 values + 16 sub-block norms
#define SPAMM_REC_BYTES 1088
// SMs of the current device (queried once per process, abi.cu); grids are sized in multiples of it
int spamm_num_sms();
#define SPAMM_NUM_SMS (spamm_num_sms())

// ---- launch bookkeeping -----------------------------------------------------
extern "C" int64_t spamm_launch_count(void);
void spamm_note_launch(int n = 1);

#define SPAMM_CHECK_LAUNCH()                                      \
    do {                                                          \
        spamm_note_launch();                                      \
        if (cudaPeekAtLastError() != cudaSuccess) {               \
            (void)cudaGetLastError();                             \
            return SPAMM_ECUDA;                                   \
        }                                                         \
    } while (0)

// ---- programmatic dependent launch ------------------------------------------------------------------
// The kernels of one multiply run back to back on one stream.  Launched with the programmatic
// stream serialization attribute, a kernel's CTAs may become resident while its predecessor is
// still running; every such kernel first waits for the predecessor's completion (and memory
// flush) with pdl_enter(), which also lets ITS successor start launching.  Only the launch latency
// and the prologue overlap; no kernel touches memory before its predecessor has finished.
__device__ __forceinline__ void pdl_enter()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool spamm_pdl_enabled();      // SPAMM_PDL=0 turns the attribute off (abi.cu)
template <typename... Params, typename... Args>
inline cudaError_t spamm_launch_pdl(void (*kernel)(Params...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                    Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = spamm_pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, Params(args)...);
}

// Level t of a level buffer starts at element spamm_level_offset(t): levels are packed root
// first, each start rounded to 4 elements so rows can be read with vector loads.
__host__ __device__ static inline int64_t spamm_level_offset(int t)
{
    return t == 0 ? 0 : 4 + ((int64_t(1) << (2 * t)) - 4) / 3;
}

// ---- Morton keys (reference morton.py:35-68: row bit above column bit) -------
__host__ __device__ __forceinline__ uint32_t spread16(uint32_t x)
{
    x &= 0xFFFFu;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}
__host__ __device__ __forceinline__ uint32_t squeeze16(uint32_t x)
{
    x &= 0x55555555u;
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0F0F0F0Fu;
    x = (x | (x >> 4)) & 0x00FF00FFu;
    x = (x | (x >> 8)) & 0x0000FFFFu;
    return x;
}
__host__ __device__ __forceinline__ uint32_t morton_encode(uint32_t i, uint32_t j)
{
    return (spread16(i) << 1) | spread16(j);
}
__host__ __device__ __forceinline__ void morton_decode(uint32_t key, uint32_t &i, uint32_t &j)
{
    i = squeeze16(key >> 1);
    j = squeeze16(key);
}

// ---- the norm test (symbolic.py:118-120, numeric.py:233-238) ------------------
// Both factors are float32 values, so the double product is exact; the comparison is
// the reference's `not (p < tau)` == `p >= tau` for non-NaN operands.  A negative norm
// marks an absent node.
__device__ __forceinline__ bool norm_test(float a, float b, double tau)
{
    return (a >= 0.0f) && (b >= 0.0f) && (__dmul_rn((double)a, (double)b) >= tau);
}

// ---- warp helpers ---------------------------------------------------------------
#define FULL_MASK 0xFFFFFFFFu
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---- mbarrier / bulk-copy (TMA 1-D) PTX wrappers ---------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// ---- flags in global memory handed between CTAs ---------------------------------------------------
__device__ __forceinline__ int ld_acquire_gpu(const int32_t *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int32_t *p, int v)
{
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// try_wait with a suspend-time hint: the warp sleeps in hardware until the phase completes or the
// hint (ns) expires, instead of coming back to the issue stage every few dozen cycles.
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t *bar, uint32_t parity, uint32_t ns)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
        : "memory");
    return ok != 0;
}
#ifndef MBAR_HINT_NS
#define MBAR_HINT_NS 20000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    if (mbar_try_wait(bar, parity)) return;
#if MBAR_HINT_NS > 0
    while (!mbar_try_wait_hint(bar, parity, MBAR_HINT_NS)) {
    }
#else
    while (!mbar_try_wait(bar, parity)) {
    }
#endif
}
// A wait that is not on anybody's critical path (the producer waiting for a stage to be handed back, two
// stages ahead of the consumers): poll rarely.  Every poll is an instruction on the producer's warp
// scheduler, which it shares with four consumer warps -- measured (ncu), the plain spin took 12 % of
// that scheduler's issue slots and made it the slowest of the team.
__device__ __forceinline__ void mbar_wait_relaxed(uint64_t *bar, uint32_t parity, uint32_t ns)
{
    while (!mbar_try_wait(bar, parity)) __nanosleep(ns);
}
// 1-D bulk copy global -> shared, completion counted on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void bulk_copy_g2s(void *smem_dst, const void *gmem_src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ---- decoupled look-back tile state ------------------------------------------------
// 64-bit word: [63:62] status, [61:31] second counter, [30:0] first counter.
#define LB_INVALID 0ull
#define LB_AGGREGATE 1ull
#define LB_PREFIX 2ull
__device__ __forceinline__ unsigned long long lb_pack(unsigned long long status, uint32_t lo, uint32_t hi)
{
    return (status << 62) | ((unsigned long long)hi << 31) | (unsigned long long)lo;
}
__device__ __forceinline__ uint32_t lb_lo(unsigned long long w) { return (uint32_t)(w & 0x7FFFFFFFull); }
__device__ __forceinline__ uint32_t lb_hi(unsigned long long w) { return (uint32_t)((w >> 31) & 0x7FFFFFFFull); }
__device__ __forceinline__ unsigned long long lb_status(unsigned long long w) { return w >> 62; }

// The same result when block b takes tile b (blocks start in index order, so every predecessor is running
// or done): every tile publishes its aggregate and reads ALL of its predecessors in batches of 256 (eight
// per lane, loads in flight together) instead of walking back 32 at a time -- one memory round trip after
// the slowest tile for up to 256 tiles.
#define PLAN_ALL_EXCLUSIVE_MAX 1024
__device__ __forceinline__ void all_exclusive_warp(volatile unsigned long long *state, int tile, uint32_t agg_lo,
                                                   uint32_t agg_hi, uint32_t &ex_lo, uint32_t &ex_hi)
{
    const int lane = (int)(threadIdx.x & 31u);
    if (lane == 0) state[tile] = lb_pack(LB_AGGREGATE, agg_lo, agg_hi);   // the word is the whole message: no fence
    uint32_t lo = 0, hi = 0;
    for (int base = 0; base < tile; base += 256) {
        unsigned long long w[8];
        bool need[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) {
            need[x] = base + lane + 32 * x < tile;
            w[x] = 0ull;
        }
        bool again;
        do {
            again = false;
#pragma unroll
            for (int x = 0; x < 8; ++x)
                if (need[x]) w[x] = state[base + lane + 32 * x];
#pragma unroll
            for (int x = 0; x < 8; ++x)
                if (need[x]) {
                    if (lb_status(w[x]) == LB_INVALID) again = true;
                    else need[x] = false;
                }
        } while (__any_sync(0xFFFFFFFFu, again));
#pragma unroll
        for (int x = 0; x < 8; ++x)
            if (base + lane + 32 * x < tile) { lo += lb_lo(w[x]); hi += lb_hi(w[x]); }
    }
    ex_lo = __reduce_add_sync(0xFFFFFFFFu, lo);
    ex_hi = __reduce_add_sync(0xFFFFFFFFu, hi);
}

// Called by ONE WARP of a tile (all 32 lanes, same arguments): publishes the tile's aggregate, then
// inspects 32 predecessors per step -- nearest first -- until one of them carries an inclusive
// prefix.  Returns the exclusive prefix (lo, hi) in every lane and publishes the inclusive one.
__device__ __forceinline__ void lb_exclusive_warp(volatile unsigned long long *state, int tile, uint32_t agg_lo,
                                                  uint32_t agg_hi, uint32_t &ex_lo, uint32_t &ex_hi)
{
    const uint32_t lane = threadIdx.x & 31u;
    if (tile == 0) {
        ex_lo = ex_hi = 0;
        if (lane == 0) {
            __threadfence();
            state[0] = lb_pack(LB_PREFIX, agg_lo, agg_hi);
        }
        return;
    }
    if (lane == 0) {
        __threadfence();
        state[tile] = lb_pack(LB_AGGREGATE, agg_lo, agg_hi);
    }
    uint32_t lo = 0, hi = 0;
    for (int base = tile - 1; base >= 0; base -= 32) {
        const int idx = base - (int)lane;                 // lane 0 looks at the nearest predecessor
        unsigned long long w = lb_pack(LB_PREFIX, 0u, 0u);   // before tile 0: an empty prefix
        if (idx >= 0) {
            do {
                w = state[idx];
            } while (lb_status(w) == LB_INVALID);
        }
        const uint32_t pref = __ballot_sync(0xFFFFFFFFu, lb_status(w) == LB_PREFIX);
        // take every lane up to and including the first one that holds a prefix
        const uint32_t take = pref ? ((2u << (__ffs(pref) - 1)) - 1u) : 0xFFFFFFFFu;
        const bool mine = (take >> lane) & 1u;
        lo += __reduce_add_sync(0xFFFFFFFFu, mine ? lb_lo(w) : 0u);
        hi += __reduce_add_sync(0xFFFFFFFFu, mine ? lb_hi(w) : 0u);
        if (pref) break;
    }
    ex_lo = lo;
    ex_hi = hi;
    if (lane == 0) {
        __threadfence();
        state[tile] = lb_pack(LB_PREFIX, lo + agg_lo, hi + agg_hi);
    }
}

// Called by ONE thread of a tile: publishes the tile's aggregate, walks back over the
// predecessors and returns the exclusive prefix (lo, hi); then publishes the inclusive one.
__device__ __forceinline__ void lb_exclusive(volatile unsigned long long *state, int tile, uint32_t agg_lo,
                                             uint32_t agg_hi, uint32_t &ex_lo, uint32_t &ex_hi)
{
    if (tile == 0) {
        ex_lo = ex_hi = 0;
        __threadfence();
        state[0] = lb_pack(LB_PREFIX, agg_lo, agg_hi);
        return;
    }
    __threadfence();
    state[tile] = lb_pack(LB_AGGREGATE, agg_lo, agg_hi);
    uint32_t lo = 0, hi = 0;
    for (int p = tile - 1; p >= 0; --p) {
        unsigned long long w;
        do {
            w = state[p];
        } while (lb_status(w) == LB_INVALID);
        lo += lb_lo(w);
        hi += lb_hi(w);
        if (lb_status(w) == LB_PREFIX) break;
    }
    ex_lo = lo;
    ex_hi = hi;
    __threadfence();
    state[tile] = lb_pack(LB_PREFIX, lo + agg_lo, hi + agg_hi);
}

// ---- the same for ONE 62-bit counter (task totals exceed 31 bits) ----------------------------------
// 64-bit word: [63:62] status, [61:0] counter.  The tile's aggregate is published first with
// lb64_publish (so that several look-backs of one tile can be in flight together), then
// lb64_exclusive_warp waits for the predecessors.
#define LB64_MASK 0x3FFFFFFFFFFFFFFFull
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v)
{
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
    return v;
}
// one lane of the tile
__device__ __forceinline__ void lb64_publish(volatile unsigned long long *state, int tile, unsigned long long agg)
{
    __threadfence();
    state[tile] = ((tile == 0 ? LB_PREFIX : LB_AGGREGATE) << 62) | (agg & LB64_MASK);
}
// one warp of the tile, all lanes, after lb64_publish: exclusive prefix in every lane
__device__ __forceinline__ unsigned long long lb64_exclusive_warp(volatile unsigned long long *state, int tile,
                                                                  unsigned long long agg)
{
    const uint32_t lane = threadIdx.x & 31u;
    if (tile == 0) return 0ull;
    unsigned long long sum = 0ull;
    for (int base = tile - 1; base >= 0; base -= 32) {
        const int idx = base - (int)lane;
        unsigned long long w = LB_PREFIX << 62;
        if (idx >= 0) {
            do {
                w = state[idx];
            } while (lb_status(w) == LB_INVALID);
        }
        const uint32_t pref = __ballot_sync(0xFFFFFFFFu, lb_status(w) == LB_PREFIX);
        const uint32_t take = pref ? ((2u << (__ffs(pref) - 1)) - 1u) : 0xFFFFFFFFu;
        sum += warp_sum_u64(((take >> lane) & 1u) ? (w & LB64_MASK) : 0ull);
        if (pref) break;
    }
    if (lane == 0) {
        __threadfence();
        state[tile] = (LB_PREFIX << 62) | ((sum + agg) & LB64_MASK);
    }
    return sum;
}
// block b takes tile b (see all_exclusive_warp): aggregates only, read in batches of 256
__device__ __forceinline__ unsigned long long all64_exclusive_warp(volatile unsigned long long *state, int tile)
{
    const int lane = (int)(threadIdx.x & 31u);
    unsigned long long s = 0ull;
    for (int base = 0; base < tile; base += 256) {
        unsigned long long w[8];
        bool need[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) {
            need[x] = base + lane + 32 * x < tile;
            w[x] = 0ull;
        }
        bool again;
        do {
            again = false;
#pragma unroll
            for (int x = 0; x < 8; ++x)
                if (need[x]) w[x] = state[base + lane + 32 * x];
#pragma unroll
            for (int x = 0; x < 8; ++x)
                if (need[x]) {
                    if (lb_status(w[x]) == LB_INVALID) again = true;
                    else need[x] = false;
                }
        } while (__any_sync(0xFFFFFFFFu, again));
#pragma unroll
        for (int x = 0; x < 8; ++x)
            if (base + lane + 32 * x < tile) s += w[x] & LB64_MASK;
    }
    return warp_sum_u64(s);
}
