// Micro-benchmark 2: cycles per warp-instruction for FFMA / FFMA2 register patterns (sm_100a).
#include <cuda_runtime.h>
#include <cstdio>
__device__ __forceinline__ unsigned long long gtime(){ unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;":"=l"(t)); return t; }

template <int MODE>
__global__ void __launch_bounds__(256) rate(float* out, long long* cyc, int iters, float a0, float b0)
{
    float acc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc[i] = threadIdx.x * 1e-3f + i;
    float a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = a0 + i; b[i] = b0 * (i + 1); }
    long long c0 = clock64();
    unsigned long long t0 = gtime();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {            // 4x4 tile scalar, 16 FFMA per k, 4 k
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i * 4 + j] = fmaf(a[i], b[j], acc[i * 4 + j]);
        } else if (MODE == 1) {     // 8x8 tile scalar, 64 FFMA per k
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i * 8 + j] = fmaf(a[i], b[j], acc[i * 8 + j]);
        } else if (MODE == 2) {     // 4x4 tile packed: 8 FFMA2 per k, 4 k
            float2* acc2 = reinterpret_cast<float2*>(acc);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        acc2[i * 4 + j] = __ffma2_rn(make_float2(a[2 * i], a[2 * i + 1]), make_float2(b[j], b[j]), acc2[i * 4 + j]);
        } else {                    // 8x8 tile packed: 32 FFMA2 per k
            float2* acc2 = reinterpret_cast<float2*>(acc);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    acc2[i * 8 + j] = __ffma2_rn(make_float2(a[2 * i], a[2 * i + 1]), make_float2(b[j], b[j]), acc2[i * 8 + j]);
        }
        a[it & 7] += 1e-9f;
    }
    unsigned long long t1 = gtime();
    long long c1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 64; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) { cyc[0] = c1 - c0; cyc[1] = (long long)(t1 - t0); }
}

int main()
{
    float* out; long long* cyc; long long h[2];
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    cudaMalloc(&cyc, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    const char* names[4] = {"FFMA 4x4", "FFMA 8x8", "FFMA2 4x4", "FFMA2 8x8"};
    for (int mode = 0; mode < 4; ++mode)
        for (int bps = 1; bps <= 2; ++bps) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (mode == 0) rate<0><<<148 * bps, 256>>>(out, cyc, iters, 1.f, 2.f);
                if (mode == 1) rate<1><<<148 * bps, 256>>>(out, cyc, iters, 1.f, 2.f);
                if (mode == 2) rate<2><<<148 * bps, 256>>>(out, cyc, iters, 1.f, 2.f);
                if (mode == 3) rate<3><<<148 * bps, 256>>>(out, cyc, iters, 1.f, 2.f);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
            }
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
            double fma = 64.0 * iters * 256.0 * 148 * bps;
            double winstr_per_smsp = (mode < 2 ? 64.0 : 32.0) * iters * (256 / 32) * bps / 4.0;
            printf("%-10s blocks/SM=%d  %.3f ms  %.1f TFLOP/s  clock %.0f MHz  %.2f cyc/warp-instr/SMSP\n", names[mode], bps, ms,
                   2 * fma / ms / 1e9, 1e3 * h[0] / (double)h[1], h[0] / winstr_per_smsp);
        }
    return 0;
}
