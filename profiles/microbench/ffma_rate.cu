// Micro-benchmark: FP32 FMA issue rate on sm_100a, scalar FFMA vs packed FFMA2 (x2 per lane).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_rate ffma_rate.cu ; run on the GPU box.
#include <cuda_runtime.h>
#include <cstdio>

template <int MODE>
__global__ void __launch_bounds__(256) rate(float* out, int iters, float a0, float b0)
{
    float acc[32];
    float2 acc2[16];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
    for (int i = 0; i < 16; ++i) acc2[i] = make_float2(threadIdx.x * 1e-3f + i, i);
    float a[4] = {a0, a0 + 1, a0 + 2, a0 + 3}, b[4] = {b0, b0 * 2, b0 * 3, b0 * 4};
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i * 4 + j] = fmaf(a[i], b[j], acc[i * 4 + j]);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        acc2[i * 4 + j] = __ffma2_rn(make_float2(a[2 * i], a[2 * i + 1]), make_float2(b[j], b[j]), acc2[i * 4 + j]);
        }
        a[it & 3] += 1e-9f;
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i] + acc[i + 16] + acc2[i].x + acc2[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
    float* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int mode = 0; mode < 2; ++mode)
        for (int blocks_per_sm = 1; blocks_per_sm <= 8; blocks_per_sm *= 2) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (mode == 0) rate<0><<<148 * blocks_per_sm, 256>>>(out, iters, 1.f, 2.f);
                else rate<1><<<148 * blocks_per_sm, 256>>>(out, iters, 1.f, 2.f);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double fma = 64.0 * iters * 256.0 * 148 * blocks_per_sm;
            printf("mode=%s blocks/SM=%d  %.3f ms  %.1f TFLOP/s\n", mode ? "FFMA2" : "FFMA ", blocks_per_sm, ms,
                   2 * fma / ms / 1e9);
        }
    return 0;
}
