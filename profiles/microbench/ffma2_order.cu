#include <cuda_runtime.h>
#include <cstdio>
// register-only 4x4 tile, 8 FFMA2 per k, different instruction orders
template <int MODE>
__global__ void __launch_bounds__(256) rate(float* out, int iters, float a0, float b0)
{
    float2 acc[2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(threadIdx.x * 1e-3f + i, j);
    float a[4][4], b[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int i = 0; i < 4; ++i) { a[u][i] = a0 + i + u; b[u][i] = b0 * (i + 1 + u); }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float2 a01 = make_float2(a[u][0], a[u][1]), a23 = make_float2(a[u][2], a[u][3]);
            if (MODE == 0) {      // row order: a01 x b0..3, a23 x b0..3
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[0][j] = __ffma2_rn(a01, make_float2(b[u][j], b[u][j]), acc[0][j]);
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[1][j] = __ffma2_rn(a23, make_float2(b[u][j], b[u][j]), acc[1][j]);
            } else if (MODE == 1) {   // snake: a01 x b0..3, a23 x b3..0
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[0][j] = __ffma2_rn(a01, make_float2(b[u][j], b[u][j]), acc[0][j]);
#pragma unroll
                for (int j = 3; j >= 0; --j) acc[1][j] = __ffma2_rn(a23, make_float2(b[u][j], b[u][j]), acc[1][j]);
            } else {              // b-major: (a01,b0),(a23,b0),(a23,b1),(a01,b1),(a01,b2),(a23,b2),(a23,b3),(a01,b3)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (j & 1) {
                        acc[1][j] = __ffma2_rn(a23, make_float2(b[u][j], b[u][j]), acc[1][j]);
                        acc[0][j] = __ffma2_rn(a01, make_float2(b[u][j], b[u][j]), acc[0][j]);
                    } else {
                        acc[0][j] = __ffma2_rn(a01, make_float2(b[u][j], b[u][j]), acc[0][j]);
                        acc[1][j] = __ffma2_rn(a23, make_float2(b[u][j], b[u][j]), acc[1][j]);
                    }
                }
            }
        }
        a[it & 3][it & 1] += 1e-9f;
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += acc[i][j].x + acc[i][j].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main()
{
    float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    for (int mode = 0; mode < 3; ++mode)
      for (int bps = 1; bps <= 4; bps *= 2) {
        float ms = 0;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) rate<0><<<148 * bps, 256>>>(out, iters, 1.f, 2.f);
            if (mode == 1) rate<1><<<148 * bps, 256>>>(out, iters, 1.f, 2.f);
            if (mode == 2) rate<2><<<148 * bps, 256>>>(out, iters, 1.f, 2.f);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        double fma = 256.0 * 148 * bps * (double)iters * 4 * 16;
        printf("mode %d blocks/SM %d: %.3f ms %.1f TFLOP/s\n", mode, bps, ms, 2 * fma / ms / 1e9);
      }
    return 0;
}
