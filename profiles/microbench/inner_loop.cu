// Micro-benchmark: upper bound of the K3 consumer inner loop (operands already in shared memory,
// no barriers, no gating).  Variants of thread tile / lane mapping / prefetch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o inner_loop inner_loop.cu
#include <cuda_runtime.h>
#include <cstdio>
#define REC 272
__device__ __forceinline__ void mac2(float2& acc, float2 a, float b) { acc = __ffma2_rn(a, make_float2(b, b), acc); }

// V0: current design: warp = 2 leaves (halves), thread = (p,q) 4x4 sub-block; lane = p1 q1 half p0 q0
template <int PREFETCH>
__global__ void __launch_bounds__(256, 2) v0(const float* __restrict__ src, float* out, int iters)
{
    extern __shared__ float sm[];
    for (int i = threadIdx.x; i < 32 * REC; i += blockDim.x) sm[i] = src[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int half = (lane >> 2) & 1, p = ((lane >> 4) & 1) << 1 | ((lane >> 1) & 1), q = ((lane >> 3) & 1) << 1 | (lane & 1);
    float2 acc[2][4];
    for (int h = 0; h < 2; ++h) for (int j = 0; j < 4; ++j) acc[h][j] = make_float2(0.f, 0.f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
        for (int kk = 0; kk < 4; ++kk) {
            const float* As = sm + ((warp >> 1) * 4 + kk) * REC;
            const float* Bs = sm + (16 + kk * 4 + (warp & 1) * 2 + half) * REC;
            if (PREFETCH == 0) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    float4 a[4], b[4];
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        a[x] = *reinterpret_cast<const float4*>(As + (4 * r + x) * 16 + 4 * p);
                        b[x] = *reinterpret_cast<const float4*>(Bs + (4 * r + x) * 16 + 4 * q);
                    }
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        float2 a01 = make_float2(a[x].x, a[x].y), a23 = make_float2(a[x].z, a[x].w);
                        float bv[4] = {b[x].x, b[x].y, b[x].z, b[x].w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) { mac2(acc[0][j], a01, bv[j]); mac2(acc[1][j], a23, bv[j]); }
                    }
                }
            } else {
                float4 a[2][4], b[2][4];
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    a[0][x] = *reinterpret_cast<const float4*>(As + x * 16 + 4 * p);
                    b[0][x] = *reinterpret_cast<const float4*>(Bs + x * 16 + 4 * q);
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (r < 3) {
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            a[(r + 1) & 1][x] = *reinterpret_cast<const float4*>(As + (4 * (r + 1) + x) * 16 + 4 * p);
                            b[(r + 1) & 1][x] = *reinterpret_cast<const float4*>(Bs + (4 * (r + 1) + x) * 16 + 4 * q);
                        }
                    }
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        float4 av = a[r & 1][x], bb = b[r & 1][x];
                        float2 a01 = make_float2(av.x, av.y), a23 = make_float2(av.z, av.w);
                        float bv[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) { mac2(acc[0][j], a01, bv[j]); mac2(acc[1][j], a23, bv[j]); }
                    }
                }
            }
        }
    }
    float s = 0;
    for (int h = 0; h < 2; ++h) for (int j = 0; j < 4; ++j) s += acc[h][j].x + acc[h][j].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// V1: warp = 2x2 quad of leaves, thread = (p,q) in the two leaves of one leaf column (half selects column):
// shares the B fragment across two tasks; 32 accumulators.
__global__ void __launch_bounds__(128, 4) v1(const float* __restrict__ src, float* out, int iters)
{
    extern __shared__ float sm[];
    for (int i = threadIdx.x; i < 32 * REC; i += blockDim.x) sm[i] = src[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int half = (lane >> 2) & 1, p = ((lane >> 4) & 1) << 1 | ((lane >> 1) & 1), q = ((lane >> 3) & 1) << 1 | (lane & 1);
    float2 acc[2][2][4];
    for (int t = 0; t < 2; ++t) for (int h = 0; h < 2; ++h) for (int j = 0; j < 4; ++j) acc[t][h][j] = make_float2(0.f, 0.f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
        for (int kk = 0; kk < 4; ++kk) {
            const float* A0 = sm + ((warp >> 1) * 8 + kk) * REC;
            const float* A1 = sm + ((warp >> 1) * 8 + 4 + kk) * REC;
            const float* Bs = sm + (16 + kk * 4 + (warp & 1) * 2 + half) * REC;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                float4 a0[4], a1[4], b[4];
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    a0[x] = *reinterpret_cast<const float4*>(A0 + (4 * r + x) * 16 + 4 * p);
                    a1[x] = *reinterpret_cast<const float4*>(A1 + (4 * r + x) * 16 + 4 * p);
                    b[x] = *reinterpret_cast<const float4*>(Bs + (4 * r + x) * 16 + 4 * q);
                }
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    float bv[4] = {b[x].x, b[x].y, b[x].z, b[x].w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        mac2(acc[0][0][j], make_float2(a0[x].x, a0[x].y), bv[j]);
                        mac2(acc[0][1][j], make_float2(a0[x].z, a0[x].w), bv[j]);
                        mac2(acc[1][0][j], make_float2(a1[x].x, a1[x].y), bv[j]);
                        mac2(acc[1][1][j], make_float2(a1[x].z, a1[x].w), bv[j]);
                    }
                }
            }
        }
    }
    float s = 0;
    for (int t = 0; t < 2; ++t) for (int h = 0; h < 2; ++h) for (int j = 0; j < 4; ++j) s += acc[t][h][j].x + acc[t][h][j].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
    float *src, *out;
    cudaMalloc(&src, 32 * REC * 4);
    cudaMemset(src, 0, 32 * REC * 4);
    cudaMalloc(&out, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 2000;
    const size_t smem = 32 * REC * 4;
    for (int variant = 0; variant < 3; ++variant)
        for (int bps = 1; bps <= 4; bps *= 2) {
            float ms = 0;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (variant == 0) v0<0><<<148 * bps, 256, smem>>>(src, out, iters);
                if (variant == 1) v0<1><<<148 * bps, 256, smem>>>(src, out, iters);
                if (variant == 2) v1<<<148 * bps, 128, smem>>>(src, out, iters);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            // flops: v0: 256 thr x 4 kk x 4 r x 4 x x 16 fma ; v1: 128 thr x ... x 32 fma
            double fma = (variant < 2 ? 256.0 * 16 : 128.0 * 32) * 4 * 4 * 4 * iters * 148.0 * bps;
            printf("variant %d (%s) blocks/SM=%d: %.3f ms  %.1f TFLOP/s  err=%s\n", variant,
                   variant == 0 ? "pair, no prefetch" : variant == 1 ? "pair, prefetch next r" : "quad-column, 32 acc", bps, ms,
                   2 * fma / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
