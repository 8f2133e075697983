// Microbenchmark: scalar FFMA vs packed FFMA2 / FADD2 throughput on sm_100a, and the SASS of a
// packed complex multiply.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float2 v) { return *reinterpret_cast<u64*>(&v); }
__device__ __forceinline__ float2 upk(u64 v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c))); return upk(r);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    u64 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b))); return upk(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    u64 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b))); return upk(r);
}
// complex multiply a*b with packed ops: (a.x*b.x, a.x*b.y) + (-a.y*b.y, a.y*b.x)
__device__ __forceinline__ float2 cmul2(float2 a, float2 b) {
    float2 t = mul2(make_float2(a.x, a.x), b);
    return fma2(make_float2(a.y, a.y), make_float2(-b.y, b.x), t);
}
__global__ void scalar_k(float* out, float s, int iters) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], s, 0.5f);
    float r = 0; for (int i = 0; i < 8; ++i) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void packed_k(float* out, float s, int iters) {
    float2 a[4];
    for (int i = 0; i < 4; ++i) a[i] = make_float2(threadIdx.x * 0.001f + i, i + 0.5f);
    const float2 ss = make_float2(s, s), h = make_float2(0.5f, 0.5f);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = fma2(a[i], ss, h);
    float r = 0; for (int i = 0; i < 4; ++i) r += a[i].x + a[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void packed8_k(float* out, float s, int iters) {
    float2 a[8];
    for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 0.001f + i, i + 0.5f);
    const float2 ss = make_float2(s, s), h = make_float2(0.5f, 0.5f);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma2(a[i], ss, h);
    float r = 0; for (int i = 0; i < 8; ++i) r += a[i].x + a[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void cm_k(float2* io, float2 w) { io[threadIdx.x] = cmul2(io[threadIdx.x], w); }
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * 8, thr = 256;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); scalar_k<<<blocks, thr>>>(out, 0.999f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8 * iters * (double)blocks * thr;
        printf("scalar FFMA : %.3f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
        cudaEventRecord(e0); packed_k<<<blocks, thr>>>(out, 0.999f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("packed FFMA2 x4: %.3f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
        cudaEventRecord(e0); packed8_k<<<blocks, thr>>>(out, 0.999f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("packed FFMA2 x8: %.3f ms  %.1f TFLOP/s\n", ms, 2 * fl / ms / 1e9);
    }
    return 0;
}
