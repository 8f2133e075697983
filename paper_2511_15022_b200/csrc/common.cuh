// Shared device/host plumbing for the holosplat-b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a tool (nsys / ncu --nvtx) is attached

#include "holosplat.h"

namespace hs {

// Host-side NVTX range (SURVEY §5 tracing row): names the C-ABI trainer calls
// and, on eager enqueues, the step's stages, so `ncu --nvtx --nvtx-include`
// can select a stage's kernels.  Inside a graph capture it marks the capture.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};


constexpr int kTile = 16;  // rasterizer.hpp:12 kTileSize
constexpr double kEpsScale = 0.1, kEpsCov = 0.1, kEpsDet = 1e-10;  // field_core.hpp:10-12
constexpr double kPowerFloor = -50.0, kAlphaCap = 0.99, kAlphaCutoff = 1.0 / 255.0;  // :13-15
constexpr double kMahalSlack = 1e-9;  // rasterizer.cpp:17
constexpr int kMaxChannels = 4;       // compiled channel specialisations 1..4

// Error carrying an hs_status; translated at the C-ABI boundary.
struct Error : std::runtime_error {
    hs_status status;
    Error(hs_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(e == cudaErrorMemoryAllocation ? HS_ENOMEM : HS_ECUDA,
                    std::string(what) + ": " + cudaGetErrorString(e));
}
#define HS_CUDA(x) ::hs::cuda_check((x), #x)

void note_launch(int n = 1);
inline void launch_check(const char* name) {
    note_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(HS_ECUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e));
}

inline void require(bool ok, const std::string& msg) {
    if (!ok) throw Error(HS_EINVAL, msg);
}

// Growable device buffer (never shrinks; reused across calls).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void reserve(size_t b) {
        if (b <= bytes) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        HS_CUDA(cudaMalloc(&p, b));
        bytes = b;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    ~DevBuf() { release(); }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

int sm_count(int device);

}  // namespace hs

struct hs_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    // reusable work buffers of the standalone C-ABI entry points (capi.cu)
    void* work = nullptr;
    // NCCL communicator of the sharded steps (comm.cu): one rank per GPU
    void* comm = nullptr;  // ncclComm_t
    int comm_size = 1, comm_rank = 0;
    bool comm_owned = false;
    void* comm_scratch = nullptr;  // device: agreement word + loss sums
};

// Device helpers ------------------------------------------------------------------
namespace hs {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// Packed fp32x2 arithmetic (sm_100 FADD2/FMUL2/FFMA2): one issue slot for two
// lanes of work.  Broadcast operands (make_float2(s, s)) map to the .F32
// operand form, so a scalar weight times a pair is one instruction.
__device__ __forceinline__ unsigned long long f2bits(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 bits2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2bits(a)), "l"(f2bits(b)), "l"(f2bits(c)));
    return bits2f(r);
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2bits(a)), "l"(f2bits(b)));
    return bits2f(r);
}
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2bits(a)), "l"(f2bits(b)));
    return bits2f(r);
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2bits(a)), "l"(f2bits(b)));
    return bits2f(r);
}
__device__ __forceinline__ float2 f2splat(float s) { return make_float2(s, s); }

// 2^x on the MUFU (ex2.approx.ftz: one instruction, rel. error ~2^-22).
__device__ __forceinline__ float ex2f(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
constexpr float kNegHalfLog2e = -0.72134752044448170368f;  // -0.5 / ln 2: e^{-m/2} = 2^{m * kNegHalfLog2e}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

inline unsigned ceil_div(size_t a, size_t b) { return static_cast<unsigned>((a + b - 1) / b); }

}  // namespace hs
