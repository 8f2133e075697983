// Training loss (recon + SSIM) and fused Adan.
#pragma once

#include "common.cuh"

namespace hs {

enum LossKind { kLossTraining = 0, kLossRecon = 1, kLossSsim = 2, kLossMse = 3 };

struct LossArgs {
    int kind;
    int L;          // planes in this call
    int L_norm;     // global plane count for the normalisers (plane sharding)
    int plane0;     // global index of the first plane in this call (mask selection)
    int C, H, W;
    const float* recon;      // L x C x H x W intensities (or nullptr when from_field)
    const float2* field;     // L x C x H x W complex fields (I = |U|^2), or nullptr
    const float* target;     // C x H x W
    const float2* tstats;    // C x (H-10) x (W-10) target window stats (ssim_target_stats)
    const uint8_t* masks;    // L_norm x H x W
    float* grad;             // dL/dI (L x C x H x W), or nullptr
    float2* du;              // dL/dU = 2 U dL/dI (L x C x H x W), or nullptr
    double* partials;        // 2 per CTA: recon-or-mse sum, ssim sum
    int C_norm = 0;          // global channel count for the normalisers (channel sharding); 0 = C
    // Row-slab sharding: this call sees a band of H rows of an image of H_norm
    // rows (the normalisers use H_norm); the loss sums count only rows
    // [own0, own1) of the band (SSIM: windows whose top row is there), the
    // gradient is produced for every row of the band.  0 / full = unsharded.
    int H_norm = 0;
    int own0 = 0, own1 = 1 << 30;
    __host__ __device__ int channels_norm() const { return C_norm > 0 ? C_norm : C; }
    __host__ __device__ int rows_norm() const { return H_norm > 0 ? H_norm : H; }
};

// Launches the loss kernel(s); returns the number of partial slots written.
int loss_launch(const LossArgs& a, cudaStream_t st);
int loss_partial_slots(int kind, int L, int C, int H, int W);
// Reduces partials into out[0] = loss, out[1] = recon sum, out[2] = ssim sum.
void loss_finalize(const LossArgs& a, int slots, double* d_out3, cudaStream_t st);

void intensity_launch(const float2* f, int64_t count, float* out, cudaStream_t st);
// clamp to [0, 1] (pipeline.cpp clipped(), used by compute_metrics)
void clip01_launch(const float* in, int64_t count, float* out, cudaStream_t st);
// (mu2, sigma2^2) of the target on the valid 11x11 grid, per channel.
void ssim_target_stats(const float* target, int C, int H, int W, float2* out, cudaStream_t st);
inline size_t ssim_target_stats_elems(int C, int H, int W) {
    return (H < 11 || W < 11) ? 1 : static_cast<size_t>(C) * (H - 10) * (W - 10);
}

// One Adan element update (Adan::step optimizer.cpp:48-72) with per-group constants
// lr, 1/bc1, beta2/bc2, 1/bc3.
struct GroupConst {
    float lr, inv_bc1, b2_bc2, inv_bc3;
};

__device__ __forceinline__ void adan_update(float& p, float g, float& m, float& v, float& n, float& gp, bool first,
                                            float b1, float b2, float b3, float eps, const GroupConst& k) {
    const float diff = first ? 0.f : g - gp;
    m = b1 * m + (1.f - b1) * g;
    v = b2 * v + (1.f - b2) * diff;
    const float u = g + b2 * diff;
    n = b3 * n + (1.f - b3) * u * u;
    const float denom = sqrtf(n * k.inv_bc3) + eps;
    p -= k.lr * (m * k.inv_bc1 + v * k.b2_bc2) / denom;
    gp = g;
}

// Fused Adan over the six groups of the parameter buffer (Adan::step optimizer.cpp:48-72).
struct AdanGroups {
    int64_t begin[6], end[6];
    float base_lr[6];
};
struct AdanDeviceStep {
    int step;          // 0-based loop step (cosine schedule input)
    int t;             // 1-based Adan step after increment
};
// d_step layout: int[4] {loop step, adan t, CTA done counter, pad} then the 6
// GroupConst of the coming step (adan_init_consts once, then kept by the kernel).
inline constexpr size_t kAdanStepBytes = 4 * sizeof(int) + 6 * sizeof(GroupConst);
void adan_init_consts(const AdanGroups& g, int total_steps, double b1, double b2, double b3, int* d_step,
                      cudaStream_t st);
// Reads the step counter from d_step and the flags
// word; advances the counter.  Position lr follows cosine_lr(step, total,
// 1e-2, 1e-3) (pipeline.cpp:254).
void adan_fused_launch(float* params, const float* grads, float* state, int64_t P,
                       const AdanGroups& g, int total_steps, double b1, double b2, double b3,
                       double eps, int* d_step, const uint32_t* d_flags, cudaStream_t st, int64_t begin = 0,
                       int64_t end = -1);
// The groups of [begin, end) of the flat buffer, re-based to begin.
AdanGroups shift_groups(const AdanGroups& G, int64_t begin, int64_t end);
// Single group, explicit lr/t (C-ABI hs_adan_step).
void adan_group_launch(float* params, const float* grads, float* state, int64_t size, int t,
                       double lr, double b1, double b2, double b3, double eps, cudaStream_t st);
// Non-finite check of a gradient array -> flag word (bit 0).
void nonfinite_launch(const float* g, int64_t n, uint32_t* flag, cudaStream_t st);
// Per-group non-finite bits of the summed gradient buffer -> *flags (reset first).
void group_nonfinite_launch(const float* g, int64_t P, const AdanGroups& G, uint32_t* flags, cudaStream_t st,
                            int64_t begin = 0, int64_t end = -1);

}  // namespace hs
