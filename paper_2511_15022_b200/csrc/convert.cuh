// Phase-only hologram conversion (convert.cpp): DPAC encode, e^{i phi}, and the
// device-resident random-POH optimisation loop.
#pragma once

#include "asm.cuh"
#include "common.cuh"

namespace hs {

// e^{i phi} of a phase raster (poh_field, convert.cpp:62-69; also the loop's u0).
void phase_to_field(const float* d_phase, int64_t n, float2* d_field, cudaStream_t st);

// dpac_encode (convert.cpp:31-60) before canonicalize_phase: mode 0 direct,
// 1 classical.  d_amax: C uints of scratch.
void dpac_encode(const float2* d_field, int C, int H, int W, int mode, unsigned* d_amax, float* d_out,
                 cudaStream_t st);

struct PohProblem {
    int C = 0, H = 0, W = 0, L = 0, pad = 2;
    const float* target = nullptr;   // device C x H x W
    const uint8_t* masks = nullptr;  // device L x H x W
};

// Device buffers of the random-POH loop (convert_random_poh_field, convert.cpp:71-174).
struct PohWork {
    PohProblem prob;
    AsmWork aw;  // transfer constants set by the caller (set_transfer with the plane distances)
    DevBuf u0, outs, du, back, gout, gint, dphi, state, partials, flag;
    int slots = 0;
    void prepare(const PohProblem& p);
    void loss_pass(const float2* d_u, float2* d_du, float* d_int, float lambda_comp, float lambda_field,
                   cudaStream_t st);
};

// Runs `steps` iterations on d_phase (in place, raw -- canonicalise on the host);
// d_loss_hist[step] receives each step's loss.  The guide field d_guide is
// C x H x W complex64.  Non-finite gradients set work.flag and stop the updates.
void random_poh_run(PohWork& w, const float2* d_guide, float* d_phase, int steps, double lambda_comp,
                    double lambda_field, double lr, double* d_loss_hist, cudaStream_t st);

}  // namespace hs
