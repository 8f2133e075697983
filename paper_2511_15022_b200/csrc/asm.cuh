// Band-limited angular spectrum propagation (K4-K6, K8-K10 of SURVEY §2.1).
#pragma once

#include "common.cuh"
#include "fft.cuh"

namespace hs {

// Per (channel, plane) transfer-function constants, built on the host in fp64
// exactly like make_band_limit (propagation.cpp:105-121).
struct TfConst {
    float kd_mod;   // fmod(k * phase_distance, 2 pi)
    float kd;       // k * phase_distance
    float bx, by;   // (2 pi / (nx pitch k))^2, (2 pi / (ny pitch k))^2
    int mx_max, my_max;  // largest |m| inside the band limit (strict <, :140)
    double a4;      // 4 * aperture^2, <= 0 disables the aperture (:149-159)
};

struct AsmWork {
    int C = 0, H = 0, W = 0, pad = 0, L = 0;
    int Px = 0, Py = 0, ox = 0, oy = 0, CC = 4, ntiles = 0;
    fft::Plan plan_x, plan_y;
    const float2* twx_ptr = nullptr;  // W_n tables (cached per device)
    const float2* twy_ptr = nullptr;
    DevBuf T1, T2;    // column-tiled intermediates
    DevBuf tf;        // TfConst [L][C]
    std::vector<TfConst> tf_host;
    size_t smem_rows = 0, smem_cols = 0;

    void prepare(int C, int H, int W, int pad, int L);
    // phase/mask distances per plane (propagate: both = d; backward: phase -d).
    void set_transfer(const hs_prop_spec& spec, const double* phase_d, const double* mask_d,
                      cudaStream_t st);
};

// forward: in C x H x W -> out L x C x H x W  (propagate_multi, :240-263)
// ev (nullable): 3 events recorded after each of the three kernels.
void asm_forward(AsmWork& w, const float2* d_in, float2* d_out, cudaStream_t st,
                 cudaEvent_t* ev = nullptr);
// backward: grads L x C x H x W -> out C x H x W (propagate_multi_backward, :265-294)
// conj = true applies conj(H) (the adjoint); the transfer constants must be
// those of the forward planes.
void asm_backward(AsmWork& w, const float2* d_grads, float2* d_out, cudaStream_t st,
                  cudaEvent_t* ev = nullptr);

fft::Plan make_plan(int n);

}  // namespace hs
