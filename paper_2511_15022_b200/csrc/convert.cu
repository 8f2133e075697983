// Phase-only hologram (POH) conversion:
// proj/core/src/convert.cpp -- dpac_encode :31-60, poh_field :62-69,
// convert_random_poh_field :71-174.
//
// The random-POH loop is device resident: per step one elementwise kernel
// turns the phase raster into e^{i phi}, the multi-plane ASM forward of
// asm_static.cu / asm.cu propagates it, one elementwise kernel forms every
// plane's loss terms and dL/dU (plane_recon_loss + the guide's squared-
// intensity and complex-L1 terms, convert.cpp:116-155), the ASM adjoint sums
// the planes, and two elementwise kernels apply the chain rule through
// e^{i phi} and the Adan update (Adan::step optimizer.cpp:48-72; non-finite gradients
// stop the updates and raise "Adan: non-finite gradient in group phase").  The
// per-step loss is reduced on the device into a history buffer read once at the
// end.  Canonicalisation into [0, 2 pi) happens on the host in fp64.
#include <cmath>
#include <vector>

#include <cub/block/block_reduce.cuh>

#include "asm.cuh"
#include "convert.cuh"
#include "loss.cuh"

namespace hs {

namespace {

constexpr int kThreads = 256;

unsigned blocks_for(int64_t n) {
    const int64_t b = (n + kThreads - 1) / kThreads;
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 8)));
}

__global__ void phase_to_field_kernel(const float* __restrict__ phase, int64_t n, float2* __restrict__ u) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float s, c;
        sincosf(phase[i], &s, &c);
        u[i] = make_float2(c, s);
    }
}

struct PohLossArgs {
    int L, C, H, W;
    const float2* u;          // L x C x H x W propagated field of the phase raster
    const float* target;      // C x H x W
    const uint8_t* masks;     // L x H x W
    const float* guide_int;   // L x C x H x W (nullable when lambda_comp == 0)
    const float2* guide_out;  // L x C x H x W (nullable when lambda_field == 0)
    float lambda_comp, lambda_field;
    float2* du;               // L x C x H x W dL/dU (nullable: loss only)
    float* intensity;         // L x C x H x W |u|^2 (nullable)
    double* partials;         // 3 per CTA: sum_l plane_recon_loss, comp sum, field sum
};

// convert.cpp:116-155 for every element of every plane.
__global__ void __launch_bounds__(kThreads) poh_loss_kernel(PohLossArgs a) {
    const int64_t hw = static_cast<int64_t>(a.H) * a.W;
    const int64_t chw = hw * a.C;
    const int64_t total = chw * a.L;
    const float w = static_cast<float>(2.0 / static_cast<double>(chw));  // plane_recon_loss, loss.cpp:341
    double s_rec = 0.0, s_comp = 0.0, s_field = 0.0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t l = i / chw, rem = i - l * chw, p = rem % hw;
        const float2 ul = a.u[i];
        const float il = ul.x * ul.x + ul.y * ul.y;
        const float t = a.target[rem];
        const float d = il - t;
        const float k = 1.f + (a.masks[l * hw + p] ? 1.f : 0.f) + t * t;
        s_rec += static_cast<double>(d * d * k);
        float gi = w * d * k;
        if (a.lambda_comp != 0.f) {
            const float dd = a.guide_int[i] - il;
            s_comp += static_cast<double>(dd * dd);
            gi += a.lambda_comp * (-2.f * dd);
        }
        float2 g = make_float2(2.f * ul.x * gi, 2.f * ul.y * gi);
        if (a.lambda_field != 0.f) {
            const float2 go = a.guide_out[i];
            const float dre = go.x - ul.x, dim = go.y - ul.y;
            s_field += static_cast<double>(fabsf(dre) + fabsf(dim));
            // subgradient of |guide - u| w.r.t. u, zero at ties
            g.x += a.lambda_field * (dre > 0.f ? -1.f : (dre < 0.f ? 1.f : 0.f));
            g.y += a.lambda_field * (dim > 0.f ? -1.f : (dim < 0.f ? 1.f : 0.f));
        }
        if (a.du) a.du[i] = g;
        if (a.intensity) a.intensity[i] = il;
    }
    using BR = cub::BlockReduce<double, kThreads>;
    __shared__ typename BR::TempStorage tmp;
    const double r = BR(tmp).Sum(s_rec);
    __syncthreads();
    const double c = BR(tmp).Sum(s_comp);
    __syncthreads();
    const double f = BR(tmp).Sum(s_field);
    if (threadIdx.x == 0) {
        a.partials[3 * blockIdx.x] = r / static_cast<double>(chw);
        a.partials[3 * blockIdx.x + 1] = c;
        a.partials[3 * blockIdx.x + 2] = f;
    }
}

// loss = guide_sum + sum_l recon_l + lambda_comp * comp + lambda_field * field (convert.cpp:114-155)
__global__ void __launch_bounds__(1024) poh_loss_finalize_kernel(const double* __restrict__ partials, int slots,
                                                                 double guide_sum, double lambda_comp,
                                                                 double lambda_field, double* __restrict__ out) {
    using BR = cub::BlockReduce<double, 1024>;
    __shared__ typename BR::TempStorage tmp;
    double r = 0.0, c = 0.0, f = 0.0;
    for (int i = threadIdx.x; i < slots; i += 1024) {
        r += partials[3 * i];
        c += partials[3 * i + 1];
        f += partials[3 * i + 2];
    }
    const double rt = BR(tmp).Sum(r);
    __syncthreads();
    const double ct = BR(tmp).Sum(c);
    __syncthreads();
    const double ft = BR(tmp).Sum(f);
    if (threadIdx.x == 0) *out = guide_sum + rt + lambda_comp * ct + lambda_field * ft;
}

// dphi = -sin(phi) back.re + cos(phi) back.im  (convert.cpp:158-160), non-finite flag
__global__ void poh_dphi_kernel(const float* __restrict__ phase, const float2* __restrict__ back, int64_t n,
                                float* __restrict__ dphi, uint32_t* __restrict__ flag) {
    bool bad = false;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float s, c;
        sincosf(phase[i], &s, &c);
        const float2 b = back[i];
        const float g = -s * b.x + c * b.y;
        dphi[i] = g;
        bad |= !isfinite(g);
    }
    if (bad) atomicOr(flag, 1u);
}

// Adan on the phase group; skipped entirely once a non-finite gradient was seen
// (the reference throws before touching the parameters, optimizer.cpp:52-54).
__global__ void poh_adan_kernel(float* __restrict__ phase, const float* __restrict__ dphi, float* __restrict__ st,
                                int64_t n, int t, GroupConst k, float b1, float b2, float b3, float eps,
                                const uint32_t* __restrict__ flag) {
    if (*flag) return;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float p = phase[i], m = st[i], v = st[n + i], nn = st[2 * n + i], gp = st[3 * n + i];
        adan_update(p, dphi[i], m, v, nn, gp, t == 1, b1, b2, b3, eps, k);
        phase[i] = p;
        st[i] = m;
        st[n + i] = v;
        st[2 * n + i] = nn;
        st[3 * n + i] = gp;
    }
}

// per-channel max |u| (dpac_encode :39-41); |u| >= 0, so float bits order like uints
__global__ void dpac_amax_kernel(const float2* __restrict__ f, int C, int64_t hw, unsigned* __restrict__ amax) {
    const int c = blockIdx.y;
    float m = 0.f;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < hw;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float2 u = f[c * hw + i];
        m = fmaxf(m, hypotf(u.x, u.y));
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomicMax(amax + c, __float_as_uint(m));
}

// dpac_encode :42-58 (value before canonicalize_phase)
__global__ void dpac_encode_kernel(const float2* __restrict__ f, int C, int H, int W,
                                   const unsigned* __restrict__ amax, int mode, float* __restrict__ out) {
    const int64_t hw = static_cast<int64_t>(H) * W, total = hw * C;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i / hw);
        const int64_t p = i - c * hw;
        const int y = static_cast<int>(p / W), x = static_cast<int>(p - static_cast<int64_t>(y) * W);
        const float2 u = f[i];
        const float am = __uint_as_float(amax[c]);
        const float amp = am > 0.f ? hypotf(u.x, u.y) / am : 0.f;
        const float phi = atan2f(u.y, u.x);
        float v;
        if (mode == 0) {  // direct
            v = ((y + x) % 2 == 0) ? amp : phi;
        } else {          // classical
            const float delta = acosf(fminf(amp, 1.f));
            v = ((y + x) % 2 == 0) ? phi + delta : phi - delta;
        }
        out[i] = v;
    }
}

}  // namespace

void phase_to_field(const float* d_phase, int64_t n, float2* d_field, cudaStream_t st) {
    if (n == 0) return;
    phase_to_field_kernel<<<blocks_for(n), kThreads, 0, st>>>(d_phase, n, d_field);
    launch_check("phase_to_field");
}

void dpac_encode(const float2* d_field, int C, int H, int W, int mode, unsigned* d_amax, float* d_out,
                 cudaStream_t st) {
    const int64_t hw = static_cast<int64_t>(H) * W;
    if (hw == 0 || C == 0) return;
    HS_CUDA(cudaMemsetAsync(d_amax, 0, sizeof(unsigned) * C, st));
    dpac_amax_kernel<<<dim3(std::max(1u, std::min(blocks_for(hw), 148u)), C), kThreads, 0, st>>>(d_field, C, hw,
                                                                                                 d_amax);
    launch_check("dpac_amax");
    dpac_encode_kernel<<<blocks_for(hw * C), kThreads, 0, st>>>(d_field, C, H, W, d_amax, mode, d_out);
    launch_check("dpac_encode");
}

void PohWork::prepare(const PohProblem& p) {
    prob = p;
    const int64_t n = static_cast<int64_t>(p.C) * p.H * p.W;
    const int64_t ln = n * p.L;
    aw.prepare(p.C, p.H, p.W, p.pad, p.L);
    u0.reserve(sizeof(float2) * n);
    outs.reserve(sizeof(float2) * ln);
    du.reserve(sizeof(float2) * ln);
    back.reserve(sizeof(float2) * n);
    gout.reserve(sizeof(float2) * ln);
    gint.reserve(sizeof(float) * ln);
    dphi.reserve(sizeof(float) * n);
    state.reserve(sizeof(float) * 4 * n);
    slots = static_cast<int>(blocks_for(ln));
    partials.reserve(sizeof(double) * 3 * slots);
    flag.reserve(sizeof(uint32_t));
}

void PohWork::loss_pass(const float2* d_u, float2* d_du, float* d_int, float lc, float lf, cudaStream_t st) {
    PohLossArgs a{prob.L, prob.C, prob.H, prob.W, d_u, prob.target, prob.masks, gint.as<float>(),
                  gout.as<float2>(), lc, lf, d_du, d_int, partials.as<double>()};
    poh_loss_kernel<<<slots, kThreads, 0, st>>>(a);
    launch_check("poh_loss");
}

void random_poh_run(PohWork& w, const float2* d_guide, float* d_phase, int steps, double lambda_comp,
                    double lambda_field, double lr, double* d_loss_hist, cudaStream_t st) {
    const PohProblem& p = w.prob;
    const int64_t n = static_cast<int64_t>(p.C) * p.H * p.W;
    // frozen guide branch: per-plane outputs, intensities and reconstruction terms
    asm_forward(w.aw, d_guide, w.gout.as<float2>(), st);
    w.loss_pass(w.gout.as<float2>(), nullptr, w.gint.as<float>(), 0.f, 0.f, st);
    DevBuf gsum;
    gsum.reserve(sizeof(double));
    poh_loss_finalize_kernel<<<1, 1024, 0, st>>>(w.partials.as<double>(), w.slots, 0.0, 0.0, 0.0,
                                                 gsum.as<double>());
    launch_check("poh_loss_finalize");
    double guide_sum = 0.0;
    HS_CUDA(cudaMemcpyAsync(&guide_sum, gsum.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));

    HS_CUDA(cudaMemsetAsync(w.state.p, 0, sizeof(float) * 4 * n, st));
    HS_CUDA(cudaMemsetAsync(w.flag.p, 0, sizeof(uint32_t), st));
    const double b1 = 0.98, b2 = 0.92, b3 = 0.99, eps = 1e-8;  // AdanConfig defaults, optimizer.hpp:10-15
    for (int step = 0; step < steps; ++step) {
        phase_to_field(d_phase, n, w.u0.as<float2>(), st);
        asm_forward(w.aw, w.u0.as<float2>(), w.outs.as<float2>(), st);
        w.loss_pass(w.outs.as<float2>(), w.du.as<float2>(), nullptr, static_cast<float>(lambda_comp),
                    static_cast<float>(lambda_field), st);
        poh_loss_finalize_kernel<<<1, 1024, 0, st>>>(w.partials.as<double>(), w.slots, guide_sum, lambda_comp,
                                                     lambda_field, d_loss_hist + step);
        launch_check("poh_loss_finalize");
        asm_backward(w.aw, w.du.as<float2>(), w.back.as<float2>(), st);
        poh_dphi_kernel<<<blocks_for(n), kThreads, 0, st>>>(d_phase, w.back.as<float2>(), n, w.dphi.as<float>(),
                                                            w.flag.as<uint32_t>());
        launch_check("poh_dphi");
        const int t = step + 1;
        const double bc1 = 1.0 - std::pow(b1, t), bc2 = 1.0 - std::pow(b2, t), bc3 = 1.0 - std::pow(b3, t);
        const GroupConst k{static_cast<float>(lr), static_cast<float>(1.0 / bc1), static_cast<float>(b2 / bc2),
                           static_cast<float>(1.0 / bc3)};
        poh_adan_kernel<<<blocks_for(n), kThreads, 0, st>>>(d_phase, w.dphi.as<float>(), w.state.as<float>(), n, t, k,
                                                            static_cast<float>(b1), static_cast<float>(b2),
                                                            static_cast<float>(b3), static_cast<float>(eps),
                                                            w.flag.as<uint32_t>());
        launch_check("poh_adan");
    }
}

}  // namespace hs
