// Training loss + gradient (K6 epilogue, K7, K12) and fused Adan (K11).
//
// Reference: proj/core/src/loss.cpp -- loss_recon_grad :317-341, ssim_channel
// :160-214 (window :89-100, corr_x/corr_y/window_mean :103-131, spread_t
// :135-152), loss_ssim_grad :361-383, training_loss_grad :389-398,
// loss_mse_grad :277-294; proj/core/src/optimizer.cpp:59-123 (cosine_lr, Adan).
//
// SSIM kernel: one CTA per 64x16 output tile of one (plane, channel).  It
// loads I (= |U|^2 when fed the propagated field directly) and the target over
// the tile plus a 10-pixel halo, computes the five 11-tap separable window
// means on the valid grid, the SSIM map and its three partial-derivative maps
// (g1, g2, g3 of ssim_channel), spreads them back with the transposed
// correlation and combines grad = sp1 + 2 I sp2 + t sp3, all in shared memory.
// The recon term (I - t)^2 (1 + M + t^2) and its gradient are fused in the
// same epilogue; in trainer mode the epilogue writes dL/dU = 2 U dL/dI
// (pipeline.cpp:265-274) directly.  Loss sums are per-CTA fp64 partials
// reduced by one deterministic final block.
#include <cmath>

#include <cub/block/block_reduce.cuh>

#include "loss.cuh"

namespace hs {

namespace {

constexpr int kTW = 64, kTH = 16, kHalo = 10, kWin = 11;
constexpr int kRW = kTW + 2 * kHalo, kRH = kTH + 2 * kHalo;  // loaded region
constexpr int kVW = kTW + kHalo, kVH = kTH + kHalo;          // valid-grid region
constexpr int kLossThreads = 256;
constexpr double kSsimC1 = 0.01 * 0.01, kSsimC2 = 0.03 * 0.03, kSsimWeight = 0.005;  // loss.hpp:12-14

struct Win {
    float g[kWin];
};

Win ssim_window_f32() {  // loss.cpp:89-100
    Win w;
    double g[kWin], sum = 0.0;
    for (int i = 0; i < kWin; ++i) {
        const double d = i - kWin / 2;
        g[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += g[i];
    }
    for (int i = 0; i < kWin; ++i) w.g[i] = static_cast<float>(g[i] / sum);
    return w;
}

template <bool FROM_FIELD>
__device__ __forceinline__ float load_I(const LossArgs& a, size_t idx) {
    if (FROM_FIELD) {
        const float2 u = a.field[idx];
        return u.x * u.x + u.y * u.y;  // intensity_of, field_core.cpp:88-93
    }
    return a.recon[idx];
}

// Target window statistics on the valid grid, per channel: (mu2, sigma2^2) =
// (E_w[t], E_w[t^2] - E_w[t]^2) -- constant over an optimisation run, so the
// trainer computes them once (ssim_channel :173-176, :190).
__global__ void ssim_target_stats_kernel(const float* __restrict__ target, int C, int H, int W, Win win,
                                         float2* __restrict__ out) {
    const int vh = H - kWin + 1, vw = W - kWin + 1;
    const int64_t total = static_cast<int64_t>(C) * vh * vw;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i / (static_cast<int64_t>(vh) * vw));
        const int rem = static_cast<int>(i - static_cast<int64_t>(c) * vh * vw);
        const int vy = rem / vw, vx = rem - vy * vw;
        const float* t = target + static_cast<size_t>(c) * H * W;
        float m = 0.f, e = 0.f;
        for (int yy = 0; yy < kWin; ++yy) {
            float rm = 0.f, re = 0.f;
            for (int xx = 0; xx < kWin; ++xx) {
                const float v = t[static_cast<size_t>(vy + yy) * W + vx + xx];
                rm = fmaf(win.g[xx], v, rm);
                re = fmaf(win.g[xx], v * v, re);
            }
            m = fmaf(win.g[yy], rm, m);
            e = fmaf(win.g[yy], re, e);
        }
        out[i] = make_float2(m, e - m * m);
    }
}

struct SsimSmem {
    float I[kRH][kRW];        // I over tile + halo
    float T[kRH][kRW];        // target over tile + halo
    float h[3][kRH][kVW];     // corr_x of I, I^2, I*t; reused for the vertical spreads
    float gm[3][kVH][kVW];    // g1, g2, g3 on the valid grid
    float2 ts[kVH][kVW];      // target window stats (mu2, sigma2^2) on the valid grid
};

// Work split of the 256 threads (register-blocked separable correlations):
constexpr int kHB = 11;  // corr_x: 36 rows x 7 runs of 11 outputs      = 252 items
constexpr int kVB = 9;   // corr_y: 74 cols x 3 runs of 9 valid rows    = 222 items
constexpr int kSX = 4;   // spread_x: 16 rows x 16 runs of 4 outputs    = 256 items

template <bool FROM_FIELD>
__global__ void __launch_bounds__(kLossThreads, 2) ssim_loss_kernel(LossArgs a, Win win) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SsimSmem& S = *reinterpret_cast<SsimSmem*>(smem_raw);
    const int plane = blockIdx.z;  // l * C + c
    const int l = plane / a.C, c = plane - l * a.C;
    const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH;
    const int H = a.H, W = a.W;
    const int vh = H - kWin + 1, vw = W - kWin + 1;
    const size_t plane_off = static_cast<size_t>(plane) * H * W;
    const float* tgt = a.target + static_cast<size_t>(c) * H * W;
    const float2* tst = a.tstats + static_cast<size_t>(c) * vh * vw;
    const uint8_t* mask = a.masks + static_cast<size_t>(a.plane0 + l) * H * W;
    const int tid = threadIdx.x;

    {  // all global loads of this thread in flight at once, then the smem stores
        constexpr int kLoads = (kRH * kRW + kLossThreads - 1) / kLossThreads;
        float iv[kLoads], tv[kLoads];
#pragma unroll
        for (int q = 0; q < kLoads; ++q) {
            const int e = tid + q * kLossThreads;
            const int ry = e / kRW, rx = e - ry * kRW;
            const int y = y0 - kHalo + ry, x = x0 - kHalo + rx;
            iv[q] = 0.f;
            tv[q] = 0.f;
            if (e < kRH * kRW && y >= 0 && y < H && x >= 0 && x < W) {
                const size_t p = static_cast<size_t>(y) * W + x;
                iv[q] = load_I<FROM_FIELD>(a, plane_off + p);
                tv[q] = tgt[p];
            }
        }
        constexpr int kTs = (kVH * kVW + kLossThreads - 1) / kLossThreads;
        float2 tsv[kTs];
#pragma unroll
        for (int q = 0; q < kTs; ++q) {
            const int e = tid + q * kLossThreads;
            const int i = e / kVW, j = e - i * kVW;
            const int vy = y0 - kHalo + i, vx = x0 - kHalo + j;
            tsv[q] = (e < kVH * kVW && vy >= 0 && vy < vh && vx >= 0 && vx < vw)
                         ? tst[static_cast<size_t>(vy) * vw + vx] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < kLoads; ++q) {
            const int e = tid + q * kLossThreads;
            if (e < kRH * kRW) {
                const int ry = e / kRW, rx = e - ry * kRW;
                S.I[ry][rx] = iv[q];
                S.T[ry][rx] = tv[q];
            }
        }
#pragma unroll
        for (int q = 0; q < kTs; ++q) {
            const int e = tid + q * kLossThreads;
            if (e < kVH * kVW) S.ts[e / kVW][e % kVW] = tsv[q];
        }
    }
    __syncthreads();
    // corr_x (loss.cpp:103-111) of I, I^2, I*t: each item a run of kHB outputs
    if (tid < kRH * 7) {
        const int ry = tid / 7, j0 = (tid - ry * 7) * kHB;
        float in_i[kHB + kWin - 1], in_t[kHB + kWin - 1];
#pragma unroll
        for (int q = 0; q < kHB + kWin - 1; ++q) {
            const int j = min(j0 + q, kRW - 1);
            in_i[q] = S.I[ry][j];
            in_t[q] = S.T[ry][j];
        }
#pragma unroll
        for (int o = 0; o < kHB; ++o) {
            float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
            for (int k = 0; k < kWin; ++k) {
                const float g = win.g[k], iv = in_i[o + k], tv = in_t[o + k];
                s0 = fmaf(g, iv, s0);
                s1 = fmaf(g, iv * iv, s1);
                s2 = fmaf(g, iv * tv, s2);
            }
            if (j0 + o < kVW) {
                S.h[0][ry][j0 + o] = s0;
                S.h[1][ry][j0 + o] = s1;
                S.h[2][ry][j0 + o] = s2;
            }
        }
    }
    __syncthreads();
    // corr_y + SSIM map + derivative maps (ssim_channel :187-205)
    double ssum = 0.0;
    const float C1 = static_cast<float>(kSsimC1), C2 = static_cast<float>(kSsimC2);
    if (tid < kVW * 3) {
        const int j = tid % kVW, i0 = (tid / kVW) * kVB;
        const int vx = x0 - kHalo + j;
        float col0[kVB + kWin - 1], col1[kVB + kWin - 1], col2[kVB + kWin - 1];
#pragma unroll
        for (int q = 0; q < kVB + kWin - 1; ++q) {
            const int i = min(i0 + q, kRH - 1);
            col0[q] = S.h[0][i][j];
            col1[q] = S.h[1][i][j];
            col2[q] = S.h[2][i][j];
        }
#pragma unroll
        for (int o = 0; o < kVB; ++o) {
            const int i = i0 + o;
            if (i >= kVH) break;
            const int vy = y0 - kHalo + i;
            float g1 = 0.f, g2 = 0.f, g3 = 0.f;
            if (vy >= 0 && vy < vh && vx >= 0 && vx < vw) {
                float m1 = 0.f, exx = 0.f, exy = 0.f;
#pragma unroll
                for (int k = 0; k < kWin; ++k) {
                    const float g = win.g[k];
                    m1 = fmaf(g, col0[o + k], m1);
                    exx = fmaf(g, col1[o + k], exx);
                    exy = fmaf(g, col2[o + k], exy);
                }
                const float2 ts = S.ts[i][j];
                const float m2 = ts.x;
                const float s12 = exy - m1 * m2;
                const float s11 = exx - m1 * m1;
                const float a1 = 2.f * m1 * m2 + C1;
                const float a2 = 2.f * s12 + C2;
                const float b1 = m1 * m1 + m2 * m2 + C1;
                const float b2 = s11 + ts.y + C2;
                // s/a1, s/a2 evaluated as a2/(b1 b2), a1/(b1 b2): equal where
                // ssim_channel's form is defined and finite when a2 rounds to
                // 0 in fp32 (a 0/0 there would poison the field via the FFT).
                const float inv = 1.f / (b1 * b2);
                const float s = a1 * a2 * inv;
                if (vy >= y0 && vy < y0 + kTH && vx >= x0 && vx < x0 + kTW) ssum += s;
                g1 = a2 * inv * 2.f * m2 - (s / b1) * 2.f * m1 + (s / b2) * 2.f * m1 - a1 * inv * 2.f * m2;
                g2 = -s / b2;
                g3 = 2.f * a1 * inv;
            }
            S.gm[0][i][j] = g1;
            S.gm[1][i][j] = g2;
            S.gm[2][i][j] = g3;
        }
    }
    __syncthreads();
    // spread_t vertical (:138-145): sv[y][vx] = sum_k g[k] gm[y - k][vx]; item = (col, map)
    float(*sv)[kVW] = reinterpret_cast<float(*)[kVW]>(&S.h[0][0][0]);  // 3 x kTH x kVW
    if (tid < kVW * 3) {
        const int j = tid % kVW, m = tid / kVW;
        float col[kVH];
#pragma unroll
        for (int q = 0; q < kVH; ++q) col[q] = S.gm[m][q][j];
#pragma unroll
        for (int oy = 0; oy < kTH; ++oy) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < kWin; ++k) acc = fmaf(win.g[k], col[oy + kHalo - k], acc);
            sv[m * kTH + oy][j] = acc;
        }
    }
    __syncthreads();
    // spread_t horizontal (:146-151) + combine (:211) + recon term + output
    const int kind = a.kind;
    const double n_el = static_cast<double>(a.C) * H * W;
    const float wr = static_cast<float>(2.0 / (n_el * a.L_norm));
    const double count = static_cast<double>(a.L_norm) * a.C * vh * vw;
    const float ws = static_cast<float>((kind == kLossTraining ? kSsimWeight : 1.0) * (-1.0 / count));
    double rsum = 0.0;
    {
        const int oy = tid / (kTW / kSX), ox0 = (tid - oy * (kTW / kSX)) * kSX;
        float o[3][kSX];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
            float row[kSX + kWin - 1];
#pragma unroll
            for (int q = 0; q < kSX + kWin - 1; ++q) row[q] = sv[m * kTH + oy][ox0 + q];
#pragma unroll
            for (int u = 0; u < kSX; ++u) {
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k < kWin; ++k) acc = fmaf(win.g[k], row[u + kHalo - k], acc);
                o[m][u] = acc;
            }
        }
        const int y = y0 + oy;
#pragma unroll
        for (int u = 0; u < kSX; ++u) {
            const int x = x0 + ox0 + u;
            if (y >= H || x >= W) continue;
            const float iv = S.I[oy + kHalo][ox0 + u + kHalo], tv = S.T[oy + kHalo][ox0 + u + kHalo];
            const float gs = o[0][u] + 2.f * iv * o[1][u] + tv * o[2][u];
            const size_t p = static_cast<size_t>(y) * W + x;
            float g = ws * gs;
            if (kind == kLossTraining) {
                const float d = iv - tv;
                const float k = 1.f + (mask[p] ? 1.f : 0.f) + tv * tv;
                rsum += static_cast<double>(d * d * k);
                g = fmaf(wr * d, k, g);
            }
            if (a.grad) a.grad[plane_off + p] = g;
            if (a.du) {
                const float2 uu = a.field[plane_off + p];
                a.du[plane_off + p] = make_float2(2.f * uu.x * g, 2.f * uu.y * g);
            }
        }
    }
    using BR = cub::BlockReduce<double, kLossThreads>;
    __shared__ typename BR::TempStorage tmp;
    const double r_tot = BR(tmp).Sum(rsum);
    __syncthreads();
    const double s_tot = BR(tmp).Sum(ssum);
    if (tid == 0) {
        const int slot = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        a.partials[2 * slot] = r_tot;
        a.partials[2 * slot + 1] = s_tot;
    }
}

// recon / mse only: elementwise
template <bool FROM_FIELD>
__global__ void __launch_bounds__(kLossThreads) pixel_loss_kernel(LossArgs a, int64_t total) {
    const double n_el = static_cast<double>(a.C) * a.H * a.W;
    const float wr = static_cast<float>(2.0 / (n_el * a.L_norm));
    const int64_t hw = static_cast<int64_t>(a.H) * a.W;
    const int64_t chw = hw * a.C;
    double rsum = 0.0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kLossThreads + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * kLossThreads) {
        const int64_t l = i / chw;
        const int64_t rem = i - l * chw;
        const int64_t c = rem / hw;
        const int64_t p = rem - c * hw;
        const float iv = load_I<FROM_FIELD>(a, i);
        const float tv = a.target[c * hw + p];
        const float d = iv - tv;
        float g;
        if (a.kind == kLossMse) {
            rsum += static_cast<double>(d * d);
            g = wr * d;
        } else {
            const float k = 1.f + (a.masks[(a.plane0 + l) * hw + p] ? 1.f : 0.f) + tv * tv;
            rsum += static_cast<double>(d * d * k);
            g = wr * d * k;
        }
        if (a.grad) a.grad[i] = g;
        if (a.du) {
            const float2 u = a.field[i];
            a.du[i] = make_float2(2.f * u.x * g, 2.f * u.y * g);
        }
    }
    using BR = cub::BlockReduce<double, kLossThreads>;
    __shared__ typename BR::TempStorage tmp;
    const double r_tot = BR(tmp).Sum(rsum);
    if (threadIdx.x == 0) {
        a.partials[2 * blockIdx.x] = r_tot;
        a.partials[2 * blockIdx.x + 1] = 0.0;
    }
}

__global__ void __launch_bounds__(1024) loss_finalize_kernel(const double* partials, int slots, int kind, double n_el,
                                     int L_norm, double count, double* out) {
    using BR = cub::BlockReduce<double, 1024>;
    __shared__ typename BR::TempStorage tmp;
    double r = 0.0, s = 0.0;
    for (int i = threadIdx.x; i < slots; i += 1024) {
        r += partials[2 * i];
        s += partials[2 * i + 1];
    }
    const double rt = BR(tmp).Sum(r);
    __syncthreads();
    const double st = BR(tmp).Sum(s);
    if (threadIdx.x == 0) {
        double v = 0.0;
        if (kind == kLossTraining) v = rt / (n_el * L_norm) + kSsimWeight * (1.0 - st / count);
        else if (kind == kLossSsim) v = 1.0 - st / count;
        else v = rt / (n_el * L_norm);
        out[0] = v;
        out[1] = rt;
        out[2] = st;
    }
}

__global__ void intensity_kernel(const float2* f, int64_t n, float* out) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float2 u = f[i];
        out[i] = u.x * u.x + u.y * u.y;
    }
}

// ---- Adan -------------------------------------------------------------------------
struct GroupConst {
    float lr, inv_bc1, b2_bc2, inv_bc3;
};

__device__ __forceinline__ void adan_update(float& p, float g, float& m, float& v, float& n,
                                            float& gp, bool first, float b1, float b2, float b3,
                                            float eps, const GroupConst& k) {
    const float diff = first ? 0.f : g - gp;
    m = b1 * m + (1.f - b1) * g;
    v = b2 * v + (1.f - b2) * diff;
    const float u = g + b2 * diff;
    n = b3 * n + (1.f - b3) * u * u;
    const float denom = sqrtf(n * k.inv_bc3) + eps;
    p -= k.lr * (m * k.inv_bc1 + v * k.b2_bc2) / denom;
    gp = g;
}

__global__ void adan_fused_kernel(float* __restrict__ p, const float* __restrict__ g,
                                  float* __restrict__ st, int64_t P, AdanGroups G, int total_steps,
                                  double b1, double b2, double b3, double eps,
                                  const int* __restrict__ step, const uint32_t* __restrict__ flags) {
    __shared__ GroupConst K[6];
    __shared__ int first_bad;
    const int t = step[1] + 1;
    if (threadIdx.x < 6) {
        const int gi = threadIdx.x;
        double lr = G.base_lr[gi];
        if (gi == 0) {  // cosine_lr(step, total, 1e-2, 1e-3), pipeline.cpp:254
            const double s = static_cast<double>(step[0]);
            lr = 1e-3 + 0.5 * (1e-2 - 1e-3) * (1.0 + cos(3.14159265358979323846 * s / total_steps));
        }
        const double bc1 = 1.0 - pow(b1, static_cast<double>(t));
        const double bc2 = 1.0 - pow(b2, static_cast<double>(t));
        const double bc3 = 1.0 - pow(b3, static_cast<double>(t));
        K[gi] = GroupConst{static_cast<float>(lr), static_cast<float>(1.0 / bc1),
                           static_cast<float>(b2 / bc2), static_cast<float>(1.0 / bc3)};
    }
    if (threadIdx.x == 0) {
        const uint32_t f = flags ? *flags : 0u;
        first_bad = f ? __ffs(f) - 1 : 6;
    }
    __syncthreads();
    const bool first = t == 1;
    float* m = st;
    float* v = st + P;
    float* n = st + 2 * P;
    float* gp = st + 3 * P;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int gi = 0;
#pragma unroll
        for (int q = 1; q < 6; ++q) gi += (i >= G.begin[q]) ? 1 : 0;
        if (gi >= first_bad) continue;
        float pv = p[i], mv = m[i], vv = v[i], nv = n[i], gpv = gp[i];
        adan_update(pv, g[i], mv, vv, nv, gpv, first, static_cast<float>(b1), static_cast<float>(b2),
                    static_cast<float>(b3), static_cast<float>(eps), K[gi]);
        p[i] = pv;
        m[i] = mv;
        v[i] = vv;
        n[i] = nv;
        gp[i] = gpv;
    }
}

__global__ void adan_advance_kernel(int* step, const uint32_t* flags) {
    if (flags && *flags) return;  // the reference aborts on a non-finite gradient
    step[0] += 1;
    step[1] += 1;
}

__global__ void adan_group_kernel(float* __restrict__ p, const float* __restrict__ g,
                                  float* __restrict__ st, int64_t P, int t, GroupConst k, float b1,
                                  float b2, float b3, float eps) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float pv = p[i], mv = st[i], vv = st[P + i], nv = st[2 * P + i], gpv = st[3 * P + i];
        adan_update(pv, g[i], mv, vv, nv, gpv, t == 1, b1, b2, b3, eps, k);
        p[i] = pv;
        st[i] = mv;
        st[P + i] = vv;
        st[2 * P + i] = nv;
        st[3 * P + i] = gpv;
    }
}

__global__ void nonfinite_kernel(const float* g, int64_t n, uint32_t* flag) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (!isfinite(g[i])) {
            atomicOr(flag, 1u);
            return;
        }
}

unsigned grid_for(int64_t n, int threads) {
    const int64_t b = (n + threads - 1) / threads;
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16)));
}

}  // namespace

int loss_partial_slots(int kind, int L, int C, int H, int W) {
    if (kind == kLossTraining || kind == kLossSsim)
        return ceil_div(W, kTW) * ceil_div(H, kTH) * L * C;
    const int64_t total = static_cast<int64_t>(L) * C * H * W;
    return static_cast<int>(grid_for(total, kLossThreads));
}

int loss_launch(const LossArgs& a, cudaStream_t st) {
    if (a.kind == kLossTraining || a.kind == kLossSsim) {
        require(a.H >= kWin && a.W >= kWin, "ssim: image smaller than the 11x11 window");
        const dim3 grid(ceil_div(a.W, kTW), ceil_div(a.H, kTH), a.L * a.C);
        const size_t smem = sizeof(SsimSmem);
        static const Win win = ssim_window_f32();
        require(a.tstats != nullptr, "ssim: target statistics missing");
        if (a.field) {
            HS_CUDA(cudaFuncSetAttribute(ssim_loss_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
            ssim_loss_kernel<true><<<grid, kLossThreads, smem, st>>>(a, win);
        } else {
            HS_CUDA(cudaFuncSetAttribute(ssim_loss_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
            ssim_loss_kernel<false><<<grid, kLossThreads, smem, st>>>(a, win);
        }
        launch_check("ssim_loss");
        return static_cast<int>(grid.x * grid.y * grid.z);
    }
    const int64_t total = static_cast<int64_t>(a.L) * a.C * a.H * a.W;
    const unsigned blocks = grid_for(total, kLossThreads);
    if (a.field) pixel_loss_kernel<true><<<blocks, kLossThreads, 0, st>>>(a, total);
    else pixel_loss_kernel<false><<<blocks, kLossThreads, 0, st>>>(a, total);
    launch_check("pixel_loss");
    return static_cast<int>(blocks);
}

void loss_finalize(const LossArgs& a, int slots, double* d_out3, cudaStream_t st) {
    const double n_el = static_cast<double>(a.C) * a.H * a.W;
    const double count = static_cast<double>(a.L_norm) * a.C * std::max(a.H - kWin + 1, 0) *
                         std::max(a.W - kWin + 1, 0);
    loss_finalize_kernel<<<1, 1024, 0, st>>>(a.partials, slots, a.kind, n_el, a.L_norm, count, d_out3);
    launch_check("loss_finalize");
}

void ssim_target_stats(const float* target, int C, int H, int W, float2* out, cudaStream_t st) {
    if (H < kWin || W < kWin) return;
    static const Win win = ssim_window_f32();
    const int64_t total = static_cast<int64_t>(C) * (H - kWin + 1) * (W - kWin + 1);
    ssim_target_stats_kernel<<<grid_for(total, 256), 256, 0, st>>>(target, C, H, W, win, out);
    launch_check("ssim_target_stats");
}

void intensity_launch(const float2* f, int64_t count, float* out, cudaStream_t st) {
    if (count == 0) return;
    intensity_kernel<<<grid_for(count, 256), 256, 0, st>>>(f, count, out);
    launch_check("intensity");
}

void adan_fused_launch(float* params, const float* grads, float* state, int64_t P,
                       const AdanGroups& g, int total_steps, double b1, double b2, double b3,
                       double eps, int* d_step, const uint32_t* d_flags, cudaStream_t st) {
    adan_fused_kernel<<<grid_for(P, 256), 256, 0, st>>>(params, grads, state, P, g, total_steps, b1, b2,
                                                        b3, eps, d_step, d_flags);
    launch_check("adan_fused");
    adan_advance_kernel<<<1, 1, 0, st>>>(d_step, d_flags);
    launch_check("adan_advance");
}

void adan_group_launch(float* params, const float* grads, float* state, int64_t size, int t,
                       double lr, double b1, double b2, double b3, double eps, cudaStream_t st) {
    if (size == 0) return;
    const double bc1 = 1.0 - std::pow(b1, t), bc2 = 1.0 - std::pow(b2, t), bc3 = 1.0 - std::pow(b3, t);
    GroupConst k{static_cast<float>(lr), static_cast<float>(1.0 / bc1), static_cast<float>(b2 / bc2),
                 static_cast<float>(1.0 / bc3)};
    adan_group_kernel<<<grid_for(size, 256), 256, 0, st>>>(params, grads, state, size, t, k,
                                                           static_cast<float>(b1), static_cast<float>(b2),
                                                           static_cast<float>(b3), static_cast<float>(eps));
    launch_check("adan_group");
}

void nonfinite_launch(const float* g, int64_t n, uint32_t* flag, cudaStream_t st) {
    if (n == 0) return;
    nonfinite_kernel<<<grid_for(n, 256), 256, 0, st>>>(g, n, flag);
    launch_check("nonfinite");
}

}  // namespace hs
