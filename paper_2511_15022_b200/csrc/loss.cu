// Training loss + gradient (K6 epilogue, K7, K12) and fused Adan (K11).
//
// Reference: proj/core/src/loss.cpp -- loss_recon_grad :248-272, ssim_channel
// :91-145 (ssim_window :20-31, corr_x/corr_y/window_mean :34-62, spread_t
// :66-83), loss_ssim_grad :292-314, training_loss_grad :320-329,
// loss_mse_grad :208-225; proj/core/src/optimizer.cpp:8-72 (cosine_lr, Adan).
//
// SSIM kernel (sliding window): one CTA of 128 threads owns a strip of 118
// output columns and SR output rows of one (plane, channel) and walks down
// it row by row.  Thread t owns column c = x0 - 10 + t of both the valid
// (H-10)x(W-10) grid and the output grid.  Per step it
//   1. correlates its input row horizontally (I, I^2, I t from a shared row),
//   2. keeps the last 11 such rows in a register ring and correlates them
//      vertically -> window means of valid row v, SSIM map and the three
//      derivative maps g1, g2, g3 (ssim_channel loss.cpp:129-135),
//   3. spreads g back horizontally from a shared row of its 10 left
//      neighbours, keeps the last 11 spread rows in a second register ring and
//      spreads vertically -> dSSIM/dI of output row v (spread_t loss.cpp:66-83),
//   4. fuses the recon term (I - t)^2 (1 + M + t^2) and, in trainer mode,
//      dL/dU = 2 U dL/dI (pipeline.cpp:265-274).
// Every input row is read once per strip (no vertical halo re-reads beyond
// the 20-row pipeline fill per CTA); one barrier per row.  Loss sums are
// per-CTA fp64 partials reduced by one deterministic final block.
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include <cub/block/block_reduce.cuh>

#include "loss.cuh"

namespace hs {

namespace {

constexpr int kWin = 11, kHalo = 10;
constexpr int kSW = 128;            // threads per CTA = valid/output columns touched per strip
constexpr int kSO = kSW - kHalo;    // output columns per strip
// output rows per CTA: SR + 20 steps must be whole 11-step ring cycles; the
// variants trade pipeline fill (20 / SR) against a single wave at MINB CTAs/SM
// (1080p x 3 channels: SR 101 -> 561 CTAs, SR 145 -> 408 CTAs)
constexpr int kSIn = kSW + kHalo;   // input columns per strip
constexpr int kLossThreads = 256;   // elementwise kernels
constexpr double kSsimC1 = 0.01 * 0.01, kSsimC2 = 0.03 * 0.03, kSsimWeight = 0.005;  // loss.hpp:12-14

struct Win {
    float g[kWin];
};

Win ssim_window_f32() {  // ssim_window, loss.cpp:20-31
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
// trainer computes them once (ssim_channel loss.cpp:105, :107).
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

// 11-tap correlation with the symmetric window: sum_j g[j] f(j).
// (two interleaved FMA chains: short dependency chains for the latency-bound SSIM kernel)
template <class F>
__device__ __forceinline__ float corr11(const Win& w, F f) {
    float a = w.g[5] * f(5);
    float b = w.g[1] * (f(1) + f(9));
    a = fmaf(w.g[0], f(0) + f(10), a);
    b = fmaf(w.g[3], f(3) + f(7), b);
    a = fmaf(w.g[2], f(2) + f(8), a);
    a = fmaf(w.g[4], f(4) + f(6), a);
    return a + b;
}

// Three 11-tap correlations at once from a loader f(j) -> float4 (x, y, z used),
// loading the symmetric pairs progressively (few live registers); x and y run
// as packed fp32x2 pairs.
template <class F>
__device__ __forceinline__ void corr11x3(const Win& w, F f, float2& a01, float& a2) {
    const float4 m = f(5);
    float2 axy = f2mul(f2splat(w.g[5]), make_float2(m.x, m.y));
    float az = w.g[5] * m.z;
    float2 bxy = make_float2(0.f, 0.f);
    float bz = 0.f;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const float4 p = f(j), q = f(10 - j);
        const float2 sxy = f2add(make_float2(p.x, p.y), make_float2(q.x, q.y));
        if (j & 1) {
            bxy = f2fma(f2splat(w.g[j]), sxy, bxy);
            bz = fmaf(w.g[j], p.z + q.z, bz);
        } else {
            axy = f2fma(f2splat(w.g[j]), sxy, axy);
            az = fmaf(w.g[j], p.z + q.z, az);
        }
    }
    a01 = f2add(axy, bxy);
    a2 = az + bz;
}

// Same for a packed ring pair and a scalar ring: f(i) -> row i of (pair, scalar).
template <class F2, class F1>
__device__ __forceinline__ void corr11x3r(const Win& w, F2 f2, F1 f1, float2& a01, float& a2) {
    float2 axy = f2mul(f2splat(w.g[5]), f2(5)), bxy = make_float2(0.f, 0.f);
    float az = w.g[5] * f1(5), bz = 0.f;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const float2 sxy = f2add(f2(j), f2(10 - j));
        if (j & 1) {
            bxy = f2fma(f2splat(w.g[j]), sxy, bxy);
            bz = fmaf(w.g[j], f1(j) + f1(10 - j), bz);
        } else {
            axy = f2fma(f2splat(w.g[j]), sxy, axy);
            az = fmaf(w.g[j], f1(j) + f1(10 - j), az);
        }
    }
    a01 = f2add(axy, bxy);
    a2 = az + bz;
}

// One 11-row register ring per thread.  Producer threads keep the horizontal
// correlations of (I, I^2 | I t) in it, consumer threads the horizontal spreads
// of (g1, g2 | g3): the same registers, role-dependent meaning.
struct SsimState {
    float2 r01[kWin];  // packed pair
    float r2[kWin];
    double sum;        // producer: SSIM map sum; consumer: recon sum (fp64, as loss.cpp:320-329)
};

// Asynchronous global->shared copies (cp.async); src_bytes = 0 zero-fills.
template <int B>
__device__ __forceinline__ void cp_async(void* dst, const void* src, bool ok) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(src), "n"(B), "r"(ok ? B : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

constexpr int kRaw = 16;  // ring of raw input rows (U or I, and t): covers rows r-12 .. r+kPD
constexpr int kPD = 2;    // prefetch distance (rows) of the cp.async pipeline (3: +1.2 us; 5 needs kTsRing > 5)
constexpr int kTsRing = 4;
static_assert(kTsRing > kPD && kRaw >= 13 + kPD, "cp.async rings must outlive the prefetch distance");

template <class Raw>
struct SsimSmem {
    Raw rawU[kRaw][kSIn];       // U (or I when the loss gets intensities)
    float rawT[kRaw][kSIn];     // target
    float2 ts[kTsRing][kSW];    // target window stats of the valid row
    float4 in[2][kSIn];         // (I, I^2, I t, -) of the row being correlated
    float4 gm[2][kSW];          // (g1, g2, g3, -) of the valid row being spread
};

template <bool FROM_FIELD, int SR, bool BAND = false>
struct SsimCta {
    using Raw = typename std::conditional<FROM_FIELD, float2, float>::type;
    const LossArgs& a;
    const Win& win;
    SsimSmem<Raw>& S;
    int t, x0, y0, y1, c, H, W, vh, vw, kind;  // output rows [y0, y1) of this CTA (at most SR)
    size_t plane_off;
    const float* tgt;
    const float2* tst;
    const uint8_t* mask;
    float wr, ws;
    // per-thread copy sources (column clamped into the image) and validity
    const Raw* srcA;     // own input column (plane base + column)
    const Raw* srcB;     // right-halo column (t < 10)
    const float* tgtA;
    const float* tgtB;
    const float2* tsA;   // target stats, own valid column
    bool okA, okB, okV;

    __device__ __forceinline__ void init_sources() {
        const int xa = x0 - kHalo + t, xb = x0 + kSO + t;
        okA = xa >= 0 && xa < W;
        okB = t < kHalo && xb < W;
        okV = c >= 0 && c < vw;
        const Raw* base = FROM_FIELD ? reinterpret_cast<const Raw*>(a.field + plane_off)
                                     : reinterpret_cast<const Raw*>(a.recon + plane_off);
        srcA = base + min(max(xa, 0), W - 1);
        srcB = base + min(max(xb, 0), W - 1);
        tgtA = tgt + min(max(xa, 0), W - 1);
        tgtB = tgt + min(max(xb, 0), W - 1);
        tsA = tst + min(max(c, 0), vw - 1);
    }

    // cp.async of input row r (own column, plus the right halo for t < 10)
    // and of the target statistics of valid row v; one commit group.
    __device__ __forceinline__ void issue(int r, int v) const {
        const bool rok = r >= 0 && r < H;
        // 32-bit row offset (a plane is < 2^32 elements); out-of-image rows
        // zero-fill from the (valid) row-0 address
        const unsigned rowp = rok ? static_cast<unsigned>(r) * static_cast<unsigned>(W) : 0u;
        const int slot = r & (kRaw - 1);
        cp_async<sizeof(Raw)>(&S.rawU[slot][t], srcA + rowp, rok && okA);
        cp_async<4>(&S.rawT[slot][t], tgtA + rowp, rok && okA);
        if (t < kHalo) {
            cp_async<sizeof(Raw)>(&S.rawU[slot][kSW + t], srcB + rowp, rok && okB);
            cp_async<4>(&S.rawT[slot][kSW + t], tgtB + rowp, rok && okB);
        }
        const bool vok = v >= 0 && v < vh;
        cp_async<8>(&S.ts[v & (kTsRing - 1)][t], tsA + (vok ? static_cast<unsigned>(v) * static_cast<unsigned>(vw) : 0u),
                    vok && okV);
        cp_commit();
    }
    __device__ __forceinline__ float intensity(Raw u) const {
        if constexpr (FROM_FIELD) return u.x * u.x + u.y * u.y;
        else return u;
    }
    // (I, I^2, I t) of raw row r -> the correlation row buffer (own columns only)
    __device__ __forceinline__ void convert(int r, int buf) const {
        const int slot = r & (kRaw - 1);
        {
            const float i = intensity(S.rawU[slot][t]), tv = S.rawT[slot][t];
            S.in[buf][t] = make_float4(i, i * i, i * tv, 0.f);
        }
        if (t < kHalo) {
            const float i = intensity(S.rawU[slot][kSW + t]), tv = S.rawT[slot][kSW + t];
            S.in[buf][kSW + t] = make_float4(i, i * i, i * tv, 0.f);
        }
    }

    // Producer half (threads 0..127) of row step s: valid row v = y0 - 20 + s,
    // ring slot U = s mod 11.  Horizontal correlation of input row r = v + 10,
    // vertical correlation of rows v..v+10, SSIM map and derivative maps of row v
    // -> gm[s & 1]; next input row -> in[(s + 1) & 1].
    template <int U>
    __device__ __forceinline__ void produce(SsimState& st, int s) const {
        const int v = y0 - 2 * kHalo + s;
        const int r = v + kHalo;
        const int buf = s & 1;
        issue(r + kPD, v + kPD);
        {  // ssim_channel corr_x (loss.cpp:34-42)
            const float4* row = &S.in[buf][t];
            corr11x3(win, [&](int j) { return row[j]; }, st.r01[U], st.r2[U]);
        }
        cp_wait<kPD - 1>();  // groups of rows <= r + 1 (and stats of v) have landed
        float4 gv = make_float4(0.f, 0.f, 0.f, 0.f);
        if (v >= 0 && v < vh && c >= 0 && c < vw) {
            float2 mm;
            float exy;
            corr11x3r(win, [&](int i) { return st.r01[(U + 1 + i) % kWin]; },
                      [&](int i) { return st.r2[(U + 1 + i) % kWin]; }, mm, exy);
            const float m1 = mm.x, exx = mm.y;
            const float2 ts = S.ts[v & (kTsRing - 1)][t];
            const float C1 = static_cast<float>(kSsimC1), C2 = static_cast<float>(kSsimC2);
            const float m2 = ts.x;
            const float s12 = exy - m1 * m2;
            const float s11 = exx - m1 * m1;
            const float a1 = 2.f * m1 * m2 + C1;
            const float a2 = 2.f * s12 + C2;
            const float b1 = m1 * m1 + m2 * m2 + C1;
            const float b2 = s11 + ts.y + C2;
            // s/a1, s/a2 evaluated as a2/(b1 b2), a1/(b1 b2): equal where
            // ssim_channel's form is defined and finite when a2 rounds to 0
            // in fp32 (a 0/0 there would poison the field via the FFT).
            const float rb1 = __fdividef(1.f, b1), rb2 = __fdividef(1.f, b2);
            const float inv = rb1 * rb2;
            const float sv = a1 * a2 * inv;
            if (t >= kHalo && v >= y0 && v < y1 &&
                (!BAND || static_cast<unsigned>(v - a.own0) < static_cast<unsigned>(a.own1 - a.own0)))
                st.sum += static_cast<double>(sv);
            gv.x = 2.f * (a2 * inv * m2 - sv * rb1 * m1 + sv * rb2 * m1 - a1 * inv * m2);
            gv.y = -sv * rb2;
            gv.z = 2.f * a1 * inv;
        }
        S.gm[buf][t] = gv;
        convert(r + 1, buf ^ 1);
    }

    // Consumer half (threads 128..255, column t = tid - 128) of row step s:
    // horizontal spread of gm[s & 1] over valid columns c-10..c, vertical spread
    // over valid rows v-10..v (spread_t, loss.cpp:66-83), output row y = v.
    template <int U>
    __device__ __forceinline__ void consume(SsimState& st, int s, float& mk_next) const {
        const int v = y0 - 2 * kHalo + s;
        const int buf = s & 1;
        const int y = v, x = c;
        const bool out_ok = t >= kHalo && y >= y0 && y < y1 && y < H && x < W;
        const float mk = mk_next;
        if (kind == kLossTraining) {  // mask of the next step's output row, one step ahead
            const int yn = y + 1;
            mk_next = (t >= kHalo && yn >= y0 && yn < y1 && yn < H && x < W)
                          ? (mask[static_cast<unsigned>(yn) * static_cast<unsigned>(W) + static_cast<unsigned>(x)] ? 1.f : 0.f)
                          : 0.f;
        }
        {
            // threads t < 10 own no output column: their spread row stays 0
            const float4* gr = &S.gm[buf][max(t, kHalo)];
            corr11x3(win, [&](int j) { return gr[-j]; }, st.r01[U], st.r2[U]);
            if (t < kHalo) {
                st.r01[U] = make_float2(0.f, 0.f);
                st.r2[U] = 0.f;
            }
        }
        if (out_ok) {
            float2 G12;
            float G3;
            corr11x3r(win, [&](int i) { return st.r01[(U + kWin - i) % kWin]; },
                      [&](int i) { return st.r2[(U + kWin - i) % kWin]; }, G12, G3);
            const float G1 = G12.x, G2 = G12.y;
            const int slot = y & (kRaw - 1);
            const Raw uu = S.rawU[slot][t];
            const float tv = S.rawT[slot][t];
            const float iv = intensity(uu);
            const float gs = G1 + 2.f * iv * G2 + tv * G3;  // loss.cpp:142
            float g = ws * gs;
            if (kind == kLossTraining) {  // loss_recon_grad, loss.cpp:248-272
                const float d = iv - tv;
                const float k = 1.f + mk + tv * tv;
                if (!BAND || static_cast<unsigned>(y - a.own0) < static_cast<unsigned>(a.own1 - a.own0)) st.sum += static_cast<double>(d * d * k);
                g = fmaf(wr * d, k, g);
            }
            const unsigned p = static_cast<unsigned>(y) * static_cast<unsigned>(W) + static_cast<unsigned>(x);
            if (a.grad) a.grad[plane_off + p] = g;
            if constexpr (FROM_FIELD) {
                if (a.du) (a.du + plane_off)[p] = make_float2(2.f * uu.x * g, 2.f * uu.y * g);
            }
        }
    }
};

// Producer/consumer warp groups: threads [0, 128) produce SSIM rows, threads
// [128, 256) consume them one step behind, so the two halves of a row step run
// concurrently and each thread carries a single 11-row register ring.
// BAND: row-slab shard, loss sums restricted to rows [own0, own1) (LossArgs)
template <bool FROM_FIELD, int MINB, int SR, bool BAND = false>
__global__ void __launch_bounds__(2 * kSW, MINB) ssim_loss_kernel(LossArgs a, Win win) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using Raw = typename SsimCta<FROM_FIELD, SR, BAND>::Raw;
    SsimSmem<Raw>& S = *reinterpret_cast<SsimSmem<Raw>*>(smem_raw);
    const int plane = blockIdx.z;  // l * C + c
    const int l = plane / a.C, ch = plane - l * a.C;
    const bool producer = threadIdx.x < kSW;
    SsimCta<FROM_FIELD, SR, BAND> K{a, win, S};
    K.t = producer ? threadIdx.x : threadIdx.x - kSW;
    K.x0 = blockIdx.x * kSO;
    // the launch's row strips split H evenly (1080 rows in 8 strips: 135 rows,
    // 155 steps instead of SR + 20 = 165)
    const int sr = (a.H + static_cast<int>(gridDim.y) - 1) / static_cast<int>(gridDim.y);
    K.y0 = blockIdx.y * sr;
    K.y1 = K.y0 + sr;
    K.c = K.x0 - kHalo + K.t;
    K.H = a.H;
    K.W = a.W;
    K.vh = a.H - kWin + 1;
    K.vw = a.W - kWin + 1;
    K.kind = a.kind;
    K.plane_off = static_cast<size_t>(plane) * a.H * a.W;
    K.tgt = a.target + static_cast<size_t>(ch) * a.H * a.W;
    K.tst = a.tstats + static_cast<size_t>(ch) * K.vh * K.vw;
    K.mask = a.masks + static_cast<size_t>(a.plane0 + l) * a.H * a.W;
    const double n_el = static_cast<double>(a.channels_norm()) * a.rows_norm() * a.W;
    K.wr = static_cast<float>(2.0 / (n_el * a.L_norm));
    const double count = static_cast<double>(a.L_norm) * a.channels_norm() * (a.rows_norm() - kWin + 1) * K.vw;
    K.ws = static_cast<float>((a.kind == kLossTraining ? kSsimWeight : 1.0) * (-1.0 / count));
    K.init_sources();

    SsimState st;
#pragma unroll
    for (int i = 0; i < kWin; ++i) {
        st.r01[i] = make_float2(0.f, 0.f);
        st.r2[i] = 0.f;
    }
    st.sum = 0.0;
    // steps s = 0 .. steps-1 cover valid rows v = y0-20 .. y0+sr-1 (output rows y0..y0+sr-1);
    // rows past the image are guarded inside the steps
    constexpr int kSteps = SR + 2 * kHalo;
    static_assert(kSteps % kWin == 0, "whole ring cycles");
    const int r0 = K.y0 - kHalo, v0 = K.y0 - 2 * kHalo;
    if (producer) {
#pragma unroll
        for (int q = 0; q < kPD; ++q) K.issue(r0 + q, v0 + q);
        cp_wait<kPD - 1>();
        K.convert(r0, 0);
    }
    float mk_next = 0.f;  // first output row comes 20 steps in
    __syncthreads();
#define HS_SSIM_STEP(U)                                      \
    if (producer) K.template produce<U>(st, sb + U);         \
    __syncthreads();                                         \
    if (!producer) K.template consume<U>(st, sb + U, mk_next); \
    if (K.y0 + sb + (U + 1 - 2 * kHalo) >= K.y1) break;  /* sr + 20 <= kSteps steps: the last ring cycle may stop part way */
#pragma unroll 1
    for (int sb = 0; sb < kSteps; sb += kWin) {
        HS_SSIM_STEP(0) HS_SSIM_STEP(1) HS_SSIM_STEP(2) HS_SSIM_STEP(3) HS_SSIM_STEP(4) HS_SSIM_STEP(5)
        HS_SSIM_STEP(6) HS_SSIM_STEP(7) HS_SSIM_STEP(8) HS_SSIM_STEP(9) HS_SSIM_STEP(10)
    }
#undef HS_SSIM_STEP
    if (producer) cp_wait<0>();
    // producers hold the SSIM sums, consumers the recon sums
    using BR = cub::BlockReduce<double, 2 * kSW>;
    __shared__ typename BR::TempStorage tmp;
    const double r_tot = BR(tmp).Sum(producer ? 0.0 : st.sum);
    __syncthreads();
    const double s_tot = BR(tmp).Sum(producer ? st.sum : 0.0);
    if (threadIdx.x == 0) {
        const int slot = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        a.partials[2 * slot] = r_tot;
        a.partials[2 * slot + 1] = s_tot;
    }
}

// recon / mse only: elementwise
template <bool FROM_FIELD>
__global__ void __launch_bounds__(kLossThreads) pixel_loss_kernel(LossArgs a, int64_t total) {
    const double n_el = static_cast<double>(a.channels_norm()) * a.H * a.W;
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

__global__ void clip01_kernel(const float* in, int64_t n, float* out) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = fminf(fmaxf(in[i], 0.f), 1.f);
}

__global__ void intensity_kernel(const float2* f, int64_t n, float* out) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float2 u = f[i];
        out[i] = u.x * u.x + u.y * u.y;
    }
}

// ---- Adan (GroupConst, adan_update: loss.cuh) -------------------------------------
// Per-group Adan constants for loop step s and Adan step t: lr (cosine for
// the position group, pipeline.cpp:254) and the bias corrections.
__device__ void adan_consts(const AdanGroups& G, int total_steps, double b1, double b2, double b3, int s, int t,
                            GroupConst* K) {
    // the bias corrections are shared by the six groups: three pow() per step
    const double bc1 = 1.0 - pow(b1, static_cast<double>(t));
    const double bc2 = 1.0 - pow(b2, static_cast<double>(t));
    const double bc3 = 1.0 - pow(b3, static_cast<double>(t));
    const float ib1 = static_cast<float>(1.0 / bc1), bb2 = static_cast<float>(b2 / bc2),
                ib3 = static_cast<float>(1.0 / bc3);
    for (int gi = 0; gi < 6; ++gi) {
        double lr = G.base_lr[gi];
        if (gi == 0)  // cosine_lr(step, total, 1e-2, 1e-3)
            lr = 1e-3 + 0.5 * (1e-2 - 1e-3) * (1.0 + cos(3.14159265358979323846 * static_cast<double>(s) / total_steps));
        K[gi] = GroupConst{static_cast<float>(lr), ib1, bb2, ib3};
    }
}

__global__ void adan_consts_kernel(AdanGroups G, int total_steps, double b1, double b2, double b3,
                                   const int* __restrict__ step, GroupConst* __restrict__ K) {
    adan_consts(G, total_steps, b1, b2, b3, step[0], step[1] + 1, K);
}

// Fused Adan over the six groups (Adan::step optimizer.cpp:48-72) with the group
// constants of this step precomputed in Kc.  VEC: every group boundary and P
// are multiples of 4, so a thread updates a float4 of one group with 16-byte
// loads/stores.  The last CTA to finish advances the device step counter (not
// after a non-finite gradient: the reference aborts) and precomputes the next
// step's constants.
constexpr int kAdanMinBlocks = 4;
template <bool VEC>
__global__ void __launch_bounds__(256, kAdanMinBlocks) adan_fused_kernel(float* __restrict__ p, const float* __restrict__ g,
                                  float* __restrict__ st, int64_t P, int64_t PS, AdanGroups G, int total_steps,
                                  double b1, double b2, double b3, double eps,
                                  int* __restrict__ step, const uint32_t* __restrict__ flags,
                                  unsigned* __restrict__ done, GroupConst* __restrict__ Kc) {
    __shared__ GroupConst K[6];
    __shared__ int first_bad;
    if (threadIdx.x < 6) K[threadIdx.x] = Kc[threadIdx.x];
    if (threadIdx.x == 0) {
        const uint32_t f = flags ? *flags : 0u;
        first_bad = f ? __ffs(f) - 1 : 6;
    }
    const bool first = step[1] == 0;  // Adan t == 1
    __syncthreads();
    const float fb1 = static_cast<float>(b1), fb2 = static_cast<float>(b2), fb3 = static_cast<float>(b3);
    const float feps = static_cast<float>(eps);
    // state moments of the P elements updated here, at stride PS (the whole
    // buffer's element count; PS > P when one rank updates its shard only)
    float* m = st;
    float* v = st + PS;
    float* n = st + 2 * PS;
    float* gp = st + 3 * PS;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    if constexpr (VEC) {
        const int64_t P4 = P / 4;
        for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < P4; q += stride) {
            const int64_t i = 4 * q;
            int gi = 0;
#pragma unroll
            for (int k = 1; k < 6; ++k) gi += (i >= G.begin[k]) ? 1 : 0;
            if (gi >= first_bad) continue;
            float4 pv = reinterpret_cast<float4*>(p)[q], gv = reinterpret_cast<const float4*>(g)[q];
            float4 mv = reinterpret_cast<float4*>(m)[q], vv = reinterpret_cast<float4*>(v)[q];
            float4 nv = reinterpret_cast<float4*>(n)[q], gpv = reinterpret_cast<float4*>(gp)[q];
            adan_update(pv.x, gv.x, mv.x, vv.x, nv.x, gpv.x, first, fb1, fb2, fb3, feps, K[gi]);
            adan_update(pv.y, gv.y, mv.y, vv.y, nv.y, gpv.y, first, fb1, fb2, fb3, feps, K[gi]);
            adan_update(pv.z, gv.z, mv.z, vv.z, nv.z, gpv.z, first, fb1, fb2, fb3, feps, K[gi]);
            adan_update(pv.w, gv.w, mv.w, vv.w, nv.w, gpv.w, first, fb1, fb2, fb3, feps, K[gi]);
            reinterpret_cast<float4*>(p)[q] = pv;
            reinterpret_cast<float4*>(m)[q] = mv;
            reinterpret_cast<float4*>(v)[q] = vv;
            reinterpret_cast<float4*>(n)[q] = nv;
            reinterpret_cast<float4*>(gp)[q] = gpv;
        }
    } else {
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P; i += stride) {
            int gi = 0;
#pragma unroll
            for (int k = 1; k < 6; ++k) gi += (i >= G.begin[k]) ? 1 : 0;
            if (gi >= first_bad) continue;
            float pv = p[i], mv = m[i], vv = v[i], nv = n[i], gpv = gp[i];
            adan_update(pv, g[i], mv, vv, nv, gpv, first, fb1, fb2, fb3, feps, K[gi]);
            p[i] = pv;
            m[i] = mv;
            v[i] = vv;
            n[i] = nv;
            gp[i] = gpv;
        }
    }
    // last CTA out (every CTA has read step and Kc) advances the counter and
    // prepares the next step's constants
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(done, 1u) == gridDim.x - 1) {
            *done = 0u;
            if (!(flags && *flags)) {
                step[0] += 1;
                step[1] += 1;
            }
            adan_consts(G, total_steps, b1, b2, b3, step[0], step[1] + 1, Kc);
        }
    }
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

// Output rows per SSIM CTA (SR + 20 steps must be whole 11-step ring
// cycles).  All CTAs walk the same number of steps and are resident 3 per SM,
// so the kernel takes about waves x (SR + 20) step-times: the row count is
// chosen per launch to minimise that (1080p x 3: 145 -> 8 row strips, one
// wave; 1080p x 24 planes: 156; a 155-row slab band x 24: 156, one CTA row
// instead of two; a small band x 3: 35).
constexpr int kSsimRowChoices[] = {35, 79, 145, 156, 167};
constexpr int kSsimMinBlocks = 3;

int ssim_rows(int planes, int H, int W) {
    static const int sms = [] {
        int dev = 0;
        HS_CUDA(cudaGetDevice(&dev));
        return sm_count(dev);
    }();
    const int64_t slots = static_cast<int64_t>(kSsimMinBlocks) * sms;
    int best = kSsimRowChoices[0];
    int64_t best_cost = -1;
    for (int sr : kSsimRowChoices) {
        const int strips = ceil_div(H, sr);
        const int64_t ctas = static_cast<int64_t>(ceil_div(W, kSO)) * strips * planes;
        const int64_t cost = (ctas + slots - 1) / slots * (ceil_div(H, strips) + 2 * kHalo);
        if (best_cost < 0 || cost < best_cost) {
            best = sr;
            best_cost = cost;
        }
    }
    return best;
}

template <bool FROM_FIELD, bool BAND, int... SR>
auto ssim_kernel_for(int sr, std::integer_sequence<int, SR...>) {
    using K = void (*)(LossArgs, Win);
    K k = nullptr;
    ((sr == SR ? (k = ssim_loss_kernel<FROM_FIELD, kSsimMinBlocks, SR, BAND>, 0) : 0), ...);
    require(k != nullptr, "ssim: no kernel for the row count");
    return k;
}
template <bool FROM_FIELD, bool BAND>
auto ssim_kernel(int sr) {
    return ssim_kernel_for<FROM_FIELD, BAND>(sr, std::integer_sequence<int, 35, 79, 145, 156, 167>{});
}

unsigned grid_for(int64_t n, int threads) {
    const int64_t b = (n + threads - 1) / threads;
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16)));
}

}  // namespace

int loss_partial_slots(int kind, int L, int C, int H, int W) {
    if (kind == kLossTraining || kind == kLossSsim)
        return ceil_div(W, kSO) * ceil_div(H, ssim_rows(L * C, H, W)) * L * C;
    const int64_t total = static_cast<int64_t>(L) * C * H * W;
    return static_cast<int>(grid_for(total, kLossThreads));
}

int loss_launch(const LossArgs& a, cudaStream_t st) {
    if (a.kind == kLossTraining || a.kind == kLossSsim) {
        require(a.H >= kWin && a.W >= kWin, "ssim: image smaller than the 11x11 window");
        const int sr = ssim_rows(a.L * a.C, a.H, a.W);
        const dim3 grid(ceil_div(a.W, kSO), ceil_div(a.H, sr), a.L * a.C);
        static const Win win = ssim_window_f32();
        require(a.tstats != nullptr, "ssim: target statistics missing");
        auto go = [&](void (*kern)(LossArgs, Win), size_t smem) {
            HS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            kern<<<grid, 2 * kSW, smem, st>>>(a, win);
        };
        const bool band = a.own0 > 0 || a.own1 < a.H;
        if (band) {
            require(a.field != nullptr, "ssim: row-band loss needs the complex field");
            go(ssim_kernel<true, true>(sr), sizeof(SsimSmem<float2>));
        } else if (a.field) {
            go(ssim_kernel<true, false>(sr), sizeof(SsimSmem<float2>));
        } else {
            go(ssim_kernel<false, false>(sr), sizeof(SsimSmem<float>));
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
    const double n_el = static_cast<double>(a.channels_norm()) * a.rows_norm() * a.W;
    const double count = static_cast<double>(a.L_norm) * a.channels_norm() * std::max(a.rows_norm() - kWin + 1, 0) *
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

void clip01_launch(const float* in, int64_t count, float* out, cudaStream_t st) {
    if (count == 0) return;
    clip01_kernel<<<grid_for(count, 256), 256, 0, st>>>(in, count, out);
    launch_check("clip01");
}

void intensity_launch(const float2* f, int64_t count, float* out, cudaStream_t st) {
    if (count == 0) return;
    intensity_kernel<<<grid_for(count, 256), 256, 0, st>>>(f, count, out);
    launch_check("intensity");
}

// float4 work items per thread of the fused Adan: a resident grid
// (kAdanMinBlocks CTAs per SM, grid-stride), no partial last wave
static unsigned adan_grid(int64_t items) {
    static const int sms = [] {
        int dev = 0;
        HS_CUDA(cudaGetDevice(&dev));
        return sm_count(dev);
    }();
    const int64_t b = (items + 255) / 256;
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(b, static_cast<int64_t>(sms) * kAdanMinBlocks)));
}

void adan_fused_launch(float* params, const float* grads, float* state, int64_t P,
                       const AdanGroups& g0, int total_steps, double b1, double b2, double b3,
                       double eps, int* d_step, const uint32_t* d_flags, cudaStream_t st, int64_t begin,
                       int64_t end) {
    // [begin, end): a rank's shard of the flat buffer (end < 0: all of it)
    if (end < 0) end = P;
    require(begin >= 0 && begin <= end && end <= P, "adan: update range outside the parameter buffer");
    const int64_t PS = P;
    const AdanGroups g = shift_groups(g0, begin, end);
    params += begin;
    grads += begin;
    state += begin;
    P = end - begin;
    bool vec = P % 4 == 0 && begin % 4 == 0 && PS % 4 == 0;
    for (int k = 0; k < 6; ++k) vec = vec && g.begin[k] % 4 == 0;
    // d_step holds {loop step, adan t, CTA done counter, pad, GroupConst[6]}
    unsigned* done = reinterpret_cast<unsigned*>(d_step + 2);
    GroupConst* kc = reinterpret_cast<GroupConst*>(d_step + 4);
    if (vec)
        adan_fused_kernel<true><<<adan_grid(P / 4), 256, 0, st>>>(params, grads, state, P, PS, g, total_steps, b1,
                                                                  b2, b3, eps, d_step, d_flags, done, kc);
    else
        adan_fused_kernel<false><<<grid_for(P, 256), 256, 0, st>>>(params, grads, state, P, PS, g, total_steps, b1,
                                                                   b2, b3, eps, d_step, d_flags, done, kc);
    launch_check("adan_fused");
}

void adan_init_consts(const AdanGroups& g, int total_steps, double b1, double b2, double b3, int* d_step,
                      cudaStream_t st) {
    adan_consts_kernel<<<1, 1, 0, st>>>(g, total_steps, b1, b2, b3, d_step, reinterpret_cast<GroupConst*>(d_step + 4));
    launch_check("adan_consts");
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

namespace {
// per-group non-finite bits of a flat gradient buffer (bit k: group k)
__global__ void group_nonfinite_kernel(const float* __restrict__ g, int64_t P, AdanGroups G, uint32_t* flags) {
    uint32_t bits = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (!isfinite(g[i])) {
            int gi = 0;
#pragma unroll
            for (int k = 1; k < 6; ++k) gi += (i >= G.begin[k]) ? 1 : 0;
            bits |= 1u << gi;
        }
    }
    bits = __reduce_or_sync(0xffffffffu, bits);
    if ((threadIdx.x & 31) == 0 && bits) atomicOr(flags, bits);
}
}  // namespace

AdanGroups shift_groups(const AdanGroups& G, int64_t begin, int64_t end) {
    AdanGroups s = G;
    for (int k = 0; k < 6; ++k) {
        s.begin[k] = std::min(std::max(G.begin[k], begin), end) - begin;
        s.end[k] = std::min(std::max(G.end[k], begin), end) - begin;
    }
    return s;
}

void group_nonfinite_launch(const float* g, int64_t P, const AdanGroups& G0, uint32_t* flags, cudaStream_t st,
                            int64_t begin, int64_t end) {
    if (end < 0) end = P;
    require(begin >= 0 && begin <= end && end <= P, "non-finite check: range outside the gradient buffer");
    const AdanGroups G = shift_groups(G0, begin, end);
    g += begin;
    P = end - begin;
    HS_CUDA(cudaMemsetAsync(flags, 0, sizeof(uint32_t), st));
    if (P == 0) return;
    group_nonfinite_kernel<<<grid_for(P, 256), 256, 0, st>>>(g, P, G, flags);
    launch_check("group_nonfinite");
}

void nonfinite_launch(const float* g, int64_t n, uint32_t* flag, cudaStream_t st) {
    if (n == 0) return;
    nonfinite_kernel<<<grid_for(n, 256), 256, 0, st>>>(g, n, flag);
    launch_check("nonfinite");
}

}  // namespace hs
