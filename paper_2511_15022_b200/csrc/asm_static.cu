// Compile-time planned angular-spectrum kernels for the benchmark grids.
//
// Same data path and numerics contract as asm.cu (propagation.cpp:135-243),
// with the FFT engine of fft_static.cuh: in-place stages, constant strides,
// first stages read straight from global memory (zero pad skipped), last
// stages write straight to global memory (crop skipped) or apply the transfer
// function H = exp(i kz d) in registers (Cody-Waite reduced fast sincos).
// The pruning assumes the centred pad of factor 2 (offset = padded length / 4),
// so these plans are only used when pad == 2.
//
// Plans (Px x Py, column tile width CC; radices with first and last % 4 == 0):
//   3840 x 2160, CC 4   cfg2/cfg3 (1920x1080, pad 2)
//    512 x  512, CC 4   cfg1 (256x256, pad 2)
//    512 x  320, CC 4   desk regression (256x160, pad 2)
//   7680 x 4320, CC 2   cfg4 (3840x2160, pad 2)
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "asm.cuh"
#include "fft_static.cuh"
#include "fft_pair.cuh"

namespace hs {

namespace {

using sfft::Radices;

// exp(i phase) of the transfer function with a 2-constant Cody-Waite
// reduction to [-pi, pi] before the MUFU sincos (|phase| <= ~200 rad here).
template <bool CONJ>
__device__ __forceinline__ float2 transfer_fast(const TfConst& t, int mx, int my) {
    if (abs(mx) > t.mx_max || abs(my) > t.my_max) return make_float2(0.f, 0.f);
    if (t.a4 > 0.0) {
        const long long ax = 2LL * mx + 1, ay = 2LL * my + 1;
        if (static_cast<double>(ax * ax + ay * ay) >= t.a4) return make_float2(0.f, 0.f);
    }
    const float fmx = static_cast<float>(mx), fmy = static_cast<float>(my);
    const float q = t.bx * fmx * fmx + t.by * fmy * fmy;
    // kz d = kd - kd * q / (1 + sqrt(1 - q)); for q < 1/32 the series
    // q/2 + q^2/8 + q^3/16 + 5q^4/128 + 7q^5/256 (truncation < 1e-9 rad here)
    // replaces the sqrt and the division.
    float ph = 0.f;
    if (q < 0.03125f) {
        const float ser = q * fmaf(q, fmaf(q, fmaf(q, fmaf(q, 0.02734375f, 0.0390625f), 0.0625f), 0.125f), 0.5f);
        ph = fmaf(-t.kd, ser, t.kd_mod);
    } else if (q < 1.f) {
        ph = t.kd_mod - t.kd * q / (1.f + sqrtf(1.f - q));
    }
    const float n = rintf(ph * 0.15915494309189535f);
    ph = fmaf(-n, 6.28318548202514648f, ph);      // 2pi rounded to fp32
    ph = fmaf(n, 1.7484555314695172e-7f, ph);     // + (fp32(2pi) - 2pi)
    float s, c;
    __sincosf(ph, &s, &c);
    return make_float2(c, CONJ ? -s : s);
}

// Row kernels: RB rows per CTA, interleaved in the engine (its CC = RB); a
// thread always serves row rr = tid % RB (NT % RB == 0), so its row pointers
// are computed once.  The forward reads only the W live inputs of each row
// (first stage pruned to the centred block) and writes the column-tiled T
// layout from the last stage; the inverse writes only the W cropped outputs.
template <int N, int RB, int NT, int CCO, class RAD>
__global__ void __launch_bounds__(NT) srows_fwd_kernel(RowArgs a, int nrows, const float2* __restrict__ tw) {
    static_assert(NT % RB == 0, "row of a thread must be fixed");
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int rho = blockIdx.x * RB + tid % RB;
    const bool ok = rho < nrows;
    const int pc = rho / a.H, y = rho - pc * a.H;
    const float2* src = a.in + static_cast<size_t>(rho) * a.W - a.ox;  // src[i], i in [ox, ox + W)
    float2* dst = a.out + (static_cast<size_t>(pc) * a.ntiles * a.H + y) * CCO;
    const size_t ts = static_cast<size_t>(a.H) * CCO;
    sfft::run<N, RB, NT, -1, sfft::Half, sfft::Full>(
        smem, tw, tid, RAD{},
        sfft::in_fn([&](int i, int) { return ok ? src[i] : make_float2(0.f, 0.f); }),
        sfft::out_fn([&](int i, int, float2 v) {
            if (ok) dst[static_cast<size_t>(i / CCO) * ts + (i % CCO)] = v;
        }));
}

// Inverse row pass gathering from the peer-major receive layout (SlabGet, asm.cuh).
template <int N, int RB, int NT, int CCO, class RAD>
__global__ void __launch_bounds__(NT) srows_inv_get_kernel(RowArgs a, int nrows, const float2* __restrict__ tw,
                                                           SlabGet sg) {
    static_assert(NT % RB == 0, "row of a thread must be fixed");
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int rho = blockIdx.x * RB + tid % RB;
    const bool ok = rho < nrows;
    const int pc = rho / a.H, y = rho - pc * a.H;
    const float2* src = a.in + (static_cast<size_t>(pc) * sg.ts * a.H + y) * CCO;
    const size_t tile_stride = static_cast<size_t>(a.H) * CCO;
    float2* dst = a.out + static_cast<size_t>(rho) * a.W - a.ox;  // dst[i], i in [ox, ox + W)
    const float sc = a.scale;
    sfft::run<N, RB, NT, +1, sfft::Full, sfft::Half>(
        smem, tw, tid, RAD{},
        sfft::in_fn([&](int i, int) {
            if (!ok) return make_float2(0.f, 0.f);
            const unsigned T = static_cast<unsigned>(i / CCO);
            unsigned r = __umulhi(T, sg.ts_magic);  // T / ts, corrected below
            if (r * sg.ts > T) --r;
            else if ((r + 1) * sg.ts <= T) ++r;
            return src[r * sg.per_src + (T - r * sg.ts) * tile_stride + (i % CCO)];
        }),
        sfft::out_fn([&](int i, int, float2 v) {
            if (ok) dst[i] = make_float2(v.x * sc, v.y * sc);
        }));
}

// Forward row pass with the peer-put epilogue (SlabPut, asm.cuh).
template <int N, int RB, int NT, int CCO, class RAD>
__global__ void __launch_bounds__(NT) srows_fwd_put_kernel(RowArgs a, int nrows, const float2* __restrict__ tw,
                                                           SlabPut sp) {
    static_assert(NT % RB == 0, "row of a thread must be fixed");
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int rho = blockIdx.x * RB + tid % RB;
    const int pc = rho / a.H, y = rho - pc * a.H;
    const int yo = y - sp.row0;
    const bool ok = rho < nrows, send = ok && yo >= 0 && yo < sp.hout;
    const float2* src = a.in + static_cast<size_t>(rho) * a.W - a.ox;  // src[i], i in [ox, ox + W)
    const size_t plane_rows = static_cast<size_t>(pc) * sp.ts;
    sfft::run<N, RB, NT, -1, sfft::Half, sfft::Full>(
        smem, tw, tid, RAD{},
        sfft::in_fn([&](int i, int) { return ok ? src[i] : make_float2(0.f, 0.f); }),
        sfft::out_fn([&](int i, int, float2 v) {
            if (!send) return;
            const unsigned T = static_cast<unsigned>(i / CCO);
            unsigned r = __umulhi(T, sp.ts_magic);  // T / ts, corrected below
            if (r * sp.ts > T) --r;
            else if ((r + 1) * sp.ts <= T) ++r;
            const size_t tl = T - r * sp.ts;
            sp.peer[r][sp.slot[r] + ((plane_rows + tl) * sp.hout + yo) * CCO + (i % CCO)] = v;
        }));
}

template <int N, int RB, int NT, int CCO, class RAD>
__global__ void __launch_bounds__(NT) srows_inv_kernel(RowArgs a, int nrows, const float2* __restrict__ tw) {
    static_assert(NT % RB == 0, "row of a thread must be fixed");
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int rho = blockIdx.x * RB + tid % RB;
    const bool ok = rho < nrows;
    const int pc = rho / a.H, y = rho - pc * a.H;
    const float2* src = a.in + (static_cast<size_t>(pc) * a.ntiles * a.H + y) * CCO;
    float2* dst = a.out + static_cast<size_t>(rho) * a.W - a.ox;  // dst[i], i in [ox, ox + W)
    const size_t ts = static_cast<size_t>(a.H) * CCO;
    const float sc = a.scale;
    sfft::run<N, RB, NT, +1, sfft::Full, sfft::Half>(
        smem, tw, tid, RAD{},
        sfft::in_fn([&](int i, int) {
            return ok ? src[static_cast<size_t>(i / CCO) * ts + (i % CCO)] : make_float2(0.f, 0.f);
        }),
        sfft::out_fn([&](int i, int, float2 v) {
            if (ok) dst[i] = make_float2(v.x * sc, v.y * sc);
        }));
}

// Column kernels: one CTA per CC-column tile of one channel.  The forward FFT
// reads the H live rows of the tile straight from T1, its last stage applies
// H(kx, ky) in registers, and the inverse's last stage writes only the H
// cropped rows to T2.  A thread always serves column cc = tid % CC.
template <int N, int CC, int NT, bool CONJ, class RAD>
__device__ __forceinline__ void col_single(const ColArgs& a, const float2* __restrict__ tw, int plane_in,
                                           int plane_out) {
    static_assert(NT % CC == 0, "column of a thread must be fixed");
    extern __shared__ float2 smem[];
    const int tile = blockIdx.x, c = blockIdx.y, tid = threadIdx.x;
    const size_t tile_elems = static_cast<size_t>(a.H) * CC;
    const size_t shift = static_cast<size_t>(a.oy) * CC;
    const float2* src = a.in + (static_cast<size_t>(plane_in) * a.ntiles + tile) * tile_elems - shift;
    float2* dst = a.out + (static_cast<size_t>(plane_out) * a.ntiles + tile) * tile_elems - shift;
    const TfConst t = a.tf[c];
    const int mx = wrapped((a.tile0 + tile) * CC + tid % CC, a.Px);
    sfft::run<N, CC, NT, -1, sfft::Half, sfft::Full>(
        smem, tw, tid, RAD{}, sfft::in_fn([&](int i, int cc) { return src[i * CC + cc]; }),
        sfft::out_smem(smem, [&](int i, int, float2 v, float2& slot) {
            slot = cmul(v, transfer_fast<CONJ>(t, mx, wrapped(i, N)));
        }));
    sfft::run<N, CC, NT, +1, sfft::Full, sfft::Half>(
        smem, tw, tid, RAD{}, sfft::in_smem(smem),
        sfft::out_fn([&](int i, int cc, float2 v) { dst[i * CC + cc] = v; }));
}

// H(kx, ky) for the two columns of a pair at once (packed fp32x2), with the
// same arithmetic as transfer_fast: q = bx mx^2 + by my^2, the series form of
// kz d for q < 1/32, 2-constant Cody-Waite, MUFU sincos.  Falls back to the
// scalar form when the aperture is on or a q of the pair is >= 1/32.
struct PairTf {
    float2 qx;       // (bx mx0^2, bx mx1^2)
    float2 inband;   // 1 / 0 per column of the |mx| band limit
    int mx0, mx1;
    bool simple;     // no aperture, every |my| in band, q < 1/32 down the whole column
};

// The pair's column constants; simple when every row takes the series branch
// (q grows with |my|, whose wrapped maximum is N/2).
template <int N>
__device__ __forceinline__ PairTf pair_tf(const TfConst& t, int mx0, int mx1) {
    PairTf p;
    p.mx0 = mx0;
    p.mx1 = mx1;
    const float f0 = static_cast<float>(mx0), f1 = static_cast<float>(mx1);
    p.qx = make_float2(t.bx * f0 * f0, t.bx * f1 * f1);
    p.inband = make_float2(abs(mx0) <= t.mx_max ? 1.f : 0.f, abs(mx1) <= t.mx_max ? 1.f : 0.f);
    const float fy = static_cast<float>(N / 2);
    const float2 qm = f2add(p.qx, f2splat(t.by * fy * fy));
    p.simple = !(t.a4 > 0.0) && t.my_max >= N / 2 && qm.x < 0.03125f && qm.y < 0.03125f;
    return p;
}
template <bool CONJ, bool SIMPLE = false>
__device__ __forceinline__ void transfer_pair(const TfConst& t, const PairTf& p, int my, float2& hc, float2& hs) {
    if (!SIMPLE && abs(my) > t.my_max) {
        hc = hs = make_float2(0.f, 0.f);
        return;
    }
    const float fmy = static_cast<float>(my);
    const float2 q = f2add(p.qx, f2splat(t.by * fmy * fmy));
    if (!SIMPLE && (t.a4 > 0.0 || q.x >= 0.03125f || q.y >= 0.03125f)) {
        const float2 h0 = transfer_fast<CONJ>(t, p.mx0, my), h1 = transfer_fast<CONJ>(t, p.mx1, my);
        hc = make_float2(h0.x, h1.x);
        hs = make_float2(h0.y, h1.y);
        return;
    }
    // ser = q/2 + q^2/8 + q^3/16 + 5q^4/128 + 7q^5/256
    float2 ser = f2fma(q, f2splat(0.02734375f), f2splat(0.0390625f));
    ser = f2fma(q, ser, f2splat(0.0625f));
    ser = f2fma(q, ser, f2splat(0.125f));
    ser = f2fma(q, ser, f2splat(0.5f));
    ser = f2mul(q, ser);
    float2 ph = f2fma(f2splat(-t.kd), ser, f2splat(t.kd_mod));
    const float2 nn = f2mul(ph, f2splat(0.15915494309189535f));
    const float2 n = make_float2(rintf(nn.x), rintf(nn.y));
    ph = f2fma(n, f2splat(-6.28318548202514648f), ph);  // 2pi rounded to fp32
    ph = f2fma(n, f2splat(1.7484555314695172e-7f), ph);  // + (fp32(2pi) - 2pi)
    float s0, c0, s1, c1;
    __sincosf(ph.x, &s0, &c0);
    __sincosf(ph.y, &s1, &c1);
    hc = f2mul(make_float2(c0, c1), p.inband);
    hs = f2mul(make_float2(CONJ ? -s0 : s0, CONJ ? -s1 : s1), p.inband);
}

// Column-pair SIMD variant of col_single (fft_pair.cuh): CC = 4 columns as two
// pairs, every thread transforms one butterfly of one pair.  The tile layout in
// global memory is the same [row][4] complex; a 16-byte load/store moves one
// pair's (re0, im0, re1, im1).
template <int N, int NT, bool CONJ, class RAD>
__device__ __forceinline__ void pcol_single(const ColArgs& a, const float2* __restrict__ tw, int plane) {
    constexpr int CC = 4, NP = 2;
    static_assert(NT % NP == 0, "pair of a thread must be fixed");
    extern __shared__ float4 smem4[];
    const int tile = blockIdx.x, c = blockIdx.y, tid = threadIdx.x;
    const size_t tile_elems = static_cast<size_t>(a.H) * CC;
    const size_t shift = static_cast<size_t>(a.oy) * CC;
    const float2* src = a.in + (static_cast<size_t>(plane) * a.ntiles + tile) * tile_elems - shift;
    float2* dst = a.out + (static_cast<size_t>(plane) * a.ntiles + tile) * tile_elems - shift;
    const TfConst t = a.tf[c];
    const int pp = tid % NP;
    const PairTf ptf = pair_tf<N>(t, wrapped((a.tile0 + tile) * CC + 2 * pp, a.Px),
                                  wrapped((a.tile0 + tile) * CC + 2 * pp + 1, a.Px));
    pfft::run<N, NP, NT, -1, pfft::Half, pfft::Full>(
        smem4, tw, tid, RAD{},
        pfft::in_fn([&](int i, int p) {
            const float4 q = *reinterpret_cast<const float4*>(src + static_cast<size_t>(i) * CC + 2 * p);
            return pfft::C2{make_float2(q.x, q.z), make_float2(q.y, q.w)};
        }),
        pfft::out_map([&](int i, int, pfft::C2 v) {
            float2 hc, hs;
            if (ptf.simple) transfer_pair<CONJ, true>(t, ptf, wrapped(i, N), hc, hs);
            else transfer_pair<CONJ>(t, ptf, wrapped(i, N), hc, hs);
            // (re + i im)(hc + i hs) per column
            return pfft::C2{f2sub(f2mul(v.re, hc), f2mul(v.im, hs)), f2fma(v.im, hc, f2mul(v.re, hs))};
        }));
    pfft::run<N, NP, NT, +1, pfft::Full, pfft::Half>(
        smem4, tw, tid, RAD{}, pfft::InSmem{},
        pfft::out_fn([&](int i, int p, pfft::C2 v) {
            *reinterpret_cast<float4*>(dst + static_cast<size_t>(i) * CC + 2 * p) =
                make_float4(v.re.x, v.im.x, v.re.y, v.im.y);
        }));
}

// ---- column-pair kernel with the tile staged by a TMA bulk copy ----
// The H live rows of a tile are one contiguous run of H * CC complex in the T
// layout, so ONE cp.async.bulk (mbarrier completion) stages it in shared
// memory and the forward FFT's first stage reads shared memory (no per-thread
// global loads).  With KT > 1 tiles per CTA the next tile is prefetched while
// the current tile's inverse FFT runs.
// tiles per CTA of the staged column kernels; measured at cfg2 (us per pass):
// 1 -> 152 (the plain kernel: 154), 2 (prefetch of the second tile overlapping
// the first tile's inverse FFT) -> 160: the global loads were not the limiter.
constexpr int kPersistTiles = 1;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra.uni WAIT_%=;\n}\n"
        ::"r"(smem_u32(bar)), "r"(parity));
}

// One tile of the prefetching column kernel: wait for its staged rows, forward
// FFT from shared memory x H, prefetch tile tn into the staging buffer, inverse
// FFT to global (cropped rows).
template <int N, int NT, bool CONJ, class RAD>
__device__ __forceinline__ void pcol_tile(float4* work, float4* stage_buf, uint64_t* bar, unsigned parity,
                                          const float2* __restrict__ tw, TfConst tf, int t, int tn, int total,
                                          int ntiles, int tile0, int Px, int oy, const float2* gin, float2* gout,
                                          size_t tile_elems, unsigned bytes) {
    constexpr int CC = 4, NP = 2;
    const int tid = threadIdx.x, pp = tid % NP;
    const int tile = t % ntiles;
    const PairTf ptf = pair_tf<N>(tf, wrapped((tile0 + tile) * CC + 2 * pp, Px),
                                  wrapped((tile0 + tile) * CC + 2 * pp + 1, Px));
    mbar_wait(bar, parity);
    const float4* stg = stage_buf - oy * NP;  // row i of the padded column
    pfft::run<N, NP, NT, -1, pfft::Half, pfft::Full>(
        work, tw, tid, RAD{},
        pfft::in_fn([stg](int i, int p) {
            const float4 q = stg[i * NP + p];
            return pfft::C2{make_float2(q.x, q.z), make_float2(q.y, q.w)};
        }),
        pfft::out_map([tf, ptf](int i, int, pfft::C2 v) {
            float2 hc, hs;
            if (ptf.simple) transfer_pair<CONJ, true>(tf, ptf, wrapped(i, N), hc, hs);
            else transfer_pair<CONJ>(tf, ptf, wrapped(i, N), hc, hs);
            return pfft::C2{f2sub(f2mul(v.re, hc), f2mul(v.im, hs)), f2fma(v.im, hc, f2mul(v.re, hs))};
        }));
    // the staging buffer is free (the forward FFT ended with a barrier): prefetch tile tn
    if (tid == 0 && tn < total) bulk_load(stage_buf, gin + static_cast<size_t>(tn) * tile_elems, bytes, bar);
    float2* dst = gout + static_cast<size_t>(t) * tile_elems - static_cast<size_t>(oy) * CC;
    pfft::run<N, NP, NT, +1, pfft::Full, pfft::Half>(
        work, tw, tid, RAD{}, pfft::InSmem{},
        pfft::out_fn([dst](int i, int p, pfft::C2 v) {
            *reinterpret_cast<float4*>(dst + static_cast<size_t>(i) * CC + 2 * p) =
                make_float4(v.re.x, v.im.x, v.re.y, v.im.y);
        }));
}

template <int N, int NT, bool CONJ, class RAD, int KT>
__device__ __forceinline__ void pcol_persist(const ColArgs& a, const float2* __restrict__ tw) {
    constexpr int CC = 4, NP = 2;
    static_assert(NT % NP == 0, "pair of a thread must be fixed");
    static_assert(KT >= 1 && KT <= 3, "tiles per CTA");
    extern __shared__ float4 smem4[];
    float4* work = smem4;
    const int H = a.H, oy = a.oy, ntiles = a.ntiles, Px = a.Px, tile0 = a.tile0;
    const int total = ntiles * a.C;
    float4* stage_buf = smem4 + pfft::padded_len4(N * NP);  // H rows x 2 pairs
    uint64_t* bar = reinterpret_cast<uint64_t*>(stage_buf + H * NP);
    const size_t tile_elems = static_cast<size_t>(H) * CC;
    const unsigned bytes = static_cast<unsigned>(tile_elems * sizeof(float2));
    const int G = gridDim.x;
    const int t0 = blockIdx.x;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        if (t0 < total) bulk_load(stage_buf, a.in + static_cast<size_t>(t0) * tile_elems, bytes, bar);
    }
    __syncthreads();
    // KT tiles per CTA (t0, t0 + G, ...) in straight-line code
    if (t0 < total)
        pcol_tile<N, NT, CONJ, RAD>(work, stage_buf, bar, 0u, tw, a.tf[t0 / ntiles], t0, KT >= 2 ? t0 + G : total,
                                    total, ntiles, tile0, Px, oy, a.in, a.out, tile_elems, bytes);
    if constexpr (KT >= 2) {
        const int t1 = t0 + G;
        __syncthreads();  // work buffer reuse
        if (t1 < total)
            pcol_tile<N, NT, CONJ, RAD>(work, stage_buf, bar, 1u, tw, a.tf[t1 / ntiles], t1, KT >= 3 ? t1 + G : total,
                                        total, ntiles, tile0, Px, oy, a.in, a.out, tile_elems, bytes);
    }
    if constexpr (KT >= 3) {
        const int t2 = t0 + 2 * G;
        __syncthreads();
        if (t2 < total)
            pcol_tile<N, NT, CONJ, RAD>(work, stage_buf, bar, 0u, tw, a.tf[t2 / ntiles], t2, total, total, ntiles,
                                        tile0, Px, oy, a.in, a.out, tile_elems, bytes);
    }
}

// ---- row-slab column kernel: segment gather in, peer put (or local) out ----
__device__ __forceinline__ void bulk_expect(uint64_t* bar, unsigned bytes) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Peer table of a row-slab column kernel, staged in shared memory at entry:
// the output rows of a thread go to different peers, and indexing the
// SlabCol kernel parameter by a per-thread peer number would serialise on the
// constant cache.
struct PeerEnt {
    float2* base;  // peer receive buffer + this rank's slot
    int g0, he;    // canvas rows [g0, g0 + he) the peer receives
};
__device__ __forceinline__ void load_peers(const SlabCol& sc, PeerEnt* tab) {
    if (static_cast<int>(threadIdx.x) < sc.R)
        tab[threadIdx.x] = PeerEnt{sc.peer[threadIdx.x] + sc.slot[threadIdx.x], sc.g0[threadIdx.x], sc.he[threadIdx.x]};
}
// Store of one element (float2, or a float4 column pair) of cropped output row
// y: into every peer whose row range holds y (the slab of y, plus a
// neighbour's loss band for halo rows), or into the local column-side layout.
template <class T>
__device__ __forceinline__ void slab_store(const SlabCol& sc, const PeerEnt* tab, float2* lout, size_t plane_tiles,
                                           int y, int CC, int off, T v) {
    if (!sc.put) {
        *reinterpret_cast<T*>(lout + static_cast<size_t>(y) * CC + off) = v;
        return;
    }
    const int d0 = __float2int_rz(static_cast<float>(y) * sc.inv_hr);
#pragma unroll
    for (int dd = -1; dd <= 1; ++dd) {
        const int d = d0 + dd;
        if (d < 0 || d >= sc.R) continue;
        const PeerEnt e = tab[d];
        const int yl = y - e.g0;
        if (yl < 0 || yl >= e.he) continue;
        *reinterpret_cast<T*>(e.base + (plane_tiles * e.he + yl) * CC + off) = v;
    }
}

template <int N, int NT, int MINB, bool CONJ, class RAD>
__global__ void __launch_bounds__(NT, MINB) pcols_slab_kernel(ColArgs a, const float2* __restrict__ tw, SlabCol sc) {
    constexpr int CC = 4, NP = 2;
    extern __shared__ float4 smem4[];
    __shared__ PeerEnt peers[kMaxPeers];
    float4* work = smem4;
    const int H = a.H, oy = a.oy, ts = a.ntiles;
    float4* stage_buf = smem4 + pfft::padded_len4(N * NP);
    uint64_t* bar = reinterpret_cast<uint64_t*>(stage_buf + H * NP);
    const int t = blockIdx.x;            // flat tile over (channel, own tile)
    const int c = t / ts, tl = t - c * ts;
    const int tid = threadIdx.x, pp = tid % NP;
    if (tid == 0) {
        mbar_init(bar, 1);
        const unsigned seg = static_cast<unsigned>(sc.hr * CC * sizeof(float2));
        bulk_expect(bar, seg * sc.R);
        for (int r = 0; r < sc.R; ++r)  // source r's rows [r hr, (r + 1) hr) of this tile
            bulk_copy(stage_buf + r * sc.hr * NP, sc.in + r * sc.per_src + static_cast<size_t>(t) * sc.hr * CC, seg, bar);
    }
    load_peers(sc, peers);
    __syncthreads();
    const TfConst tf = a.tf[c];
    const PairTf ptf = pair_tf<N>(tf, wrapped((a.tile0 + tl) * CC + 2 * pp, a.Px),
                                  wrapped((a.tile0 + tl) * CC + 2 * pp + 1, a.Px));
    mbar_wait(bar, 0u);
    const float4* stg = stage_buf - oy * NP;
    pfft::run<N, NP, NT, -1, pfft::Half, pfft::Full>(
        work, tw, tid, RAD{},
        pfft::in_fn([stg](int i, int p) {
            const float4 q = stg[i * NP + p];
            return pfft::C2{make_float2(q.x, q.z), make_float2(q.y, q.w)};
        }),
        pfft::out_map([tf, ptf](int i, int, pfft::C2 v) {
            float2 hc, hs;
            if (ptf.simple) transfer_pair<CONJ, true>(tf, ptf, wrapped(i, N), hc, hs);
            else transfer_pair<CONJ>(tf, ptf, wrapped(i, N), hc, hs);
            return pfft::C2{f2sub(f2mul(v.re, hc), f2mul(v.im, hs)), f2fma(v.im, hc, f2mul(v.re, hs))};
        }));
    float2* lout = a.out + static_cast<size_t>(t) * H * CC;
    const size_t plane_tiles = static_cast<size_t>(c) * ts + tl;
    pfft::run<N, NP, NT, +1, pfft::Full, pfft::Half>(
        work, tw, tid, RAD{}, pfft::InSmem{},
        pfft::out_fn([&](int i, int p, pfft::C2 v) {
            slab_store(sc, peers, lout, plane_tiles, i - oy, CC, 2 * p, make_float4(v.re.x, v.im.x, v.re.y, v.im.y));
        }));
}

// Row-slab column kernel on the scalar engine (plans without the pair engine,
// e.g. the 4K CC 2 plan): the same segment gather in (R TMA bulk copies) and
// peer put (or local) out as pcols_slab_kernel.
template <int N, int CC, int NT, int MINB, bool CONJ, class RAD>
__global__ void __launch_bounds__(NT, MINB) scols_slab_kernel(ColArgs a, const float2* __restrict__ tw, SlabCol sc) {
    static_assert(NT % CC == 0, "column of a thread must be fixed");
    extern __shared__ float2 smem[];
    __shared__ PeerEnt peers[kMaxPeers];
    float2* work = smem;
    const int H = a.H, oy = a.oy, ts = a.ntiles;
    float2* stage_buf = smem + fft::padded_len(N * CC);
    uint64_t* bar = reinterpret_cast<uint64_t*>(stage_buf + H * CC);
    const int t = blockIdx.x;  // flat tile over (channel, own tile)
    const int c = t / ts, tl = t - c * ts;
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bar, 1);
        const unsigned seg = static_cast<unsigned>(sc.hr * CC * sizeof(float2));
        bulk_expect(bar, seg * sc.R);
        for (int r = 0; r < sc.R; ++r)
            bulk_copy(stage_buf + r * sc.hr * CC, sc.in + r * sc.per_src + static_cast<size_t>(t) * sc.hr * CC, seg, bar);
    }
    load_peers(sc, peers);
    __syncthreads();
    const TfConst tf = a.tf[c];
    const int mx = wrapped((a.tile0 + tl) * CC + tid % CC, a.Px);
    mbar_wait(bar, 0u);
    const float2* stg = stage_buf - oy * CC;
    sfft::run<N, CC, NT, -1, sfft::Half, sfft::Full>(
        work, tw, tid, RAD{}, sfft::in_fn([&](int i, int cc) { return stg[i * CC + cc]; }),
        sfft::out_smem(work, [&](int i, int, float2 v, float2& slot) {
            slot = cmul(v, transfer_fast<CONJ>(tf, mx, wrapped(i, N)));
        }));
    float2* lout = a.out + static_cast<size_t>(t) * H * CC;
    const size_t plane_tiles = static_cast<size_t>(c) * ts + tl;
    sfft::run<N, CC, NT, +1, sfft::Full, sfft::Half>(
        work, tw, tid, RAD{}, sfft::in_smem(work),
        sfft::out_fn([&](int i, int cc, float2 v) { slab_store(sc, peers, lout, plane_tiles, i - oy, CC, cc, v); }));
}

// Multi-plane row-slab column kernels (scalar engine, one CTA per (channel,
// own tile)): the exchange is fused at both ends as in scols_slab_kernel.
// Forward: gather the tile's H rows from the R source segments (R TMA bulk
// copies on one mbarrier), one forward FFT into the spectrum buffer, then per
// plane l the inverse FFT of H_l x spectrum stores its cropped rows straight
// into the loss bands of the peers (plane l C + c of the exchange layout).
template <int N, int CC, int NT, bool CONJ, class RAD>
__global__ void __launch_bounds__(NT, 1) scols_fwdL_slab_kernel(ColArgs a, const float2* __restrict__ tw, SlabCol sc) {
    static_assert(NT % CC == 0, "column of a thread must be fixed");
    extern __shared__ float2 smem[];
    __shared__ PeerEnt peers[kMaxPeers];
    float2* A = smem;
    float2* Sp = smem + fft::padded_len(N * CC);
    float2* stage_buf = Sp + fft::padded_len(N * CC);
    const int H = a.H, oy = a.oy, ts = a.ntiles;
    uint64_t* bar = reinterpret_cast<uint64_t*>(stage_buf + H * CC);
    const int t = blockIdx.x;  // flat tile over (channel, own tile)
    const int c = t / ts, tl = t - c * ts;
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bar, 1);
        const unsigned seg = static_cast<unsigned>(sc.hr * CC * sizeof(float2));
        bulk_expect(bar, seg * sc.R);
        for (int r = 0; r < sc.R; ++r)
            bulk_copy(stage_buf + r * sc.hr * CC, sc.in + r * sc.per_src + static_cast<size_t>(t) * sc.hr * CC, seg, bar);
    }
    load_peers(sc, peers);
    __syncthreads();
    const int mx = wrapped((a.tile0 + tl) * CC + tid % CC, a.Px);
    mbar_wait(bar, 0u);
    const float2* stg = stage_buf - oy * CC;
    sfft::run<N, CC, NT, -1, sfft::Half, sfft::Full>(
        Sp, tw, tid, RAD{}, sfft::in_fn([&](int i, int cc) { return stg[i * CC + cc]; }), sfft::out_smem(Sp));
#pragma unroll 1
    for (int l = 0; l < a.L; ++l) {
        const TfConst tf = a.tf[l * a.C + c];
        const size_t plane_tiles = (static_cast<size_t>(l) * a.C + c) * ts + tl;
        float2* lout = a.out + plane_tiles * H * CC;
        sfft::run<N, CC, NT, +1, sfft::Full, sfft::Half>(
            A, sfft::launder(tw), sfft::launder(tid), RAD{},
            sfft::in_smem(Sp, [&](int i, int, float2 v) { return cmul(v, transfer_fast<CONJ>(tf, mx, wrapped(i, N))); }),
            sfft::out_fn([&](int i, int cc, float2 v) { slab_store(sc, peers, lout, plane_tiles, i - oy, CC, cc, v); }));
    }
}

// Adjoint: per plane l, the tile's rows of plane l C + c arrive from the R
// source segments (double-buffered: plane l + 1 is copied while plane l is
// transformed); each plane's forward FFT accumulates conj(H_l) x spectrum from
// its last stage; one inverse FFT stores the own-slab rows into the peers.
template <int N, int CC, int NT, class RAD>
__global__ void __launch_bounds__(NT, 1) scols_bwdL_slab_kernel(ColArgs a, const float2* __restrict__ tw, SlabCol sc) {
    static_assert(NT % CC == 0, "column of a thread must be fixed");
    extern __shared__ float2 smem[];
    __shared__ PeerEnt peers[kMaxPeers];
    float2* A = smem;
    float2* Z = smem + fft::padded_len(N * CC);
    const int H = a.H, oy = a.oy, ts = a.ntiles;
    float2* stage0 = Z + fft::padded_len(N * CC);
    uint64_t* bar = reinterpret_cast<uint64_t*>(stage0 + 2 * H * CC);  // bar[0], bar[1]
    const int t = blockIdx.x;  // flat tile over (channel, own tile)
    const int c = t / ts, tl = t - c * ts;
    const int tid = threadIdx.x;
    const unsigned seg = static_cast<unsigned>(sc.hr * CC * sizeof(float2));
    auto fetch = [&](int l) {  // thread 0: plane l's segments -> stage buffer l & 1
        float2* dst = stage0 + (l & 1) * H * CC;
        const size_t p = (static_cast<size_t>(l) * a.C + c) * ts + tl;
        bulk_expect(bar + (l & 1), seg * sc.R);
        for (int r = 0; r < sc.R; ++r)
            bulk_copy(dst + r * sc.hr * CC, sc.in + r * sc.per_src + p * sc.hr * CC, seg, bar + (l & 1));
    };
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fetch(0);
    }
    load_peers(sc, peers);
    __syncthreads();
    const int mx = wrapped((a.tile0 + tl) * CC + tid % CC, a.Px);
#pragma unroll 1
    for (int l = 0; l < a.L; ++l) {
        // the other buffer was last read by plane l - 1, whose FFT ended with a barrier
        if (tid == 0 && l + 1 < a.L) fetch(l + 1);
        mbar_wait(bar + (l & 1), static_cast<unsigned>((l >> 1) & 1));
        const TfConst tf = a.tf[l * a.C + c];
        const float2* stg = sfft::launder(stage0 + (l & 1) * H * CC) - oy * CC;
        const bool first = l == 0;
        sfft::run<N, CC, NT, -1, sfft::Half, sfft::Full>(
            A, sfft::launder(tw), sfft::launder(tid), RAD{}, sfft::in_fn([&](int i, int cc) { return stg[i * CC + cc]; }),
            sfft::out_smem(Z, [&](int i, int, float2 v, float2& slot) {
                const float2 w = cmul(v, transfer_fast<true>(tf, mx, wrapped(i, N)));
                slot = first ? w : cadd(slot, w);
            }));
    }
    const size_t plane_tiles = static_cast<size_t>(c) * ts + tl;
    float2* lout = a.out + plane_tiles * H * CC;
    sfft::run<N, CC, NT, +1, sfft::Full, sfft::Half>(
        Z, tw, tid, RAD{}, sfft::in_smem(Z),
        sfft::out_fn([&](int i, int cc, float2 v) { slab_store(sc, peers, lout, plane_tiles, i - oy, CC, cc, v); }));
}

template <int N, int NT, int MINB, class RAD>
__global__ void __launch_bounds__(NT, MINB) pcols_fwdP_kernel(ColArgs a, const float2* __restrict__ tw) {
    pcol_persist<N, NT, false, RAD, kPersistTiles>(a, tw);
}
template <int N, int NT, int MINB, class RAD>
__global__ void __launch_bounds__(NT, MINB) pcols_bwdP_kernel(ColArgs a, const float2* __restrict__ tw) {
    pcol_persist<N, NT, true, RAD, kPersistTiles>(a, tw);
}

template <int N, int NT, int MINB, class RAD>
__global__ void __launch_bounds__(NT, MINB) pcols_fwd1_kernel(ColArgs a, const float2* __restrict__ tw) {
    pcol_single<N, NT, false, RAD>(a, tw, blockIdx.y);
}

template <int N, int NT, int MINB, class RAD>
__global__ void __launch_bounds__(NT, MINB) pcols_bwd1_kernel(ColArgs a, const float2* __restrict__ tw) {
    pcol_single<N, NT, true, RAD>(a, tw, blockIdx.y);
}

// Single plane (the benchmark case).
template <int N, int CC, int NT, int MINB, class RAD>
__global__ void __launch_bounds__(NT, MINB) scols_fwd1_kernel(ColArgs a, const float2* __restrict__ tw) {
    col_single<N, CC, NT, false, RAD>(a, tw, blockIdx.y, blockIdx.y);
}

template <int N, int CC, int NT, int MINB, class RAD>
__global__ void __launch_bounds__(NT, MINB) scols_bwd1_kernel(ColArgs a, const float2* __restrict__ tw) {
    col_single<N, CC, NT, true, RAD>(a, tw, blockIdx.y, blockIdx.y);
}

// Multi-plane: one forward FFT per tile shared by all planes (spectrum kept in
// a second shared buffer; each plane's inverse reads it through H_l); the
// adjoint accumulates every plane's conj(H_l)-weighted spectrum straight from
// its FFT's last stage before one inverse FFT (propagate_multi_backward propagation.cpp:214-243).
template <int N, int CC, int NT, int MINB, class RAD>
__global__ void __launch_bounds__(NT, MINB) scols_fwdL_kernel(ColArgs a, const float2* __restrict__ tw) {
    static_assert(NT % CC == 0, "column of a thread must be fixed");
    extern __shared__ float2 smem[];
    float2* A = smem;
    float2* Sp = smem + fft::padded_len(N * CC);
    const int tile = blockIdx.x, c = blockIdx.y, tid = threadIdx.x;
    const size_t tile_elems = static_cast<size_t>(a.H) * CC;
    const size_t shift = static_cast<size_t>(a.oy) * CC;
    const float2* src = a.in + (static_cast<size_t>(c) * a.ntiles + tile) * tile_elems - shift;
    const int mx = wrapped((a.tile0 + tile) * CC + tid % CC, a.Px);
    sfft::run<N, CC, NT, -1, sfft::Half, sfft::Full>(
        Sp, tw, tid, RAD{}, sfft::in_fn([&](int i, int cc) { return src[i * CC + cc]; }), sfft::out_smem(Sp));
#pragma unroll 1
    for (int l = 0; l < a.L; ++l) {
        const TfConst t = a.tf[l * a.C + c];
        float2* dst = a.out + ((static_cast<size_t>(l) * a.C + c) * a.ntiles + tile) * tile_elems - shift;
        sfft::run<N, CC, NT, +1, sfft::Full, sfft::Half>(
            A, sfft::launder(tw), sfft::launder(tid), RAD{},
            sfft::in_smem(Sp, [&](int i, int, float2 v) { return cmul(v, transfer_fast<false>(t, mx, wrapped(i, N))); }),
            sfft::out_fn([&](int i, int cc, float2 v) { dst[i * CC + cc] = v; }));
    }
}

template <int N, int CC, int NT, int MINB, class RAD>
__global__ void __launch_bounds__(NT, MINB) scols_bwdL_kernel(ColArgs a, const float2* __restrict__ tw) {
    static_assert(NT % CC == 0, "column of a thread must be fixed");
    extern __shared__ float2 smem[];
    float2* A = smem;
    float2* Z = smem + fft::padded_len(N * CC);
    const int tile = blockIdx.x, c = blockIdx.y, tid = threadIdx.x;
    const size_t tile_elems = static_cast<size_t>(a.H) * CC;
    const size_t shift = static_cast<size_t>(a.oy) * CC;
    const int mx = wrapped((a.tile0 + tile) * CC + tid % CC, a.Px);
#pragma unroll 1
    for (int l = 0; l < a.L; ++l) {
        const TfConst t = a.tf[l * a.C + c];
        const float2* src = a.in + ((static_cast<size_t>(l) * a.C + c) * a.ntiles + tile) * tile_elems - shift;
        const bool first = l == 0;
        sfft::run<N, CC, NT, -1, sfft::Half, sfft::Full>(
            A, sfft::launder(tw), sfft::launder(tid), RAD{}, sfft::in_fn([&](int i, int cc) { return src[i * CC + cc]; }),
            sfft::out_smem(Z, [&](int i, int, float2 v, float2& slot) {
                const float2 w = cmul(v, transfer_fast<true>(t, mx, wrapped(i, N)));
                slot = first ? w : cadd(slot, w);
            }));
    }
    float2* dst = a.out + (static_cast<size_t>(c) * a.ntiles + tile) * tile_elems - shift;
    sfft::run<N, CC, NT, +1, sfft::Full, sfft::Half>(
        Z, tw, tid, RAD{}, sfft::in_smem(Z), sfft::out_fn([&](int i, int cc, float2 v) { dst[i * CC + cc] = v; }));
}

// ---- plan table -------------------------------------------------------------------------------
struct RowPlan {
    void (*fwd)(RowArgs, int, const float2*);
    void (*inv)(RowArgs, int, const float2*);
    int nt, rb;
    std::vector<float2> (*table)(int);
    void (*fwd_put)(RowArgs, int, const float2*, SlabPut) = nullptr;
    void (*inv_get)(RowArgs, int, const float2*, SlabGet) = nullptr;
};
struct ColPlan {
    void (*fwd)(ColArgs, const float2*);
    void (*bwd)(ColArgs, const float2*);
    void (*fwdL)(ColArgs, const float2*);
    void (*bwdL)(ColArgs, const float2*);
    int nt, cc;
    std::vector<float2> (*table)(int);
    int nt1 = 0;        // threads of the single-plane kernels (0: nt)
    bool pair = false;  // single-plane kernels use the column-pair SIMD engine (float4 smem)
    void (*fwdS)(ColArgs, const float2*, SlabCol) = nullptr;  // row-slab column kernels
    void (*bwdS)(ColArgs, const float2*, SlabCol) = nullptr;
    void (*fwdSL)(ColArgs, const float2*, SlabCol) = nullptr;  // multi-plane row-slab column kernels
    void (*bwdSL)(ColArgs, const float2*, SlabCol) = nullptr;
    void (*fwdP)(ColArgs, const float2*) = nullptr;  // bulk-copy staged single-plane kernels
    void (*bwdP)(ColArgs, const float2*) = nullptr;
};

template <int N, int RB, int NT, int CCO, class RAD>
RowPlan row_plan() {
    return RowPlan{srows_fwd_kernel<N, RB, NT, CCO, RAD>, srows_inv_kernel<N, RB, NT, CCO, RAD>, NT, RB,
                   [](int n) { return sfft::twiddle_table(n, RAD{}); }, srows_fwd_put_kernel<N, RB, NT, CCO, RAD>,
                   srows_inv_get_kernel<N, RB, NT, CCO, RAD>};
}
// Column-pair SIMD single-plane kernels (CC = 4), standard multi-plane kernels.
template <int N, int NT1, int MINB1, int NTL, class RAD>
ColPlan pcol_plan() {
    ColPlan p{pcols_fwd1_kernel<N, NT1, MINB1, RAD>, pcols_bwd1_kernel<N, NT1, MINB1, RAD>,
              scols_fwdL_kernel<N, 4, NTL, 1, RAD>, scols_bwdL_kernel<N, 4, NTL, 1, RAD>, NTL, 4,
              [](int n) { return sfft::twiddle_table(n, RAD{}); }};
    p.nt1 = NT1;
    p.pair = true;
    p.fwdP = pcols_fwdP_kernel<N, NT1, MINB1, RAD>;
    p.bwdP = pcols_bwdP_kernel<N, NT1, MINB1, RAD>;
    p.fwdS = pcols_slab_kernel<N, NT1, MINB1, false, RAD>;
    p.bwdS = pcols_slab_kernel<N, NT1, MINB1, true, RAD>;
    p.fwdSL = scols_fwdL_slab_kernel<N, 4, NTL, false, RAD>;
    p.bwdSL = scols_bwdL_slab_kernel<N, 4, NTL, RAD>;
    return p;
}

// The multi-plane kernels hold two tiles in shared memory (spectrum + work),
// so they run one CTA per SM regardless of MINB: they get the full register file.
template <int N, int CC, int NT, int MINB, class RAD>
ColPlan col_plan() {
    ColPlan p{scols_fwd1_kernel<N, CC, NT, MINB, RAD>, scols_bwd1_kernel<N, CC, NT, MINB, RAD>,
              scols_fwdL_kernel<N, CC, NT, 1, RAD>, scols_bwdL_kernel<N, CC, NT, 1, RAD>, NT, CC,
              [](int n) { return sfft::twiddle_table(n, RAD{}); }};
    p.fwdS = scols_slab_kernel<N, CC, NT, MINB, false, RAD>;
    p.bwdS = scols_slab_kernel<N, CC, NT, MINB, true, RAD>;
    p.fwdSL = scols_fwdL_slab_kernel<N, CC, NT, false, RAD>;
    p.bwdSL = scols_bwdL_slab_kernel<N, CC, NT, RAD>;
    return p;
}

struct Plans {
    int Px, Py, cc;
    RowPlan row;
    ColPlan col;
};

const std::vector<Plans>& plans() {
    static const std::vector<Plans> p = {
        {3840, 2160, 4, row_plan<3840, 1, 256, 4, Radices<16, 15, 16>>(),
         pcol_plan<2160, 360, 2, 720, Radices<12, 15, 12>>()},
        {512, 512, 4, row_plan<512, 1, 64, 4, Radices<8, 8, 8>>(), col_plan<512, 4, 128, 2, Radices<8, 8, 8>>()},
        {512, 320, 4, row_plan<512, 1, 64, 4, Radices<8, 8, 8>>(), col_plan<320, 4, 128, 2, Radices<16, 20>>()},
        {7680, 4320, 2, row_plan<7680, 2, 512, 2, Radices<16, 30, 16>>(),
         col_plan<4320, 2, 360, 2, Radices<12, 30, 12>>()},
    };
    return p;
}

const Plans* find(int Px, int Py) {
    for (const auto& p : plans())
        if (p.Px == Px && p.Py == Py) return &p;
    return nullptr;
}

struct STwCache {
    std::mutex mu;
    std::map<std::tuple<int, int, int>, float2*> t;  // (device, plan index, axis)
};
STwCache g_stw;

const float2* stable(int plan_idx, int axis, const std::vector<float2>& h) {
    int dev = 0;
    HS_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_stw.mu);
    auto key = std::make_tuple(dev, plan_idx, axis);
    auto it = g_stw.t.find(key);
    if (it != g_stw.t.end()) return it->second;
    float2* d = nullptr;
    HS_CUDA(cudaMalloc(&d, sizeof(float2) * h.size()));
    HS_CUDA(cudaMemcpy(d, h.data(), sizeof(float2) * h.size(), cudaMemcpyHostToDevice));
    g_stw.t[key] = d;
    return d;
}

size_t rows_smem(const Plans& p) { return sizeof(float2) * fft::padded_len(p.Px * p.row.rb); }
size_t cols_smem(const Plans& p, int L) {
    if (L == 1 && p.col.pair) return sizeof(float4) * pfft::padded_len4(p.Py * p.col.cc / 2);
    return sizeof(float2) * fft::padded_len(p.Py * p.col.cc) * (L > 1 ? 2 : 1);
}
int cols_threads(const Plans& p, int L) { return (L == 1 && p.col.nt1) ? p.col.nt1 : p.col.nt; }

// multi-plane slab kernels: work + spectrum buffers, one (forward) or two
// (adjoint) staging buffers of H rows, mbarriers
size_t cols_smem_slabL(const Plans& p, int H, bool backward) {
    return sizeof(float2) * (2 * static_cast<size_t>(fft::padded_len(p.Py * p.col.cc)) +
                             (backward ? 2 : 1) * static_cast<size_t>(H) * p.col.cc) + 16;
}

size_t cols_smem_persist(const Plans& p, int H) {
    return cols_smem(p, 1) + sizeof(float2) * static_cast<size_t>(H) * p.col.cc + 16;
}

// Column pass launch: the staged kernels for a single plane when the plan has
// them (KT tiles per CTA), else one CTA per (tile, channel).
void launch_cols(const Plans* p, const AsmWork& w, bool backward, const ColArgs& c, cudaStream_t st) {
    if (w.L == 1 && p->col.fwdP) {
        const int total = c.ntiles * c.C;
        const int grid = (total + kPersistTiles - 1) / kPersistTiles;
        (backward ? p->col.bwdP : p->col.fwdP)<<<grid, p->col.nt1, cols_smem_persist(*p, w.H), st>>>(c, w.stw_y);
    } else {
        const size_t cs = cols_smem(*p, w.L);
        auto k = backward ? (w.L > 1 ? p->col.bwdL : p->col.bwd) : (w.L > 1 ? p->col.fwdL : p->col.fwd);
        k<<<dim3(c.ntiles, c.C), cols_threads(*p, w.L), cs, st>>>(c, w.stw_y);
    }
    launch_check(backward ? "scols_bwd" : "scols_fwd");
}


}  // namespace

bool static_plan_cc(int Px, int Py, int pad, int L, int* cc) {
    if (pad != 2 || Px % 4 != 0 || Py % 4 != 0) return false;  // pruned stages need offset = P / 4
    const Plans* p = find(Px, Py);
    if (!p) return false;
    if (cols_smem(*p, L) > 220 * 1024) return false;
    *cc = p->cc;
    return true;
}

void static_prepare(AsmWork& w) {
    const Plans* p = find(w.Px, w.Py);
    const int idx = static_cast<int>(p - plans().data());
    w.stw_x = stable(idx, 0, p->row.table(w.Px));
    w.stw_y = stable(idx, 1, p->col.table(w.Py));
    const size_t rs = rows_smem(*p), cs = cols_smem(*p, w.L);
    HS_CUDA(cudaFuncSetAttribute(p->row.fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rs)));
    HS_CUDA(cudaFuncSetAttribute(p->row.inv, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rs)));
    if (p->row.fwd_put)
        HS_CUDA(cudaFuncSetAttribute(p->row.fwd_put, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rs)));
    if (p->row.inv_get)
        HS_CUDA(cudaFuncSetAttribute(p->row.inv_get, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rs)));
    for (auto k : {p->col.fwd, p->col.bwd, p->col.fwdL, p->col.bwdL})
        HS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cs)));
    if (p->col.fwdP) {
        const int csp = static_cast<int>(cols_smem_persist(*p, w.H));
        for (auto k : {p->col.fwdP, p->col.bwdP}) {
            HS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, csp));
            HS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        }
    }
    if (p->col.fwdS && cols_smem_persist(*p, w.H) <= 227 * 1024) {
        const int css = static_cast<int>(cols_smem_persist(*p, w.H));
        for (auto k : {p->col.fwdS, p->col.bwdS}) {
            HS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, css));
            HS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        }
    }
}


bool static_forward(AsmWork& w, const float2* d_in, float2* d_out, cudaStream_t st, cudaEvent_t* ev) {
    const Plans* p = find(w.Px, w.Py);
    if (!p || p->cc != w.CC) return false;
    const size_t rs = rows_smem(*p);
    const int rows1 = w.C * w.H;
    RowArgs r{d_in, w.T1.as<float2>(), w.W, w.H, w.Px, w.ox, w.ntiles, 1.f, w.plan_x, nullptr};
    p->row.fwd<<<(rows1 + p->row.rb - 1) / p->row.rb, p->row.nt, rs, st>>>(r, rows1, w.stw_x);
    launch_check("srows_fwd");
    if (ev) HS_CUDA(cudaEventRecordWithFlags(ev[0], st, cudaEventRecordExternal));
    ColArgs c{w.T1.as<float2>(), w.T2.as<float2>(), w.C, w.H, w.Py, w.Px, w.oy, w.ntiles, w.L, w.plan_y, nullptr,
              w.tf.as<TfConst>()};
    launch_cols(p, w, false, c, st);
    if (ev) HS_CUDA(cudaEventRecordWithFlags(ev[1], st, cudaEventRecordExternal));
    const int rows2 = w.L * w.C * w.H;
    RowArgs ri{w.T2.as<float2>(), d_out, w.W, w.H, w.Px, w.ox, w.ntiles,
               static_cast<float>(1.0 / (static_cast<double>(w.Px) * w.Py)), w.plan_x, nullptr};
    p->row.inv<<<(rows2 + p->row.rb - 1) / p->row.rb, p->row.nt, rs, st>>>(ri, rows2, w.stw_x);
    launch_check("srows_inv");
    if (ev) HS_CUDA(cudaEventRecordWithFlags(ev[2], st, cudaEventRecordExternal));
    return true;
}

bool static_backward(AsmWork& w, const float2* d_grads, float2* d_out, cudaStream_t st, cudaEvent_t* ev) {
    const Plans* p = find(w.Px, w.Py);
    if (!p || p->cc != w.CC) return false;
    const size_t rs = rows_smem(*p);
    const int rows1 = w.L * w.C * w.H;
    RowArgs r{d_grads, w.T2.as<float2>(), w.W, w.H, w.Px, w.ox, w.ntiles, 1.f, w.plan_x, nullptr};
    p->row.fwd<<<(rows1 + p->row.rb - 1) / p->row.rb, p->row.nt, rs, st>>>(r, rows1, w.stw_x);
    launch_check("srows_fwd");
    if (ev) HS_CUDA(cudaEventRecordWithFlags(ev[0], st, cudaEventRecordExternal));
    ColArgs c{w.T2.as<float2>(), w.T1.as<float2>(), w.C, w.H, w.Py, w.Px, w.oy, w.ntiles, w.L, w.plan_y, nullptr,
              w.tf.as<TfConst>()};
    launch_cols(p, w, true, c, st);
    if (ev) HS_CUDA(cudaEventRecordWithFlags(ev[1], st, cudaEventRecordExternal));
    const int rows2 = w.C * w.H;
    RowArgs ri{w.T1.as<float2>(), d_out, w.W, w.H, w.Px, w.ox, w.ntiles,
               static_cast<float>(1.0 / (static_cast<double>(w.Px) * w.Py)), w.plan_x, nullptr};
    p->row.inv<<<(rows2 + p->row.rb - 1) / p->row.rb, p->row.nt, rs, st>>>(ri, rows2, w.stw_x);
    launch_check("srows_inv");
    if (ev) HS_CUDA(cudaEventRecordWithFlags(ev[2], st, cudaEventRecordExternal));
    return true;
}

bool static_rows_pass(AsmWork& w, bool inverse, const float2* in, float2* out, int planes, int h, cudaStream_t st) {
    const Plans* p = find(w.Px, w.Py);
    if (!p || p->cc != w.CC) return false;
    const size_t rs = rows_smem(*p);
    const int rows = planes * h;
    const float scale = inverse ? static_cast<float>(1.0 / (static_cast<double>(w.Px) * w.Py)) : 1.f;
    RowArgs r{in, out, w.W, h, w.Px, w.ox, w.ntiles, scale, w.plan_x, nullptr};
    (inverse ? p->row.inv : p->row.fwd)<<<(rows + p->row.rb - 1) / p->row.rb, p->row.nt, rs, st>>>(r, rows, w.stw_x);
    launch_check(inverse ? "srows_inv" : "srows_fwd");
    return true;
}

bool static_cols_pass(AsmWork& w, bool backward, const float2* in, float2* out, int tile0, int ntiles_local,
                      cudaStream_t st) {
    const Plans* p = find(w.Px, w.Py);
    if (!p || p->cc != w.CC) return false;
    ColArgs c{in, out, w.C, w.H, w.Py, w.Px, w.oy, ntiles_local, w.L, w.plan_y, nullptr, w.tf.as<TfConst>()};
    c.tile0 = tile0;
    launch_cols(p, w, backward, c, st);
    return true;
}

bool asm_rows_fwd_put(AsmWork& w, const float2* in, int planes, int h, const SlabPut& sp, cudaStream_t st) {
    if (!w.use_static) return false;
    const Plans* p = find(w.Px, w.Py);
    if (!p || p->cc != w.CC || !p->row.fwd_put) return false;
    const int rows = planes * h;
    if (rows == 0) return true;
    RowArgs r{in, nullptr, w.W, h, w.Px, w.ox, w.ntiles, 1.f, w.plan_x, nullptr};
    p->row.fwd_put<<<(rows + p->row.rb - 1) / p->row.rb, p->row.nt, rows_smem(*p), st>>>(r, rows, w.stw_x, sp);
    launch_check("srows_fwd_put");
    return true;
}

bool asm_rows_inv_get(AsmWork& w, const float2* recv, float2* out, int planes, int h, const SlabGet& sg,
                      cudaStream_t st) {
    if (!w.use_static) return false;
    const Plans* p = find(w.Px, w.Py);
    if (!p || p->cc != w.CC || !p->row.inv_get) return false;
    const int rows = planes * h;
    if (rows == 0) return true;
    RowArgs r{recv, out, w.W, h, w.Px, w.ox, w.ntiles, static_cast<float>(1.0 / (static_cast<double>(w.Px) * w.Py)),
              w.plan_x, nullptr};
    p->row.inv_get<<<(rows + p->row.rb - 1) / p->row.rb, p->row.nt, rows_smem(*p), st>>>(r, rows, w.stw_x, sg);
    launch_check("srows_inv_get");
    return true;
}

bool asm_cols_slab(AsmWork& w, bool backward, const SlabCol& sc, float2* out, int tile0, int ntiles_local,
                   cudaStream_t st) {
    if (!w.use_static) return false;
    if (w.L > 1) {
        const Plans* p = find(w.Px, w.Py);
        if (!p || p->cc != w.CC || !p->col.fwdSL) return false;
        const size_t sm = cols_smem_slabL(*p, w.H, backward);
        if (sm > 227 * 1024 || w.H % sc.R != 0 || sc.hr * sc.R != w.H) return false;
        auto k = backward ? p->col.bwdSL : p->col.fwdSL;
        static std::mutex mu;
        {
            std::lock_guard<std::mutex> lock(mu);
            HS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
        }
        ColArgs c{nullptr, out, w.C, w.H, w.Py, w.Px, w.oy, ntiles_local, w.L, w.plan_y, nullptr, w.tf.as<TfConst>()};
        c.tile0 = tile0;
        k<<<ntiles_local * w.C, p->col.nt, sm, st>>>(c, w.stw_y, sc);
        launch_check(backward ? "scols_bwdL_slab" : "scols_fwdL_slab");
        return true;
    }
    const Plans* p = find(w.Px, w.Py);
    if (!p || p->cc != w.CC || !p->col.fwdS || cols_smem_persist(*p, w.H) > 227 * 1024) return false;
    if (w.H % sc.R != 0 || sc.hr * sc.R != w.H) return false;
    ColArgs c{nullptr, out, w.C, w.H, w.Py, w.Px, w.oy, ntiles_local, w.L, w.plan_y, nullptr, w.tf.as<TfConst>()};
    c.tile0 = tile0;
    (backward ? p->col.bwdS : p->col.fwdS)<<<ntiles_local * w.C, p->col.nt1 ? p->col.nt1 : p->col.nt,
                                             cols_smem_persist(*p, w.H), st>>>(c, w.stw_y, sc);
    launch_check(backward ? "scols_bwd_slab" : "scols_fwd_slab");
    return true;
}

}  // namespace hs
