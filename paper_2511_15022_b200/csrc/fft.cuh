// Shared-memory mixed-radix Stockham FFT engine (fp32) for sm_100a.
//
// Replaces the reference's FFTW3 fft2_inplace (proj/core/src/propagation.cpp:
// 21-40): unnormalised DFT, sign -1 forward (FFTW_FORWARD), +1 inverse.
// A CTA runs CC independent transforms of length n held interleaved in shared
// memory ([n][CC] float2, one pad slot per 16 entries against bank conflicts).
// Each stage is a radix-R Stockham autosort pass (natural-order output):
//   for butterfly j:  v[r] = in[j + r*n/R] * W_{ns R}^{r (j mod ns)}
//                     DFT_R(v);  out[(j - j mod ns) R + j mod ns + r ns] = v[r]
// Small DFTs are fully unrolled with compile-time twiddle constants
// (constexpr fp64 trig rounded to fp32); composite radices use an in-register
// Cooley-Tukey split.  Stage twiddles come from a per-length fp64-accurate
// table W_n[k] = exp(-2 pi i k / n) (conjugated for the inverse).
#pragma once

#include <utility>

#include "common.cuh"

namespace hs {
namespace fft {

constexpr double kPi = 3.141592653589793238462643383279502884;

constexpr double cx_reduce(double x) {
    const double k = x / (2.0 * kPi);
    const long long n = static_cast<long long>(k + (k >= 0 ? 0.5 : -0.5));
    return x - static_cast<double>(n) * 2.0 * kPi;
}
constexpr double cx_sin(double x) {
    x = cx_reduce(x);
    double term = x, sum = x;
    for (int i = 1; i < 30; ++i) {
        term *= -x * x / ((2.0 * i) * (2.0 * i + 1.0));
        sum += term;
    }
    return sum;
}
constexpr double cx_cos(double x) {
    x = cx_reduce(x);
    double term = 1.0, sum = 1.0;
    for (int i = 1; i < 30; ++i) {
        term *= -x * x / ((2.0 * i - 1.0) * (2.0 * i));
        sum += term;
    }
    return sum;
}

// exp(S * 2 pi i * num / den) as compile-time floats
template <int S, int NUM, int DEN>
struct W {
    static constexpr int m = ((NUM % DEN) + DEN) % DEN;
    static constexpr float re = static_cast<float>(cx_cos(2.0 * kPi * m / DEN));
    static constexpr float im = static_cast<float>(S * cx_sin(2.0 * kPi * m / DEN));
};

template <class F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

template <int S, int NUM, int DEN>
__device__ __forceinline__ float2 mul_w(float2 a) {
    using w = W<S, NUM, DEN>;
    constexpr int m = w::m;
    if constexpr (m == 0) {
        return a;
    } else if constexpr (4 * m == DEN) {  // S*i
        return S < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
    } else if constexpr (2 * m == DEN) {
        return make_float2(-a.x, -a.y);
    } else if constexpr (4 * m == 3 * DEN) {  // -S*i
        return S < 0 ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
    } else {
        return make_float2(a.x * w::re - a.y * w::im, a.x * w::im + a.y * w::re);
    }
}

template <int R>
struct Factor {  // smallest proper factor split R = A * B (A = 4 preferred)
    static constexpr int A = (R % 4 == 0 && R > 4) ? 4
                           : (R % 2 == 0 && R > 2) ? 2
                           : (R % 3 == 0 && R > 3) ? 3
                           : (R % 5 == 0 && R > 5) ? 5
                           : (R % 7 == 0 && R > 7) ? 7 : 1;
    static constexpr int B = A == 1 ? R : R / A;
};

template <int R, int S>
__device__ __forceinline__ void dft(float2 (&v)[R]);

template <int R, int S>
__device__ __forceinline__ void dft_naive(float2 (&v)[R]) {
    float2 out[R];
    static_for<R>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        float2 acc = v[0];
        static_for<R - 1>([&](auto jc) {
            constexpr int j = decltype(jc)::value + 1;
            const float2 t = mul_w<S, j * k, R>(v[j]);
            acc.x += t.x;
            acc.y += t.y;
        });
        out[k] = acc;
    });
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = out[k];
}

template <int A, int B, int S>
__device__ __forceinline__ void dft_ct(float2 (&v)[A * B]) {
    // n = B n1 + n2, k = k1 + A k2
    float2 y[A * B];  // y[n2 * A + k1]
    static_for<B>([&](auto n2c) {
        constexpr int n2 = decltype(n2c)::value;
        float2 u[A];
        static_for<A>([&](auto n1c) {
            constexpr int n1 = decltype(n1c)::value;
            u[n1] = v[B * n1 + n2];
        });
        dft<A, S>(u);
        static_for<A>([&](auto k1c) {
            constexpr int k1 = decltype(k1c)::value;
            y[n2 * A + k1] = mul_w<S, n2 * k1, A * B>(u[k1]);
        });
    });
    static_for<A>([&](auto k1c) {
        constexpr int k1 = decltype(k1c)::value;
        float2 z[B];
        static_for<B>([&](auto n2c) {
            constexpr int n2 = decltype(n2c)::value;
            z[n2] = y[n2 * A + k1];
        });
        dft<B, S>(z);
        static_for<B>([&](auto k2c) {
            constexpr int k2 = decltype(k2c)::value;
            v[k1 + A * k2] = z[k2];
        });
    });
}

template <int R, int S>
__device__ __forceinline__ void dft(float2 (&v)[R]) {
    if constexpr (R == 1) {
        return;
    } else if constexpr (R == 2) {
        const float2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    } else if constexpr (R == 3) {
        constexpr float c1 = -0.5f;
        constexpr float s1 = static_cast<float>(S * 0.86602540378443864676);
        const float2 t = cadd(v[1], v[2]);
        const float2 d = csub(v[1], v[2]);
        const float2 m = make_float2(v[0].x + c1 * t.x, v[0].y + c1 * t.y);
        v[0] = cadd(v[0], t);
        // v1 = m + s1*i*d, v2 = m - s1*i*d
        v[1] = make_float2(m.x - s1 * d.y, m.y + s1 * d.x);
        v[2] = make_float2(m.x + s1 * d.y, m.y - s1 * d.x);
    } else if constexpr (R == 4) {
        const float2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
        const float2 b0 = cadd(v[1], v[3]), b1 = csub(v[1], v[3]);
        const float2 jb1 = S < 0 ? make_float2(b1.y, -b1.x) : make_float2(-b1.y, b1.x);
        v[0] = cadd(a0, b0);
        v[2] = csub(a0, b0);
        v[1] = cadd(a1, jb1);
        v[3] = csub(a1, jb1);
    } else if constexpr (R == 5) {
        constexpr float c1 = static_cast<float>(0.30901699437494742410);   // cos(2pi/5)
        constexpr float c2 = static_cast<float>(-0.80901699437494742410);  // cos(4pi/5)
        constexpr float s1 = static_cast<float>(S * 0.95105651629515357212);
        constexpr float s2 = static_cast<float>(S * 0.58778525229247312917);
        const float2 t1 = cadd(v[1], v[4]), d1 = csub(v[1], v[4]);
        const float2 t2 = cadd(v[2], v[3]), d2 = csub(v[2], v[3]);
        const float2 m1 = make_float2(v[0].x + c1 * t1.x + c2 * t2.x, v[0].y + c1 * t1.y + c2 * t2.y);
        const float2 m2 = make_float2(v[0].x + c2 * t1.x + c1 * t2.x, v[0].y + c2 * t1.y + c1 * t2.y);
        // i*(s1 d1 + s2 d2), i*(s2 d1 - s1 d2)
        const float2 n1 = make_float2(s1 * d1.x + s2 * d2.x, s1 * d1.y + s2 * d2.y);
        const float2 n2 = make_float2(s2 * d1.x - s1 * d2.x, s2 * d1.y - s1 * d2.y);
        v[0] = make_float2(v[0].x + t1.x + t2.x, v[0].y + t1.y + t2.y);
        v[1] = make_float2(m1.x - n1.y, m1.y + n1.x);
        v[4] = make_float2(m1.x + n1.y, m1.y - n1.x);
        v[2] = make_float2(m2.x - n2.y, m2.y + n2.x);
        v[3] = make_float2(m2.x + n2.y, m2.y - n2.x);
    } else if constexpr (Factor<R>::A == 1) {
        dft_naive<R, S>(v);
    } else {
        dft_ct<Factor<R>::A, Factor<R>::B, S>(v);
    }
}

// Padded shared-memory index (one pad per 16 float2).
__device__ __forceinline__ int pidx(int q) { return q + (q >> 4); }
__host__ __device__ constexpr int padded_len(int q) { return q + (q >> 4) + 16; }

constexpr int kMaxStages = 12;
struct Plan {
    int n = 0;
    int nst = 0;
    int radix[kMaxStages];
    int ns[kMaxStages];
};

template <int R, int CC, int S>
__device__ __forceinline__ void stage(const float2* __restrict__ in, float2* __restrict__ out, int n,
                                      int ns, const float2* __restrict__ tw, int tid, int nthr) {
    const int m = n / R;
    const int span = n / (ns * R);
    for (int b = tid; b < m * CC; b += nthr) {
        const int cc = b % CC;
        const int j = b / CC;
        const int k = j % ns;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = in[pidx((j + r * m) * CC + cc)];
        if (k != 0) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                float2 w = __ldg(tw + r * k * span);
                if (S > 0) w.y = -w.y;
                v[r] = cmul(v[r], w);
            }
        }
        dft<R, S>(v);
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) out[pidx((base + r * ns) * CC + cc)] = v[r];
    }
}

// Any radix (runtime R): each thread computes one output of one butterfly.
template <int CC, int S>
__device__ void stage_any(const float2* __restrict__ in, float2* __restrict__ out, int n, int R,
                          int ns, const float2* __restrict__ tw, int tid, int nthr) {
    const int m = n / R;
    const int span = n / (ns * R);
    const int stride_r = n / R;  // W_R^{q} = W_n^{q * n/R}
    for (int e = tid; e < n * CC; e += nthr) {
        const int cc = e % CC;
        const int rest = e / CC;
        const int o = rest % R;  // output index within the butterfly
        const int j = rest / R;
        const int k = j % ns;
        float2 acc = make_float2(0.f, 0.f);
        for (int r = 0; r < R; ++r) {
            float2 v = in[pidx((j + r * m) * CC + cc)];
            int idx = (r * k * span + ((r * o) % R) * stride_r) % n;
            float2 w = __ldg(tw + idx);
            if (S > 0) w.y = -w.y;
            const float2 t = cmul(v, w);
            acc.x += t.x;
            acc.y += t.y;
        }
        out[pidx(((j - k) * R + k + o * ns) * CC + cc)] = acc;
    }
}

template <int CC, int S>
__device__ __forceinline__ void run_stage(const float2* in, float2* out, const Plan& P, int s,
                                          const float2* tw, int tid, int nthr) {
    const int n = P.n, ns = P.ns[s];
    switch (P.radix[s]) {
        case 2: stage<2, CC, S>(in, out, n, ns, tw, tid, nthr); break;
        case 3: stage<3, CC, S>(in, out, n, ns, tw, tid, nthr); break;
        case 4: stage<4, CC, S>(in, out, n, ns, tw, tid, nthr); break;
        case 5: stage<5, CC, S>(in, out, n, ns, tw, tid, nthr); break;
        case 6: stage<6, CC, S>(in, out, n, ns, tw, tid, nthr); break;
        case 7: stage<7, CC, S>(in, out, n, ns, tw, tid, nthr); break;
        case 8: stage<8, CC, S>(in, out, n, ns, tw, tid, nthr); break;
        case 9: stage<9, CC, S>(in, out, n, ns, tw, tid, nthr); break;
        case 10: stage<10, CC, S>(in, out, n, ns, tw, tid, nthr); break;
        case 12: stage<12, CC, S>(in, out, n, ns, tw, tid, nthr); break;
        case 15: stage<15, CC, S>(in, out, n, ns, tw, tid, nthr); break;
        case 16: stage<16, CC, S>(in, out, n, ns, tw, tid, nthr); break;
        default: stage_any<CC, S>(in, out, n, P.radix[s], ns, tw, tid, nthr); break;
    }
}

// Runs all stages ping-ponging between a and b; returns the buffer holding the
// result.  Starts and ends with __syncthreads.
template <int CC, int S>
__device__ float2* run(float2* a, float2* b, const Plan& P, const float2* tw, int tid, int nthr) {
    float2* in = a;
    float2* out = b;
    for (int s = 0; s < P.nst; ++s) {
        __syncthreads();
        run_stage<CC, S>(in, out, P, s, tw, tid, nthr);
        float2* t = in;
        in = out;
        out = t;
    }
    __syncthreads();
    return in;
}

}  // namespace fft
}  // namespace hs
