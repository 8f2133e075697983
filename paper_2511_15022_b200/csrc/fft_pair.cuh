// Column-pair SIMD FFT engine (fp32): the compile-time-planned in-place
// Stockham FFT of fft_static.cuh, but every thread transforms the SAME
// butterfly of TWO adjacent columns at once, with the two columns' real parts
// in one register pair and their imaginary parts in another.  Every complex
// add is then one packed FADD2 for two columns, a multiply by a known or
// tabulated twiddle two FMUL2/FFMA2 pairs, and a multiply by +-i is free (the
// re/im registers swap roles and the following add becomes a subtract) -- no
// register swizzles, unlike packing re/im of one value.  Twiddles are shared by
// the pair, so their loads halve too.
//
// Shared memory holds float4 (re0, re1, im0, im1) per (row, column pair):
// element (i, pp) at pidx4(i * NP + pp), one pad per 8 float4 against bank
// conflicts of the strided first-stage stores.
#pragma once

#include "fft_static.cuh"  // sfft::Radices, twiddle_table (same stage-twiddle layout)

namespace hs {
namespace pfft {

struct C2 {
    float2 re, im;  // (column 2p, column 2p + 1)
};

__device__ __forceinline__ C2 c2(float4 v) { return C2{make_float2(v.x, v.y), make_float2(v.z, v.w)}; }
__device__ __forceinline__ float4 f4(C2 a) { return make_float4(a.re.x, a.re.y, a.im.x, a.im.y); }
// store as two 8-byte halves: the re and im pairs need not sit in four
// consecutive registers (which would cost MOVs per STS.128)
__device__ __forceinline__ void st2(float4* dst, C2 a) {
    float2* d = reinterpret_cast<float2*>(dst);
    d[0] = a.re;
    d[1] = a.im;
}
__device__ __forceinline__ C2 zero2() { return C2{make_float2(0.f, 0.f), make_float2(0.f, 0.f)}; }
__device__ __forceinline__ C2 add(C2 a, C2 b) { return C2{f2add(a.re, b.re), f2add(a.im, b.im)}; }
__device__ __forceinline__ C2 sub(C2 a, C2 b) { return C2{f2sub(a.re, b.re), f2sub(a.im, b.im)}; }
// a * (wr + i wi), scalar twiddle shared by the pair
__device__ __forceinline__ C2 mulc(C2 a, float wr, float wi) {
    return C2{f2fma(a.im, f2splat(-wi), f2mul(a.re, f2splat(wr))), f2fma(a.im, f2splat(wr), f2mul(a.re, f2splat(wi)))};
}
// a * s (real scalar)
__device__ __forceinline__ C2 scale(C2 a, float s) { return C2{f2mul(a.re, f2splat(s)), f2mul(a.im, f2splat(s))}; }
// a + s * b
__device__ __forceinline__ C2 fma_s(C2 b, float s, C2 a) {
    return C2{f2fma(b.re, f2splat(s), a.re), f2fma(b.im, f2splat(s), a.im)};
}
// a + s * i * b = (a.re - s b.im, a.im + s b.re)
__device__ __forceinline__ C2 fma_si(C2 b, float s, C2 a) {
    return C2{f2fma(b.im, f2splat(-s), a.re), f2fma(b.re, f2splat(s), a.im)};
}
// a * (S i)
template <int S>
__device__ __forceinline__ C2 mul_si(C2 a) {
    return S < 0 ? C2{a.im, f2mul(a.re, f2splat(-1.f))} : C2{f2mul(a.im, f2splat(-1.f)), a.re};
}

template <int S, int NUM, int DEN>
__device__ __forceinline__ C2 mul_w(C2 a) {
    using w = fft::W<S, NUM, DEN>;
    constexpr int m = w::m;
    if constexpr (m == 0) {
        return a;
    } else if constexpr (4 * m == DEN) {
        return mul_si<S>(a);
    } else if constexpr (2 * m == DEN) {
        return scale(a, -1.f);
    } else if constexpr (4 * m == 3 * DEN) {
        return mul_si<-S>(a);
    } else {
        return mulc(a, w::re, w::im);
    }
}

template <int R>
struct Factor {  // R = A * B (A = 4 preferred)
    static constexpr int A = (R % 4 == 0 && R > 4) ? 4
                           : (R % 2 == 0 && R > 2) ? 2
                           : (R % 3 == 0 && R > 3) ? 3
                           : (R % 5 == 0 && R > 5) ? 5 : 1;
    static constexpr int B = A == 1 ? R : R / A;
};

template <int R, int S>
__device__ __forceinline__ void dft(C2 (&v)[R]);

template <int A, int B, int S>
__device__ __forceinline__ void dft_ct(C2 (&v)[A * B]) {
    // n = B n1 + n2, k = k1 + A k2
    C2 y[A * B];
    fft::static_for<B>([&](auto n2c) {
        constexpr int n2 = decltype(n2c)::value;
        C2 u[A];
        fft::static_for<A>([&](auto n1c) {
            constexpr int n1 = decltype(n1c)::value;
            u[n1] = v[B * n1 + n2];
        });
        dft<A, S>(u);
        fft::static_for<A>([&](auto k1c) {
            constexpr int k1 = decltype(k1c)::value;
            y[n2 * A + k1] = mul_w<S, n2 * k1, A * B>(u[k1]);
        });
    });
    fft::static_for<A>([&](auto k1c) {
        constexpr int k1 = decltype(k1c)::value;
        C2 z[B];
        fft::static_for<B>([&](auto n2c) {
            constexpr int n2 = decltype(n2c)::value;
            z[n2] = y[n2 * A + k1];
        });
        dft<B, S>(z);
        fft::static_for<B>([&](auto k2c) {
            constexpr int k2 = decltype(k2c)::value;
            v[k1 + A * k2] = z[k2];
        });
    });
}

template <int R, int S>
__device__ __forceinline__ void dft(C2 (&v)[R]) {
    if constexpr (R == 1) {
        return;
    } else if constexpr (R == 2) {
        const C2 a = v[0], b = v[1];
        v[0] = add(a, b);
        v[1] = sub(a, b);
    } else if constexpr (R == 3) {
        constexpr float s1 = static_cast<float>(S * 0.86602540378443864676);
        const C2 t = add(v[1], v[2]);
        const C2 d = sub(v[1], v[2]);
        const C2 m = fma_s(t, -0.5f, v[0]);
        v[0] = add(v[0], t);
        v[1] = fma_si(d, s1, m);
        v[2] = fma_si(d, -s1, m);
    } else if constexpr (R == 4) {
        const C2 a0 = add(v[0], v[2]), a1 = sub(v[0], v[2]);
        const C2 b0 = add(v[1], v[3]), b1 = sub(v[1], v[3]);
        v[0] = add(a0, b0);
        v[2] = sub(a0, b0);
        // v1 = a1 + (S i) b1, v3 = a1 - (S i) b1; (S i) b1 = (-S b1.im, S b1.re)
        if constexpr (S < 0) {
            v[1] = C2{f2add(a1.re, b1.im), f2sub(a1.im, b1.re)};
            v[3] = C2{f2sub(a1.re, b1.im), f2add(a1.im, b1.re)};
        } else {
            v[1] = C2{f2sub(a1.re, b1.im), f2add(a1.im, b1.re)};
            v[3] = C2{f2add(a1.re, b1.im), f2sub(a1.im, b1.re)};
        }
    } else if constexpr (R == 5) {
        constexpr float c1 = static_cast<float>(0.30901699437494742410);   // cos(2pi/5)
        constexpr float c2 = static_cast<float>(-0.80901699437494742410);  // cos(4pi/5)
        constexpr float s1 = static_cast<float>(S * 0.95105651629515357212);
        constexpr float s2 = static_cast<float>(S * 0.58778525229247312917);
        const C2 t1 = add(v[1], v[4]), d1 = sub(v[1], v[4]);
        const C2 t2 = add(v[2], v[3]), d2 = sub(v[2], v[3]);
        const C2 m1 = fma_s(t2, c2, fma_s(t1, c1, v[0]));
        const C2 m2 = fma_s(t2, c1, fma_s(t1, c2, v[0]));
        // n1 = s1 d1 + s2 d2, n2 = s2 d1 - s1 d2;  v1,4 = m1 +- i n1;  v2,3 = m2 +- i n2
        const C2 n1 = fma_s(d2, s2, scale(d1, s1));
        const C2 n2 = fma_s(d2, -s1, scale(d1, s2));
        v[0] = add(v[0], add(t1, t2));
        v[1] = fma_si(n1, 1.f, m1);
        v[4] = fma_si(n1, -1.f, m1);
        v[2] = fma_si(n2, 1.f, m2);
        v[3] = fma_si(n2, -1.f, m2);
    } else {
        static_assert(Factor<R>::A != 1, "pair engine: radix needs a 2/3/4/5 factorisation");
        dft_ct<Factor<R>::A, Factor<R>::B, S>(v);
    }
}

// Padded float4 index: one pad per 8 entries (1/16 was measured slower: bank
// conflicts of the strided first-stage stores).
constexpr int kPadShift = 3;
__device__ __forceinline__ int pidx4(int q) { return q + (q >> kPadShift); }
__host__ __device__ constexpr int padded_len4(int q) { return q + (q >> kPadShift) + 16; }

struct Full {
    template <int R>
    static constexpr int lo = 0;
    template <int R>
    static constexpr int hi = R;
};
struct Half {  // centred pad / crop of factor 2: digits [R/4, 3R/4)
    template <int R>
    static constexpr int lo = R / 4;
    template <int R>
    static constexpr int hi = 3 * R / 4;
};

// I/O policies (element i along the FFT axis, column pair pp):
//  InSmem / OutSmem: the in-place float4 buffer; InFn f(i, pp) -> C2; OutFn g(i, pp, C2);
//  OutMap g(i, pp, C2) -> C2 written back into the buffer.
struct InSmem {};
template <class F>
struct InFn {
    F f;
};
struct OutSmem {};
template <class G>
struct OutFn {
    G g;
};
template <class G>
struct OutMap {
    G g;
};
template <class F>
__device__ __forceinline__ InFn<F> in_fn(F f) { return InFn<F>{f}; }
template <class G>
__device__ __forceinline__ OutFn<G> out_fn(G g) { return OutFn<G>{g}; }
template <class G>
__device__ __forceinline__ OutMap<G> out_map(G g) { return OutMap<G>{g}; }
template <class T>
struct is_in_smem : std::false_type {};
template <>
struct is_in_smem<InSmem> : std::true_type {};
template <class T>
struct is_out_smem : std::false_type {};
template <>
struct is_out_smem<OutSmem> : std::true_type {};
template <class G>
struct is_out_smem<OutMap<G>> : std::true_type {};

// One radix-R stage over NP column pairs of length N with NT threads; thread
// bi serves pair bi % NP of butterfly bi / NP.
template <int N, int NP, int NT, int S, int R, int NS, class LIN, class LOUT, class IN, class OUT>
__device__ __forceinline__ void stage(float4* buf, const float2* __restrict__ tw, int tid, IN in, OUT out) {
    constexpr int M = N / R;
    constexpr int NB = M * NP;
    constexpr int BPT = (NB + NT - 1) / NT;
    constexpr int I0 = LIN::template lo<R>, I1 = LIN::template hi<R>;
    constexpr int O0 = LOUT::template lo<R>, O1 = LOUT::template hi<R>;
    constexpr bool smem_in = is_in_smem<IN>::value, smem_out = is_out_smem<OUT>::value;
    C2 v[BPT][R];
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int bi = tid + b * NT;
        if (NB % NT == 0 || bi < NB) {
            const int pp = bi % NP, j = bi / NP;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (r < I0 || r >= I1) {
                    v[b][r] = zero2();
                } else if constexpr (smem_in) {
                    if constexpr ((M * NP) % (1 << kPadShift) == 0)  // linear padded stride
                        v[b][r] = c2(buf[pidx4(j * NP + pp) + r * ((M * NP) >> kPadShift) * ((1 << kPadShift) + 1)]);
                    else
                        v[b][r] = c2(buf[pidx4((j + r * M) * NP + pp)]);
                } else {
                    v[b][r] = in.f(j + r * M, pp);
                }
            }
        }
    }
    if constexpr (smem_in && smem_out) __syncthreads();
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int bi = tid + b * NT;
        if (NB % NT == 0 || bi < NB) {
            const int pp = bi % NP, j = bi / NP;
            const int k = j % NS;
            if constexpr (NS > 1) {
                const float2* t = tw + (NS - 1) + k;
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    if (r < I0 || r >= I1) continue;
                    const float2 w = __ldg(t + (r - 1) * NS);
                    v[b][r] = mulc(v[b][r], w.x, S > 0 ? -w.y : w.y);
                }
            }
            dft<R, S>(v[b]);
            const int i0 = (j - k) * R + k;
#pragma unroll
            for (int r = O0; r < O1; ++r) {
                const int i = i0 + r * NS;
                if constexpr (is_out_smem<OUT>::value) {
                    const int q = (NS * NP) % (1 << kPadShift) == 0
                                      ? pidx4(i0 * NP + pp) + r * ((NS * NP) >> kPadShift) * ((1 << kPadShift) + 1)
                                      : pidx4(i * NP + pp);
                    if constexpr (std::is_same<OUT, OutSmem>::value) st2(buf + q, v[b][r]);
                    else st2(buf + q, out.g(i, pp, v[b][r]));
                } else {
                    out.g(i, pp, v[b][r]);
                }
            }
        }
    }
    if constexpr (smem_out) __syncthreads();
}

template <int N, int NP, int NT, int S, int NS, class LIN, class LOUT, class IN, class OUT, int R, int... Rest>
__device__ __forceinline__ void chain(float4* buf, const float2* tw, int tid, IN in, OUT out) {
    if constexpr (sizeof...(Rest) == 0) {
        stage<N, NP, NT, S, R, NS, LIN, LOUT>(buf, tw, tid, in, out);
    } else {
        stage<N, NP, NT, S, R, NS, LIN, Full>(buf, tw, tid, in, OutSmem{});
        chain<N, NP, NT, S, NS * R, Full, LOUT, InSmem, OUT, Rest...>(buf, tw, tid, InSmem{}, out);
    }
}

template <int N, int NP, int NT, int S, class LIN, class LOUT, class IN, class OUT, int... R>
__device__ __forceinline__ void run(float4* buf, const float2* tw, int tid, sfft::Radices<R...>, IN in, OUT out) {
    chain<N, NP, NT, S, 1, LIN, LOUT, IN, OUT, R...>(buf, tw, tid, in, out);
}

}  // namespace pfft
}  // namespace hs
