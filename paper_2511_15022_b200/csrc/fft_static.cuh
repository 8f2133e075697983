// Compile-time-planned shared-memory Stockham FFT (fp32) for the hot sizes.
//
// Same transform as fft.cuh (unnormalised DFT, sign S = -1 forward / +1
// inverse, natural-order output), but every size, radix, stride and trip count
// is a template constant, and every stage is written as
//
//     load R inputs of each butterfly  ->  twiddle  ->  radix-R DFT  ->  store R outputs
//
// where "load" and "store" are either the in-place shared buffer or a caller
// functor.  That lets a kernel
//   * read its first stage straight from global memory into registers, skipping
//     the inputs that are known zero (the centred zero pad: with a pad factor
//     of 2 the live input block is [N/4, 3N/4), i.e. radix digits [R/4, 3R/4)
//     of the first stage), and
//   * write its last stage straight to global memory, skipping the outputs the
//     crop discards (again digits [R/4, 3R/4) of the last stage), or apply the
//     transfer function to them in registers,
// so a transform costs (stages - 1) shared-memory round trips instead of
// stages + 1.  In-place stages synchronise between their loads and stores.
//
// Shared memory is addressed through the kernel's own `extern __shared__`
// symbol with 32-bit offsets (LDS/STS with immediate offsets); element q of
// the CC interleaved transforms lives at pidx(q) = q + q/16.
//
// Stage twiddles W_{NS R}^{r k} (k = j mod NS) live in one global table per
// plan, laid out stage by stage as [r-1][k] (offset NS-1 for the stage with
// stride NS); all CTAs read it through L1.
#pragma once

#include "fft.cuh"

namespace hs {
namespace sfft {

template <int... R>
struct Radices {};

// Live digit range of a pruned first/last stage (pad factor 2: [R/4, 3R/4)).
struct Full {
    template <int R>
    static constexpr int lo = 0;
    template <int R>
    static constexpr int hi = R;
};
struct Half {
    template <int R>
    static constexpr int lo = R / 4;
    template <int R>
    static constexpr int hi = 3 * R / 4;
};

// Shared-memory access with the linear-stride shortcut: when the stride of
// digit r is a multiple of 16 elements the padded index is pidx(q0) + r * s*17/16.
template <int CC, int STRIDE>
struct SmemView {
    float2* base;
    __device__ __forceinline__ int p0(int q0) const { return fft::pidx(q0); }
    __device__ __forceinline__ float2 get(int q0, int p, int r) const {
        if constexpr ((STRIDE * CC) % 16 == 0) return base[p + r * (STRIDE * CC / 16 * 17)];
        else return base[fft::pidx(q0 + r * STRIDE * CC)];
    }
    __device__ __forceinline__ void put(int q0, int p, int r, float2 v) const {
        if constexpr ((STRIDE * CC) % 16 == 0) base[p + r * (STRIDE * CC / 16 * 17)] = v;
        else base[fft::pidx(q0 + r * STRIDE * CC)] = v;
    }
};

// I/O policies ----------------------------------------------------------------------------
//  InSmem{src, f}: read shared buffer `src` (may be the stage's own buffer), value f(i, cc, v).
//  InFn{f}:        arbitrary loader f(i, cc) -> float2 (e.g. global memory).
//  OutSmem{dst, g}: g(i, cc, v, slot) writes the shared slot of element i (plain store,
//                   transfer multiply, accumulate ...).
//  OutFn{g}:       arbitrary sink g(i, cc, v) (e.g. global memory).
// Element i of transform cc is the natural-order index along the FFT axis.
struct Ident {
    __device__ __forceinline__ float2 operator()(int, int, float2 v) const { return v; }
};
struct Put {
    __device__ __forceinline__ void operator()(int, int, float2 v, float2& slot) const { slot = v; }
};
template <class F = Ident>
struct InSmem {
    const float2* src;
    F f;
};
template <class F>
struct InFn {
    F f;
};
template <class G = Put>
struct OutSmem {
    float2* dst;
    G g;
};
template <class G>
struct OutFn {
    G g;
};
template <class F>
__device__ __forceinline__ InSmem<F> in_smem(const float2* src, F f) { return InSmem<F>{src, f}; }
__device__ __forceinline__ InSmem<Ident> in_smem(const float2* src) { return InSmem<Ident>{src, Ident{}}; }
template <class F>
__device__ __forceinline__ InFn<F> in_fn(F f) { return InFn<F>{f}; }
template <class G>
__device__ __forceinline__ OutSmem<G> out_smem(float2* dst, G g) { return OutSmem<G>{dst, g}; }
__device__ __forceinline__ OutSmem<Put> out_smem(float2* dst) { return OutSmem<Put>{dst, Put{}}; }
template <class G>
__device__ __forceinline__ OutFn<G> out_fn(G g) { return OutFn<G>{g}; }

template <class T>
struct is_smem_in : std::false_type {};
template <class F>
struct is_smem_in<InSmem<F>> : std::true_type {};
template <class T>
struct is_smem_out : std::false_type {};
template <class G>
struct is_smem_out<OutSmem<G>> : std::true_type {};

// One radix-R Stockham stage of CC interleaved length-N transforms, NT threads.
// LIVE_IN / LIVE_OUT restrict the digits that are loaded / stored.  A stage
// that reads and writes shared memory synchronises between its loads and its
// stores (in-place safe); every shared-memory write is followed by a barrier.
template <int N, int CC, int NT, int S, int R, int NS, class LIVE_IN, class LIVE_OUT, class IN, class OUT>
__device__ __forceinline__ void stage(const float2* __restrict__ tw, int tid, IN in, OUT out) {
    constexpr int M = N / R;       // butterflies per transform
    constexpr int NB = M * CC;     // butterflies per CTA
    constexpr int BPT = (NB + NT - 1) / NT;
    constexpr int I0 = LIVE_IN::template lo<R>, I1 = LIVE_IN::template hi<R>;
    constexpr int O0 = LIVE_OUT::template lo<R>, O1 = LIVE_OUT::template hi<R>;
    static_assert(N % R == 0, "radix must divide N");
    constexpr bool smem_in = is_smem_in<IN>::value, smem_out = is_smem_out<OUT>::value;
    float2 v[BPT][R];
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int bi = tid + b * NT;
        if (NB % NT == 0 || bi < NB) {
            const int cc = bi % CC, j = bi / CC;
            const int q0 = j * CC + cc;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (r < I0 || r >= I1) {
                    v[b][r] = make_float2(0.f, 0.f);
                } else if constexpr (smem_in) {
                    const SmemView<CC, M> vin{const_cast<float2*>(in.src)};
                    v[b][r] = in.f(j + r * M, cc, vin.get(q0, vin.p0(q0), r));
                } else {
                    v[b][r] = in.f(j + r * M, cc);
                }
            }
        }
    }
    if constexpr (smem_in && smem_out) __syncthreads();
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int bi = tid + b * NT;
        if (NB % NT == 0 || bi < NB) {
            const int cc = bi % CC, j = bi / CC;
            const int k = j % NS;
            if constexpr (NS > 1) {
                const float2* t = tw + (NS - 1) + k;
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    if (r < I0 || r >= I1) continue;
                    float2 w = __ldg(t + (r - 1) * NS);
                    if (S > 0) w.y = -w.y;
                    v[b][r] = cmul(v[b][r], w);
                }
            }
            fft::dft<R, S>(v[b]);
            const int i0 = (j - k) * R + k;  // output element of digit 0
#pragma unroll
            for (int r = O0; r < O1; ++r) {
                if constexpr (smem_out) {
                    const int qs = i0 * CC + cc;
                    if constexpr ((NS * CC) % 16 == 0)
                        out.g(i0 + r * NS, cc, v[b][r], out.dst[fft::pidx(qs) + r * (NS * CC / 16 * 17)]);
                    else
                        out.g(i0 + r * NS, cc, v[b][r], out.dst[fft::pidx(qs + r * NS * CC)]);
                } else {
                    out.g(i0 + r * NS, cc, v[b][r]);
                }
            }
        }
    }
    if constexpr (smem_out) __syncthreads();
}

// Chains the stages of RAD over one in-place buffer `buf`: the first stage reads
// through IN (live digits LIN), the last writes through OUT (live digits LOUT).
template <int N, int CC, int NT, int S, int NS, class LIN, class LOUT, class IN, class OUT, int R, int... Rest>
__device__ __forceinline__ void chain(float2* buf, const float2* tw, int tid, IN in, OUT out) {
    if constexpr (sizeof...(Rest) == 0) {
        stage<N, CC, NT, S, R, NS, LIN, LOUT>(tw, tid, in, out);
    } else {
        stage<N, CC, NT, S, R, NS, LIN, Full>(tw, tid, in, out_smem(buf));
        chain<N, CC, NT, S, NS * R, Full, LOUT, InSmem<Ident>, OUT, Rest...>(buf, tw, tid, in_smem(buf), out);
    }
}

template <int N, int CC, int NT, int S, class LIN, class LOUT, class IN, class OUT, int... R>
__device__ __forceinline__ void run(float2* buf, const float2* tw, int tid, Radices<R...>, IN in, OUT out) {
    chain<N, CC, NT, S, 1, LIN, LOUT, IN, OUT, R...>(buf, tw, tid, in, out);
}

// Opaque copies of a value / pointer: inside loops over planes they stop the
// compiler from hoisting every stage's (loop-invariant) twiddle loads and smem
// offsets out of the loop, which pins ~100 registers and spills.
template <class T>
__device__ __forceinline__ T* launder(T* p) {
    T* q;
    asm volatile("mov.b64 %0, %1;" : "=l"(q) : "l"(p));
    return q;
}
__device__ __forceinline__ int launder(int v) {
    int q;
    asm volatile("mov.b32 %0, %1;" : "=r"(q) : "r"(v));
    return q;
}

// Host: stage twiddle table for a plan (N - 1 entries, forward sign).
template <int... R>
std::vector<float2> twiddle_table(int N, Radices<R...>) {
    std::vector<float2> t(static_cast<size_t>(N > 1 ? N - 1 : 1));
    const int rad[] = {R...};
    int ns = 1;
    for (int r : rad) {
        for (int q = 1; q < r; ++q)
            for (int k = 0; k < ns; ++k) {
                const long long num = static_cast<long long>(q) * k;
                const double a = -2.0 * fft::kPi * static_cast<double>(num % (ns * r)) / (ns * r);
                t[(ns - 1) + static_cast<size_t>(q - 1) * ns + k] =
                    make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
            }
        ns *= r;
    }
    return t;
}

}  // namespace sfft
}  // namespace hs
