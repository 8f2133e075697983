// Compile-time-planned shared-memory Stockham FFT (fp32) for the hot sizes.
//
// Same transform as fft.cuh (unnormalised DFT, sign S = -1 forward / +1
// inverse, natural-order output), but every size, radix, stride and trip count
// is a template constant: index math folds to shifts/multiply-adds, loops
// unroll, and each stage runs IN PLACE in one shared buffer -- every thread
// first pulls all inputs of its butterflies into registers, the CTA
// synchronises, then the twiddled radix-R DFTs are written back.  One buffer
// instead of two halves the shared memory per transform, which is what lets
// several CTAs share an SM.
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

template <int N, int CC, int NT, int S, int R, int NS>
__device__ __forceinline__ void stage(float2* __restrict__ buf, const float2* __restrict__ tw, int tid) {
    constexpr int M = N / R;       // butterflies per transform
    constexpr int NB = M * CC;     // butterflies per CTA
    constexpr int BPT = (NB + NT - 1) / NT;
    static_assert(N % R == 0, "radix must divide N");
    float2 v[BPT][R];
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int bi = tid + b * NT;
        if (NB % NT == 0 || bi < NB) {
            const int cc = bi % CC, j = bi / CC;
            const int q0 = j * CC + cc;
            if constexpr ((M * CC) % 16 == 0) {  // padded stride is linear: one index, immediate offsets
                const int p0 = fft::pidx(q0);
#pragma unroll
                for (int r = 0; r < R; ++r) v[b][r] = buf[p0 + r * (M * CC / 16 * 17)];
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) v[b][r] = buf[fft::pidx(q0 + r * M * CC)];
            }
        }
    }
    __syncthreads();
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
                    float2 w = __ldg(t + (r - 1) * NS);
                    if (S > 0) w.y = -w.y;
                    v[b][r] = cmul(v[b][r], w);
                }
            }
            fft::dft<R, S>(v[b]);
            const int qs = ((j - k) * R + k) * CC + cc;
            if constexpr ((NS * CC) % 16 == 0) {
                const int ps = fft::pidx(qs);
#pragma unroll
                for (int r = 0; r < R; ++r) buf[ps + r * (NS * CC / 16 * 17)] = v[b][r];
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) buf[fft::pidx(qs + r * NS * CC)] = v[b][r];
            }
        }
    }
    __syncthreads();
}

template <int N, int CC, int NT, int S, int NS, int R, int... Rest>
__device__ __forceinline__ void run_stages(float2* buf, const float2* tw, int tid) {
    stage<N, CC, NT, S, R, NS>(buf, tw, tid);
    if constexpr (sizeof...(Rest) > 0) run_stages<N, CC, NT, S, NS * R, Rest...>(buf, tw, tid);
}

// Opaque copy of a pointer: stops the compiler from hoisting the (loop-
// invariant) twiddle loads of every stage out of persistent loops, which
// would pin ~100 registers per thread and spill.
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

// The thread index, the buffer and the table are laundered per call: inside
// persistent loops the compiler would otherwise hoist every stage's smem
// offsets and twiddle loads out of the loop and spill them.
template <int N, int CC, int NT, int S, int... R>
__device__ __forceinline__ void run(float2* buf, const float2* tw, int tid, Radices<R...>) {
    run_stages<N, CC, NT, S, 1, R...>(launder(buf), launder(tw), launder(tid));
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
