// Compile-time planned angular-spectrum kernels for the benchmark grids.
//
// Same data path and numerics contract as asm.cu (propagation.cpp:186-294),
// with the FFT engine of fft_static.cuh: in-place stages, constant strides,
// persistent CTAs looping over rows / column tiles, and the transfer function
// H = exp(i kz d) evaluated with a Cody-Waite reduced fast sincos.
//
// Plans (Px x Py, column tile width CC):
//   3840 x 2160, CC 4   cfg2/cfg3 (1920x1080, pad 2)
//    512 x  512, CC 4   cfg1 (256x256, pad 2)
//    512 x  320, CC 4   desk regression (256x160, pad 2)
//   7680 x 4320, CC 2   cfg4 (3840x2160, pad 2)
#include <map>
#include <mutex>
#include <tuple>

#include "asm.cuh"
#include "fft_static.cuh"

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

// One work item per CTA throughout: a loop around the unrolled FFT makes
// ptxas spill heavily (measured), so persistence is traded for more CTAs.
// Per-row bases are hoisted out of the element loops (a runtime division by
// H per element was ~15% of the row kernels' instructions).
template <int N, int RB, int NT, int CCO, class RAD>
__global__ void __launch_bounds__(NT) srows_fwd_kernel(RowArgs a, int nrows, const float2* __restrict__ tw) {
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int rho0 = blockIdx.x * RB;
    const float2* src[RB];
    float2* dst[RB];
    bool ok[RB];
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
        const int rho = rho0 + rr;
        ok[rr] = rho < nrows;
        const int pc = rho / a.H, y = rho - pc * a.H;
        src[rr] = a.in + static_cast<size_t>(rho) * a.W - a.ox;
        dst[rr] = a.out + (static_cast<size_t>(pc) * a.ntiles * a.H + y) * CCO;
    }
    const size_t tile_stride = static_cast<size_t>(a.H) * CCO;
#pragma unroll 4
    for (int i = tid; i < N; i += NT) {
        const bool in = i >= a.ox && i < a.ox + a.W;
#pragma unroll
        for (int rr = 0; rr < RB; ++rr)
            smem[fft::pidx(i * RB + rr)] = (in && ok[rr]) ? src[rr][i] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    sfft::run<N, RB, NT, -1>(smem, tw, tid, RAD{});
#pragma unroll 4
    for (int i = tid; i < N; i += NT) {
        const size_t off = static_cast<size_t>(i / CCO) * tile_stride + (i % CCO);
#pragma unroll
        for (int rr = 0; rr < RB; ++rr)
            if (ok[rr]) dst[rr][off] = smem[fft::pidx(i * RB + rr)];
    }
}

template <int N, int RB, int NT, int CCO, class RAD>
__global__ void __launch_bounds__(NT) srows_inv_kernel(RowArgs a, int nrows, const float2* __restrict__ tw) {
    extern __shared__ float2 smem[];
    const int tid = threadIdx.x;
    const int rho0 = blockIdx.x * RB;
    const float2* src[RB];
    float2* dst[RB];
    bool ok[RB];
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
        const int rho = rho0 + rr;
        ok[rr] = rho < nrows;
        const int pc = rho / a.H, y = rho - pc * a.H;
        src[rr] = a.in + (static_cast<size_t>(pc) * a.ntiles * a.H + y) * CCO;
        dst[rr] = a.out + static_cast<size_t>(rho) * a.W - a.ox;
    }
    const size_t tile_stride = static_cast<size_t>(a.H) * CCO;
#pragma unroll 4
    for (int i = tid; i < N; i += NT) {
        const size_t off = static_cast<size_t>(i / CCO) * tile_stride + (i % CCO);
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) smem[fft::pidx(i * RB + rr)] = ok[rr] ? src[rr][off] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    sfft::run<N, RB, NT, +1>(smem, tw, tid, RAD{});
    const float sc = a.scale;
#pragma unroll 4
    for (int i = a.ox + tid; i < a.ox + a.W; i += NT) {
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) {
            if (!ok[rr]) continue;
            const float2 v = smem[fft::pidx(i * RB + rr)];
            dst[rr][i] = make_float2(v.x * sc, v.y * sc);
        }
    }
}

template <int N, int CC, int NT>
__device__ __forceinline__ void load_tile(float2* A, const float2* __restrict__ src, int H, int oy) {
    for (int e = threadIdx.x; e < N * CC; e += NT) {
        const int i = e / CC, y = i - oy;
        A[fft::pidx(e)] = (y >= 0 && y < H) ? src[static_cast<size_t>(y) * CC + (e - i * CC)] : make_float2(0.f, 0.f);
    }
}

template <int N, int CC, int NT>
__device__ __forceinline__ void store_tile(float2* __restrict__ dst, const float2* A, int H, int oy) {
    for (int e = threadIdx.x; e < H * CC; e += NT) dst[e] = A[fft::pidx(e + oy * CC)];
}

template <bool CONJ, int N, int CC, int NT>
__device__ __forceinline__ void apply_transfer(float2* dst, const float2* src, const TfConst& t, int tile, int Px,
                                               bool accumulate) {
    for (int e = threadIdx.x; e < N * CC; e += NT) {
        const int ky = e / CC, kx = tile * CC + (e - ky * CC);
        const float2 v = cmul(src[fft::pidx(e)], transfer_fast<CONJ>(t, wrapped(kx, Px), wrapped(ky, N)));
        dst[fft::pidx(e)] = accumulate ? cadd(dst[fft::pidx(e)], v) : v;
    }
}

// Single plane (the benchmark case): no loops around the FFTs.
template <int N, int CC, int NT, class RAD>
__global__ void __launch_bounds__(NT, 2) scols_fwd1_kernel(ColArgs a, const float2* __restrict__ tw) {
    extern __shared__ float2 smem[];
    const int tile = blockIdx.x, c = blockIdx.y;
    const size_t tile_elems = static_cast<size_t>(a.H) * CC;
    load_tile<N, CC, NT>(smem, a.in + (static_cast<size_t>(c) * a.ntiles + tile) * tile_elems, a.H, a.oy);
    __syncthreads();
    sfft::run<N, CC, NT, -1>(smem, tw, threadIdx.x, RAD{});
    apply_transfer<false, N, CC, NT>(smem, smem, a.tf[c], tile, a.Px, false);
    __syncthreads();
    sfft::run<N, CC, NT, +1>(smem, tw, threadIdx.x, RAD{});
    store_tile<N, CC, NT>(a.out + (static_cast<size_t>(c) * a.ntiles + tile) * tile_elems, smem, a.H, a.oy);
}

template <int N, int CC, int NT, class RAD>
__global__ void __launch_bounds__(NT, 2) scols_bwd1_kernel(ColArgs a, const float2* __restrict__ tw) {
    extern __shared__ float2 smem[];
    const int tile = blockIdx.x, c = blockIdx.y;
    const size_t tile_elems = static_cast<size_t>(a.H) * CC;
    load_tile<N, CC, NT>(smem, a.in + (static_cast<size_t>(c) * a.ntiles + tile) * tile_elems, a.H, a.oy);
    __syncthreads();
    sfft::run<N, CC, NT, -1>(smem, tw, threadIdx.x, RAD{});
    apply_transfer<true, N, CC, NT>(smem, smem, a.tf[c], tile, a.Px, false);
    __syncthreads();
    sfft::run<N, CC, NT, +1>(smem, tw, threadIdx.x, RAD{});
    store_tile<N, CC, NT>(a.out + (static_cast<size_t>(c) * a.ntiles + tile) * tile_elems, smem, a.H, a.oy);
}

// Multi-plane: one forward FFT per tile shared by all planes (spectrum kept in
// a second shared buffer); the adjoint sums the planes' spectra before one
// inverse FFT (propagation.cpp:240-294).
template <int N, int CC, int NT, class RAD>
__global__ void __launch_bounds__(NT, 2) scols_fwdL_kernel(ColArgs a, const float2* __restrict__ tw) {
    extern __shared__ float2 smem[];
    float2* A = smem;
    float2* Sp = smem + fft::padded_len(N * CC);
    const int tile = blockIdx.x, c = blockIdx.y;
    const size_t tile_elems = static_cast<size_t>(a.H) * CC;
    load_tile<N, CC, NT>(Sp, a.in + (static_cast<size_t>(c) * a.ntiles + tile) * tile_elems, a.H, a.oy);
    __syncthreads();
    sfft::run<N, CC, NT, -1>(Sp, tw, threadIdx.x, RAD{});
#pragma unroll 1
    for (int l = 0; l < a.L; ++l) {
        apply_transfer<false, N, CC, NT>(A, Sp, a.tf[l * a.C + c], tile, a.Px, false);
        __syncthreads();
        sfft::run<N, CC, NT, +1>(A, tw, threadIdx.x, RAD{});
        store_tile<N, CC, NT>(a.out + ((static_cast<size_t>(l) * a.C + c) * a.ntiles + tile) * tile_elems, A,
                              a.H, a.oy);
        __syncthreads();
    }
}

template <int N, int CC, int NT, class RAD>
__global__ void __launch_bounds__(NT, 2) scols_bwdL_kernel(ColArgs a, const float2* __restrict__ tw) {
    extern __shared__ float2 smem[];
    float2* A = smem;
    float2* Z = smem + fft::padded_len(N * CC);
    const int tile = blockIdx.x, c = blockIdx.y;
    const size_t tile_elems = static_cast<size_t>(a.H) * CC;
#pragma unroll 1
    for (int l = 0; l < a.L; ++l) {
        load_tile<N, CC, NT>(A, a.in + ((static_cast<size_t>(l) * a.C + c) * a.ntiles + tile) * tile_elems, a.H,
                             a.oy);
        __syncthreads();
        sfft::run<N, CC, NT, -1>(A, tw, threadIdx.x, RAD{});
        apply_transfer<true, N, CC, NT>(Z, A, a.tf[l * a.C + c], tile, a.Px, l > 0);
        __syncthreads();
    }
    sfft::run<N, CC, NT, +1>(Z, tw, threadIdx.x, RAD{});
    store_tile<N, CC, NT>(a.out + (static_cast<size_t>(c) * a.ntiles + tile) * tile_elems, Z, a.H, a.oy);
}

// ---- plan table -------------------------------------------------------------------------------
struct RowPlan {
    void (*fwd)(RowArgs, int, const float2*);
    void (*inv)(RowArgs, int, const float2*);
    int nt, rb;
    std::vector<float2> (*table)(int);
};
struct ColPlan {
    void (*fwd)(ColArgs, const float2*);
    void (*bwd)(ColArgs, const float2*);
    void (*fwdL)(ColArgs, const float2*);
    void (*bwdL)(ColArgs, const float2*);
    int nt, cc;
    std::vector<float2> (*table)(int);
};

template <int N, int RB, int NT, int CCO, class RAD>
RowPlan row_plan() {
    return RowPlan{srows_fwd_kernel<N, RB, NT, CCO, RAD>, srows_inv_kernel<N, RB, NT, CCO, RAD>, NT, RB,
                   [](int n) { return sfft::twiddle_table(n, RAD{}); }};
}
template <int N, int CC, int NT, class RAD>
ColPlan col_plan() {
    return ColPlan{scols_fwd1_kernel<N, CC, NT, RAD>, scols_bwd1_kernel<N, CC, NT, RAD>,
                   scols_fwdL_kernel<N, CC, NT, RAD>, scols_bwdL_kernel<N, CC, NT, RAD>, NT, CC,
                   [](int n) { return sfft::twiddle_table(n, RAD{}); }};
}

struct Plans {
    int Px, Py, cc;
    RowPlan row;
    ColPlan col;
};

const std::vector<Plans>& plans() {
    static const std::vector<Plans> p = {
        {3840, 2160, 4, row_plan<3840, 1, 256, 4, Radices<16, 16, 15>>(),
         col_plan<2160, 4, 736, Radices<12, 12, 15>>()},
        {512, 512, 4, row_plan<512, 1, 64, 4, Radices<8, 8, 8>>(), col_plan<512, 4, 128, Radices<8, 8, 8>>()},
        {512, 320, 4, row_plan<512, 1, 64, 4, Radices<8, 8, 8>>(), col_plan<320, 4, 128, Radices<16, 20>>()},
        {7680, 4320, 2, row_plan<7680, 2, 512, 2, Radices<16, 16, 30>>(),
         col_plan<4320, 2, 576, Radices<16, 18, 15>>()},
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
    return sizeof(float2) * fft::padded_len(p.Py * p.col.cc) * (L > 1 ? 2 : 1);
}


}  // namespace

bool static_plan_cc(int Px, int Py, int L, int* cc) {
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
    for (auto k : {p->col.fwd, p->col.bwd, p->col.fwdL, p->col.bwdL})
        HS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cs)));
}


bool static_forward(AsmWork& w, const float2* d_in, float2* d_out, cudaStream_t st, cudaEvent_t* ev) {
    const Plans* p = find(w.Px, w.Py);
    if (!p || p->cc != w.CC) return false;
    const size_t rs = rows_smem(*p), cs = cols_smem(*p, w.L);
    const int rows1 = w.C * w.H;
    RowArgs r{d_in, w.T1.as<float2>(), w.W, w.H, w.Px, w.ox, w.ntiles, 1.f, w.plan_x, nullptr};
    p->row.fwd<<<(rows1 + p->row.rb - 1) / p->row.rb, p->row.nt, rs, st>>>(r, rows1, w.stw_x);
    launch_check("srows_fwd");
    if (ev) HS_CUDA(cudaEventRecord(ev[0], st));
    ColArgs c{w.T1.as<float2>(), w.T2.as<float2>(), w.C, w.H, w.Py, w.Px, w.oy, w.ntiles, w.L, w.plan_y, nullptr,
              w.tf.as<TfConst>()};
    (w.L > 1 ? p->col.fwdL : p->col.fwd)<<<dim3(w.ntiles, w.C), p->col.nt, cs, st>>>(c, w.stw_y);
    launch_check("scols_fwd");
    if (ev) HS_CUDA(cudaEventRecord(ev[1], st));
    const int rows2 = w.L * w.C * w.H;
    RowArgs ri{w.T2.as<float2>(), d_out, w.W, w.H, w.Px, w.ox, w.ntiles,
               static_cast<float>(1.0 / (static_cast<double>(w.Px) * w.Py)), w.plan_x, nullptr};
    p->row.inv<<<(rows2 + p->row.rb - 1) / p->row.rb, p->row.nt, rs, st>>>(ri, rows2, w.stw_x);
    launch_check("srows_inv");
    if (ev) HS_CUDA(cudaEventRecord(ev[2], st));
    return true;
}

bool static_backward(AsmWork& w, const float2* d_grads, float2* d_out, cudaStream_t st, cudaEvent_t* ev) {
    const Plans* p = find(w.Px, w.Py);
    if (!p || p->cc != w.CC) return false;
    const size_t rs = rows_smem(*p), cs = cols_smem(*p, w.L);
    const int rows1 = w.L * w.C * w.H;
    RowArgs r{d_grads, w.T2.as<float2>(), w.W, w.H, w.Px, w.ox, w.ntiles, 1.f, w.plan_x, nullptr};
    p->row.fwd<<<(rows1 + p->row.rb - 1) / p->row.rb, p->row.nt, rs, st>>>(r, rows1, w.stw_x);
    launch_check("srows_fwd");
    if (ev) HS_CUDA(cudaEventRecord(ev[0], st));
    ColArgs c{w.T2.as<float2>(), w.T1.as<float2>(), w.C, w.H, w.Py, w.Px, w.oy, w.ntiles, w.L, w.plan_y, nullptr,
              w.tf.as<TfConst>()};
    (w.L > 1 ? p->col.bwdL : p->col.bwd)<<<dim3(w.ntiles, w.C), p->col.nt, cs, st>>>(c, w.stw_y);
    launch_check("scols_bwd");
    if (ev) HS_CUDA(cudaEventRecord(ev[1], st));
    const int rows2 = w.C * w.H;
    RowArgs ri{w.T1.as<float2>(), d_out, w.W, w.H, w.Px, w.ox, w.ntiles,
               static_cast<float>(1.0 / (static_cast<double>(w.Px) * w.Py)), w.plan_x, nullptr};
    p->row.inv<<<(rows2 + p->row.rb - 1) / p->row.rb, p->row.nt, rs, st>>>(ri, rows2, w.stw_x);
    launch_check("srows_inv");
    if (ev) HS_CUDA(cudaEventRecord(ev[2], st));
    return true;
}

}  // namespace hs
