// Band-limited angular spectrum method on B200: pad-aware row FFT, fused
// column FFT x H(fx,fy,z,lambda) x column IFFT (all planes from one load), and
// crop-aware row IFFT.
//
// Reference: proj/core/src/propagation.cpp -- pad_center/crop_center :111-127,
// apply_transfer :79-109, make_band_limit/kz_of :54-75, propagate_impl
// :135-153, propagate_multi :189-212, propagate_multi_backward :214-243.
//
// Data path per channel (Px = pad W, Py = pad H, centred offsets ox, oy):
//   rows_fwd : H rows, zero-padded to Px, FFT_x          -> T1 (H x Px, column-tiled)
//   cols_fwd : Px columns, zero-padded to Py, FFT_y, then per plane
//              x H_l, IFFT_y, keep rows [oy, oy+H)      -> T2_l
//   rows_inv : per plane, H rows IFFT_x, x 1/(Px Py), keep cols [ox, ox+W)
// The backward (adjoint) runs the same three passes with conj(H_l) and sums
// the planes inside the column kernel before its single IFFT_y.
// Intermediates use a column-tiled layout [tile][row][CC] so that the column
// kernel streams contiguous memory and the row kernels touch CC*8-byte runs.
#include <cmath>
#include <map>
#include <mutex>

#include "asm.cuh"

namespace hs {

namespace {

// F1 / B1: one CTA per input row.  Row rho = pc * H + y of a stack of
// C x H x W (or L x C x H x W) fields -> tiled output block pc.
template <int CC>
__global__ void __launch_bounds__(256) rows_fwd_kernel(RowArgs a) {
    extern __shared__ float2 smem[];
    const int n = a.Px;
    float2* A = smem;
    float2* B = smem + fft::padded_len(n);
    const int rho = blockIdx.x;
    const int pc = rho / a.H, y = rho - pc * a.H;
    const float2* src = a.in + static_cast<size_t>(rho) * a.W;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int x = i - a.ox;
        A[fft::pidx(i)] = (x >= 0 && x < a.W) ? src[x] : make_float2(0.f, 0.f);
    }
    const float2* res = fft::run<1, -1>(A, B, a.plan, a.tw, threadIdx.x, blockDim.x);
    float2* dst = a.out + (static_cast<size_t>(pc) * a.ntiles * a.H + y) * CC;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int tile = i / CC, cc = i - tile * CC;
        dst[static_cast<size_t>(tile) * a.H * CC + cc] = res[fft::pidx(i)];
    }
}

// F3 / B3: one CTA per output row; reads the tiled row, IFFT_x, crops, scales.
template <int CC>
__global__ void __launch_bounds__(256) rows_inv_kernel(RowArgs a) {
    extern __shared__ float2 smem[];
    const int n = a.Px;
    float2* A = smem;
    float2* B = smem + fft::padded_len(n);
    const int rho = blockIdx.x;
    const int pc = rho / a.H, y = rho - pc * a.H;
    const float2* src = a.in + (static_cast<size_t>(pc) * a.ntiles * a.H + y) * CC;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int tile = i / CC, cc = i - tile * CC;
        A[fft::pidx(i)] = src[static_cast<size_t>(tile) * a.H * CC + cc];
    }
    const float2* res = fft::run<1, +1>(A, B, a.plan, a.tw, threadIdx.x, blockDim.x);
    float2* dst = a.out + static_cast<size_t>(rho) * a.W;
    for (int x = threadIdx.x; x < a.W; x += blockDim.x) {
        const float2 v = res[fft::pidx(x + a.ox)];
        dst[x] = make_float2(v.x * a.scale, v.y * a.scale);
    }
}


template <int CC>
__device__ __forceinline__ void load_col_tile(float2* A, const float2* src, int H, int Py, int oy) {
    const int total = Py * CC;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int i = e / CC;
        const int y = i - oy;
        A[fft::pidx(e)] = (y >= 0 && y < H) ? src[static_cast<size_t>(y) * CC + (e - i * CC)]
                                            : make_float2(0.f, 0.f);
    }
}

template <int CC>
__device__ __forceinline__ void store_col_tile(float2* dst, const float2* res, int H, int oy) {
    const int total = H * CC;
    for (int e = threadIdx.x; e < total; e += blockDim.x) dst[e] = res[fft::pidx(e + oy * CC)];
}

// F2: grid (tiles, C).  Column FFT, per plane x H_l and IFFT, crop rows.
template <int CC>
__global__ void __launch_bounds__(256) cols_fwd_kernel(ColArgs a) {
    extern __shared__ float2 smem[];
    const int n = a.Py;
    const int plen = fft::padded_len(n * CC);
    float2* A = smem;
    float2* B = smem + plen;
    float2* S = smem + 2 * plen;  // spectrum copy (L > 1)
    const int tile = blockIdx.x, c = blockIdx.y;
    const size_t tile_elems = static_cast<size_t>(a.H) * CC;
    load_col_tile<CC>(A, a.in + (static_cast<size_t>(c) * a.ntiles + tile) * tile_elems, a.H, n, a.oy);
    float2* spec = fft::run<CC, -1>(A, B, a.plan, a.tw, threadIdx.x, blockDim.x);
    if (a.L > 1) {
        for (int e = threadIdx.x; e < n * CC; e += blockDim.x) S[fft::pidx(e)] = spec[fft::pidx(e)];
    }
    for (int l = 0; l < a.L; ++l) {
        const TfConst t = a.tf[l * a.C + c];
        float2* work = (a.L > 1) ? A : spec;
        const float2* from = (a.L > 1) ? S : spec;
        __syncthreads();
        for (int e = threadIdx.x; e < n * CC; e += blockDim.x) {
            const int ky = e / CC;
            const int kx = (a.tile0 + tile) * CC + (e - ky * CC);
            const float2 h = transfer<false>(t, wrapped(kx, a.Px), wrapped(ky, n));
            work[fft::pidx(e)] = cmul(from[fft::pidx(e)], h);
        }
        float2* other = (work == A) ? B : A;
        const float2* res = fft::run<CC, +1>(work, other, a.plan, a.tw, threadIdx.x, blockDim.x);
        store_col_tile<CC>(a.out + ((static_cast<size_t>(l) * a.C + c) * a.ntiles + tile) * tile_elems,
                           res, a.H, a.oy);
    }
}

// B2: grid (tiles, C).  Per plane column FFT x conj(H_l), summed; one IFFT.
template <int CC>
__global__ void __launch_bounds__(256) cols_bwd_kernel(ColArgs a) {
    extern __shared__ float2 smem[];
    const int n = a.Py;
    const int plen = fft::padded_len(n * CC);
    float2* A = smem;
    float2* B = smem + plen;
    float2* Z = smem + 2 * plen;  // accumulator (L > 1)
    const int tile = blockIdx.x, c = blockIdx.y;
    const size_t tile_elems = static_cast<size_t>(a.H) * CC;
    float2* acc = nullptr;
    for (int l = 0; l < a.L; ++l) {
        __syncthreads();
        load_col_tile<CC>(A, a.in + ((static_cast<size_t>(l) * a.C + c) * a.ntiles + tile) * tile_elems,
                          a.H, n, a.oy);
        float2* spec = fft::run<CC, -1>(A, B, a.plan, a.tw, threadIdx.x, blockDim.x);
        const TfConst t = a.tf[l * a.C + c];
        float2* dst = (a.L > 1) ? Z : spec;
        for (int e = threadIdx.x; e < n * CC; e += blockDim.x) {
            const int ky = e / CC;
            const int kx = (a.tile0 + tile) * CC + (e - ky * CC);
            const float2 h = transfer<true>(t, wrapped(kx, a.Px), wrapped(ky, n));
            const float2 v = cmul(spec[fft::pidx(e)], h);
            if (a.L > 1 && l > 0) dst[fft::pidx(e)] = cadd(dst[fft::pidx(e)], v);
            else dst[fft::pidx(e)] = v;
        }
        acc = dst;
    }
    float2* pong = (acc == A) ? B : A;
    const float2* res = fft::run<CC, +1>(acc, pong, a.plan, a.tw, threadIdx.x, blockDim.x);
    store_col_tile<CC>(a.out + (static_cast<size_t>(c) * a.ntiles + tile) * tile_elems, res, a.H, a.oy);
}

struct TwCache {
    std::mutex mu;
    std::map<std::pair<int, int>, float2*> tables;  // (device, n) -> W_n
};
TwCache g_tw;

const float2* twiddles(int n) {
    int dev = 0;
    HS_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_tw.mu);
    auto it = g_tw.tables.find({dev, n});
    if (it != g_tw.tables.end()) return it->second;
    std::vector<float2> h(n);
    for (int k = 0; k < n; ++k) {
        // exact reduction of k/n to a quarter period keeps the table fp64-accurate
        const double a = -2.0 * fft::kPi * static_cast<double>(k) / n;
        h[k] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
    }
    float2* d = nullptr;
    HS_CUDA(cudaMalloc(&d, sizeof(float2) * n));
    HS_CUDA(cudaMemcpy(d, h.data(), sizeof(float2) * n, cudaMemcpyHostToDevice));
    g_tw.tables[{dev, n}] = d;
    return d;
}

template <class K>
void allow_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024)
        HS_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(bytes)));
}

constexpr size_t kSmemBudget = 220 * 1024;

}  // namespace

template <int CC>
static void set_smem_attrs(const AsmWork& w);

fft::Plan make_plan(int n) {
    require(n >= 1, "fft: non-positive length");
    fft::Plan p;
    p.n = n;
    int rest = n;
    int e2 = 0;
    while (rest % 2 == 0) { rest /= 2; ++e2; }
    int e3 = 0, e5 = 0;
    while (rest % 3 == 0) { rest /= 3; ++e3; }
    while (rest % 5 == 0) { rest /= 5; ++e5; }
    std::vector<int> rad;
    while (e3 >= 1 && e5 >= 1) { rad.push_back(15); --e3; --e5; }
    while (e3 >= 2) { rad.push_back(9); e3 -= 2; }
    while (e5 >= 1) { rad.push_back(5); --e5; }
    while (e2 >= 4) { rad.push_back(16); e2 -= 4; }
    if (e3 == 1) {
        if (e2 >= 2) { rad.push_back(12); e2 -= 2; }
        else if (e2 == 1) { rad.push_back(6); e2 = 0; }
        else rad.push_back(3);
    }
    if (e2 == 3) rad.push_back(8);
    else if (e2 == 2) rad.push_back(4);
    else if (e2 == 1) rad.push_back(2);
    for (int q = 7; rest > 1; q += 2) {
        while (rest % q == 0) { rad.push_back(q); rest /= q; }
        if (q > rest && rest > 1) { rad.push_back(rest); rest = 1; }
    }
    require(static_cast<int>(rad.size()) <= fft::kMaxStages, "fft: too many stages");
    int ns = 1;
    for (size_t s = 0; s < rad.size(); ++s) {
        p.radix[s] = rad[s];
        p.ns[s] = ns;
        ns *= rad[s];
    }
    p.nst = static_cast<int>(rad.size());
    return p;
}

void AsmWork::prepare(int C_, int H_, int W_, int pad_, int L_) {
    require(pad_ >= 1, "propagation: pad_factor must be >= 1");
    require(C_ >= 1 && H_ >= 1 && W_ >= 1 && L_ >= 1, "propagation: bad dims");
    const bool same = C_ == C && H_ == H && W_ == W && pad_ == pad && L_ <= L;
    C = C_;
    H = H_;
    W = W_;
    pad = pad_;
    if (!same) L = L_;
    Px = W * pad;
    Py = H * pad;
    ox = (Px - W) / 2;
    oy = (Py - H) / 2;
    const int nbuf = L_ > 1 ? 3 : 2;
    CC = 4;
    use_static = static_plan_cc(Px, Py, pad, std::max(L, L_), &CC);
    if (!use_static) CC = 4;
    while (!use_static && CC > 1 &&
           nbuf * static_cast<size_t>(fft::padded_len(Py * CC)) * sizeof(float2) > kSmemBudget)
        CC /= 2;
    require(nbuf * static_cast<size_t>(fft::padded_len(Py * CC)) * sizeof(float2) <= kSmemBudget &&
                2 * static_cast<size_t>(fft::padded_len(Px)) * sizeof(float2) <= kSmemBudget,
            "propagation: padded grid too large for the shared-memory FFT");
    ntiles = (Px + CC - 1) / CC;
    plan_x = make_plan(Px);
    plan_y = make_plan(Py);
    twx_ptr = twiddles(Px);
    twy_ptr = twiddles(Py);
    smem_rows = 2 * static_cast<size_t>(fft::padded_len(Px)) * sizeof(float2);
    smem_cols = nbuf * static_cast<size_t>(fft::padded_len(Py * CC)) * sizeof(float2);
    switch (CC) {
        case 4: set_smem_attrs<4>(*this); break;
        case 2: set_smem_attrs<2>(*this); break;
        default: set_smem_attrs<1>(*this); break;
    }
    if (use_static) static_prepare(*this);
    const size_t tiled = static_cast<size_t>(ntiles) * H * CC * sizeof(float2);
    T1.reserve(tiled * C);
    T2.reserve(tiled * C * std::max(L, L_));
    tf.reserve(sizeof(TfConst) * C * std::max(L, L_));
    L = std::max(L, L_);
}

void AsmWork::set_transfer(const hs_prop_spec& spec, const double* phase_d, const double* mask_d,
                           cudaStream_t st) {
    require(spec.n_wavelengths == C, "propagation: channel count does not match wavelengths");
    require(spec.pad_factor >= 1, "propagation: pad_factor must be >= 1");
    tf_host.assign(static_cast<size_t>(L) * C, TfConst{});
    const double two_pi = 2.0 * fft::kPi;
    for (int l = 0; l < L; ++l) {
        for (int c = 0; c < C; ++c) {
            const double lambda = spec.wavelengths[c];
            require(lambda > 0.0 && spec.pixel_pitch > 0.0,
                    "propagation: non-positive wavelength or pitch");
            // make_band_limit (propagation.cpp:54-70)
            const double k = two_pi / lambda;
            const double lx = Px * spec.pixel_pitch, ly = Py * spec.pixel_pitch;
            const double inv_lx = 1.0 / lx, inv_ly = 1.0 / ly;
            const double md = mask_d[l];
            const double fx_max = 1.0 / (lambda * std::sqrt((2.0 * md / lx) * (2.0 * md / lx) + 1.0));
            const double fy_max = 1.0 / (lambda * std::sqrt((2.0 * md / ly) * (2.0 * md / ly) + 1.0));
            auto max_m = [](double inv_l, double fmax, int nn) {
                int m = 0;
                // |m * inv_l| < fmax  (strict, propagation.cpp:84 and :89)
                while (m <= nn && std::abs(static_cast<double>(m) * inv_l) < fmax) ++m;
                return m - 1;  // -1: even DC is outside
            };
            TfConst t;
            t.mx_max = max_m(inv_lx, fx_max, Px);
            t.my_max = max_m(inv_ly, fy_max, Py);
            const double kd = k * phase_d[l];
            t.kd = static_cast<float>(kd);
            t.kd_mod = static_cast<float>(std::fmod(kd, two_pi));
            t.bx = static_cast<float>((two_pi * inv_lx / k) * (two_pi * inv_lx / k));
            t.by = static_cast<float>((two_pi * inv_ly / k) * (two_pi * inv_ly / k));
            t.a4 = spec.aperture_radius > 0.0 ? 4.0 * (spec.aperture_radius * spec.aperture_radius) : -1.0;
            tf_host[static_cast<size_t>(l) * C + c] = t;
        }
    }
    HS_CUDA(cudaMemcpyAsync(tf.p, tf_host.data(), sizeof(TfConst) * tf_host.size(),
                            cudaMemcpyHostToDevice, st));
}

template <int CC>
static void set_smem_attrs(const AsmWork& w) {
    allow_smem(rows_fwd_kernel<CC>, w.smem_rows);
    allow_smem(rows_inv_kernel<CC>, w.smem_rows);
    allow_smem(cols_fwd_kernel<CC>, w.smem_cols);
    allow_smem(cols_bwd_kernel<CC>, w.smem_cols);
}

template <int CC>
static void launch_forward(AsmWork& w, const float2* d_in, float2* d_out, cudaStream_t st,
                           cudaEvent_t* ev) {
    RowArgs r{d_in, w.T1.as<float2>(), w.W, w.H, w.Px, w.ox, w.ntiles, 1.f, w.plan_x, w.twx_ptr};
    rows_fwd_kernel<CC><<<w.C * w.H, 256, w.smem_rows, st>>>(r);
    launch_check("rows_fwd");
    if (ev) HS_CUDA(cudaEventRecordWithFlags(ev[0], st, cudaEventRecordExternal));
    ColArgs c{w.T1.as<float2>(), w.T2.as<float2>(), w.C, w.H, w.Py, w.Px, w.oy, w.ntiles, w.L,
              w.plan_y, w.twy_ptr, w.tf.as<TfConst>()};
    cols_fwd_kernel<CC><<<dim3(w.ntiles, w.C), 256, w.smem_cols, st>>>(c);
    launch_check("cols_fwd");
    if (ev) HS_CUDA(cudaEventRecordWithFlags(ev[1], st, cudaEventRecordExternal));
    RowArgs ri{w.T2.as<float2>(), d_out, w.W, w.H, w.Px, w.ox, w.ntiles,
               static_cast<float>(1.0 / (static_cast<double>(w.Px) * w.Py)), w.plan_x, w.twx_ptr};
    rows_inv_kernel<CC><<<w.L * w.C * w.H, 256, w.smem_rows, st>>>(ri);
    launch_check("rows_inv");
    if (ev) HS_CUDA(cudaEventRecordWithFlags(ev[2], st, cudaEventRecordExternal));
}

template <int CC>
static void launch_backward(AsmWork& w, const float2* d_grads, float2* d_out, cudaStream_t st,
                            cudaEvent_t* ev) {
    RowArgs r{d_grads, w.T2.as<float2>(), w.W, w.H, w.Px, w.ox, w.ntiles, 1.f, w.plan_x,
              w.twx_ptr};
    rows_fwd_kernel<CC><<<w.L * w.C * w.H, 256, w.smem_rows, st>>>(r);
    launch_check("rows_fwd");
    if (ev) HS_CUDA(cudaEventRecordWithFlags(ev[0], st, cudaEventRecordExternal));
    ColArgs c{w.T2.as<float2>(), w.T1.as<float2>(), w.C, w.H, w.Py, w.Px, w.oy, w.ntiles, w.L,
              w.plan_y, w.twy_ptr, w.tf.as<TfConst>()};
    cols_bwd_kernel<CC><<<dim3(w.ntiles, w.C), 256, w.smem_cols, st>>>(c);
    launch_check("cols_bwd");
    if (ev) HS_CUDA(cudaEventRecordWithFlags(ev[1], st, cudaEventRecordExternal));
    RowArgs ri{w.T1.as<float2>(), d_out, w.W, w.H, w.Px, w.ox, w.ntiles,
               static_cast<float>(1.0 / (static_cast<double>(w.Px) * w.Py)), w.plan_x, w.twx_ptr};
    rows_inv_kernel<CC><<<w.C * w.H, 256, w.smem_rows, st>>>(ri);
    launch_check("rows_inv");
    if (ev) HS_CUDA(cudaEventRecordWithFlags(ev[2], st, cudaEventRecordExternal));
}

void asm_forward(AsmWork& w, const float2* d_in, float2* d_out, cudaStream_t st, cudaEvent_t* ev) {
    if (w.use_static && static_forward(w, d_in, d_out, st, ev)) return;
    switch (w.CC) {
        case 4: launch_forward<4>(w, d_in, d_out, st, ev); break;
        case 2: launch_forward<2>(w, d_in, d_out, st, ev); break;
        default: launch_forward<1>(w, d_in, d_out, st, ev); break;
    }
}

void asm_backward(AsmWork& w, const float2* d_grads, float2* d_out, cudaStream_t st, cudaEvent_t* ev) {
    if (w.use_static && static_backward(w, d_grads, d_out, st, ev)) return;
    switch (w.CC) {
        case 4: launch_backward<4>(w, d_grads, d_out, st, ev); break;
        case 2: launch_backward<2>(w, d_grads, d_out, st, ev); break;
        default: launch_backward<1>(w, d_grads, d_out, st, ev); break;
    }
}

// ---- row-slab passes and the exchange block copy ----------------------------------------
template <int CC>
static void rows_pass_generic(AsmWork& w, bool inverse, const float2* in, float2* out, int planes, int h,
                              cudaStream_t st) {
    const float scale = inverse ? static_cast<float>(1.0 / (static_cast<double>(w.Px) * w.Py)) : 1.f;
    RowArgs r{in, out, w.W, h, w.Px, w.ox, w.ntiles, scale, w.plan_x, w.twx_ptr};
    if (inverse) rows_inv_kernel<CC><<<planes * h, 256, w.smem_rows, st>>>(r);
    else rows_fwd_kernel<CC><<<planes * h, 256, w.smem_rows, st>>>(r);
    launch_check(inverse ? "rows_inv" : "rows_fwd");
}

template <int CC>
static void cols_pass_generic(AsmWork& w, bool backward, const float2* in, float2* out, int tile0, int nt,
                              cudaStream_t st) {
    ColArgs c{in, out, w.C, w.H, w.Py, w.Px, w.oy, nt, w.L, w.plan_y, w.twy_ptr, w.tf.as<TfConst>()};
    c.tile0 = tile0;
    if (backward) cols_bwd_kernel<CC><<<dim3(nt, w.C), 256, w.smem_cols, st>>>(c);
    else cols_fwd_kernel<CC><<<dim3(nt, w.C), 256, w.smem_cols, st>>>(c);
    launch_check(backward ? "cols_bwd" : "cols_fwd");
}

void asm_rows_pass(AsmWork& w, bool inverse, const float2* in, float2* out, int planes, int h, cudaStream_t st) {
    if (planes * h == 0) return;
    if (w.use_static && static_rows_pass(w, inverse, in, out, planes, h, st)) return;
    switch (w.CC) {
        case 4: rows_pass_generic<4>(w, inverse, in, out, planes, h, st); break;
        case 2: rows_pass_generic<2>(w, inverse, in, out, planes, h, st); break;
        default: rows_pass_generic<1>(w, inverse, in, out, planes, h, st); break;
    }
}

void asm_cols_pass(AsmWork& w, bool backward, const float2* in, float2* out, int tile0, int ntiles_local,
                   cudaStream_t st) {
    require(tile0 >= 0 && ntiles_local >= 1 && tile0 + ntiles_local <= w.ntiles, "propagation: column slab out of range");
    if (w.use_static && static_cols_pass(w, backward, in, out, tile0, ntiles_local, st)) return;
    switch (w.CC) {
        case 4: cols_pass_generic<4>(w, backward, in, out, tile0, ntiles_local, st); break;
        case 2: cols_pass_generic<2>(w, backward, in, out, tile0, ntiles_local, st); break;
        default: cols_pass_generic<1>(w, backward, in, out, tile0, ntiles_local, st); break;
    }
}

namespace {
// One warp per chunk; 16-byte moves when the chunk's offsets and length are even.
__global__ void __launch_bounds__(256) chunk_copy_kernel(const float2* __restrict__ src, float2* __restrict__ dst,
                                                         ChunkMap m) {
    const int64_t nchunks = static_cast<int64_t>(m.A) * m.B * m.T;
    const int lane = threadIdx.x & 31;
    for (int64_t k = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; k < nchunks;
         k += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const int t = static_cast<int>(k % m.T);
        const int64_t ab = k / m.T;
        const int b = static_cast<int>(ab % m.B), a = static_cast<int>(ab / m.B);
        const int64_t so = m.sA[a] + b * m.sB[a] + t * m.sT[a];
        const int64_t dof = m.dA[a] + b * m.dB[a] + t * m.dT[a];
        const int64_t len = m.len[a];
        float2* out = m.dptr[a] ? m.dptr[a] : dst;  // a peer's buffer: the stores travel over NVLink
        if (((so | dof | len) & 1) == 0) {
            const float4* s4 = reinterpret_cast<const float4*>(src + so);
            float4* d4 = reinterpret_cast<float4*>(out + dof);
            for (int64_t i = lane; i < len / 2; i += 32) d4[i] = s4[i];
        } else {
            for (int64_t i = lane; i < len; i += 32) out[dof + i] = src[so + i];
        }
    }
}
struct PeerFlags {
    uint32_t* f[kMaxPeers];
};

__global__ void slab_signal_kernel(PeerFlags pf, int ranks, int me, uint32_t* epoch_ctr) {
    const int a = threadIdx.x;
    const uint32_t epoch = *epoch_ctr + 1u;
    __syncwarp();
    if (a == 0) *epoch_ctr = epoch;
    if (a >= ranks) return;
    // every store of the preceding pack kernel (stream order) is made visible
    // system-wide before the flag
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pf.f[a] + me), "r"(epoch) : "memory");
}

__global__ void slab_wait_kernel(const uint32_t* flags, int ranks, const uint32_t* epoch_ctr, uint32_t* error) {
    const int a = threadIdx.x;
    const uint32_t epoch = *epoch_ctr;
    if (a < ranks) {
        const long long t0 = clock64();
        uint32_t v = 0;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + a) : "memory");
            if (static_cast<int32_t>(v - epoch) >= 0) break;
            if (clock64() - t0 > 4000000000LL) {  // ~2 s at 1.97 GHz: a peer never signalled
                atomicExch(error, 1u);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncthreads();
}
}  // namespace

void slab_signal(uint32_t* const* peer_flags, int ranks, int me, uint32_t* epoch, cudaStream_t st) {
    PeerFlags pf{};
    for (int a = 0; a < ranks; ++a) pf.f[a] = peer_flags[a];
    slab_signal_kernel<<<1, 32, 0, st>>>(pf, ranks, me, epoch);
    launch_check("slab_signal");
}

void slab_wait(const uint32_t* flags, int ranks, const uint32_t* epoch, uint32_t* error, cudaStream_t st) {
    slab_wait_kernel<<<1, 32, 0, st>>>(flags, ranks, epoch, error);
    launch_check("slab_wait");
}

void chunk_copy(const float2* src, float2* dst, const ChunkMap& m, cudaStream_t st) {
    require(m.A >= 1 && m.A <= kMaxPeers, "slab exchange: peer count outside 1..16");
    const int64_t nchunks = static_cast<int64_t>(m.A) * m.B * m.T;
    if (nchunks == 0) return;
    const int64_t blocks = std::min<int64_t>((nchunks + 7) / 8, 148 * 8);
    chunk_copy_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(src, dst, m);
    launch_check("chunk_copy");
}

}  // namespace hs
