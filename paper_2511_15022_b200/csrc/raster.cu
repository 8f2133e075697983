// K0 projection, K1 tile binning, K2 tile-parallel forward splat, K3 backward.
//
// Reference: proj/core/src/rasterizer.cpp (activate_flat :33-88, build_index
// :90-119, rasterize_forward :128-190, rasterize_backward :192-286) and the
// scalar math of proj/core/src/field_core.cpp:11-68.
//
// Numerics
//  * Projection (K0) runs in fp64 on the fp32 parameters with the reference's
//    exact operation order and no FMA contraction (__dmul_rn/__dadd_rn), so the
//    cull radius and tile bounds -- hence the (tile,id) pair list -- are
//    bit-identical with holo::build_tile_index on the same values.
//  * Shading (K2/K3) runs in fp32.  The two skip tests of the reference
//    (mahal > cutoff, alpha_eff < 1/255; rasterizer.cpp:166-169,222-228) are
//    decided in fp32 outside a per-Gaussian error band `tol` and re-decided in
//    fp64 with the reference arithmetic inside it, so the set of contributing
//    (pixel, Gaussian) pairs matches the reference.
//  * Forward accumulates each pixel in ascending Gaussian id (the sorted
//    per-tile list), like the reference, so results are run-to-run identical.
//  * Backward is a per-Gaussian gather (the reference's own decomposition,
//    rasterizer.cpp:201-284): one warp per Gaussian walks the exact ellipse
//    footprint row by row, lanes own pixels, a warp-shuffle reduction folds
//    the 7 + 2C partial sums and lane 0 applies the fp64 chain rule.  No
//    atomics: the gradients are deterministic.
#include <cstdlib>
#include <type_traits>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "raster.cuh"

namespace hs {

namespace {

// ---------------------------------------------------------------------------
// K0: projection (activate_flat, rasterizer.cpp:33-88; field_core.cpp:11-68)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ bool finite(double v) { return isfinite(v); }

struct ProjParams {
    const float* params;
    int n, c, width, height, tiles_x, tiles_y;
    float4* rec;
    float4* shade;
    double* p64;
    int4* pbox;
    int4* tbox;
    uint32_t* tcount;  // Gaussians per tile (atomics)
    uint32_t* status;
    int fuse_shade;    // also write the per-channel shading record
    uint4* trows;      // tight binning: touched tile columns per box row (nullptr: off)
};

// Per-channel shading (rasterizer.cpp:78-85).  fp32: the record is only
// consumed in fp32, and sincosf has accurate range reduction (~1 ulp).
__device__ __forceinline__ void shade_one(const float* __restrict__ params, int g, int n, int c,
                                          float4* __restrict__ shade, uint32_t* __restrict__ status) {
    const size_t N = n;
    const float* amp = params + 5 * N;       // after pre_position 2N | pre_scale 2N | rotation N
    const float* pha = amp + N * c;
    for (int ch = 0; ch < c; ++ch) {
        const size_t i = static_cast<size_t>(g) * c + ch;
        const float a = fminf(fmaxf(amp[i], 0.f), 1.f);
        const float ph = pha[i];
        if (!isfinite(ph) || !isfinite(amp[i])) atomicOr(status + 2, 1u);
        float sp, cp;
        sincosf(ph, &sp, &cp);
        shade[static_cast<size_t>(ch) * N + g] = make_float4(a * cp, a * sp, cp, sp);
    }
}

// Its own kernel when the amplitude/phase groups can still be in flight
// (host-resident parameter upload) while the geometry is binned.
__global__ void shade_kernel(const float* __restrict__ params, int n, int c, float4* __restrict__ shade,
                             uint32_t* __restrict__ status) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) shade_one(params, g, n, c, shade, status);
}

// Conservative x-extent [xlo, xhi] (pixels) of the Gaussian's skip-test region
// (the ellipse mahal <= cut + tol, widened by 1e-2 px) over the row band
// [cy0, cy0 + ch]: the widest chord (band row closest to the centre) around the
// centre line shifted to both band edges.  False when no band row meets it.
__device__ __forceinline__ bool row_band_extent(float4 r0, float4 r1, float4 r2, float cy0, float ch, float& xlo,
                                                float& xhi) {
    const float M = r1.w + r2.y;
    const float px = r0.x + r0.z, py = r0.y + r0.w;
    const float dya = cy0 - py, dyb = dya + ch;
    const float dyc = fminf(fmaxf(0.f, dya), dyb);
    const float D = r1.x * M - r2.z * dyc * dyc;
    if (D < 0.f) return false;
    const float hw = sqrtf(D) * r2.w + 1e-2f;
    const float ratio = r1.y * r2.w;
    const float ca = -ratio * dya, cb = -ratio * dyb;
    xlo = px + fminf(ca, cb) - hw;
    xhi = px + fmaxf(ca, cb) + hw;
    return true;
}

// Can any pixel of the cell [cx0, cx0 + cw] x [cy0, cy0 + ch] pass the exact tests?
__device__ __forceinline__ bool cell_hit(float4 r0, float4 r1, float4 r2, float cx0, float cy0,
                                         float cw, float ch) {
    float xlo, xhi;
    if (!row_band_extent(r0, r1, r2, cy0, ch, xlo, xhi)) return false;
    return xhi >= cx0 && xlo <= cx0 + cw;
}

// Tight binning (trainer and forward paths): a (tile, Gaussian) pair of the
// reference's box list (rasterizer.cpp:95-108) is kept only if the ellipse can
// reach the tile.  Dropped pairs contribute exactly zero to every pixel of the
// tile (their pixels all fail mahal <= cutoff), and the kept ids stay ascending,
// so the forward field is bit-identical; build_tile_index (the exported,
// reference-exact list) bins with tight off.  The projection stores, for the
// first kTightRows tile rows of the box, the touched tile-column range relative
// to the box (one byte each for lo and hi, lo > hi = none); rows beyond that,
// or boxes wider than 255 tiles, keep the whole box row.
constexpr int kTightRows = 8;

__device__ __forceinline__ uint4 tight_rows(float4 r0, float4 r1, float4 r2, int tx0, int tx1, int ty0, int ty1) {
    uint32_t lo[2] = {0u, 0u}, hi[2] = {0xffffffffu, 0xffffffffu};  // default: whole row
    if (tx1 - tx0 > 254) return make_uint4(lo[0], lo[1], hi[0], hi[1]);
    for (int r = 0; r < kTightRows && ty0 + r <= ty1; ++r) {
        float xlo, xhi;
        int a = 255, b = 0;  // empty
        if (row_band_extent(r0, r1, r2, static_cast<float>((ty0 + r) * kTile), static_cast<float>(kTile - 1), xlo,
                            xhi)) {
            // tiles tx with xlo <= tx*16 + 15 and tx*16 <= xhi: cell_hit over the tile, exactly
            // (xlo - 15 and the scalings by 1/16 are exact in fp32 on the canvas range)
            a = max(static_cast<int>(ceilf((xlo - static_cast<float>(kTile - 1)) * (1.f / kTile))), tx0) - tx0;
            b = min(static_cast<int>(floorf(xhi * (1.f / kTile))), tx1) - tx0;
            if (a > b) a = 255, b = 0;
        }
        const int w = r >> 2, sh = 8 * (r & 3);
        lo[w] = (lo[w] & ~(0xffu << sh)) | (static_cast<uint32_t>(a) << sh);
        hi[w] = (hi[w] & ~(0xffu << sh)) | (static_cast<uint32_t>(b) << sh);
    }
    return make_uint4(lo[0], lo[1], hi[0], hi[1]);
}

// Is tile (tx, ty) of the box (origin tx0, ty0) in the tight set?
__device__ __forceinline__ bool tight_has(uint4 t, int tx, int ty, int tx0, int ty0) {
    const int r = ty - ty0;
    if (r >= kTightRows) return true;
    const int sh = 8 * (r & 3);
    const uint32_t lo = ((r < 4 ? t.x : t.y) >> sh) & 0xffu, hi = ((r < 4 ? t.z : t.w) >> sh) & 0xffu;
    const uint32_t o = static_cast<uint32_t>(tx - tx0);
    return o >= lo && o <= hi;
}

__global__ void project_kernel(ProjParams P) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= P.n) return;
    const size_t N = P.n;
    const float* pp = P.params;                 // pre_position 2N
    const float* ps = pp + 2 * N;               // pre_scale 2N
    const float* rot = ps + 2 * N;              // rotation N
    const float* opa = rot + N + 2 * N * P.c;   // pre_opacity N (after amplitude, phase N*C each)

    const double prx = pp[2 * g], pry = pp[2 * g + 1];
    const double psx = ps[2 * g], psy = ps[2 * g + 1];
    const double th = rot[g], po = opa[g];
    if (!(finite(prx) && finite(pry) && finite(psx) && finite(psy) && finite(po)))
        atomicOr(P.status + 2, 1u);

    // activate_position: (tanh(pre) + 1) * 0.5 * extent   (field_core.cpp:11-14)
    const double px = dmul(dmul(dadd(tanh(prx), 1.0), 0.5), static_cast<double>(P.width));
    const double py = dmul(dmul(dadd(tanh(pry), 1.0), 0.5), static_cast<double>(P.height));
    // activate_scale: exp(pre) + 0.1   (:21-24)
    const double sx = dadd(exp(psx), kEpsScale);
    const double sy = dadd(exp(psy), kEpsScale);
    // covariance (:46-54)
    const double cth = cos(th), sth = sin(th);
    const double sx2 = dmul(sx, sx), sy2 = dmul(sy, sy);
    const double sxx = dadd(dadd(dmul(dmul(sx2, cth), cth), dmul(dmul(sy2, sth), sth)), kEpsCov);
    const double sxy = dmul(dmul(dsub(sx2, sy2), cth), sth);
    const double syy = dadd(dadd(dmul(dmul(sx2, sth), sth), dmul(dmul(sy2, cth), cth)), kEpsCov);
    // invert_covariance (:56-68)
    const double det = dsub(dmul(sxx, syy), dmul(sxy, sxy));
    const double det_safe = fmax(det, kEpsDet);
    const double i00 = ddiv(syy, det_safe), i01 = ddiv(-sxy, det_safe), i11 = ddiv(sxx, det_safe);
    const double mid = dmul(0.5, dadd(sxx, syy));
    const double half_diff = dmul(0.5, dsub(sxx, syy));
    const double lmax = dadd(mid, __dsqrt_rn(fmax(dadd(dmul(half_diff, half_diff), dmul(sxy, sxy)), 0.0)));
    const double radius3 = dmul(3.0, __dsqrt_rn(fmax(lmax, 0.0)));
    // activate_opacity: 1 / (1 + exp(-pre))   (:26-29)
    const double alpha = ddiv(1.0, dadd(1.0, exp(-po)));
    // rasterizer.cpp:74-77
    const double cutoff = dmul(2.0, fmax(log(dmul(255.0, alpha)), 0.0));
    const double mahal_cutoff = dadd(cutoff, kMahalSlack);
    const double sigma = ddiv(radius3, 3.0);
    const double r = dadd(dmul(sigma, __dsqrt_rn(fmax(9.0, cutoff))), 1.0);

    // build_index bounds (rasterizer.cpp:95-103)
    int tx0 = static_cast<int>(floor(ddiv(dsub(px, r), static_cast<double>(kTile))));
    int tx1 = static_cast<int>(floor(ddiv(dadd(px, r), static_cast<double>(kTile))));
    int ty0 = static_cast<int>(floor(ddiv(dsub(py, r), static_cast<double>(kTile))));
    int ty1 = static_cast<int>(floor(ddiv(dadd(py, r), static_cast<double>(kTile))));
    tx0 = max(tx0, 0);
    ty0 = max(ty0, 0);
    tx1 = min(tx1, P.tiles_x - 1);
    ty1 = min(ty1, P.tiles_y - 1);
    P.tbox[g] = make_int4(tx0, tx1, ty0, ty1);  // per-tile counts: count_tiles_kernel
    // pixel bbox (rasterizer.cpp:157-160, 209-212)
    const int x0 = max(0, static_cast<int>(ceil(dsub(px, r))));
    const int x1 = min(P.width - 1, static_cast<int>(floor(dadd(px, r))));
    const int y0 = max(0, static_cast<int>(ceil(dsub(py, r))));
    const int y1 = min(P.height - 1, static_cast<int>(floor(dadd(py, r))));
    P.pbox[g] = make_int4(x0, x1, y0, y1);

    // fp32 shading record.  px = px_hi + px_lo so (x - px_hi) - px_lo is the
    // correctly-rounded fp32 offset of an integer pixel.
    const float px_hi = static_cast<float>(px), py_hi = static_cast<float>(py);
    const float px_lo = static_cast<float>(px - static_cast<double>(px_hi));
    const float py_lo = static_cast<float>(py - static_cast<double>(py_hi));
    // fp32 error band of the quadratic form: a few ulp of its largest term,
    // whose size relative to mahal is bounded by the condition number.
    const double lmin = fmax(mid - sqrt(fmax(half_diff * half_diff + sxy * sxy, 0.0)), 1e-300);
    const double cond = fmin(lmax / lmin, 1e12);
    const double tol = 5e-7 * (1.0 + cond) * (1.0 + cutoff) + 1e-6;
    const double det_inv = i00 * i11 - i01 * i01;
    // SoA records (coalesced stores; the kernels gather them by Gaussian id)
    P.rec[g] = make_float4(px_hi, py_hi, px_lo, py_lo);
    P.rec[N + g] = make_float4(static_cast<float>(i00), static_cast<float>(i01),
                               static_cast<float>(i11), static_cast<float>(mahal_cutoff));
    const float4 q0 = make_float4(px_hi, py_hi, px_lo, py_lo);
    const float4 q1 = make_float4(static_cast<float>(i00), static_cast<float>(i01), static_cast<float>(i11),
                                  static_cast<float>(mahal_cutoff));
    const float4 q2 = make_float4(static_cast<float>(log2(alpha)), static_cast<float>(tol),
                                  static_cast<float>(det_inv), static_cast<float>(1.0 / i00));
    P.rec[2 * N + g] = q2;
    if (P.trows) P.trows[g] = tight_rows(q0, q1, q2, tx0, tx1, ty0, ty1);
    double* q = P.p64 + g;
    q[0] = px; q[N] = py; q[2 * N] = i00; q[3 * N] = i01; q[4 * N] = i11; q[5 * N] = mahal_cutoff;
    q[6 * N] = alpha; q[7 * N] = r;
    if (!finite(th)) atomicOr(P.status + 2, 1u);
    // per-channel shading (rasterizer.cpp:78-85), fused unless the amplitude /
    // phase groups may still be uploading (then shade_kernel runs after them)
    if (P.fuse_shade) shade_one(P.params, g, P.n, P.c, P.shade, P.status);
}

// ---------------------------------------------------------------------------
// K1: tile binning (build_index, rasterizer.cpp:90-119).  The projection
// kernel counts the Gaussians of every tile (atomics); one CTA scans the
// counts into per-tile offsets and writes ranges ({0,0} for empty tiles, as
// the reference); a scatter drops each Gaussian id into its tiles' segments;
// each tile's segment is then sorted ascending in shared memory.  (tile, id)
// pairs are unique, so the result equals the reference's std::sort order
// exactly, independent of the scatter order.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) tile_scan_kernel(const uint32_t* __restrict__ tcount, int tiles,
                                                                 uint32_t* __restrict__ toffset,
                                                                 uint2* __restrict__ ranges,
                                                                 uint32_t* __restrict__ status, int64_t cap) {
    // each thread scans a contiguous run of tiles (16-byte loads and stores
    // when the run is a whole number of 4-tile groups: the counts are read
    // twice, from L1/L2, instead of being held in registers); one block scan
    // joins the runs
    using BSc = cub::BlockScan<unsigned long long, kScanThreads>;
    __shared__ typename BSc::TempStorage tmp;
    const int per = (tiles + kScanThreads - 1) / kScanThreads;
    const int t0 = threadIdx.x * per, t1 = min(t0 + per, tiles);
    const bool vec = (per % 4) == 0 && t1 - t0 == per;
    unsigned long long run = 0;
    if (vec) {
#pragma unroll 4
        for (int i = 0; i < per; i += 4) {
            const uint4 q = *reinterpret_cast<const uint4*>(tcount + t0 + i);
            run += static_cast<unsigned long long>(q.x) + q.y + q.z + q.w;
        }
    } else {
        for (int t = t0; t < t1; ++t) run += tcount[t];
    }
    unsigned long long ex, agg;
    BSc(tmp).ExclusiveSum(run, ex, agg);
    auto range = [](unsigned long long e, uint32_t c) {
        return c ? make_uint2(static_cast<uint32_t>(e), static_cast<uint32_t>(e + c)) : make_uint2(0u, 0u);
    };
    if (vec) {
#pragma unroll 2
        for (int i = 0; i < per; i += 4) {
            const uint4 q = *reinterpret_cast<const uint4*>(tcount + t0 + i);
            const unsigned long long e0 = ex, e1 = e0 + q.x, e2 = e1 + q.y, e3 = e2 + q.z;
            ex = e3 + q.w;
            *reinterpret_cast<uint4*>(toffset + t0 + i) = make_uint4(static_cast<uint32_t>(e0), static_cast<uint32_t>(e1),
                                                                     static_cast<uint32_t>(e2), static_cast<uint32_t>(e3));
            const uint2 r0 = range(e0, q.x), r1 = range(e1, q.y), r2 = range(e2, q.z), r3 = range(e3, q.w);
            reinterpret_cast<uint4*>(ranges + t0 + i)[0] = make_uint4(r0.x, r0.y, r1.x, r1.y);
            reinterpret_cast<uint4*>(ranges + t0 + i)[1] = make_uint4(r2.x, r2.y, r3.x, r3.y);
        }
    } else {
        for (int t = t0; t < t1; ++t) {
            const uint32_t v = tcount[t];
            toffset[t] = static_cast<uint32_t>(ex);
            ranges[t] = range(ex, v);
            ex += v;
        }
    }
    if (threadIdx.x == 0) {
        status[0] = static_cast<uint32_t>(agg > 0xffffffffull ? 0xffffffffull : agg);
        status[1] = agg > static_cast<unsigned long long>(cap) ? 1u : 0u;
    }
}

// Scatter (duplicate-with-keys, :94-108): tcount is consumed as a countdown.
// Per-tile Gaussian counts: 16 threads per Gaussian, one fire-and-forget
// atomic per (Gaussian, tile) pair.
constexpr int kScatterSub = 16;
// Tile rows [ty_lo, ty_hi] only (a row-slab rank bins its own band).
__device__ __forceinline__ int4 band_box(int4 b, int ty_lo, int ty_hi) {
    b.z = max(b.z, ty_lo);
    b.w = min(b.w, ty_hi);
    return b;
}
__device__ __forceinline__ int box_count(const int4& b) {
    const int nx = b.y - b.x + 1, ny = b.w - b.z + 1;
    return (nx > 0 && ny > 0) ? nx * ny : 0;
}

// Row-slab band: ids of the Gaussians whose pixel box meets rows [y0, y1]
// (warp-aggregated slots; the order is irrelevant: binning sorts each tile,
// the backward writes per id).
__global__ void band_list_kernel(int n, const int4* __restrict__ pbox, int y0, int y1, uint32_t* __restrict__ list,
                                 uint32_t* __restrict__ list_n) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    bool in = false;
    if (g < n) {
        const int4 b = pbox[g];
        in = b.z <= y1 && b.w >= y0 && b.x <= b.y;
    }
    const unsigned m = __ballot_sync(0xffffffffu, in);
    if (!m) return;
    unsigned base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(list_n, static_cast<unsigned>(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (in) list[base + __popc(m & ((1u << lane) - 1u))] = static_cast<uint32_t>(g);
}

// list (nullable): the Gaussians to bin, *list_n of them (a row-slab rank's band)
__device__ __forceinline__ int pick(int idx, int n, const uint32_t* list, const uint32_t* list_n) {
    if (list) return idx < static_cast<int>(*list_n) ? static_cast<int>(list[idx]) : -1;
    return idx < n ? idx : -1;
}

__global__ void __launch_bounds__(256) count_tiles_kernel(int n, const int4* __restrict__ tbox, int tiles_x,
                                                          uint32_t* __restrict__ tcount, int ty_lo, int ty_hi,
                                                          const uint32_t* __restrict__ list,
                                                          const uint32_t* __restrict__ list_n,
                                                          const uint4* __restrict__ trows) {
    const int g = pick(blockIdx.x * (256 / kScatterSub) + threadIdx.x / kScatterSub, n, list, list_n);
    const int sub = threadIdx.x % kScatterSub;
    if (g < 0) return;
    const int4 b0 = tbox[g];
    const int4 b = band_box(b0, ty_lo, ty_hi);
    const int nx = b.y - b.x + 1, cnt = box_count(b);
    const uint4 tr = trows ? trows[g] : make_uint4(0u, 0u, ~0u, ~0u);
    for (int k = sub; k < cnt; k += kScatterSub) {
        const int tx = b.x + k % nx, ty = b.z + k / nx;
        if (!tight_has(tr, tx, ty, b0.x, b0.z)) continue;
        atomicAdd(tcount + ty * tiles_x + tx, 1u);
    }
}

// 16 threads per Gaussian, thread k handling tiles k, k + 16, ... of its tile
// box: one slot atomic per thread in the common case, so the atomics' round
// trips overlap across many resident threads instead of chaining per Gaussian.
__global__ void __launch_bounds__(256) scatter_ids_kernel(int n, const int4* __restrict__ tbox, int tiles_x,
                                                          const uint32_t* __restrict__ toffset,
                                                          uint32_t* __restrict__ tcount,
                                                          const uint32_t* __restrict__ status,
                                                          uint32_t* __restrict__ ids, int ty_lo, int ty_hi,
                                                          const uint32_t* __restrict__ list,
                                                          const uint32_t* __restrict__ list_n,
                                                          const uint4* __restrict__ trows) {
    const int g = pick(blockIdx.x * (256 / kScatterSub) + threadIdx.x / kScatterSub, n, list, list_n);
    const int sub = threadIdx.x % kScatterSub;
    if (g < 0 || status[1]) return;
    const int4 b0 = tbox[g];
    const int4 b = band_box(b0, ty_lo, ty_hi);
    const int nx = b.y - b.x + 1, cnt = box_count(b);
    const uint4 tr = trows ? trows[g] : make_uint4(0u, 0u, ~0u, ~0u);
    for (int k = sub; k < cnt; k += kScatterSub) {
        const int tx = b.x + k % nx, ty = b.z + k / nx;
        if (!tight_has(tr, tx, ty, b0.x, b0.z)) continue;
        const int t = ty * tiles_x + tx;
        const uint32_t slot = atomicSub(tcount + t, 1u) - 1u;
        ids[toffset[t] + slot] = static_cast<uint32_t>(g);
    }
}

constexpr int kSegSmem = 4096;  // ids sorted in shared memory per tile

__device__ __forceinline__ void bitonic_smem(uint32_t* s, int P) {
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint32_t a = s[i], b = s[ixj];
                    if ((a > b) == ((i & k) == 0)) {
                        s[i] = b;
                        s[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
}

// Warp per tile for segments of <= 512 ids: an in-register bitonic network,
// PER ids per lane (element e = lane * PER + i); distances < PER are register
// swaps, larger ones use shuffles.
constexpr int kWarpSeg = 512;

template <int PER>
__device__ __forceinline__ void warp_bitonic(uint32_t* __restrict__ seg, int n, int lane) {
    constexpr int P = 32 * PER;
    uint32_t v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = lane * PER + i;
        v[i] = e < n ? seg[e] : 0xffffffffu;
    }
#pragma unroll
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= PER) {
                const int lj = j / PER;  // partner lane distance
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const int e = lane * PER + i;
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, v[i], lj);
                    const bool lower = (e & j) == 0;
                    const bool up = (e & k) == 0;
                    // keep min if (lower == up) else max
                    v[i] = (lower == up) ? min(v[i], o) : max(v[i], o);
                }
            } else {
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const int e = lane * PER + i;
                        const bool up = (e & k) == 0;
                        const uint32_t a = v[i], b = v[ixj];
                        const bool sw = (a > b) == up;
                        v[i] = sw ? b : a;
                        v[ixj] = sw ? a : b;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = lane * PER + i;
        if (e < n) seg[e] = v[i];
    }
}

__device__ void sort_big_tile(const uint2 r, uint32_t* __restrict__ ids, uint32_t* __restrict__ scratch) {
    __shared__ uint32_t s[kSegSmem];
    const int n = static_cast<int>(r.y - r.x);
    int P = 1;
    while (P < n) P <<= 1;
    if (P <= kSegSmem) {
        for (int i = threadIdx.x; i < P; i += blockDim.x) s[i] = i < n ? ids[r.x + i] : 0xffffffffu;
        __syncthreads();
        bitonic_smem(s, P);
        for (int i = threadIdx.x; i < n; i += blockDim.x) ids[r.x + i] = s[i];
        return;
    }
    // pathological tile (> kSegSmem Gaussians): same network in global memory,
    // on a private padded copy at scratch[2*begin, 2*begin + P)
    uint32_t* g = scratch + 2 * static_cast<size_t>(r.x);
    for (int i = threadIdx.x; i < P; i += blockDim.x) g[i] = i < n ? ids[r.x + i] : 0xffffffffu;
    __syncthreads();
    bitonic_smem(g, P);
    for (int i = threadIdx.x; i < n; i += blockDim.x) ids[r.x + i] = g[i];
}

// Warp per tile; tiles with more than kWarpSeg ids (rare) are collected and
// then sorted one after another by the whole CTA (8 tiles per CTA).
__global__ void __launch_bounds__(256) segment_sort_kernel(const uint2* __restrict__ ranges, int tiles,
                                                           uint32_t* __restrict__ ids, uint32_t* __restrict__ scratch,
                                                           const uint32_t* __restrict__ status) {
    __shared__ int s_big[8];
    __shared__ int s_nbig;
    if (status[1]) return;  // grid-uniform
    if (threadIdx.x == 0) s_nbig = 0;
    __syncthreads();
    const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (t < tiles) {
        const uint2 r = ranges[t];
        const int n = static_cast<int>(r.y - r.x);
        // network size by segment length (tight binning: ~100 ids per tile at cfg2)
        if (n > kWarpSeg) {
            if (lane == 0) s_big[atomicAdd(&s_nbig, 1)] = t;
        } else if (n > 1) {
            if (n <= 32) warp_bitonic<1>(ids + r.x, n, lane);
            else if (n <= 64) warp_bitonic<2>(ids + r.x, n, lane);
            else if (n <= 128) warp_bitonic<4>(ids + r.x, n, lane);
            else if (n <= 256) warp_bitonic<8>(ids + r.x, n, lane);
            else warp_bitonic<16>(ids + r.x, n, lane);
        }
    }
    __syncthreads();
    const int nb = s_nbig;
    for (int i = 0; i < nb; ++i) {
        sort_big_tile(ranges[s_big[i]], ids, scratch);
        __syncthreads();
    }
}

// build_tile_index export: CTA per tile writes its (tile, id) pairs + range.
__global__ void export_kernel(const uint32_t* __restrict__ ids, const uint2* __restrict__ ranges,
                              uint32_t* __restrict__ tiles_out, uint32_t* __restrict__ ids_out,
                              uint64_t* __restrict__ ranges_out) {
    const int t = blockIdx.x;
    const uint2 r = ranges[t];
    if (threadIdx.x == 0) {
        ranges_out[2 * static_cast<size_t>(t)] = r.x;
        ranges_out[2 * static_cast<size_t>(t) + 1] = r.y;
    }
    for (uint32_t i = r.x + threadIdx.x; i < r.y; i += blockDim.x) {
        tiles_out[i] = static_cast<uint32_t>(t);
        ids_out[i] = ids[i];
    }
}

// ---------------------------------------------------------------------------
// Exact fp64 contribution test (rasterizer.cpp:164-169 / :220-228).  Returns
// false when skipped; else G, saturation flag and alpha_eff in fp64.
// ---------------------------------------------------------------------------
// q = p64 + g, fields at stride n (SoA: px, py, i00, i01, i11, mahal_cutoff, alpha, r).
// Returns (G, alpha_eff, saturated, contributes) by value: the out-values stay
// in registers on the callers' fast paths (no local-memory round trip).
__device__ __noinline__ float4 exact_contrib4(const double* __restrict__ q, size_t n, int x, int y) {
    const double dx = dsub(static_cast<double>(x), q[0]);
    const double dy = dsub(static_cast<double>(y), q[n]);
    // dx * dx * i00 + 2.0 * dx * dy * i01 + dy * dy * i11
    const double mahal = dadd(dadd(dmul(dmul(dx, dx), q[2 * n]), dmul(dmul(dmul(2.0, dx), dy), q[3 * n])),
                              dmul(dmul(dy, dy), q[4 * n]));
    if (mahal > q[5 * n]) return make_float4(0.f, 0.f, 0.f, 0.f);
    const double power = fmax(dmul(-0.5, mahal), kPowerFloor);
    const double G = exp(power);
    const double aG = dmul(q[6 * n], G);
    const bool saturated = aG > kAlphaCap;
    const double aeff = saturated ? kAlphaCap : aG;
    return make_float4(static_cast<float>(G), static_cast<float>(aeff), saturated ? 1.f : 0.f,
                       aeff < kAlphaCutoff ? 0.f : 1.f);
}

// ---------------------------------------------------------------------------
// K2: forward.  One CTA per 16x16 tile, 4 warps, each warp an 8x8 cell (a
// lane owns two pixels of a column).  The tile's sorted Gaussian list is
// staged in shared memory 128 at a time; the staging thread of a Gaussian
// tests it against the tile's four cells (exact row-band ellipse bound,
// conservative) and stores the cell bits with Sigma^-1 repacked as aligned
// pairs and the cutoff band precomputed; each warp ballots its cell's bit over
// a 32-batch, walks the hits in ascending order and every lane evaluates its
// pixels.
// ---------------------------------------------------------------------------
constexpr int kFwdThreads = 128;  // 4 warps per 16x16 tile, each an 8x8 cell
constexpr int kFwdBatch = 128;


// staged Gaussian of the forward kernel (shared memory)
template <int C>
struct alignas(16) FwdRec {
    float4 r0;     // projection record r0 (centre, split)
    float4 iq;     // (i00, i01, i01, i11): both rows of Sigma^-1 as aligned pairs
    float4 q;      // (cut - tol, cut + tol, log2 alpha, bits: cells of the tile it can reach)
    float2 sh[C];  // (amp cos, amp sin) per channel
    uint32_t id;
};

template <int C>
__global__ void __launch_bounds__(kFwdThreads) raster_fwd_kernel(
    const uint32_t* __restrict__ ids, const uint2* __restrict__ ranges,
    const float4* __restrict__ rec, const float4* __restrict__ shade,
    const double* __restrict__ p64, int N, int tiles_x, int W, int H, float2* __restrict__ field, int y0,
    int hs, int ty0) {
    // one contiguous record per staged Gaussian: a hit reads it through one
    // base address with immediate offsets (lanes broadcast the same record)
    __shared__ FwdRec<C> s_g[kFwdBatch];
    // row band [y0, y0 + hs) of the canvas (the whole canvas unless row-slab
    // sharded); the grid covers its tile rows from ty0, the field holds its rows
    const int tile = blockIdx.x + ty0 * tiles_x;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cx0 = tx * kTile + (warp & 1) * 8;
    const int cy0 = ty * kTile + (warp >> 1) * 8;
    // each lane owns two pixels of its column: rows ly and ly + 4 of the cell
    const int x = cx0 + (lane & 7), y = cy0 + (lane >> 3);
    const float fx = static_cast<float>(x), fy = static_cast<float>(y);
    float2 accA[C], accB[C];
#pragma unroll
    for (int c = 0; c < C; ++c) accA[c] = accB[c] = make_float2(0.f, 0.f);
    const uint2 rg = ranges[tile];
    for (uint32_t base = rg.x; base < rg.y; base += kFwdBatch) {
        const int cnt = min(static_cast<int>(rg.y - base), kFwdBatch);
        __syncthreads();
        if (static_cast<int>(threadIdx.x) < cnt) {
            const uint32_t g = ids[base + threadIdx.x];
            FwdRec<C>& d = s_g[threadIdx.x];
            d.id = g;
            const float4 r0 = rec[g], r1 = rec[static_cast<size_t>(N) + g], r2 = rec[2 * static_cast<size_t>(N) + g];
            // the cells (warps) of this tile the Gaussian can reach
            uint32_t cm = 0u;
#pragma unroll
            for (int cl = 0; cl < 4; ++cl)
                if (cell_hit(r0, r1, r2, static_cast<float>(tx * kTile + (cl & 1) * 8),
                             static_cast<float>(ty * kTile + (cl >> 1) * 8), 7.f, 7.f))
                    cm |= 1u << cl;
            d.r0 = r0;
            d.iq = make_float4(r1.x, r1.y, r1.y, r1.z);
            d.q = make_float4(r1.w - r2.y, r1.w + r2.y, r2.x, __uint_as_float(cm));
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const float4 sh = shade[static_cast<size_t>(c) * N + g];
                d.sh[c] = make_float2(sh.x, sh.y);
            }
        }
        __syncthreads();
        for (int sub = 0; sub < cnt; sub += 32) {
            const int j = sub + lane;
            bool hit = false;
            if (j < cnt) hit = (__float_as_uint(s_g[j].q.w) >> warp) & 1u;
            uint32_t mask = __ballot_sync(0xffffffffu, hit);
            // fast fp32 alphas of hit jj for both pixels (rows y, y + 4); band = inside
            // the error band [cut - tol, cut + tol] (decided exactly afterwards)
            auto fast = [&](int jj, float& aA, float& aB, bool& bA, bool& bB) {
                const FwdRec<C>& G = s_g[jj];
                const float4 r0 = G.r0, iq = G.iq, q = G.q;
                const float dx = (fx - r0.x) - r0.z;
                const float dyA = (fy - r0.y) - r0.w;
                // both pixels (rows y, y + 4) as one fp32x2 pair: Sigma^-1 (dx, dy)
                // by component, then the quadratic forms and the exponents
                const float2 dy2 = make_float2(dyA, dyA + 4.f);
                const float2 ex = f2fma(dy2, f2splat(iq.y), f2splat(dx * iq.x));  // i00 dx + i01 dy
                const float2 ey = f2fma(dy2, f2splat(iq.w), f2splat(dx * iq.z));  // i01 dx + i11 dy
                const float2 m = f2fma(f2splat(dx), ex, f2mul(dy2, ey));
                const float2 arg = f2fma(m, f2splat(kNegHalfLog2e), f2splat(q.z));
                const float mA = m.x, mB = m.y;
                // alpha e^{-m/2} = 2^(log2 alpha - m / (2 ln 2))
                const float lo = q.x, hi = q.y;
                aA = mA <= lo ? fminf(0.99f, ex2f(arg.x)) : 0.f;
                aB = mB <= lo ? fminf(0.99f, ex2f(arg.y)) : 0.f;
                bA = mA > lo && mA <= hi;
                bB = mB > lo && mB <= hi;
            };
            auto exact = [&](int jj, float& aA, float& aB, bool bA, bool bB) {  // rare: fp64 decision
                const double* q = p64 + s_g[jj].id;
                if (bA) {
                    const float4 e4 = exact_contrib4(q, N, x, y);
                    aA = e4.w != 0.f ? e4.y : 0.f;
                }
                if (bB) {
                    const float4 e4 = exact_contrib4(q, N, x, y + 4);
                    aB = e4.w != 0.f ? e4.y : 0.f;
                }
            };
            auto accum = [&](int jj, float aA, float aB) {
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const float2 sh = s_g[jj].sh[c];
                    accA[c] = f2fma(f2splat(aA), sh, accA[c]);
                    accB[c] = f2fma(f2splat(aB), sh, accB[c]);
                }
            };
            while (mask) {  // warp-uniform: hits in ascending id order, two per iteration
                const int j1 = sub + __ffs(mask) - 1;
                mask &= mask - 1;
                float a1A, a1B;
                bool b1A, b1B;
                fast(j1, a1A, a1B, b1A, b1B);
                if (mask) {
                    const int j2 = sub + __ffs(mask) - 1;
                    mask &= mask - 1;
                    float a2A, a2B;
                    bool b2A, b2B;
                    fast(j2, a2A, a2B, b2A, b2B);
                    if (__any_sync(0xffffffffu, b1A || b1B || b2A || b2B)) {
                        exact(j1, a1A, a1B, b1A, b1B);
                        exact(j2, a2A, a2B, b2A, b2B);
                    }
                    accum(j1, a1A, a1B);
                    accum(j2, a2A, a2B);
                } else {
                    if (__any_sync(0xffffffffu, b1A || b1B)) exact(j1, a1A, a1B, b1A, b1B);
                    accum(j1, a1A, a1B);
                }
            }
        }
    }
    (void)H;
    if (x < W) {
        const int ya = y - y0, yb = y + 4 - y0;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (ya >= 0 && ya < hs) field[(static_cast<size_t>(c) * hs + ya) * W + x] = accA[c];
            if (yb >= 0 && yb < hs) field[(static_cast<size_t>(c) * hs + yb) * W + x] = accB[c];
        }
    }
}

// ---------------------------------------------------------------------------
// K3: backward, one warp per Gaussian (rasterize_backward :201-284).
//
// The warp walks the Gaussian's exact ellipse footprint in bands of 32 rows:
// lane r computes row r's x-interval, the nonempty rows are compacted into a
// per-warp shared table (y, x - flat index), and the band's pixels are
// flattened so that every lane always has a pixel.  A lane finds the row of
// its flat pixel with two warp reductions per 32-pixel chunk (row starts
// inside the chunk as a bitmask, rows before it as a count) and one popc.
// The per-pixel math runs on packed fp32x2 pairs: (dx, dy), the rows of
// Sigma^-1 (dx, dy), per channel (d_amp, d_phase), (gmx, gmy) and (ga, gc).
// ---------------------------------------------------------------------------
// One warp per CTA: footprints differ per Gaussian, and single-warp CTAs let
// every SM refill a finished warp's slot at once (32 resident, 64 registers).
// Measured at cfg2: 256-thread CTAs 312 us, 128: 296, 64: 290, 32: 282.
constexpr int kBwdThreads = 32;
constexpr int kBwdWarps = kBwdThreads / 32;
constexpr int kBwdGrab = 4;  // Gaussians per work-counter atomic

// LIST: a row-slab rank walks only the Gaussians of its band list (the
// other raw sums were zeroed before the launch).
// One Gaussian of the backward walk (one warp).
template <int C, bool LIST>
__device__ __forceinline__ void raster_bwd_one(int g, int N, const float4* __restrict__ rec,
                                               const float4* __restrict__ shade, const double* __restrict__ p64,
                                               const int4* __restrict__ pbox, int W, int H,
                                               const float2* __restrict__ gfield, float* __restrict__ raw, int y0,
                                               int hs) {
    __shared__ int4 s_rows[kBwdWarps][32];  // compact nonempty rows (see the walk)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const float4 r0 = rec[g];
    const float4 r1 = rec[static_cast<size_t>(N) + g];
    const float4 r2 = rec[2 * static_cast<size_t>(N) + g];
    float2 S[C];  // (amp cos, amp sin) per channel
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const float4 sh = shade[static_cast<size_t>(c) * N + g];
        S[c] = make_float2(sh.x, sh.y);
    }
    const int4 bb = pbox[g];
    const float px = r0.x + r0.z, py = r0.y + r0.w;
    const float2 p_hi = make_float2(r0.x, r0.y), p_lo = make_float2(r0.z, r0.w);
    const float i00 = r1.x, i01 = r1.y, i11 = r1.z, cut = r1.w;
    const float2 row0 = make_float2(i00, i01), row1 = make_float2(i01, i11);
    const float alpha = exp2f(r2.x), tol = r2.y, detI = r2.z, inv_i00 = r2.w;  // r2.x = log2 alpha
    const float M = cut + tol;
    const float ratio = i01 * inv_i00;
    // channel planes of the gradient field: rows [y0, y0 + hs) of the canvas
    // (the whole canvas unless row-slab sharded), indexed by the band offset
    // (y - y0) W + x (32-bit) from the kernel parameter; channel c is c * cs further on
    (void)H;
    const unsigned cs = static_cast<unsigned>(hs) * static_cast<unsigned>(W);

    // Sg[c] = sum of alpha_eff * g_c over the footprint.  (d_amp, d_phase) are
    // linear in it with per-Gaussian coefficients, so they are formed once after
    // the walk: d_amp = cos Sg.re + sin Sg.im, d_phase = amp (cos Sg.im - sin Sg.re).
    float2 Sg[C];
#pragma unroll
    for (int c = 0; c < C; ++c) Sg[c] = make_float2(0.f, 0.f);
    float2 gm = make_float2(0.f, 0.f), gac = make_float2(0.f, 0.f);
    float d_alpha = 0.f, gb = 0.f;

    const float ext = sqrtf(fmaxf(i00 * M / detI, 0.f)) + 1e-2f;
    const int ya = max(max(bb.z, y0), static_cast<int>(ceilf(py - ext)));
    const int yb = min(min(bb.w, y0 + hs - 1), static_cast<int>(floorf(py + ext)));
    const double* q = p64 + g;
    const unsigned lanemask_le = 0xffffffffu >> (31 - lane);

    for (int ybase = ya; ybase <= yb; ybase += 32) {
        const int row = ybase + lane;
        int xl = 0, wdt = 0;
        if (row <= yb) {
            const float dy = static_cast<float>(row) - py;
            const float D = i00 * M - detI * dy * dy;
            if (D >= 0.f) {
                const float hw = sqrtf(D) * inv_i00 + 1e-2f;
                const float cen = px - ratio * dy;
                xl = max(bb.x, static_cast<int>(ceilf(cen - hw)));
                const int xr = min(bb.y, static_cast<int>(floorf(cen + hw)));
                wdt = max(0, xr - xl + 1);
            }
        }
        int incl = wdt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) continue;
        const int excl = incl - wdt;
        const unsigned nonempty = __ballot_sync(0xffffffffu, wdt > 0);
        __syncwarp();
        // row table: flat pixel f of this row sits at band offset f + .x and
        // column f + .y; .z = the row's exact dy = (y - py_hi) - py_lo, .w = y
        if (wdt > 0)
            s_rows[wid][__popc(nonempty & (lanemask_le >> 1))] =
                make_int4((row - y0) * W + xl - excl, xl - excl,
                          __float_as_int((static_cast<float>(row) - p_hi.y) - p_lo.y), row);
        __syncwarp();
        for (int cb = 0; cb < total; cb += 32) {
            const unsigned d = static_cast<unsigned>(excl - cb - 1);  // start strictly inside the chunk
            const unsigned bit = (wdt > 0 && d < 31u) ? 2u << d : 0u;
            const unsigned starts = __reduce_or_sync(0xffffffffu, bit);
            const int k0 = static_cast<int>(__reduce_add_sync(0xffffffffu, (wdt > 0 && excl <= cb) ? 1u : 0u)) - 1;
            const int f = cb + lane;
            if (f >= total) continue;
            const int4 info = s_rows[wid][k0 + __popc(starts & lanemask_le)];
            const int x = f + info.y;
            const float dxf = (static_cast<float>(x) - p_hi.x) - p_lo.x;
            const float2 dxy = make_float2(dxf, __int_as_float(info.z));
            const float2 e = f2fma(f2splat(dxy.x), row0, f2mul(f2splat(dxy.y), row1));  // Sigma^-1 (dx, dy)
            const float m = fmaf(dxy.x, e.x, dxy.y * e.y);
            if (m > M) continue;
            const float2* p = gfield + static_cast<unsigned>(f + info.x);
            float2 gv[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                gv[c] = __ldg(p);
                p += cs;
            }
            float G = ex2f(m * kNegHalfLog2e), aeff;
            bool sat;
            float aG = alpha * G;
            if (m <= cut - tol && fabsf(aG - 0.99f) > 1e-5f) {
                sat = aG > 0.99f;
                aeff = sat ? 0.99f : aG;
            } else {
                const float4 e4 = exact_contrib4(q, N, x, info.w);
                if (e4.w == 0.f) continue;
                G = e4.x;
                aG = alpha * G;
                aeff = e4.y;
                sat = e4.z != 0.f;
            }
            // s_amp = sum_c Re(conj(amp e^{i phi}) g_c), as packed pairs
            float2 sa = f2mul(S[0], gv[0]);
            Sg[0] = f2fma(f2splat(aeff), gv[0], Sg[0]);
#pragma unroll
            for (int c = 1; c < C; ++c) {
                Sg[c] = f2fma(f2splat(aeff), gv[c], Sg[c]);
                sa = f2fma(S[c], gv[c], sa);
            }
            const float s_amp = sa.x + sa.y;
            if (!sat) {
                d_alpha = fmaf(s_amp, G, d_alpha);
                const float qv = s_amp * aG;  // = -2 w of the reference (w = s_amp alpha G / -2)
                gm = f2fma(f2splat(qv), e, gm);
                gac = f2fma(f2splat(-0.5f * qv), f2mul(dxy, dxy), gac);
                gb = fmaf(-qv * dxy.x, dxy.y, gb);
            }
        }
    }
    // Transpose reduction: 16 shuffles fold the 7 + 2C partial sums (padded
    // to 16); afterwards lanes 2k, 2k+1 hold the warp total of value k.
    float v[16];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const float4 sh = shade[static_cast<size_t>(c) * N + g];  // (amp cos, amp sin, cos, sin)
        v[c] = fmaf(sh.z, Sg[c].x, sh.w * Sg[c].y);
        v[C + c] = fmaf(sh.x, Sg[c].y, -sh.y * Sg[c].x);
    }
    v[2 * C + 0] = d_alpha;
    v[2 * C + 1] = gm.x;
    v[2 * C + 2] = gm.y;
    v[2 * C + 3] = gac.x;
    v[2 * C + 4] = gb;
    v[2 * C + 5] = gac.y;
#pragma unroll
    for (int i = 2 * C + 6; i < 16; ++i) v[i] = 0.f;
#pragma unroll
    for (int half = 8; half >= 1; half >>= 1) {
        const bool hi = (lane & (2 * half)) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const float send = hi ? v[i] : v[i + half];
            const float keep = hi ? v[i + half] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * half);
        }
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    const int k = lane >> 1;
    if ((lane & 1) == 0 && k < 2 * C + 6) raw[static_cast<size_t>(k) * N + g] = v[0];
}

template <int C, int MINB, bool LIST = false>
__global__ void __launch_bounds__(kBwdThreads, MINB) raster_bwd_kernel(
    int N, const float4* __restrict__ rec, const float4* __restrict__ shade,
    const double* __restrict__ p64, const int4* __restrict__ pbox, int W, int H,
    const float2* __restrict__ gfield, float* __restrict__ raw, int y0, int hs,
    const uint32_t* __restrict__ list, const uint32_t* __restrict__ list_n, uint32_t* __restrict__ work) {
    // Band list (row-slab rank): persistent warps, each grabbing kBwdGrab list
    // entries per atomic on the work counter, so a short list launches no
    // empty CTAs (the list length is only known on the device).
    const int lane = threadIdx.x & 31;
    const int limit = LIST ? static_cast<int>(*list_n) : N;
    if constexpr (!LIST) {  // the whole set: one Gaussian per one-warp CTA (measured faster than persistent)
        if (static_cast<int>(blockIdx.x) < limit)
            raster_bwd_one<C, LIST>(blockIdx.x, N, rec, shade, p64, pbox, W, H, gfield, raw, y0, hs);
        return;
    }
    for (;;) {
        int base = 0;
        if (lane == 0) base = static_cast<int>(atomicAdd(work, static_cast<uint32_t>(kBwdGrab)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= limit) return;
        const int end = min(base + kBwdGrab, limit);
        for (int i = base; i < end; ++i)
            raster_bwd_one<C, LIST>(LIST ? static_cast<int>(list[i]) : i, N, rec, shade, p64, pbox, W, H, gfield,
                                    raw, y0, hs);
    }
}

// ---------------------------------------------------------------------------
// K3t: backward, per tile (the north_star form; the default trainer path).
// One warp per 16x16 tile, cells of 8x8 pixels as the forward.  The warp
// stages the tile's gradient (C channels) in shared memory and walks the
// tile's sorted Gaussian list 32 candidates at a time: each lane tests one
// candidate against the four cells (the forward's row-band bound) and the hits
// are compacted into one queue of (Gaussian, cell) entries.  Every 32 queued
// entries run as one batch with LANE = (GAUSSIAN, CELL): the lane walks the 64
// pixels of its cell row by row (gradient values from shared memory, staged
// pair-transposed -- (re0, re1, im0, im1) per pixel pair and channel, cells at
// a 4-bank shift -- so a pixel pair is one 16-byte load per channel and its
// weights, Sigma S.g and moments run as packed fp32x2; no global gathers),
// evaluates its Gaussian there with the fast fp32 decision (rows holding a
// pixel inside the error band, or a saturating one, are flagged and their
// band pixels redone with the fp64 decision afterwards, as K3) and
// accumulates the 7 + 2C partial sums in registers.  Only the tile's
// last batch runs partly empty.  The sums over the cell go to the Gaussian's
// row of an AoS [N][16] buffer with 16-byte vector atomics
// (red.global.add.v4.f32): the reduction over the cell's pixels happens in
// registers before one atomic per (cell, Gaussian, 4 values).  The last bits
// depend on the atomic order; K3 is the deterministic path.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void red_add_v4(float* dst, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

constexpr int kTb1Stride = 66;  // float2 per staged cell (64 + 2 pad: 16-byte pixel pairs, 4-bank shift per cell)
constexpr int kTb1Q = 160;      // queue: < 32 left over + 4 x 32 new entries

template <int C>
__global__ void __launch_bounds__(32, 16) raster_bwd_tile1w_kernel(
    const uint32_t* __restrict__ ids, const uint2* __restrict__ ranges, const float4* __restrict__ rec,
    const float4* __restrict__ shade, const double* __restrict__ p64, int N, int tiles_x, int W, int H,
    const float2* __restrict__ gfield, float* __restrict__ raw16, int y0, int hs, int ty0) {
    static_assert(2 * C + 6 <= 16, "AoS row of 16 floats");
    __shared__ __align__(16) float2 s_t[C][4 * kTb1Stride];
    __shared__ uint32_t s_q[kTb1Q];
    const int tile = blockIdx.x + ty0 * tiles_x;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int lane = threadIdx.x;
    const int ylo = max(y0, 0), yhi = min(y0 + hs, H);  // valid rows [ylo, yhi)
    const unsigned cs = static_cast<unsigned>(hs) * static_cast<unsigned>(W);
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // stage the tile's 256 pixels: cell = pix >> 6
        const int pix = lane + 32 * j, cell = pix >> 6, p = pix & 63;
        const int x = tx * kTile + (cell & 1) * 8 + (p & 7), y = ty * kTile + (cell >> 1) * 8 + (p >> 3);
        const bool ok = x < W && y >= ylo && y < yhi;
        const float2* src = gfield + (ok ? static_cast<unsigned>(y - y0) * static_cast<unsigned>(W) + x : 0u);
#pragma unroll
        for (int c = 0; c < C; ++c)
        {
            float* sc = reinterpret_cast<float*>(&s_t[c][cell * kTb1Stride]) + (p >> 1) * 4 + (p & 1);
            const float2 v = ok ? __ldg(src + static_cast<size_t>(c) * cs) : make_float2(0.f, 0.f);
            sc[0] = v.x;
            sc[2] = v.y;
        }
    }
    // cells with at least one valid pixel (warp-uniform)
    unsigned cell_ok = 0u;
#pragma unroll
    for (int cell = 0; cell < 4; ++cell) {
        const int cx = tx * kTile + (cell & 1) * 8, cy = ty * kTile + (cell >> 1) * 8;
        if (cx < W && max(cy, ylo) < min(cy + 8, yhi)) cell_ok |= 1u << cell;
    }
    __syncwarp();
    const uint2 rg = ranges[tile];
    int qn = 0;
    const unsigned lanemask_lt = (1u << lane) - 1u;
    auto batch = [&](int nb) {  // process s_q[0, nb)
        const bool act = lane < nb;
        const uint32_t e = act ? s_q[lane] : s_q[0];
        const uint32_t g = e >> 2;
        const int cell = static_cast<int>(e & 3u);
        const int cx0 = tx * kTile + (cell & 1) * 8, cy0 = ty * kTile + (cell >> 1) * 8;
        const float4 r0 = rec[g];
        const float4 r1 = rec[static_cast<size_t>(N) + g];
        const float4 r2 = rec[2 * static_cast<size_t>(N) + g];
        float2 S[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const float4 sh = shade[static_cast<size_t>(c) * N + g];
            S[c] = make_float2(sh.x, sh.y);
        }
        const float i00 = r1.x, i01 = r1.y, i11 = r1.z;
        const float cut = r1.w, tol = r2.y, l2a = r2.x, alpha = exp2f(r2.x);
        const float M = act ? cut + tol : -1.f;  // idle lanes never pass m <= M
        const float Mfast = cut - tol;
        const double* q = p64 + g;
        // per channel: (sum over even pixels, sum over odd pixels) of alpha_eff g re / im
        float2 SgRe[C], SgIm[C];
#pragma unroll
        for (int c = 0; c < C; ++c) SgRe[c] = SgIm[c] = make_float2(0.f, 0.f);
        float2 T1 = make_float2(0.f, 0.f), T2 = make_float2(0.f, 0.f);
        float QA = 0.f, T3 = 0.f;
        const float* gcell = reinterpret_cast<const float*>(&s_t[0][cell * kTb1Stride]);  // pair-transposed
        float dxk[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) dxk[k] = (static_cast<float>(cx0 + k) - r0.x) - r0.z;
        const float2 i00_2 = f2splat(i00), kx2 = f2splat(kNegHalfLog2e), l2a2 = f2splat(l2a);
        // the row terms of m = (i00 dx + bq) dx + cq: shared by the fast walk and
        // the exact pass so that both see the same fp32 m for a pixel
        auto row_terms = [&](float dy, float& bq, float& cq) {
            bq = 2.f * i01 * dy;
            cq = i11 * dy * dy;
        };
        // pixel fast/band decision (same in both passes): fast = inside the
        // cutoff by more than the tolerance and not saturating (SAT: the lane
        // can saturate at all); band = could contribute but not fast
        auto decide = [&](auto satc, float m, float aG, float Mfr, float Mr, bool& fast, bool& band) {
            fast = m <= Mfr;
            if constexpr (decltype(satc)::value) fast = fast && aG < 0.99f - 1e-5f;
            band = m <= Mr && !fast;
        };
        // rows holding a band pixel (bit r): redone exactly afterwards
        uint32_t rowmask = 0u;
        auto walk = [&](auto satc) {
#pragma unroll 1
            for (int r = 0; r < 8; ++r) {
                const int y = cy0 + r;
                const bool rowok = y >= ylo && y < yhi;
                const float Mr = rowok ? M : -1.f, Mfr = rowok ? Mfast : -1.f;
                const float dy = (static_cast<float>(y) - r0.y) - r0.w;
                float bq, cq;
                row_terms(dy, bq, cq);
                const float2 bq2 = f2splat(bq), cq2 = f2splat(cq);
                const float* gp = gcell + (r << 4);
                bool rb = false;
                float2 R0p = make_float2(0.f, 0.f), R1p = R0p, R2p = R0p;
#pragma unroll
                for (int k = 0; k < 8; k += 2) {
                    const float2 dxp = make_float2(dxk[k], dxk[k + 1]);
                    const float2 m2 = f2fma(f2fma(i00_2, dxp, bq2), dxp, cq2);
                    const float2 arg = f2fma(m2, kx2, l2a2);
                    const float aG0 = ex2f(arg.x), aG1 = ex2f(arg.y);  // alpha e^{-m/2}
                    // the pixel pair's gradient per channel: (re0, re1, im0, im1), one 16-byte load
                    float4 g4[C];
#pragma unroll
                    for (int c = 0; c < C; ++c) g4[c] = *reinterpret_cast<const float4*>(gp + c * 8 * kTb1Stride + 2 * k);
                    bool f0, b0, f1, b1;
                    decide(satc, m2.x, aG0, Mfr, Mr, f0, b0);
                    decide(satc, m2.y, aG1, Mfr, Mr, f1, b1);
                    rb = rb || b0 || b1;
                    const float2 w = make_float2(f0 ? aG0 : 0.f, f1 ? aG1 : 0.f);
                    float2 sx = f2mul(f2splat(S[0].x), make_float2(g4[0].x, g4[0].y));
                    float2 sy = f2mul(f2splat(S[0].y), make_float2(g4[0].z, g4[0].w));
                    SgRe[0] = f2fma(w, make_float2(g4[0].x, g4[0].y), SgRe[0]);
                    SgIm[0] = f2fma(w, make_float2(g4[0].z, g4[0].w), SgIm[0]);
#pragma unroll
                    for (int c = 1; c < C; ++c) {
                        const float2 gre = make_float2(g4[c].x, g4[c].y), gim = make_float2(g4[c].z, g4[c].w);
                        SgRe[c] = f2fma(w, gre, SgRe[c]);
                        SgIm[c] = f2fma(w, gim, SgIm[c]);
                        sx = f2fma(f2splat(S[c].x), gre, sx);
                        sy = f2fma(f2splat(S[c].y), gim, sy);
                    }
                    const float2 qv = f2mul(f2add(sx, sy), w);
                    R0p = f2add(R0p, qv);
                    R1p = f2fma(qv, dxp, R1p);
                    R2p = f2fma(qv, f2mul(dxp, dxp), R2p);
                }
                const float R0 = R0p.x + R0p.y;
                const float2 R12 = make_float2(R1p.x + R1p.y, R2p.x + R2p.y);
                QA += R0;
                T1 = f2add(T1, make_float2(R12.x, dy * R0));
                T2 = f2add(T2, make_float2(R12.y, dy * dy * R0));
                T3 = fmaf(dy, R12.x, T3);
                if (rb) rowmask |= 1u << r;
            }
        };
        // a Gaussian whose peak alpha is clearly below the cap cannot saturate
        // (alpha e^{-m/2} <= alpha, with margin for the fp32 m near 0)
        const bool sat_free = __all_sync(0xffffffffu, !act || alpha * 1.001f < 0.99f - 1e-5f);
        if (sat_free) walk(std::false_type{});
        else walk(std::true_type{});
        // rare: the exact fp64 decision for the band pixels of the flagged rows
        // (rasterizer.cpp:220-228)
        if (__any_sync(0xffffffffu, rowmask != 0u)) {
            const int xmax = W - cx0;
            for (uint32_t rm = rowmask; rm; rm &= rm - 1) {
                const int r = __ffs(rm) - 1, y = cy0 + r;
                const float dy = (static_cast<float>(y) - r0.y) - r0.w;
                float bq, cq;
                row_terms(dy, bq, cq);
                for (int k = 0; k < 8; ++k) {
                    if (k >= xmax) break;  // outside the canvas
                    const float dx = dxk[k];
                    const float m = fmaf(fmaf(i00, dx, bq), dx, cq);
                    const float aG = ex2f(fmaf(m, kNegHalfLog2e, l2a));
                    bool fast, band;
                    decide(std::true_type{}, m, aG, Mfast, M, fast, band);  // rows of the mask are valid rows
                    if (!band) continue;
                    const int pix = (r << 3) + k, x = cx0 + k;
                    const float4 e4 = exact_contrib4(q, N, x, y);
                    if (e4.w == 0.f) continue;
                    const float w = e4.y, qv0 = e4.z != 0.f ? 0.f : alpha * e4.x;
                    float2 gv[C];
                    const float* gq = gcell + (pix >> 1) * 4 + (pix & 1);
#pragma unroll
                    for (int c = 0; c < C; ++c) gv[c] = make_float2(gq[c * 8 * kTb1Stride], gq[c * 8 * kTb1Stride + 2]);
                    float2 sa = f2mul(S[0], gv[0]);
                    SgRe[0].x = fmaf(w, gv[0].x, SgRe[0].x);
                    SgIm[0].x = fmaf(w, gv[0].y, SgIm[0].x);
#pragma unroll
                    for (int c = 1; c < C; ++c) {
                        SgRe[c].x = fmaf(w, gv[c].x, SgRe[c].x);
                        SgIm[c].x = fmaf(w, gv[c].y, SgIm[c].x);
                        sa = f2fma(S[c], gv[c], sa);
                    }
                    const float qv = (sa.x + sa.y) * qv0;
                    QA += qv;
                    const float2 dxy = make_float2(dx, dy);
                    const float2 t = f2mul(f2splat(qv), dxy);
                    T1 = f2add(T1, t);
                    T2 = f2fma(t, dxy, T2);
                    T3 = fmaf(t.x, dy, T3);
                }
            }
        }
        if (act) {
            float v[16];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                v[c] = SgRe[c].x + SgRe[c].y;
                v[C + c] = SgIm[c].x + SgIm[c].y;
            }
            v[2 * C + 0] = alpha > 0.f ? QA / alpha : 0.f;
            v[2 * C + 1] = fmaf(i00, T1.x, i01 * T1.y);
            v[2 * C + 2] = fmaf(i01, T1.x, i11 * T1.y);
            v[2 * C + 3] = -0.5f * T2.x;
            v[2 * C + 4] = -T3;
            v[2 * C + 5] = -0.5f * T2.y;
#pragma unroll
            for (int i = 2 * C + 6; i < 16; ++i) v[i] = 0.f;
            float* dst = raw16 + static_cast<size_t>(g) * 16;
#pragma unroll
            for (int k = 0; k < (2 * C + 6 + 3) / 4; ++k) red_add_v4(dst + 4 * k, v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        }
    };
    for (uint32_t base = rg.x; base < rg.y; base += 32) {
        const uint32_t i = base + lane;
        uint32_t g = 0;
        float4 r0, r1, r2;
        const bool valid = i < rg.y;
        if (valid) {
            g = ids[i];
            r0 = rec[g];
            r1 = rec[static_cast<size_t>(N) + g];
            r2 = rec[2 * static_cast<size_t>(N) + g];
        }
#pragma unroll
        for (int cell = 0; cell < 4; ++cell) {
            const bool hit = valid && ((cell_ok >> cell) & 1u) &&
                             cell_hit(r0, r1, r2, static_cast<float>(tx * kTile + (cell & 1) * 8),
                                      static_cast<float>(ty * kTile + (cell >> 1) * 8), 7.f, 7.f);
            const unsigned mask = __ballot_sync(0xffffffffu, hit);
            if (hit) s_q[qn + __popc(mask & lanemask_lt)] = (g << 2) | static_cast<uint32_t>(cell);
            qn += __popc(mask);
        }
        __syncwarp();
        while (qn >= 32) {
            batch(32);
            __syncwarp();
            qn -= 32;
            for (int j = lane; j < qn; j += 32) s_q[j] = s_q[32 + j];
            __syncwarp();
        }
    }
    if (qn > 0) batch(qn);
}

// 1 - tanh^2 x = 4 e / (1 + e)^2 with e = e^{-2|x|}: relative accuracy of expf
// over the whole range (1 - tanhf^2 loses it once tanhf rounds near 1)
__device__ __forceinline__ double sech2_fd(float x) {
    const double e = expf(-2.f * fabsf(x));
    return 4.0 * e / ((1.0 + e) * (1.0 + e));
}
// e^x of an fp32 argument: expf where the result is a normal fp32, fp64 exp beyond
__device__ __forceinline__ double exp_fd(float x) {
    return fabsf(x) < 80.f ? static_cast<double>(expf(x)) : exp(static_cast<double>(x));
}

// AOS: the per-tile backward's [N][16] rows (sum alpha_eff g_c re/im instead of
// (d_amp, d_phase), converted here with the Gaussian's shading record).
template <int C, bool LIST = false, bool AOS = false>
__global__ void __launch_bounds__(256) raster_finalize_kernel(int N, const float* __restrict__ raw,
                                                               const float* __restrict__ params, int W, int H,
                                                               float* __restrict__ grads, uint32_t* flags,
                                                               const uint32_t* __restrict__ list = nullptr,
                                                               const uint32_t* __restrict__ list_n = nullptr,
                                                               const float4* __restrict__ shade = nullptr) {
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if constexpr (LIST) {  // row-slab rank: its band's Gaussians (the other gradients were zeroed)
        if (g >= static_cast<int>(*list_n)) return;
        g = static_cast<int>(list[g]);
    } else {
        if (g >= N) return;
    }
    const size_t Ns = N;
    // AoS: the Gaussian's 16-float row as four 16-byte loads
    float row[AOS ? 16 : 1];
    if constexpr (AOS) {
        const float4* r4 = reinterpret_cast<const float4*>(raw + static_cast<size_t>(g) * 16);
#pragma unroll
        for (int i = 0; i < (2 * C + 6 + 3) / 4; ++i) {
            const float4 v = r4[i];
            row[4 * i] = v.x;
            row[4 * i + 1] = v.y;
            row[4 * i + 2] = v.z;
            row[4 * i + 3] = v.w;
        }
    }
    auto R = [&](int k) {
        if constexpr (AOS) return static_cast<double>(row[k]);
        else return static_cast<double>(raw[static_cast<size_t>(k) * Ns + g]);
    };
    // (d_amp, d_phase) of channel c: stored (K3), or from sum alpha_eff g_c (K3t):
    // d_amp = cos Sg.re + sin Sg.im, d_phase = amp (cos Sg.im - sin Sg.re)
    auto DA = [&](int c) {
        if constexpr (!AOS) return R(c);
        const float4 sh = shade[static_cast<size_t>(c) * Ns + g];
        return static_cast<double>(sh.z) * R(c) + static_cast<double>(sh.w) * R(C + c);
    };
    auto DP = [&](int c) {
        if constexpr (!AOS) return R(C + c);
        const float4 sh = shade[static_cast<size_t>(c) * Ns + g];
        return static_cast<double>(sh.x) * R(C + c) - static_cast<double>(sh.y) * R(c);
    };
    const double d_alpha = R(2 * C), gmx = R(2 * C + 1), gmy = R(2 * C + 2);
    const double ga = R(2 * C + 3), gb = R(2 * C + 4), gc = R(2 * C + 5);
    const float* pp = params;
    const float* ps = pp + 2 * Ns;
    const float* rot = ps + 2 * Ns;
    const float* amp = rot + Ns;
    const float* pha = amp + Ns * C;
    const float* opa = pha + Ns * C;
    (void)pha;
    float* gpp = grads;
    float* gps = gpp + 2 * Ns;
    float* grot = gps + 2 * Ns;
    float* gamp = grot + Ns;
    float* gpha = gamp + Ns * C;
    float* gopa = gpha + Ns * C;
    uint32_t bad = 0;
    auto put = [&](float* dst, double v, int group) {
        const float f = static_cast<float>(v);
        if (!isfinite(f)) bad |= 1u << group;
        *dst = f;
    };
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const size_t i = static_cast<size_t>(g) * C + c;
        const float rawp = amp[i];
        put(gamp + i, (rawp >= 0.f && rawp <= 1.f) ? DA(c) : 0.0, 3);
        put(gpha + i, DP(c), 4);
    }
    // Transcendentals of the fp32 parameters in fp32 (correctly rounded to
    // ~1 ulp: perturbs every derived fp64 quantity by ~1e-7 relative, far
    // inside the 1e-3 gradient tolerance; the covariance algebra below stays
    // fp64, so det keeps its fp64 cancellation behaviour); exp falls back to
    // fp64 where fp32 would overflow.  One fp64 division instead of six (all forms).
    // (trainer's per-tile form only: the stand-alone rasterize_backward and the
    // deterministic gather keep the fp64 transcendentals of the reference)
    const double sig = 1.0 / (1.0 + (AOS ? exp_fd(-opa[g]) : exp(-static_cast<double>(opa[g]))));
    put(gopa + g, d_alpha * (sig * (1.0 - sig)), 5);
    auto sech2 = [](float x) {
        if constexpr (AOS) return sech2_fd(x);
        const double t = tanh(static_cast<double>(x));
        return 1.0 - t * t;
    };
    auto expd = [](float x) {
        if constexpr (AOS) return exp_fd(x);
        return exp(static_cast<double>(x));
    };
    put(gpp + 2 * g, gmx * (0.5 * W * sech2(pp[2 * g])), 0);
    put(gpp + 2 * g + 1, gmy * (0.5 * H * sech2(pp[2 * g + 1])), 0);
    const double esx = expd(ps[2 * g]), esy = expd(ps[2 * g + 1]);
    const double sx = esx + kEpsScale, sy = esy + kEpsScale;
    double ct, st;
    if constexpr (AOS) {
        float sf, cf;
        sincosf(rot[g], &sf, &cf);
        ct = cf;
        st = sf;
    } else {
        sincos(static_cast<double>(rot[g]), &st, &ct);
    }
    const double sx2 = sx * sx, sy2 = sy * sy;
    const double c00 = sx2 * ct * ct + sy2 * st * st + kEpsCov;
    const double c01 = (sx2 - sy2) * ct * st;
    const double c11 = sx2 * st * st + sy2 * ct * ct + kEpsCov;
    const double det = c00 * c11 - c01 * c01;
    const double dsafe = fmax(det, kEpsDet);
    const double t_adj = ga * c11 - gb * c01 + gc * c00;
    const double clamped = det > kEpsDet ? 1.0 : 0.0;
    const double inv = 1.0 / dsafe;
    const double ti2 = t_adj * clamped * (inv * inv);
    const double gS00 = gc * inv - ti2 * c11;
    const double gS01 = -gb * inv + ti2 * 2.0 * c01;
    const double gS11 = ga * inv - ti2 * c00;
    const double dsx = 2.0 * sx * (ct * ct * gS00 + ct * st * gS01 + st * st * gS11);
    const double dsy = 2.0 * sy * (st * st * gS00 - ct * st * gS01 + ct * ct * gS11);
    put(gps + 2 * g, dsx * esx, 1);
    put(gps + 2 * g + 1, dsy * esy, 1);
    put(grot + g, 2.0 * (sy2 - sx2) * ct * st * gS00 + (sx2 - sy2) * (ct * ct - st * st) * gS01 +
                      2.0 * (sx2 - sy2) * ct * st * gS11,
        2);
    if (bad && flags) atomicOr(flags, bad);
}

int bits_for(int64_t v) {
    int b = 1;
    while ((int64_t(1) << b) <= v) ++b;
    return b;
}

}  // namespace

void RasterWork::prepare(int n_, int c_, int w_, int h_) {
    require(c_ >= 1 && c_ <= kMaxChannels,
            "rasterizer: channel count " + std::to_string(c_) + " outside 1..4");
    n = n_;
    c = c_;
    width = w_;
    height = h_;
    tiles_x = (w_ + kTile - 1) / kTile;
    tiles_y = (h_ + kTile - 1) / kTile;
    tile_bits = bits_for(static_cast<int64_t>(tiles_x) * tiles_y - 1);
    const size_t N = std::max(n, 1);
    rec.reserve(N * 3 * sizeof(float4));
    shade.reserve(N * c * sizeof(float4));
    p64.reserve(N * 8 * sizeof(double));
    pbox.reserve(N * sizeof(int4));
    tbox.reserve(N * sizeof(int4));
    trows.reserve(N * sizeof(uint4));
    raw.reserve(N * (2 * c + 6) * sizeof(float));
    tcount.reserve(static_cast<size_t>(tiles_x) * tiles_y * sizeof(uint32_t));
    toffset.reserve(static_cast<size_t>(tiles_x) * tiles_y * sizeof(uint32_t));
    ranges.reserve(static_cast<size_t>(tiles_x) * tiles_y * sizeof(uint2));
    status.reserve(4 * sizeof(uint32_t));
    work.reserve(sizeof(uint32_t));
    raw16.reserve(N * 16 * sizeof(float));
    if (sms == 0) {
        int dev = 0;
        HS_CUDA(cudaGetDevice(&dev));
        sms = sm_count(dev);
    }
    if (cap == 0) reserve_pairs(std::max<int64_t>(int64_t(1) << 20, 16 * static_cast<int64_t>(N)));
}

void RasterWork::reserve_pairs(int64_t cap_) {
    if (cap_ <= cap) return;
    cap = cap_;
    ids.reserve(static_cast<size_t>(cap) * sizeof(uint32_t));
    scratch.reserve(2 * static_cast<size_t>(cap) * sizeof(uint32_t));
}

void RasterWork::project_and_bin(const float* d_params, cudaStream_t st, cudaEvent_t shading_ready) {
    uint32_t* stat = status.as<uint32_t>();
    HS_CUDA(cudaMemsetAsync(stat, 0, 4 * sizeof(uint32_t), st));
    const int tiles = tiles_x * tiles_y;
    if (n == 0) {
        HS_CUDA(cudaMemsetAsync(ranges.p, 0, static_cast<size_t>(tiles) * sizeof(uint2), st));
        return;
    }
    HS_CUDA(cudaMemsetAsync(tcount.p, 0, static_cast<size_t>(tiles) * sizeof(uint32_t), st));
    ProjParams P{d_params, n,  c,  width, height, tiles_x, tiles_y, rec.as<float4>(),
                 shade.as<float4>(), p64.as<double>(), pbox.as<int4>(), tbox.as<int4>(),
                 tcount.as<uint32_t>(), stat, shading_ready ? 0 : 1, tight ? trows.as<uint4>() : nullptr};
    project_kernel<<<ceil_div(n, 128), 128, 0, st>>>(P);
    launch_check("project");
    const uint32_t* lst = nullptr;
    const uint32_t* lst_n = nullptr;
    if (banded()) {
        band_list.reserve(sizeof(uint32_t) * n);
        band_n.reserve(sizeof(uint32_t));
        HS_CUDA(cudaMemsetAsync(band_n.p, 0, sizeof(uint32_t), st));
        band_list_kernel<<<ceil_div(n, 256), 256, 0, st>>>(n, pbox.as<int4>(), band_y0, band_y1,
                                                             band_list.as<uint32_t>(), band_n.as<uint32_t>());
        launch_check("band_list");
        lst = band_list.as<uint32_t>();
        lst_n = band_n.as<uint32_t>();
    }
    count_tiles_kernel<<<ceil_div(n, 256 / kScatterSub), 256, 0, st>>>(n, tbox.as<int4>(), tiles_x,
                                                                       tcount.as<uint32_t>(), band_ty0, band_ty1, lst,
                                                                       lst_n, tight ? trows.as<uint4>() : nullptr);
    launch_check("count_tiles");
    tile_scan_kernel<<<1, kScanThreads, 0, st>>>(tcount.as<uint32_t>(), tiles, toffset.as<uint32_t>(), ranges.as<uint2>(),
                                         stat, cap);
    launch_check("tile_scan");
    scatter_ids_kernel<<<ceil_div(n, 256 / kScatterSub), 256, 0, st>>>(n, tbox.as<int4>(), tiles_x, toffset.as<uint32_t>(),
                                                         tcount.as<uint32_t>(), stat, ids.as<uint32_t>(), band_ty0,
                                                         band_ty1, lst, lst_n, tight ? trows.as<uint4>() : nullptr);
    launch_check("scatter_ids");
    segment_sort_kernel<<<ceil_div(tiles, 8), 256, 0, st>>>(ranges.as<uint2>(), tiles, ids.as<uint32_t>(),
                                                             scratch.as<uint32_t>(), stat);
    launch_check("segment_sort");
    if (shading_ready) {  // amplitude/phase uploaded: shade now (else project_kernel did)
        HS_CUDA(cudaStreamWaitEvent(st, shading_ready, 0));
        shade_kernel<<<ceil_div(n, 256), 256, 0, st>>>(d_params, n, c, shade.as<float4>(), stat);
        launch_check("shade");
    }
}

void export_tile_index(const RasterWork& rw, int64_t k, uint32_t* d_tiles, uint32_t* d_ids,
                       uint64_t* d_ranges, cudaStream_t st) {
    (void)k;
    const int tiles = rw.tiles_x * rw.tiles_y;
    if (tiles == 0) return;
    export_kernel<<<tiles, 128, 0, st>>>(rw.ids.as<uint32_t>(), rw.ranges.as<uint2>(), d_tiles, d_ids, d_ranges);
    launch_check("export_tile_index");
}

template <int C>
static void fwd_launch(const RasterWork& rw, float2* d_field, int y0, int hs, cudaStream_t st) {
    const int ty0 = y0 / kTile, ty1 = (y0 + hs - 1) / kTile;
    raster_fwd_kernel<C><<<rw.tiles_x * (ty1 - ty0 + 1), kFwdThreads, 0, st>>>(
        rw.ids.as<uint32_t>(), rw.ranges.as<uint2>(), rw.rec.as<float4>(), rw.shade.as<float4>(),
        rw.p64.as<double>(), rw.n, rw.tiles_x, rw.width, rw.height, d_field, y0, hs, ty0);
    launch_check("raster_fwd");
}

void raster_forward(const RasterWork& rw, float2* d_field, cudaStream_t st, int y0, int hs) {
    if (hs < 0) hs = rw.height - y0;
    require(y0 >= 0 && hs >= 1 && y0 + hs <= rw.height, "rasterizer: row band outside the canvas");
    switch (rw.c) {
        case 1: fwd_launch<1>(rw, d_field, y0, hs, st); break;
        case 2: fwd_launch<2>(rw, d_field, y0, hs, st); break;
        case 3: fwd_launch<3>(rw, d_field, y0, hs, st); break;
        case 4: fwd_launch<4>(rw, d_field, y0, hs, st); break;
        default: throw Error(HS_EINVAL, "rasterizer: unsupported channel count");
    }
}

template <int C>
static void bwd_launch(const RasterWork& rw, const float* d_params, const float2* d_gf,
                       float* d_grads, uint32_t* d_flags, int y0, int hs, cudaStream_t st) {
    // persistent: 32 one-warp CTAs per SM (the register-limited residency)
    const int grid = std::max(1, std::min(static_cast<int>(ceil_div(rw.n, kBwdGrab)), 32 * rw.sms));
    uint32_t* work = rw.work.as<uint32_t>();
    if (rw.banded()) {
        HS_CUDA(cudaMemsetAsync(work, 0, sizeof(uint32_t), st));  // row-slab rank: only the band's Gaussians; the others' gradients are zero
        const int64_t P = static_cast<int64_t>(rw.n) * (6 + 2 * C);
        HS_CUDA(cudaMemsetAsync(d_grads, 0, sizeof(float) * P, st));
        if (rw.tile_bwd) {  // the band's tiles (binned for the band only) with the per-tile backward
            const int ty0 = y0 / kTile, ty1 = (y0 + hs - 1) / kTile;
            float* r16 = rw.raw16.as<float>();
            HS_CUDA(cudaMemsetAsync(r16, 0, sizeof(float) * 16 * static_cast<size_t>(rw.n), st));
            raster_bwd_tile1w_kernel<C><<<rw.tiles_x * (ty1 - ty0 + 1), 32, 0, st>>>(
                rw.ids.as<uint32_t>(), rw.ranges.as<uint2>(), rw.rec.as<float4>(), rw.shade.as<float4>(),
                rw.p64.as<double>(), rw.n, rw.tiles_x, rw.width, rw.height, d_gf, r16, y0, hs, ty0);
            launch_check("raster_bwd_tile");
            raster_finalize_kernel<C, true, true><<<ceil_div(rw.n, 256), 256, 0, st>>>(
                rw.n, r16, d_params, rw.width, rw.height, d_grads, d_flags, rw.band_list.as<uint32_t>(),
                rw.band_n.as<uint32_t>(), rw.shade.as<float4>());
            launch_check("raster_finalize");
            return;
        }
        raster_bwd_kernel<C, 32, true><<<grid, kBwdThreads, 0, st>>>(
            rw.n, rw.rec.as<float4>(), rw.shade.as<float4>(), rw.p64.as<double>(), rw.pbox.as<int4>(), rw.width,
            rw.height, d_gf, rw.raw.as<float>(), y0, hs, rw.band_list.as<uint32_t>(), rw.band_n.as<uint32_t>(), work);
        launch_check("raster_bwd");
        raster_finalize_kernel<C, true><<<ceil_div(rw.n, 256), 256, 0, st>>>(
            rw.n, rw.raw.as<float>(), d_params, rw.width, rw.height, d_grads, d_flags, rw.band_list.as<uint32_t>(),
            rw.band_n.as<uint32_t>());
        launch_check("raster_finalize");
        return;
    }
    if (rw.tile_bwd) {  // per-tile backward with vector atomics into the AoS rows
        const int ty0 = y0 / kTile, ty1 = (y0 + hs - 1) / kTile;
        float* r16 = rw.raw16.as<float>();
        HS_CUDA(cudaMemsetAsync(r16, 0, sizeof(float) * 16 * static_cast<size_t>(rw.n), st));
        raster_bwd_tile1w_kernel<C><<<rw.tiles_x * (ty1 - ty0 + 1), 32, 0, st>>>(
            rw.ids.as<uint32_t>(), rw.ranges.as<uint2>(), rw.rec.as<float4>(), rw.shade.as<float4>(),
            rw.p64.as<double>(), rw.n, rw.tiles_x, rw.width, rw.height, d_gf, r16, y0, hs, ty0);
        launch_check("raster_bwd_tile");
        raster_finalize_kernel<C, false, true><<<ceil_div(rw.n, 256), 256, 0, st>>>(
            rw.n, r16, d_params, rw.width, rw.height, d_grads, d_flags, nullptr, nullptr, rw.shade.as<float4>());
        launch_check("raster_finalize");
        return;
    }
    raster_bwd_kernel<C, 32><<<rw.n, kBwdThreads, 0, st>>>(
        rw.n, rw.rec.as<float4>(), rw.shade.as<float4>(), rw.p64.as<double>(), rw.pbox.as<int4>(), rw.width,
        rw.height, d_gf, rw.raw.as<float>(), y0, hs, nullptr, nullptr, work);
    launch_check("raster_bwd");
    raster_finalize_kernel<C><<<ceil_div(rw.n, 256), 256, 0, st>>>(rw.n, rw.raw.as<float>(), d_params, rw.width,
                                                                   rw.height, d_grads, d_flags);
    launch_check("raster_finalize");
}

void raster_backward(const RasterWork& rw, const float* d_params, const float2* d_grad_field,
                     float* d_grads, uint32_t* d_flags, cudaStream_t st, int y0, int hs) {
    if (rw.n == 0) return;
    if (hs < 0) hs = rw.height - y0;
    require(y0 >= 0 && hs >= 1 && y0 + hs <= rw.height, "rasterizer: row band outside the canvas");
    switch (rw.c) {
        case 1: bwd_launch<1>(rw, d_params, d_grad_field, d_grads, d_flags, y0, hs, st); break;
        case 2: bwd_launch<2>(rw, d_params, d_grad_field, d_grads, d_flags, y0, hs, st); break;
        case 3: bwd_launch<3>(rw, d_params, d_grad_field, d_grads, d_flags, y0, hs, st); break;
        case 4: bwd_launch<4>(rw, d_params, d_grad_field, d_grads, d_flags, y0, hs, st); break;
        default: throw Error(HS_EINVAL, "rasterizer: unsupported channel count");
    }
}

}  // namespace hs
