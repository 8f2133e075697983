// holosplat-b200 C++ drop-in (libholo_b200.so): the reference's holo:: API
// (proj/core/include/holo/*.hpp) implemented over the C ABI of
// libholosplat.so.  Host containers stay fp64 like the reference; values are
// rounded to fp32 for the device, results are widened back.  The hot-path
// calls (rasterizer, propagation, loss, Adan) always run on the B200 -- there
// is no CPU fallback; the scalar helpers of field_core and the transfer
// function sampler are host code, as in the reference.
#include <algorithm>
#include <cmath>
#include <iterator>
#include <fstream>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "holo/complex_field.hpp"
#include "holo/convert.hpp"
#include "holo/field_core.hpp"
#include "holo/gaussian_set.hpp"
#include "holo/io.hpp"
#include "holo/loss.hpp"
#include "holo/optimizer.hpp"
#include "holo/parallel.hpp"
#include "holo/pipeline.hpp"
#include "holo/propagation.hpp"
#include "holo/rasterizer.hpp"
#include "holosplat.h"

namespace holo {

namespace {

void check(hs_status s) {
    if (s == HS_OK) return;
    const std::string msg = hs_last_error();
    if (s == HS_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

hs_ctx* ctx() {
    static std::once_flag once;
    static hs_ctx* c = nullptr;
    std::call_once(once, [] {
        const char* env = std::getenv("HOLO_B200_DEVICE");
        check(hs_ctx_create(env ? std::atoi(env) : 0, &c));
    });
    return c;
}

// Device buffers of the value-semantics calls come from a grow-only cache
// (power-of-two size classes): after the first call of a given size the drop-in
// performs no cudaMalloc/cudaFree (which would also synchronise the device).
class DevPool {
  public:
    void* take(size_t bytes, size_t* cls) {
        *cls = size_class(bytes);
        {
            std::lock_guard<std::mutex> lock(mu_);
            auto it = free_.find(*cls);
            if (it != free_.end() && !it->second.empty()) {
                void* p = it->second.back();
                it->second.pop_back();
                return p;
            }
        }
        void* p = nullptr;
        check(hs_device_alloc(ctx(), *cls, &p));
        return p;
    }
    void give(void* p, size_t cls) {
        std::lock_guard<std::mutex> lock(mu_);
        free_[cls].push_back(p);
    }

  private:
    static size_t size_class(size_t b) {
        size_t c = 256;
        while (c < b) c <<= 1;
        return c;
    }
    std::mutex mu_;
    std::map<size_t, std::vector<void*>> free_;
};

DevPool& pool() {
    static DevPool* p = new DevPool;  // never destroyed: outlives every Dev, no teardown-order hazards
    return *p;
}

// RAII device buffer from the pool.
struct Dev {
    void* p = nullptr;
    size_t bytes = 0, cls = 0;
    explicit Dev(size_t b) : bytes(b) { p = pool().take(std::max<size_t>(b, 4), &cls); }
    ~Dev() {
        if (p) pool().give(p, cls);
    }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    Dev(Dev&& o) noexcept : p(o.p), bytes(o.bytes), cls(o.cls) { o.p = nullptr; }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    void upload(const void* h, size_t b) { check(hs_copy_h2d(ctx(), p, h, b)); }
    void download(void* h, size_t b) const { check(hs_copy_d2h(ctx(), h, p, b)); }
};

std::vector<float> flat_params(const GaussianSet& s) {
    std::vector<float> f;
    f.reserve(s.pre_position.size() + s.pre_scale.size() + s.rotation.size() + s.amplitude.size() +
              s.phase.size() + s.pre_opacity.size());
    for (const auto* v : {&s.pre_position, &s.pre_scale, &s.rotation, &s.amplitude, &s.phase, &s.pre_opacity})
        for (double x : *v) f.push_back(static_cast<float>(x));
    return f;
}

GaussianSet unflatten(const std::vector<float>& f, int n, int c) {
    GaussianSet g(n, c);
    size_t o = 0;
    for (auto* v : {&g.pre_position, &g.pre_scale, &g.rotation, &g.amplitude, &g.phase, &g.pre_opacity})
        for (double& x : *v) x = f[o++];
    return g;
}

Dev upload_params(const GaussianSet& s) {
    s.validate();
    const std::vector<float> f = flat_params(s);
    Dev d(f.size() * sizeof(float));
    d.upload(f.data(), f.size() * sizeof(float));
    return d;
}

// planar fp64 (re, im) -> interleaved complex64 on the device
Dev upload_field(const std::vector<const ComplexField*>& fs) {
    size_t n = 0;
    for (auto* f : fs) n += f->size();
    std::vector<float> h(2 * n);
    size_t o = 0;
    for (auto* f : fs)
        for (size_t i = 0; i < f->size(); ++i, ++o) {
            h[2 * o] = static_cast<float>(f->real[i]);
            h[2 * o + 1] = static_cast<float>(f->imag[i]);
        }
    Dev d(h.size() * sizeof(float));
    d.upload(h.data(), h.size() * sizeof(float));
    return d;
}

void download_field(const Dev& d, size_t offset_elems, ComplexField& f) {
    std::vector<float> h(2 * f.size());
    check(hs_copy_d2h(ctx(), h.data(), static_cast<float*>(d.p) + 2 * offset_elems, h.size() * sizeof(float)));
    for (size_t i = 0; i < f.size(); ++i) {
        f.real[i] = h[2 * i];
        f.imag[i] = h[2 * i + 1];
    }
}

struct SpecHolder {
    hs_prop_spec s{};
    std::vector<double> wl;
    explicit SpecHolder(const PropagationSpec& p) : wl(p.wavelengths) {
        s.wavelengths = wl.data();
        s.n_wavelengths = static_cast<int>(wl.size());
        s.pixel_pitch = p.pixel_pitch;
        s.pad_factor = p.pad_factor;
        s.aperture_radius = p.aperture_radius;
    }
};

}  // namespace

// ---- gaussian_set (gaussian_set.cpp:9-57) -----------------------------------------------------
GaussianSet::GaussianSet(int n, int c) : count(n), channels(c) {
    if (n < 0 || c <= 0) throw std::invalid_argument("GaussianSet: invalid N or C");
    const size_t N = static_cast<size_t>(n);
    pre_position.assign(2 * N, 0.0);
    pre_scale.assign(2 * N, 0.0);
    rotation.assign(N, 0.0);
    amplitude.assign(N * c, 0.0);
    phase.assign(N * c, 0.0);
    pre_opacity.assign(N, 0.0);
}

void GaussianSet::validate() const {
    if (count < 0 || channels <= 0) throw std::invalid_argument("GaussianSet: invalid N or C");
    const size_t n = static_cast<size_t>(count);
    const struct {
        const std::vector<double>* v;
        size_t want;
        const char* name;
    } groups[] = {{&pre_position, 2 * n, "pre_position"}, {&pre_scale, 2 * n, "pre_scale"},
                  {&rotation, n, "rotation"},           {&amplitude, n * channels, "amplitude"},
                  {&phase, n * channels, "phase"},      {&pre_opacity, n, "pre_opacity"}};
    for (const auto& g : groups) {
        if (g.v->size() != g.want) throw std::invalid_argument(std::string("GaussianSet: bad size for ") + g.name);
        for (double x : *g.v)
            if (!std::isfinite(x))
                throw std::invalid_argument(std::string("GaussianSet: non-finite entry in ") + g.name);
    }
}

GaussianSet GaussianSet::concat(const GaussianSet& a, const GaussianSet& b) {
    if (a.channels != b.channels) throw std::invalid_argument("GaussianSet::concat: channel mismatch");
    GaussianSet out(a.count + b.count, a.channels);
    auto join = [](std::vector<double>& d, const std::vector<double>& x, const std::vector<double>& y) {
        std::copy(x.begin(), x.end(), d.begin());
        std::copy(y.begin(), y.end(), d.begin() + x.size());
    };
    join(out.pre_position, a.pre_position, b.pre_position);
    join(out.pre_scale, a.pre_scale, b.pre_scale);
    join(out.rotation, a.rotation, b.rotation);
    join(out.amplitude, a.amplitude, b.amplitude);
    join(out.phase, a.phase, b.phase);
    join(out.pre_opacity, a.pre_opacity, b.pre_opacity);
    return out;
}

// ---- field_core (field_core.cpp:11-93), host scalar math ------------------------------------------
double activate_position(double pre, double extent) {
    if (!std::isfinite(pre)) throw std::invalid_argument("activate_position: non-finite input");
    return (std::tanh(pre) + 1.0) * 0.5 * extent;
}
double activate_position_deriv(double pre, double extent) {
    const double t = std::tanh(pre);
    return 0.5 * extent * (1.0 - t * t);
}
double activate_scale(double pre) {
    if (!std::isfinite(pre)) throw std::invalid_argument("activate_scale: non-finite input");
    return std::exp(pre) + kEpsScale;
}
double activate_scale_deriv(double pre) { return std::exp(pre); }
double activate_opacity(double pre) {
    if (!std::isfinite(pre)) throw std::invalid_argument("activate_opacity: non-finite input");
    return 1.0 / (1.0 + std::exp(-pre));
}
double activate_opacity_deriv(double pre) {
    const double s = activate_opacity(pre);
    return s * (1.0 - s);
}
double activate_amplitude(double raw) { return std::min(std::max(raw, 0.0), 1.0); }
double activate_amplitude_deriv(double raw) { return (raw >= 0.0 && raw <= 1.0) ? 1.0 : 0.0; }
double unactivate_position(double value, double extent) { return std::atanh(2.0 * value / extent - 1.0); }

Covariance2 covariance(double sx, double sy, double theta) {
    const double c = std::cos(theta), s = std::sin(theta), a = sx * sx, b = sy * sy;
    return Covariance2{a * c * c + b * s * s + kEpsCov, (a - b) * c * s, a * s * s + b * c * c + kEpsCov};
}

CovarianceInverse invert_covariance(const Covariance2& cv) {
    const double det = cv.sxx * cv.syy - cv.sxy * cv.sxy;
    const double d = std::max(det, kEpsDet);
    CovarianceInverse o;
    o.inv = InverseCovariance2{cv.syy / d, -cv.sxy / d, cv.sxx / d};
    const double mid = 0.5 * (cv.sxx + cv.syy), half = 0.5 * (cv.sxx - cv.syy);
    const double lmax = mid + std::sqrt(std::max(half * half + cv.sxy * cv.sxy, 0.0));
    o.radius = 3.0 * std::sqrt(std::max(lmax, 0.0));
    return o;
}

ActivatedGaussian activate(const GaussianSet& set, int n, int width, int height) {
    if (n < 0 || n >= set.count) throw std::out_of_range("activate: primitive index");
    ActivatedGaussian g;
    g.position[0] = activate_position(set.pre_position[2 * n], width);
    g.position[1] = activate_position(set.pre_position[2 * n + 1], height);
    g.scale[0] = activate_scale(set.pre_scale[2 * n]);
    g.scale[1] = activate_scale(set.pre_scale[2 * n + 1]);
    g.rotation = set.rotation[n];
    g.opacity = activate_opacity(set.pre_opacity[n]);
    for (int c = 0; c < set.channels; ++c) {
        const size_t i = static_cast<size_t>(n) * set.channels + c;
        g.amplitude.push_back(activate_amplitude(set.amplitude[i]));
        g.phase.push_back(set.phase[i]);
    }
    return g;
}

RealField intensity_of(const ComplexField& u) {
    RealField out(u.channels, u.height, u.width);
    Dev f = upload_field({&u});
    Dev o(u.size() * sizeof(float));
    check(hs_intensity(ctx(), f.as<float>(), static_cast<int64_t>(u.size()), o.as<float>()));
    std::vector<float> h(u.size());
    o.download(h.data(), h.size() * sizeof(float));
    std::copy(h.begin(), h.end(), out.values.begin());
    return out;
}

// ---- rasterizer ---------------------------------------------------------------------------------------
TileIndex build_tile_index(const GaussianSet& set, int width, int height) {
    if (width <= 0 || height <= 0) throw std::invalid_argument("build_tile_index: empty canvas");
    Dev p = upload_params(set);
    int64_t k = 0;
    int txy[2] = {0, 0};
    check(hs_build_tile_index(ctx(), p.as<float>(), set.count, set.channels, width, height, nullptr, nullptr,
                              nullptr, -1, &k, txy));
    TileIndex idx;
    idx.tiles_x = txy[0];
    idx.tiles_y = txy[1];
    const size_t tiles = static_cast<size_t>(txy[0]) * txy[1];
    Dev dt(std::max<int64_t>(k, 1) * 4), di(std::max<int64_t>(k, 1) * 4), dr(tiles * 16);
    check(hs_build_tile_index(ctx(), p.as<float>(), set.count, set.channels, width, height, dt.as<uint32_t>(),
                              di.as<uint32_t>(), dr.as<uint64_t>(), k, &k, txy));
    std::vector<uint32_t> t(k), id(k);
    std::vector<uint64_t> r(2 * tiles);
    if (k) {
        dt.download(t.data(), k * 4);
        di.download(id.data(), k * 4);
    }
    dr.download(r.data(), r.size() * 8);
    idx.pairs.resize(k);
    for (int64_t i = 0; i < k; ++i) idx.pairs[i] = {t[i], id[i]};
    idx.ranges.resize(tiles);
    for (size_t i = 0; i < tiles; ++i) idx.ranges[i] = {static_cast<size_t>(r[2 * i]), static_cast<size_t>(r[2 * i + 1])};
    return idx;
}

ComplexField rasterize_forward(const GaussianSet& set, int width, int height) {
    if (width <= 0 || height <= 0) throw std::invalid_argument("rasterize_forward: empty canvas");
    ComplexField out(set.channels, height, width);
    if (set.count == 0) return out;
    Dev p = upload_params(set);
    Dev f(out.size() * 2 * sizeof(float));
    check(hs_rasterize_forward(ctx(), p.as<float>(), set.count, set.channels, width, height, f.as<float>()));
    download_field(f, 0, out);
    return out;
}

GaussianSetGrads rasterize_backward(const GaussianSet& set, const RealField& grad_real,
                                    const RealField& grad_imag) {
    if (!grad_real.same_shape(grad_imag) || grad_real.channels != set.channels)
        throw std::invalid_argument("rasterize_backward: gradient shape mismatch");
    if (set.count == 0) return GaussianSetGrads(0, set.channels);
    ComplexField g(grad_real.channels, grad_real.height, grad_real.width);
    g.real = grad_real.values;
    g.imag = grad_imag.values;
    Dev p = upload_params(set);
    Dev gf = upload_field({&g});
    const size_t np = p.bytes / sizeof(float);
    Dev out(np * sizeof(float));
    check(hs_rasterize_backward(ctx(), p.as<float>(), set.count, set.channels, grad_real.width, grad_real.height,
                                gf.as<float>(), out.as<float>()));
    std::vector<float> h(np);
    out.download(h.data(), np * sizeof(float));
    return unflatten(h, set.count, set.channels);
}

// ---- propagation ----------------------------------------------------------------------------------------
std::vector<TransferFunctionSample> transfer_function(const PropagationSpec& spec, double distance, int channel,
                                                      int padded_nx, int padded_ny) {
    // transfer_function, propagation.cpp:157-172 (make_band_limit :54-70, kz_of :72-75) on the host (test-facing sampler)
    if (padded_nx <= 0 || padded_ny <= 0) throw std::invalid_argument("transfer_function: non-positive dims");
    if (channel < 0 || channel >= static_cast<int>(spec.wavelengths.size()))
        throw std::invalid_argument("propagation: channel has no wavelength");
    const double lambda = spec.wavelengths[channel];
    if (lambda <= 0.0 || spec.pixel_pitch <= 0.0)
        throw std::invalid_argument("propagation: non-positive wavelength or pitch");
    const double two_pi = 6.283185307179586476925286766559;
    const double k = two_pi / lambda, lx = padded_nx * spec.pixel_pitch, ly = padded_ny * spec.pixel_pitch;
    const double fx_max = 1.0 / (lambda * std::sqrt((2.0 * distance / lx) * (2.0 * distance / lx) + 1.0));
    const double fy_max = 1.0 / (lambda * std::sqrt((2.0 * distance / ly) * (2.0 * distance / ly) + 1.0));
    std::vector<TransferFunctionSample> grid(static_cast<size_t>(padded_nx) * padded_ny);
    for (int iy = 0; iy < padded_ny; ++iy)
        for (int ix = 0; ix < padded_nx; ++ix) {
            auto& s = grid[static_cast<size_t>(iy) * padded_nx + ix];
            s.fx = (ix - padded_nx / 2) * (1.0 / lx);
            s.fy = (iy - padded_ny / 2) * (1.0 / ly);
            const double kz2 = k * k - two_pi * two_pi * (s.fx * s.fx + s.fy * s.fy);
            s.kz = kz2 > 0.0 ? std::sqrt(kz2) : 0.0;
            s.inside_bandlimit = std::abs(s.fx) < fx_max && std::abs(s.fy) < fy_max;
        }
    return grid;
}

static ComplexField propagate_mode(const ComplexField& field, const PropagationSpec& spec, int mode, double d,
                                   double md) {
    SpecHolder sh(spec);
    if (field.channels != sh.s.n_wavelengths)
        throw std::invalid_argument("propagation: channel count does not match wavelengths");
    Dev in = upload_field({&field});
    Dev out(in.bytes);
    check(hs_propagate(ctx(), &sh.s, mode, d, md, in.as<float>(), field.channels, field.height, field.width,
                       out.as<float>()));
    ComplexField o(field.channels, field.height, field.width);
    download_field(out, 0, o);
    return o;
}

ComplexField propagate(const ComplexField& field, const PropagationSpec& spec, double distance) {
    return propagate_mode(field, spec, 0, distance, distance);
}
ComplexField propagate_with_mask_distance(const ComplexField& field, const PropagationSpec& spec, double distance,
                                          double mask_distance) {
    return propagate_mode(field, spec, 1, distance, mask_distance);
}
ComplexField propagate_backward(const ComplexField& grad_out, const PropagationSpec& spec, double distance) {
    return propagate_mode(grad_out, spec, 2, distance, distance);
}

std::vector<ComplexField> propagate_multi(const ComplexField& field, const PropagationSpec& spec,
                                          const std::vector<double>& distances) {
    SpecHolder sh(spec);
    const int L = static_cast<int>(distances.size());
    Dev in = upload_field({&field});
    Dev out(in.bytes * std::max(L, 1));
    check(hs_propagate_multi(ctx(), &sh.s, distances.data(), L, in.as<float>(), field.channels, field.height,
                             field.width, out.as<float>()));
    std::vector<ComplexField> o(distances.size(), ComplexField(field.channels, field.height, field.width));
    for (int l = 0; l < L; ++l) download_field(out, static_cast<size_t>(l) * field.size(), o[l]);
    return o;
}

ComplexField propagate_multi_backward(const std::vector<ComplexField>& grads, const PropagationSpec& spec,
                                      const std::vector<double>& distances) {
    if (grads.empty() || grads.size() != distances.size())
        throw std::invalid_argument("propagate_multi_backward: plane count mismatch");
    std::vector<const ComplexField*> ptrs;
    for (const auto& g : grads) {
        if (!g.same_shape(grads[0])) throw std::invalid_argument("propagate_multi_backward: gradient shape mismatch");
        ptrs.push_back(&g);
    }
    SpecHolder sh(spec);
    Dev in = upload_field(ptrs);
    Dev out(grads[0].size() * 2 * sizeof(float));
    check(hs_propagate_multi_backward(ctx(), &sh.s, distances.data(), static_cast<int>(distances.size()),
                                      in.as<float>(), grads[0].channels, grads[0].height, grads[0].width,
                                      out.as<float>()));
    ComplexField o(grads[0].channels, grads[0].height, grads[0].width);
    download_field(out, 0, o);
    return o;
}

// ---- loss ---------------------------------------------------------------------------------------------------
DepthPlaneSet make_depth_planes(int count, double center_distance, double spacing) {
    if (count < 1) throw std::invalid_argument("make_depth_planes: count must be >= 1");
    DepthPlaneSet p{count, center_distance, spacing, {}};
    for (int l = 0; l < count; ++l) p.distances.push_back(center_distance + (l - (count - 1) * 0.5) * spacing);
    return p;
}

MaskStack build_masks(const RealField& depth, int plane_count, bool near_is_high) {
    if (plane_count < 1) throw std::invalid_argument("build_masks: plane count must be >= 1");
    const size_t n = static_cast<size_t>(depth.height) * depth.width;
    if (depth.channels != 1 || depth.values.size() != n)
        throw std::invalid_argument("build_masks: depth must be a single plane");
    std::vector<uint8_t> flat(n * plane_count);
    check(hs_build_masks(depth.values.data(), depth.height, depth.width, plane_count, near_is_high ? 1 : 0,
                         flat.data()));
    MaskStack m(plane_count);
    for (int l = 0; l < plane_count; ++l) m[l].assign(flat.begin() + l * n, flat.begin() + (l + 1) * n);
    return m;
}

TargetStack make_target_stack(const RealField& intensity, const RealField& depth, int plane_count,
                              bool near_is_high) {
    if (depth.height != intensity.height || depth.width != intensity.width)
        throw std::invalid_argument("make_target_stack: depth/intensity size mismatch");
    return TargetStack{intensity, depth, build_masks(depth, plane_count, near_is_high)};
}

static double run_loss(int kind, const std::vector<RealField>& recon, const TargetStack& target,
                       std::vector<RealField>* grads) {
    if (recon.empty()) throw std::invalid_argument("loss: no reconstruction planes");
    if (recon.size() != target.masks.size()) throw std::invalid_argument("loss: plane count does not match masks");
    for (const auto& r : recon)
        if (!r.same_shape(target.intensity)) throw std::invalid_argument("loss: reconstruction shape mismatch");
    const int L = static_cast<int>(recon.size());
    const RealField& t = target.intensity;
    const size_t n = t.values.size(), hw = static_cast<size_t>(t.height) * t.width;
    std::vector<float> hr(n * L), ht(n);
    for (int l = 0; l < L; ++l)
        for (size_t i = 0; i < n; ++i) hr[l * n + i] = static_cast<float>(recon[l].values[i]);
    for (size_t i = 0; i < n; ++i) ht[i] = static_cast<float>(t.values[i]);
    std::vector<uint8_t> hm(hw * L);
    for (int l = 0; l < L; ++l) std::copy(target.masks[l].begin(), target.masks[l].end(), hm.begin() + l * hw);
    Dev dr(hr.size() * 4), dt(ht.size() * 4), dm(hm.size()), dg(hr.size() * 4);
    dr.upload(hr.data(), hr.size() * 4);
    dt.upload(ht.data(), ht.size() * 4);
    dm.upload(hm.data(), hm.size());
    double v = 0.0;
    check(hs_loss(ctx(), kind, L, t.channels, t.height, t.width, dr.as<float>(), dt.as<float>(), dm.as<uint8_t>(),
                  grads ? dg.as<float>() : nullptr, &v));
    if (grads) {
        std::vector<float> hg(hr.size());
        dg.download(hg.data(), hg.size() * 4);
        grads->assign(L, RealField(t.channels, t.height, t.width));
        for (int l = 0; l < L; ++l)
            for (size_t i = 0; i < n; ++i) (*grads)[l].values[i] = hg[l * n + i];
    }
    return v;
}

double loss_mse(const std::vector<RealField>& r, const TargetStack& t) { return run_loss(3, r, t, nullptr); }
double loss_recon(const std::vector<RealField>& r, const TargetStack& t) { return run_loss(1, r, t, nullptr); }
double loss_ssim(const std::vector<RealField>& r, const TargetStack& t) { return run_loss(2, r, t, nullptr); }
double training_loss(const std::vector<RealField>& r, const TargetStack& t) { return run_loss(0, r, t, nullptr); }
double loss_mse_grad(const std::vector<RealField>& r, const TargetStack& t, std::vector<RealField>& g) {
    return run_loss(3, r, t, &g);
}
double loss_recon_grad(const std::vector<RealField>& r, const TargetStack& t, std::vector<RealField>& g) {
    return run_loss(1, r, t, &g);
}
double loss_ssim_grad(const std::vector<RealField>& r, const TargetStack& t, std::vector<RealField>& g) {
    return run_loss(2, r, t, &g);
}
double training_loss_grad(const std::vector<RealField>& r, const TargetStack& t, std::vector<RealField>& g) {
    return run_loss(0, r, t, &g);
}

double plane_recon_loss(const RealField& recon, const TargetStack& target, size_t plane, RealField* grad) {
    // plane_recon_loss, loss.cpp:331-354: the single-plane recon term (w = 2/n)
    if (!recon.same_shape(target.intensity)) throw std::invalid_argument("plane_recon_loss: shape mismatch");
    if (plane >= target.masks.size()) throw std::invalid_argument("plane_recon_loss: plane out of range");
    TargetStack one{target.intensity, target.depth, MaskStack{target.masks[plane]}};
    std::vector<RealField> g;
    const double v = run_loss(1, {recon}, one, grad ? &g : nullptr);
    if (grad) *grad = g[0];
    return v;
}

double ssim_value(const RealField& a, const RealField& b) {
    // ssim_value, loss.cpp:356-369 = 1 - loss_ssim of one plane
    if (!a.same_shape(b)) throw std::invalid_argument("ssim_value: shape mismatch");
    TargetStack t{b, RealField(1, b.height, b.width), MaskStack(1, std::vector<uint8_t>(
                                                                  static_cast<size_t>(b.height) * b.width, 0))};
    return 1.0 - run_loss(2, {a}, t, nullptr);
}

// ---- optimizer -------------------------------------------------------------------------------------------------
double cosine_lr(int step, int total_steps, double lr_max, double lr_min) {
    double v = 0.0;
    check(hs_cosine_lr(step, total_steps, lr_max, lr_min, &v));
    return v;
}

struct Adan::Impl {
    struct Group {
        std::string name;
        double lr = 0.0;
        int t = 0;
        size_t size = 0;
        void* state = nullptr;  // 4 * size floats on the device
    };
    std::vector<Group> groups;
    ~Impl() {
        for (auto& g : groups)
            if (g.state) hs_device_free(ctx(), g.state);
    }
    Group& find(const std::string& n) {
        for (auto& g : groups)
            if (g.name == n) return g;
        throw std::invalid_argument("Adan: unknown group " + n);
    }
};

Adan::Adan(AdanConfig cfg) : cfg_(cfg), impl_(std::make_unique<Impl>()) {}
Adan::~Adan() = default;
Adan::Adan(Adan&&) noexcept = default;
Adan& Adan::operator=(Adan&&) noexcept = default;

void Adan::add_group(const std::string& name, size_t size, double lr) {
    for (const auto& g : impl_->groups)
        if (g.name == name) throw std::invalid_argument("Adan: duplicate group " + name);
    Impl::Group g;
    g.name = name;
    g.lr = lr;
    g.size = size;
    check(hs_device_alloc(ctx(), std::max<size_t>(4 * size, 1) * sizeof(float), &g.state));
    std::vector<float> zeros(4 * size, 0.f);
    if (size) check(hs_copy_h2d(ctx(), g.state, zeros.data(), zeros.size() * sizeof(float)));
    impl_->groups.push_back(std::move(g));
}
void Adan::set_lr(const std::string& name, double lr) { impl_->find(name).lr = lr; }
double Adan::lr(const std::string& name) const { return impl_->find(name).lr; }
int Adan::step_count(const std::string& name) const { return impl_->find(name).t; }

// The moments live on the device in fp32; the caller's fp64 parameters never
// pass through fp32: the kernel runs on a zero "parameter" buffer, so it
// returns -update, which is then applied to the fp64 values on the host
// (optimizer.cpp:69: params[i] -= lr * (...) / denom).
void Adan::step(const std::string& name, std::span<double> params, std::span<const double> grads) {
    Impl::Group& g = impl_->find(name);
    if (params.size() != g.size || grads.size() != g.size)
        throw std::invalid_argument("Adan: size mismatch for group " + name);
    std::vector<float> gr(grads.begin(), grads.end()), d(g.size, 0.f);
    Dev dd(d.size() * 4), dg(gr.size() * 4);
    dd.upload(d.data(), d.size() * 4);
    dg.upload(gr.data(), gr.size() * 4);
    hs_adan_config c{cfg_.beta1, cfg_.beta2, cfg_.beta3, cfg_.eps};
    check(hs_adan_step(ctx(), &c, name.c_str(), dd.as<float>(), dg.as<float>(), static_cast<float*>(g.state),
                       static_cast<int64_t>(g.size), g.t + 1, g.lr));
    g.t += 1;
    dd.download(d.data(), d.size() * 4);
    for (size_t i = 0; i < g.size; ++i) params[i] += static_cast<double>(d[i]);
}

// ---- parallel (parallel.cpp:11-44) ---------------------------------------------------------------------------------
namespace {
int g_threads = 0;
}
void set_thread_count(int n) { g_threads = n < 0 ? 0 : n; }
int thread_count() {
    int n = g_threads;
    if (n == 0) n = std::max(1u, std::thread::hardware_concurrency());
    return n;
}
void parallel_for(int64_t begin, int64_t end, const std::function<void(int64_t, int64_t)>& fn) {
    const int64_t count = end - begin;
    if (count <= 0) return;
    const int workers = static_cast<int>(std::min<int64_t>(thread_count(), count));
    const int64_t chunk = (count + workers - 1) / workers;
    std::vector<std::thread> pool;
    for (int w = 1; w < workers; ++w) {
        const int64_t lo = begin + w * chunk, hi = std::min(end, lo + chunk);
        if (lo < hi) pool.emplace_back(fn, lo, hi);
    }
    fn(begin, std::min(end, begin + chunk));
    for (auto& t : pool) t.join();
}

// ---- phase-only hologram conversion (convert.hpp; convert.cpp:20-184) ----------------------------
namespace {
constexpr double kTwoPi = 2.0 * std::numbers::pi;
}  // namespace

double canonicalize_phase(double value) {  // convert.cpp:20-25 (fp64, like the reference)
    double r = std::fmod(value, kTwoPi);
    if (r < 0.0) r += kTwoPi;
    if (r >= kTwoPi) r -= kTwoPi;
    return r;
}

void canonicalize_phase(RealField& raster) {
    for (double& v : raster.values) v = canonicalize_phase(v);
}

PhaseOnlyHologram dpac_encode(const ComplexField& field, DpacMode mode) {
    Dev in = upload_field({&field});
    Dev out(field.size() * sizeof(float));
    check(hs_dpac_encode(ctx(), in.as<float>(), field.channels, field.height, field.width,
                         mode == DpacMode::direct ? 0 : 1, out.as<float>()));
    std::vector<float> h(field.size());
    out.download(h.data(), h.size() * sizeof(float));
    PhaseOnlyHologram poh;
    poh.format = PohFormat::smooth;
    poh.phase = RealField(field.channels, field.height, field.width);
    for (size_t i = 0; i < h.size(); ++i) poh.phase.values[i] = canonicalize_phase(static_cast<double>(h[i]));
    return poh;
}

ComplexField poh_field(const PhaseOnlyHologram& poh) {
    const RealField& ph = poh.phase;
    std::vector<float> h(ph.values.size());
    for (size_t i = 0; i < h.size(); ++i) h[i] = static_cast<float>(ph.values[i]);
    Dev in(h.size() * sizeof(float));
    in.upload(h.data(), h.size() * sizeof(float));
    Dev out(h.size() * 2 * sizeof(float));
    check(hs_poh_field(ctx(), in.as<float>(), static_cast<int64_t>(h.size()), out.as<float>()));
    ComplexField f(ph.channels, ph.height, ph.width);
    download_field(out, 0, f);
    return f;
}

RandomPohResult convert_random_poh_field(const ComplexField& guide_field, const DepthPlaneSet& planes,
                                         const TargetStack& target, const PropagationSpec& spec,
                                         const RandomPohOptions& opt) {
    const int ch = guide_field.channels, h = guide_field.height, w = guide_field.width;
    if (ch != target.intensity.channels || h != target.intensity.height || w != target.intensity.width)
        throw std::invalid_argument("convert_random_poh: guide/target shape mismatch");
    if (planes.distances.empty()) throw std::invalid_argument("convert_random_poh: no depth planes");
    if (target.masks.size() != planes.distances.size())
        throw std::invalid_argument("convert_random_poh: plane/mask count mismatch");
    if (opt.steps < 1) throw std::invalid_argument("convert_random_poh: steps must be >= 1");
    const size_t n = guide_field.size(), hw = static_cast<size_t>(h) * w;
    const int L = static_cast<int>(planes.distances.size());
    // initial phase: the reference's Rng (mt19937_64, 53-bit uniform) in element order
    std::mt19937_64 eng(opt.seed);
    std::vector<float> phase(n);
    for (float& v : phase) {
        const double u = static_cast<double>(eng() >> 11) * 0x1.0p-53;
        v = static_cast<float>(-std::numbers::pi + 2.0 * std::numbers::pi * u);
    }
    std::vector<float> tgt(target.intensity.values.size());
    for (size_t i = 0; i < tgt.size(); ++i) tgt[i] = static_cast<float>(target.intensity.values[i]);
    std::vector<uint8_t> masks(hw * L);
    for (int l = 0; l < L; ++l) {
        if (target.masks[l].size() != hw) throw std::invalid_argument("convert_random_poh: mask shape mismatch");
        std::copy(target.masks[l].begin(), target.masks[l].end(), masks.begin() + l * hw);
    }
    SpecHolder sh(spec);
    hs_poh_config cfg{ch, h, w, L, planes.distances.data(), sh.s, tgt.data(), masks.data(), opt.steps,
                      opt.lambda_comp, opt.lambda_field, opt.lr};
    Dev guide = upload_field({&guide_field});
    Dev dph(n * sizeof(float));
    dph.upload(phase.data(), n * sizeof(float));
    std::vector<double> loss(opt.steps);
    check(hs_convert_random_poh_field(ctx(), &cfg, guide.as<float>(), dph.as<float>(), loss.data()));
    dph.download(phase.data(), n * sizeof(float));
    RandomPohResult result;
    for (int step = 0; step < opt.steps; ++step) {  // convert.cpp:165-166
        const bool logged = opt.log_every > 0 && (step + 1) % opt.log_every == 0;
        if (logged || step + 1 == opt.steps) result.loss_history.push_back(loss[step]);
    }
    result.poh.phase = RealField(ch, h, w);
    for (size_t i = 0; i < n; ++i) result.poh.phase.values[i] = canonicalize_phase(static_cast<double>(phase[i]));
    result.poh.format = PohFormat::random;
    return result;
}

RandomPohResult convert_random_poh(const GaussianSet& guide, const DepthPlaneSet& planes,
                                   const TargetStack& target, const PropagationSpec& spec,
                                   const RandomPohOptions& opt) {
    const ComplexField guide_field = rasterize_forward(guide, target.intensity.width, target.intensity.height);
    return convert_random_poh_field(guide_field, planes, target, spec, opt);
}

// ---- end-of-run metrics (pipeline.hpp:47-57, pipeline.cpp:135-163) -------------------------------
double psnr_value(const RealField& recon, const RealField& target) {
    if (!recon.same_shape(target)) throw std::invalid_argument("psnr: shape mismatch");
    double mse = 0.0;
    for (size_t i = 0; i < recon.values.size(); ++i) {
        const double d = std::clamp(recon.values[i], 0.0, 1.0) - std::clamp(target.values[i], 0.0, 1.0);
        mse += d * d;
    }
    mse /= static_cast<double>(recon.values.size());
    if (mse <= 0.0) return std::numeric_limits<double>::infinity();
    return -10.0 * std::log10(mse);
}

Metrics compute_metrics(const std::vector<RealField>& recon, const RealField& target) {
    if (recon.empty()) throw std::invalid_argument("compute_metrics: no planes");
    for (const auto& r : recon)
        if (!r.same_shape(target)) throw std::invalid_argument("psnr: shape mismatch");
    const size_t n = target.values.size();
    std::vector<float> h(n * (recon.size() + 1));
    for (size_t i = 0; i < n; ++i) h[i] = static_cast<float>(target.values[i]);
    for (size_t l = 0; l < recon.size(); ++l)
        for (size_t i = 0; i < n; ++i) h[n * (l + 1) + i] = static_cast<float>(recon[l].values[i]);
    Dev d(h.size() * sizeof(float));
    d.upload(h.data(), h.size() * sizeof(float));
    Metrics m;
    m.psnr.resize(recon.size());
    m.ssim.resize(recon.size());
    check(hs_compute_metrics(ctx(), static_cast<int>(recon.size()), target.channels, target.height, target.width,
                             d.as<float>() + n, d.as<float>(), m.psnr.data(), m.ssim.data()));
    for (double v : m.psnr) m.mean_psnr += v;
    for (double v : m.ssim) m.mean_ssim += v;
    m.mean_psnr /= static_cast<double>(m.psnr.size());
    m.mean_ssim /= static_cast<double>(m.ssim.size());
    return m;
}

// ---- artifact formats (io.hpp; io.cpp:237-335) ----------------------------------------------------
namespace {
template <class T>
void put_le(std::string& out, T v) {  // little-endian, like the reference's append_* helpers
    unsigned char b[sizeof(T)];
    std::memcpy(b, &v, sizeof(T));
    out.append(reinterpret_cast<const char*>(b), sizeof(T));  // x86-64 / aarch64 hosts are little-endian
}

struct ByteReader {
    const std::string& path;
    const unsigned char* p;
    size_t left;
    void need(size_t n) const {
        if (left < n) throw std::runtime_error("truncated file");  // io.cpp:44-47 (no path)
    }
    template <class T>
    T get() {
        need(sizeof(T));
        T v;
        std::memcpy(&v, p, sizeof(T));
        p += sizeof(T);
        left -= sizeof(T);
        return v;
    }
    void magic(const char* m, const char* what) {
        need(4);
        if (std::memcmp(p, m, 4) != 0) throw std::runtime_error(path + ": not a " + what + " file");
        p += 4;
        left -= 4;
    }
};

std::string slurp_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}
}  // namespace

void atomic_write(const std::string& path, const std::string& bytes) {
    const std::string tmp = path + ".tmp";
    {
        std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
        if (!out) throw std::runtime_error("cannot write " + tmp);
        out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
        if (!out) throw std::runtime_error("short write to " + tmp);
    }
    if (std::rename(tmp.c_str(), path.c_str()) != 0) throw std::runtime_error("cannot rename into " + path);
}

void write_field(const std::string& path, const ComplexField& field, bool as_f64) {
    std::string out;
    out.reserve(19 + field.size() * 2 * (as_f64 ? 8 : 4));
    out += "CGHF";
    put_le<uint16_t>(out, 1);
    put_le<uint32_t>(out, static_cast<uint32_t>(field.channels));
    put_le<uint32_t>(out, static_cast<uint32_t>(field.height));
    put_le<uint32_t>(out, static_cast<uint32_t>(field.width));
    out.push_back(as_f64 ? 1 : 0);
    for (const auto* plane : {&field.real, &field.imag})
        for (double v : *plane) {
            if (as_f64) put_le<double>(out, v);
            else put_le<float>(out, static_cast<float>(v));
        }
    atomic_write(path, out);
}

ComplexField read_field(const std::string& path) {
    const std::string bytes = slurp_file(path);
    ByteReader r{path, reinterpret_cast<const unsigned char*>(bytes.data()), bytes.size()};
    r.magic("CGHF", "CGHF");
    if (r.get<uint16_t>() != 1) throw std::runtime_error(path + ": unsupported CGHF version");
    const uint32_t c = r.get<uint32_t>(), h = r.get<uint32_t>(), w = r.get<uint32_t>();
    const uint8_t dtype = r.get<uint8_t>();
    if (dtype > 1) throw std::runtime_error(path + ": unknown CGHF dtype");
    ComplexField f(static_cast<int>(c), static_cast<int>(h), static_cast<int>(w));
    r.need(f.size() * 2 * (dtype ? 8 : 4));
    for (auto* plane : {&f.real, &f.imag})
        for (double& v : *plane) v = dtype ? r.get<double>() : static_cast<double>(r.get<float>());
    if (r.left != 0) throw std::runtime_error(path + ": trailing bytes");
    return f;
}

void write_gaussians(const std::string& path, const GaussianSet& set) {
    std::string out = "CGGS";
    put_le<uint16_t>(out, 1);
    put_le<uint32_t>(out, static_cast<uint32_t>(set.count));
    put_le<uint32_t>(out, static_cast<uint32_t>(set.channels));
    for (const auto* v : {&set.pre_position, &set.pre_scale, &set.rotation, &set.amplitude, &set.phase,
                          &set.pre_opacity})
        for (double x : *v) put_le<float>(out, static_cast<float>(x));
    atomic_write(path, out);
}

GaussianSet read_gaussians(const std::string& path) {
    const std::string bytes = slurp_file(path);
    ByteReader r{path, reinterpret_cast<const unsigned char*>(bytes.data()), bytes.size()};
    r.magic("CGGS", "CGGS");
    if (r.get<uint16_t>() != 1) throw std::runtime_error(path + ": unsupported CGGS version");
    const uint32_t n = r.get<uint32_t>(), c = r.get<uint32_t>();
    GaussianSet set(static_cast<int>(n), static_cast<int>(c));
    for (auto* v : {&set.pre_position, &set.pre_scale, &set.rotation, &set.amplitude, &set.phase, &set.pre_opacity})
        for (double& x : *v) x = static_cast<double>(r.get<float>());
    if (r.left != 0) throw std::runtime_error(path + ": trailing bytes");
    return set;
}

}  // namespace holo
