// Test infrastructure (oracle) -- NOT part of the product path.
//
// extern "C" adaptor over the UNMODIFIED reference library (holo:: API in
// /root/reference/proj/core, compiled by oracle/Makefile into
// oracle/_ref/libholoref.so).  Python tests and bench.py's cpu_baseline /
// --impl reference arm drive the reference through these entry points:
//   * per-function parity (rasterizer.hpp:24-36, propagation.hpp:25-49,
//     loss.hpp:44-67, optimizer.hpp:18-49, oracles.hpp),
//   * the reference's own fixture generators (tests/test_util.hpp,
//     pipeline.cpp:175-200 init_gaussians),
//   * RefTrainer: the step-loop body of pipeline.cpp:253-297, verbatim call
//     order, used for full-step parity and for the CPU baseline timing.
// Every entry point returns 0 on success, or a negative code with the
// exception text retrievable from ref_last_error().
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "holo/complex_field.hpp"
#include "holo/field_core.hpp"
#include "holo/gaussian_set.hpp"
#include "holo/io.hpp"
#include "holo/convert.hpp"
#include "holo/loss.hpp"
#include "holo/optimizer.hpp"
#include "holo/oracles.hpp"
#include "holo/parallel.hpp"
#include "holo/pipeline.hpp"
#include "holo/propagation.hpp"
#include "holo/rasterizer.hpp"
#include "test_util.hpp"

using namespace holo;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return -2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -3;
    }
}

GaussianSet make_set(int n, int c, const double* pos, const double* scale, const double* rot,
                     const double* amp, const double* phase, const double* opac) {
    GaussianSet s(n, c);
    const size_t N = static_cast<size_t>(n), NC = N * c;
    if (N) {
        std::memcpy(s.pre_position.data(), pos, 2 * N * sizeof(double));
        std::memcpy(s.pre_scale.data(), scale, 2 * N * sizeof(double));
        std::memcpy(s.rotation.data(), rot, N * sizeof(double));
        std::memcpy(s.amplitude.data(), amp, NC * sizeof(double));
        std::memcpy(s.phase.data(), phase, NC * sizeof(double));
        std::memcpy(s.pre_opacity.data(), opac, N * sizeof(double));
    }
    return s;
}

void unpack_set(const GaussianSet& s, double* pos, double* scale, double* rot, double* amp,
                double* phase, double* opac) {
    auto cp = [](double* dst, const std::vector<double>& v) {
        if (!v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
    };
    cp(pos, s.pre_position);
    cp(scale, s.pre_scale);
    cp(rot, s.rotation);
    cp(amp, s.amplitude);
    cp(phase, s.phase);
    cp(opac, s.pre_opacity);
}

PropagationSpec make_spec(int c, const double* wl, double pitch, int pad, double aperture) {
    PropagationSpec s;
    s.wavelengths.assign(wl, wl + c);
    s.pixel_pitch = pitch;
    s.pad_factor = pad;
    s.aperture_radius = aperture;
    return s;
}

ComplexField make_field(int c, int h, int w, const double* re, const double* im) {
    ComplexField f(c, h, w);
    std::memcpy(f.real.data(), re, f.size() * sizeof(double));
    std::memcpy(f.imag.data(), im, f.size() * sizeof(double));
    return f;
}

void store_field(const ComplexField& f, double* re, double* im) {
    std::memcpy(re, f.real.data(), f.size() * sizeof(double));
    std::memcpy(im, f.imag.data(), f.size() * sizeof(double));
}

RealField make_real(int c, int h, int w, const double* v) {
    RealField f(c, h, w);
    std::memcpy(f.values.data(), v, f.values.size() * sizeof(double));
    return f;
}

}  // namespace

#define SET_ARGS int n, int c, const double *pos, const double *scale, const double *rot, \
                 const double *amp, const double *phase, const double *opac
#define SET_OUT double *o_pos, double *o_scale, double *o_rot, double *o_amp, double *o_phase, \
                double *o_opac

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_thread_count(int t) { set_thread_count(t); }
int ref_thread_count() { return thread_count(); }

// ---- artifact formats (io.cpp:237-335, the reference's own writers/readers) ----
int ref_write_field(const char* path, int c, int h, int w, const double* re, const double* im, int as_f64) {
    return guard([&] {
        ComplexField f(c, h, w);
        std::memcpy(f.real.data(), re, f.size() * sizeof(double));
        std::memcpy(f.imag.data(), im, f.size() * sizeof(double));
        write_field(path, f, as_f64 != 0);
    });
}
// shape query (re == nullptr) or read into re/im of the caller's size
int ref_read_field(const char* path, int* chw, double* re, double* im) {
    return guard([&] {
        const ComplexField f = read_field(path);
        chw[0] = f.channels;
        chw[1] = f.height;
        chw[2] = f.width;
        if (re) store_field(f, re, im);
    });
}
int ref_write_gaussians(const char* path, SET_ARGS) {
    return guard([&] { write_gaussians(path, make_set(n, c, pos, scale, rot, amp, phase, opac)); });
}
int ref_read_gaussians(const char* path, int* nc, SET_OUT) {
    return guard([&] {
        const GaussianSet s = read_gaussians(path);
        nc[0] = s.count;
        nc[1] = s.channels;
        if (o_pos) unpack_set(s, o_pos, o_scale, o_rot, o_amp, o_phase, o_opac);
    });
}

// ---- fixtures (tests/test_util.hpp, pipeline.cpp:165-200) -----------------
int ref_random_set(uint64_t seed, int count, int channels, int width, int height, SET_OUT) {
    return guard([&] {
        unpack_set(testutil::random_set(seed, count, channels, width, height), o_pos, o_scale,
                   o_rot, o_amp, o_phase, o_opac);
    });
}
int ref_random_field(uint64_t seed, int c, int h, int w, double amp, double* re, double* im) {
    return guard([&] { store_field(testutil::random_field(seed, c, h, w, amp), re, im); });
}
int ref_random_real(uint64_t seed, int c, int h, int w, double lo, double hi, double* out) {
    return guard([&] {
        const RealField f = testutil::random_real(seed, c, h, w, lo, hi);
        std::memcpy(out, f.values.data(), f.values.size() * sizeof(double));
    });
}
int ref_synthetic_image(uint64_t seed, int c, int h, int w, double* out) {
    return guard([&] {
        const RealField f = testutil::synthetic_image(seed, c, h, w);
        std::memcpy(out, f.values.data(), f.values.size() * sizeof(double));
    });
}
int ref_synthetic_depth(uint64_t seed, int h, int w, double* out) {
    return guard([&] {
        const RealField f = testutil::synthetic_depth(seed, h, w);
        std::memcpy(out, f.values.data(), f.values.size() * sizeof(double));
    });
}
int ref_init_gaussians(int count, int channels, int width, int height, uint64_t seed, SET_OUT) {
    return guard([&] {
        unpack_set(init_gaussians(count, channels, width, height, seed), o_pos, o_scale, o_rot,
                   o_amp, o_phase, o_opac);
    });
}
int ref_resolve_gaussian_count(double ratio, int count, int channels, int width, int height) {
    RunConfig cfg;
    cfg.parameter_ratio = ratio;
    cfg.gaussian_count = count;
    int out = -1;
    guard([&] { out = resolve_gaussian_count(cfg, channels, width, height); });
    return out;
}

// ---- field_core (field_core.cpp) --------------------------------------------
int ref_activations(double pre, double extent, double* out8) {
    return guard([&] {
        out8[0] = activate_position(pre, extent);
        out8[1] = activate_position_deriv(pre, extent);
        out8[2] = activate_scale(pre);
        out8[3] = activate_scale_deriv(pre);
        out8[4] = activate_opacity(pre);
        out8[5] = activate_opacity_deriv(pre);
        out8[6] = activate_amplitude(pre);
        out8[7] = activate_amplitude_deriv(pre);
    });
}
int ref_covariance(double sx, double sy, double theta, double* out7) {
    return guard([&] {
        const Covariance2 cv = covariance(sx, sy, theta);
        const CovarianceInverse ci = invert_covariance(cv);
        out7[0] = cv.sxx; out7[1] = cv.sxy; out7[2] = cv.syy;
        out7[3] = ci.inv.inv00; out7[4] = ci.inv.inv01; out7[5] = ci.inv.inv11;
        out7[6] = ci.radius;
    });
}

// ---- rasterizer (rasterizer.cpp) ---------------------------------------------
// Returns the pair count K; pairs are written only when K <= cap.  ranges is
// 2*tiles_x*tiles_y uint64 (begin,end).
int64_t ref_build_tile_index(SET_ARGS, int width, int height, uint32_t* tiles, uint32_t* ids,
                             uint64_t* ranges, int64_t cap, int* tiles_xy) {
    int64_t k = -1;
    const int rc = guard([&] {
        const TileIndex idx = build_tile_index(make_set(n, c, pos, scale, rot, amp, phase, opac),
                                               width, height);
        tiles_xy[0] = idx.tiles_x;
        tiles_xy[1] = idx.tiles_y;
        k = static_cast<int64_t>(idx.pairs.size());
        if (k <= cap) {
            for (size_t i = 0; i < idx.pairs.size(); ++i) {
                tiles[i] = idx.pairs[i].first;
                ids[i] = idx.pairs[i].second;
            }
            for (size_t t = 0; t < idx.ranges.size(); ++t) {
                ranges[2 * t] = idx.ranges[t].first;
                ranges[2 * t + 1] = idx.ranges[t].second;
            }
        }
    });
    return rc ? rc : k;
}
int ref_rasterize_forward(SET_ARGS, int width, int height, double* re, double* im) {
    return guard([&] {
        store_field(rasterize_forward(make_set(n, c, pos, scale, rot, amp, phase, opac), width, height),
                    re, im);
    });
}
int ref_brute_rasterize(SET_ARGS, int width, int height, double* re, double* im, int64_t* counters3) {
    return guard([&] {
        oracle::BruteCounters bc;
        store_field(oracle::brute_rasterize_counted(make_set(n, c, pos, scale, rot, amp, phase, opac),
                                                    width, height, bc),
                    re, im);
        counters3[0] = bc.skipped;
        counters3[1] = bc.saturated;
        counters3[2] = bc.floored;
    });
}
int ref_rasterize_backward(SET_ARGS, int width, int height, const double* gre, const double* gim,
                           SET_OUT) {
    return guard([&] {
        const GaussianSet s = make_set(n, c, pos, scale, rot, amp, phase, opac);
        const GaussianSetGrads g = rasterize_backward(s, make_real(c, height, width, gre),
                                                      make_real(c, height, width, gim));
        unpack_set(g, o_pos, o_scale, o_rot, o_amp, o_phase, o_opac);
    });
}

// ---- propagation (propagation.cpp) -------------------------------------------
// mode 0 propagate, 1 propagate_with_mask_distance, 2 propagate_backward,
// 3 oracle::direct_dft_propagate
int ref_propagate(int mode, int c, int h, int w, const double* re, const double* im,
                  const double* wl, double pitch, int pad, double aperture, double distance,
                  double mask_distance, double* out_re, double* out_im) {
    return guard([&] {
        const ComplexField f = make_field(c, h, w, re, im);
        const PropagationSpec s = make_spec(c, wl, pitch, pad, aperture);
        ComplexField o;
        if (mode == 0) o = propagate(f, s, distance);
        else if (mode == 1) o = propagate_with_mask_distance(f, s, distance, mask_distance);
        else if (mode == 2) o = propagate_backward(f, s, distance);
        else o = oracle::direct_dft_propagate(f, s, distance);
        store_field(o, out_re, out_im);
    });
}
int ref_propagate_multi(int c, int h, int w, const double* re, const double* im, const double* wl,
                        double pitch, int pad, double aperture, const double* dist, int L,
                        double* out_re, double* out_im) {
    return guard([&] {
        const auto outs = propagate_multi(make_field(c, h, w, re, im),
                                          make_spec(c, wl, pitch, pad, aperture),
                                          std::vector<double>(dist, dist + L));
        const size_t plane = static_cast<size_t>(c) * h * w;
        for (int l = 0; l < L; ++l) store_field(outs[l], out_re + l * plane, out_im + l * plane);
    });
}
int ref_propagate_multi_backward(int c, int h, int w, const double* re, const double* im,
                                 const double* wl, double pitch, int pad, double aperture,
                                 const double* dist, int L, double* out_re, double* out_im) {
    return guard([&] {
        const size_t plane = static_cast<size_t>(c) * h * w;
        std::vector<ComplexField> g;
        for (int l = 0; l < L; ++l) g.push_back(make_field(c, h, w, re + l * plane, im + l * plane));
        store_field(propagate_multi_backward(g, make_spec(c, wl, pitch, pad, aperture),
                                             std::vector<double>(dist, dist + L)),
                    out_re, out_im);
    });
}
int ref_transfer_function(const double* wl, int nwl, double pitch, int pad, double aperture,
                          double distance, int channel, int pnx, int pny, double* out4) {
    return guard([&] {
        const auto g = transfer_function(make_spec(nwl, wl, pitch, pad, aperture), distance,
                                         channel, pnx, pny);
        for (size_t i = 0; i < g.size(); ++i) {
            out4[4 * i] = g[i].fx;
            out4[4 * i + 1] = g[i].fy;
            out4[4 * i + 2] = g[i].kz;
            out4[4 * i + 3] = g[i].inside_bandlimit ? 1.0 : 0.0;
        }
    });
}

// ---- end-of-run metrics (pipeline.cpp:135-163) ------------------------------------
int ref_compute_metrics(int L, int c, int h, int w, const double* recon, const double* target, double* psnr,
                        double* ssim) {
    return guard([&] {
        const size_t plane = static_cast<size_t>(c) * h * w;
        std::vector<RealField> r;
        for (int l = 0; l < L; ++l) r.push_back(make_real(c, h, w, recon + l * plane));
        const Metrics m = compute_metrics(r, make_real(c, h, w, target));
        for (int l = 0; l < L; ++l) {
            psnr[l] = m.psnr[l];
            ssim[l] = m.ssim[l];
        }
    });
}

// ---- POH conversion (convert.cpp) -------------------------------------------------
int ref_dpac_encode(int c, int h, int w, const double* re, const double* im, int mode, double* out) {
    return guard([&] {
        const PhaseOnlyHologram p = dpac_encode(make_field(c, h, w, re, im),
                                                mode == 0 ? DpacMode::direct : DpacMode::classical);
        std::memcpy(out, p.phase.values.data(), p.phase.values.size() * sizeof(double));
    });
}
int ref_poh_field(int c, int h, int w, const double* phase, double* re, double* im) {
    return guard([&] {
        PhaseOnlyHologram p;
        p.phase = make_real(c, h, w, phase);
        store_field(poh_field(p), re, im);
    });
}
// convert_random_poh_field with the target stack built from (target, depth, L,
// near_is_high) like make_target_stack; phase_out C x H x W, loss_out
// (n_loss capacity) receives the loss history, returns its length.
int ref_convert_random_poh_field(int c, int h, int w, const double* gre, const double* gim,
                                 const double* target, const double* depth, int near_is_high,
                                 const double* dist, int L, const double* wl, double pitch, int pad,
                                 double aperture, int steps, uint64_t seed, double lambda_comp,
                                 double lambda_field, double lr, int log_every, double* phase_out,
                                 double* loss_out, int n_loss) {
    int len = 0;
    const int rc = guard([&] {
        DepthPlaneSet planes;
        planes.count = L;
        planes.distances.assign(dist, dist + L);
        const TargetStack t = make_target_stack(make_real(c, h, w, target), make_real(1, h, w, depth), L,
                                                near_is_high != 0);
        RandomPohOptions o;
        o.steps = steps;
        o.seed = seed;
        o.lambda_comp = lambda_comp;
        o.lambda_field = lambda_field;
        o.lr = lr;
        o.log_every = log_every;
        const RandomPohResult r = convert_random_poh_field(make_field(c, h, w, gre, gim), planes, t,
                                                           make_spec(c, wl, pitch, pad, aperture), o);
        std::memcpy(phase_out, r.poh.phase.values.data(), r.poh.phase.values.size() * sizeof(double));
        len = static_cast<int>(r.loss_history.size());
        for (int i = 0; i < std::min(len, n_loss); ++i) loss_out[i] = r.loss_history[i];
    });
    return rc < 0 ? rc : len;
}

// ---- loss (loss.cpp) -----------------------------------------------------------
int ref_build_masks(const double* depth, int h, int w, int L, int near_is_high, uint8_t* out) {
    return guard([&] {
        const MaskStack m = build_masks(make_real(1, h, w, depth), L, near_is_high != 0);
        for (int l = 0; l < L; ++l) std::memcpy(out + static_cast<size_t>(l) * h * w, m[l].data(), m[l].size());
    });
}
int ref_make_depth_planes(int count, double d0, double dz, double* out) {
    return guard([&] {
        const DepthPlaneSet p = make_depth_planes(count, d0, dz);
        for (int l = 0; l < count; ++l) out[l] = p.distances[l];
    });
}
// kind: 0 training_loss_grad, 1 loss_recon_grad, 2 loss_ssim_grad, 3 loss_mse_grad,
//       10..13 the value-only variants (grads untouched), 20 oracle::loop_recon,
//       21 oracle::loop_ssim, 22 oracle::loop_mse
int ref_loss(int kind, int L, int c, int h, int w, const double* recon, const double* target,
             const double* depth, int near_is_high, double* grads, double* loss) {
    return guard([&] {
        const size_t plane = static_cast<size_t>(c) * h * w;
        std::vector<RealField> r;
        for (int l = 0; l < L; ++l) r.push_back(make_real(c, h, w, recon + l * plane));
        const TargetStack t = make_target_stack(make_real(c, h, w, target), make_real(1, h, w, depth),
                                                L, near_is_high != 0);
        std::vector<RealField> g;
        double v = 0.0;
        switch (kind) {
            case 0: v = training_loss_grad(r, t, g); break;
            case 1: v = loss_recon_grad(r, t, g); break;
            case 2: v = loss_ssim_grad(r, t, g); break;
            case 3: v = loss_mse_grad(r, t, g); break;
            case 10: v = training_loss(r, t); break;
            case 11: v = loss_recon(r, t); break;
            case 12: v = loss_ssim(r, t); break;
            case 13: v = loss_mse(r, t); break;
            case 20: v = oracle::loop_recon(r, t); break;
            case 21: v = oracle::loop_ssim(r, t); break;
            case 22: v = oracle::loop_mse(r, t); break;
            default: throw std::invalid_argument("ref_loss: unknown kind");
        }
        if (kind < 10)
            for (int l = 0; l < L; ++l)
                std::memcpy(grads + l * plane, g[l].values.data(), plane * sizeof(double));
        *loss = v;
    });
}

// ---- optimizer (optimizer.cpp) ---------------------------------------------------
double ref_cosine_lr(int step, int total, double lr_max, double lr_min, int* rc) {
    double v = 0.0;
    *rc = guard([&] { v = cosine_lr(step, total, lr_max, lr_min); });
    return v;
}
void* ref_adan_create() { return new Adan(); }
void ref_adan_destroy(void* a) { delete static_cast<Adan*>(a); }
int ref_adan_add_group(void* a, const char* name, int64_t size, double lr) {
    return guard([&] { static_cast<Adan*>(a)->add_group(name, static_cast<size_t>(size), lr); });
}
int ref_adan_set_lr(void* a, const char* name, double lr) {
    return guard([&] { static_cast<Adan*>(a)->set_lr(name, lr); });
}
int ref_adan_step(void* a, const char* name, double* params, const double* grads, int64_t np,
                  int64_t ng) {
    return guard([&] {
        static_cast<Adan*>(a)->step(name, std::span<double>(params, static_cast<size_t>(np)),
                                    std::span<const double>(grads, static_cast<size_t>(ng)));
    });
}

// ---- the step loop (pipeline.cpp:243-297) -------------------------------------------
struct RefTrainer {
    int w = 0, h = 0, ch = 0;
    int total_steps = 0;
    int step = 0;
    GaussianSet set;
    TargetStack target;
    DepthPlaneSet planes;
    PropagationSpec spec;
    Adan adan;
    double stage_ms[7] = {0, 0, 0, 0, 0, 0, 0};
};

void* ref_trainer_create(SET_ARGS, int width, int height, const double* target, const double* depth,
                         int L, double d0, double dz, int near_is_high, const double* wl,
                         double pitch, int pad, double aperture, int total_steps) {
    RefTrainer* t = nullptr;
    const int rc = guard([&] {
        t = new RefTrainer;
        t->w = width;
        t->h = height;
        t->ch = c;
        t->total_steps = total_steps;
        t->set = make_set(n, c, pos, scale, rot, amp, phase, opac);
        t->target = make_target_stack(make_real(c, height, width, target),
                                      make_real(1, height, width, depth), L, near_is_high != 0);
        t->planes = make_depth_planes(L, d0, dz);
        t->spec = make_spec(c, wl, pitch, pad, aperture);
        // pipeline.cpp:243-249
        t->adan.add_group("position", t->set.pre_position.size(), 1e-2);
        t->adan.add_group("scale", t->set.pre_scale.size(), 5e-3);
        t->adan.add_group("rotation", t->set.rotation.size(), 1e-3);
        t->adan.add_group("amplitude", t->set.amplitude.size(), 2.5e-3);
        t->adan.add_group("phase", t->set.phase.size(), 2.5e-3);
        t->adan.add_group("opacity", t->set.pre_opacity.size(), 2.5e-2);
    });
    if (rc) {
        delete t;
        return nullptr;
    }
    return t;
}

void ref_trainer_destroy(void* p) { delete static_cast<RefTrainer*>(p); }

// One iteration of pipeline.cpp:253-297 in the reference's call order.  When
// grads_out is non-null it receives the six gradient groups (before Adan).
int ref_trainer_step(void* p, double* loss_out, SET_OUT) {
    RefTrainer* t = static_cast<RefTrainer*>(p);
    return guard([&] {
        using clk = std::chrono::steady_clock;
        auto ms = [](clk::time_point a, clk::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        const int w = t->w, h = t->h, ch = t->ch;
        const size_t planes_n = t->planes.distances.size();
        auto t0 = clk::now();
        t->adan.set_lr("position", cosine_lr(t->step, t->total_steps, 1e-2, 1e-3));
        const ComplexField field = rasterize_forward(t->set, w, h);
        auto t1 = clk::now();
        const std::vector<ComplexField> outs = propagate_multi(field, t->spec, t->planes.distances);
        std::vector<RealField> intens;
        intens.reserve(planes_n);
        for (const auto& u : outs) intens.push_back(intensity_of(u));
        auto t2 = clk::now();
        std::vector<RealField> gi;
        const double loss = training_loss_grad(intens, t->target, gi);
        auto t3 = clk::now();
        std::vector<ComplexField> du;
        du.reserve(planes_n);
        for (size_t l = 0; l < planes_n; ++l) {
            ComplexField g(ch, h, w);
            for (size_t i = 0; i < g.size(); ++i) {
                g.real[i] = 2.0 * outs[l].real[i] * gi[l].values[i];
                g.imag[i] = 2.0 * outs[l].imag[i] * gi[l].values[i];
            }
            du.push_back(std::move(g));
        }
        ComplexField back = propagate_multi_backward(du, t->spec, t->planes.distances);
        auto t4 = clk::now();
        RealField grad_re(ch, h, w), grad_im(ch, h, w);
        grad_re.values = std::move(back.real);
        grad_im.values = std::move(back.imag);
        const GaussianSetGrads grads = rasterize_backward(t->set, grad_re, grad_im);
        auto t5 = clk::now();
        if (o_pos) unpack_set(grads, o_pos, o_scale, o_rot, o_amp, o_phase, o_opac);
        t->adan.step("position", t->set.pre_position, grads.pre_position);
        t->adan.step("scale", t->set.pre_scale, grads.pre_scale);
        t->adan.step("rotation", t->set.rotation, grads.rotation);
        t->adan.step("amplitude", t->set.amplitude, grads.amplitude);
        t->adan.step("phase", t->set.phase, grads.phase);
        t->adan.step("opacity", t->set.pre_opacity, grads.pre_opacity);
        auto t6 = clk::now();
        t->stage_ms[0] += ms(t0, t1);
        t->stage_ms[1] += ms(t1, t2);
        t->stage_ms[2] += ms(t2, t3);
        t->stage_ms[3] += ms(t3, t4);
        t->stage_ms[4] += ms(t4, t5);
        t->stage_ms[5] += ms(t5, t6);
        t->stage_ms[6] += ms(t0, t6);
        t->step += 1;
        *loss_out = loss;
    });
}

int ref_trainer_params(void* p, SET_OUT) {
    RefTrainer* t = static_cast<RefTrainer*>(p);
    return guard([&] { unpack_set(t->set, o_pos, o_scale, o_rot, o_amp, o_phase, o_opac); });
}

void ref_trainer_stage_ms(void* p, double* out7) {
    RefTrainer* t = static_cast<RefTrainer*>(p);
    for (int i = 0; i < 7; ++i) out7[i] = t->stage_ms[i];
}

}  // extern "C"
