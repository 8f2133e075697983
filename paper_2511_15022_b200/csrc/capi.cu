// C ABI (include/holosplat.h) and the device-resident trainer that replaces the
// step-loop body of proj/core/src/pipeline.cpp:253-297.
#include <atomic>
#include <cmath>
#include <limits>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "asm.cuh"
#include "loss.cuh"
#include "convert.cuh"
#include "raster.cuh"
#include "trainer.cuh"

namespace hs {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

const char* kGroupNames[6] = {"position", "scale", "rotation", "amplitude", "phase", "opacity"};

struct CtxWork {
    CtxWork() { rw.tile_bwd = false; }  // the stand-alone rasterize_backward: deterministic by default
    RasterWork rw;
    AsmWork aw;
    DevBuf flags, partials, out3, tstats;
    PohWork poh;
    DevBuf amax, poh_target, poh_masks, poh_loss, metric_buf;
};

}  // namespace

void note_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n), std::memory_order_relaxed); }

hs_status fail(hs_status s, const std::string& m) {
    g_last_error = m;
    return s;
}

int sm_count(int device) {
    int v = 0;
    HS_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
    return v;
}

}  // namespace hs

using namespace hs;

// ctx-owned reusable work buffers for the standalone entry points
static CtxWork& work_of(hs_ctx* ctx) {
    if (!ctx->work) ctx->work = new CtxWork();
    return *static_cast<CtxWork*>(ctx->work);
}


extern "C" {

const char* hs_last_error(void) { return g_last_error.c_str(); }
uint64_t hs_kernel_launch_count(void) { return g_launches.load(); }

hs_status hs_ctx_create(int device, hs_ctx** out) {
    return guard([&] {
        int ndev = 0;
        HS_CUDA(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, "hs_ctx_create: no such device");
        HS_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop{};
        HS_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            throw Error(HS_ECUDA, std::string("holosplat-b200 needs sm_100a (B200); found ") + prop.name);
        auto* c = new hs_ctx;
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        *out = c;
    });
}

void hs_ctx_destroy(hs_ctx* ctx) {
    if (!ctx) return;
    hs_ctx_comm_destroy(ctx);
    delete static_cast<CtxWork*>(ctx->work);
    ctx->work = nullptr;
    delete ctx;
}

hs_status hs_ctx_set_stream(hs_ctx* ctx, void* stream) {
    ctx->stream = static_cast<cudaStream_t>(stream);
    return HS_OK;
}

hs_status hs_ctx_synchronize(hs_ctx* ctx) {
    return guard([&] { HS_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

hs_status hs_device_alloc(hs_ctx* ctx, size_t bytes, void** d_out) {
    return guard([&] {
        HS_CUDA(cudaSetDevice(ctx->device));
        HS_CUDA(cudaMalloc(d_out, std::max<size_t>(bytes, 1)));
    });
}
hs_status hs_device_free(hs_ctx*, void* d_ptr) {
    return guard([&] { HS_CUDA(cudaFree(d_ptr)); });
}
hs_status hs_copy_h2d(hs_ctx* ctx, void* d_dst, const void* h_src, size_t bytes) {
    return guard([&] {
        HS_CUDA(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, ctx->stream));
        HS_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
hs_status hs_copy_d2h(hs_ctx* ctx, void* h_dst, const void* d_src, size_t bytes) {
    return guard([&] {
        HS_CUDA(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        HS_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"

// ---- rasterizer ----------------------------------------------------------------------
[[maybe_unused]] static void check_params_finite(RasterWork& rw, cudaStream_t st) {
    uint32_t stat[4];
    HS_CUDA(cudaMemcpyAsync(stat, rw.status.p, sizeof(stat), cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));
    // field_core.cpp:12,22,29 / gaussian_set.cpp:30-39
    if (stat[2]) throw Error(HS_EINVAL, "activate: non-finite input");
}

extern "C" hs_status hs_build_tile_index(hs_ctx* ctx, const float* d_params, int n, int c, int width,
                              int height, uint32_t* d_tiles, uint32_t* d_ids, uint64_t* d_ranges,
                              int64_t cap, int64_t* npairs, int* tiles_xy) {
    return guard([&] {
        require(width > 0 && height > 0, "build_tile_index: empty canvas");  // rasterizer.cpp:124
        require(n >= 0, "GaussianSet: invalid N or C");
        RasterWork& rw = work_of(ctx).rw;
        rw.prepare(n, c, width, height);
        tiles_xy[0] = rw.tiles_x;
        tiles_xy[1] = rw.tiles_y;
        cudaStream_t st = ctx->stream;
        rw.tight = false;  // the reference's exact (tile, id) list (rasterizer.cpp:90-119)
        struct Restore {
            RasterWork& r;
            ~Restore() { r.tight = true; }
        } restore{rw};  // (back to the default: tight)
        for (int attempt = 0; attempt < 2; ++attempt) {
            rw.project_and_bin(d_params, st);
            uint32_t stat[4] = {0, 0, 0, 0};
            HS_CUDA(cudaMemcpyAsync(stat, rw.status.p, sizeof(stat), cudaMemcpyDeviceToHost, st));
            HS_CUDA(cudaStreamSynchronize(st));
            if (stat[2]) throw Error(HS_EINVAL, "activate: non-finite input");
            if (stat[1]) {  // grow to the exact total (status[0], saturated) and redo
                const int64_t need = stat[0];
                require(need < 0xffffffffll, "build_tile_index: more than 2^32 pairs");
                rw.reserve_pairs(need + 1);
                continue;
            }
            *npairs = n == 0 ? 0 : stat[0];
            if (*npairs <= cap && (d_tiles || d_ranges)) {
                if (n == 0) {
                    HS_CUDA(cudaMemsetAsync(d_ranges, 0, sizeof(uint64_t) * 2 * rw.tiles_x * rw.tiles_y, st));
                } else {
                    export_tile_index(rw, *npairs, d_tiles, d_ids, d_ranges, st);
                }
                HS_CUDA(cudaStreamSynchronize(st));
            }
            return;
        }
        throw Error(HS_EOVERFLOW, "build_tile_index: pair capacity");
    });
}

extern "C" hs_status hs_ctx_set_tight_binning(hs_ctx* ctx, int tight) {
    return guard([&] { work_of(ctx).rw.tight = tight != 0; });
}

static void raster_prepare_and_bin(hs_ctx* ctx, RasterWork& rw, const float* d_params, int n, int c,
                                   int width, int height) {
    rw.prepare(n, c, width, height);
    cudaStream_t st = ctx->stream;
    for (int attempt = 0; attempt < 2; ++attempt) {
        rw.project_and_bin(d_params, st);
        uint32_t stat[4];
        HS_CUDA(cudaMemcpyAsync(stat, rw.status.p, sizeof(stat), cudaMemcpyDeviceToHost, st));
        HS_CUDA(cudaStreamSynchronize(st));
        if (stat[2]) throw Error(HS_EINVAL, "activate: non-finite input");
        if (!stat[1]) return;
        const int64_t need = stat[0];
        require(need < 0xffffffffll, "rasterizer: more than 2^32 tile pairs");
        rw.reserve_pairs(need + 1);
    }
    throw Error(HS_EOVERFLOW, "rasterizer: pair capacity");
}

extern "C" hs_status hs_rasterize_forward(hs_ctx* ctx, const float* d_params, int n, int c, int width,
                               int height, float* d_field) {
    return guard([&] {
        require(width > 0 && height > 0, "rasterize_forward: empty canvas");  // rasterizer.cpp:129
        require(c >= 1, "ComplexField: non-positive dims");
        const size_t bytes = sizeof(float2) * static_cast<size_t>(c) * width * height;
        if (n == 0) {
            HS_CUDA(cudaMemsetAsync(d_field, 0, bytes, ctx->stream));
            return;
        }
        RasterWork& rw = work_of(ctx).rw;
        raster_prepare_and_bin(ctx, rw, d_params, n, c, width, height);
        raster_forward(rw, reinterpret_cast<float2*>(d_field), ctx->stream);
    });
}

extern "C" hs_status hs_rasterize_backward(hs_ctx* ctx, const float* d_params, int n, int c, int width,
                                int height, const float* d_grad_field, float* d_grads) {
    return guard([&] {
        require(width > 0 && height > 0 && c >= 1, "rasterize_backward: gradient shape mismatch");
        if (n == 0) return;
        RasterWork& rw = work_of(ctx).rw;
        raster_prepare_and_bin(ctx, rw, d_params, n, c, width, height);
        raster_backward(rw, d_params, reinterpret_cast<const float2*>(d_grad_field), d_grads, nullptr,
                        ctx->stream);
    });
}

// ---- propagation ------------------------------------------------------------------------
static void check_spec(const hs_prop_spec* spec, int c) {
    require(spec && spec->n_wavelengths == c, "propagation: channel count does not match wavelengths");
    require(spec->pad_factor >= 1, "propagation: pad_factor must be >= 1");
}

extern "C" hs_status hs_propagate(hs_ctx* ctx, const hs_prop_spec* spec, int mode, double distance,
                       double mask_distance, const float* d_in, int c, int h, int w, float* d_out) {
    return guard([&] {
        check_spec(spec, c);
        if (mode == 0 || mode == 2)
            require(std::isfinite(distance), "propagate: non-finite distance");  // propagation.cpp:175
        double pd = distance, md = distance;
        if (mode == 1) md = mask_distance;
        if (mode == 2) pd = -distance;  // propagate_backward: phase -d, mask d (:237)
        AsmWork& aw = work_of(ctx).aw;
        aw.prepare(c, h, w, spec->pad_factor, 1);
        aw.L = 1;
        aw.set_transfer(*spec, &pd, &md, ctx->stream);
        asm_forward(aw, reinterpret_cast<const float2*>(d_in), reinterpret_cast<float2*>(d_out), ctx->stream);
        HS_CUDA(cudaStreamSynchronize(ctx->stream));  // tf_host lifetime
    });
}

extern "C" hs_status hs_propagate_multi(hs_ctx* ctx, const hs_prop_spec* spec, const double* h_distances,
                             int L, const float* d_in, int c, int h, int w, float* d_out) {
    return guard([&] {
        check_spec(spec, c);
        require(L >= 1, "propagate_multi: no distances");
        AsmWork& aw = work_of(ctx).aw;
        aw.prepare(c, h, w, spec->pad_factor, L);
        aw.L = L;
        aw.set_transfer(*spec, h_distances, h_distances, ctx->stream);
        asm_forward(aw, reinterpret_cast<const float2*>(d_in), reinterpret_cast<float2*>(d_out), ctx->stream);
        HS_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" hs_status hs_propagate_multi_backward(hs_ctx* ctx, const hs_prop_spec* spec,
                                      const double* h_distances, int L, const float* d_grads, int c,
                                      int h, int w, float* d_out) {
    return guard([&] {
        require(L >= 1, "propagate_multi_backward: plane count mismatch");  // propagation.cpp:217-218
        check_spec(spec, c);
        AsmWork& aw = work_of(ctx).aw;
        aw.prepare(c, h, w, spec->pad_factor, L);
        aw.L = L;
        aw.set_transfer(*spec, h_distances, h_distances, ctx->stream);
        asm_backward(aw, reinterpret_cast<const float2*>(d_grads), reinterpret_cast<float2*>(d_out),
                     ctx->stream);
        HS_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ---- end-of-run metrics (pipeline.cpp:135-163) ------------------------------------------------
extern "C" hs_status hs_compute_metrics(hs_ctx* ctx, int L, int c, int h, int w, const float* d_recon,
                                        const float* d_target, double* h_psnr, double* h_ssim) {
    return guard([&] {
        require(L >= 1, "compute_metrics: no planes");
        require(h >= 11 && w >= 11, "ssim: image smaller than the 11x11 window");
        CtxWork& cw = work_of(ctx);
        cudaStream_t st = ctx->stream;
        const int64_t chw = static_cast<int64_t>(c) * h * w;
        cw.metric_buf.reserve(sizeof(float) * chw * (L + 1));
        float* tclip = cw.metric_buf.as<float>();
        float* rclip = tclip + chw;
        clip01_launch(d_target, chw, tclip, st);
        clip01_launch(d_recon, chw * L, rclip, st);
        cw.tstats.reserve(sizeof(float2) * ssim_target_stats_elems(c, h, w));
        ssim_target_stats(tclip, c, h, w, cw.tstats.as<float2>(), st);
        const int slots = std::max(loss_partial_slots(kLossSsim, 1, c, h, w), loss_partial_slots(kLossMse, 1, c, h, w));
        cw.partials.reserve(sizeof(double) * 2 * std::max(slots, 1));
        cw.out3.reserve(sizeof(double) * 3 * 2 * L);
        for (int l = 0; l < L; ++l) {
            for (int kind : {kLossMse, kLossSsim}) {
                LossArgs a{kind, 1, 1, 0, c, h, w, rclip + l * chw, nullptr, tclip, cw.tstats.as<float2>(), nullptr,
                           nullptr, nullptr, cw.partials.as<double>()};
                const int used = loss_launch(a, st);
                loss_finalize(a, used, cw.out3.as<double>() + 3 * (2 * l + (kind == kLossSsim ? 1 : 0)), st);
            }
        }
        std::vector<double> out(6 * static_cast<size_t>(L));
        HS_CUDA(cudaMemcpyAsync(out.data(), cw.out3.p, sizeof(double) * out.size(), cudaMemcpyDeviceToHost, st));
        HS_CUDA(cudaStreamSynchronize(st));
        for (int l = 0; l < L; ++l) {
            const double mse = out[6 * l];  // loss_mse of one plane: mean squared difference
            h_psnr[l] = mse <= 0.0 ? std::numeric_limits<double>::infinity() : -10.0 * std::log10(mse);
            h_ssim[l] = 1.0 - out[6 * l + 3];  // loss_ssim = 1 - ssim_value
        }
    });
}

// ---- POH conversion ---------------------------------------------------------------------------
extern "C" hs_status hs_dpac_encode(hs_ctx* ctx, const float* d_field, int c, int h, int w, int mode,
                                    float* d_phase) {
    return guard([&] {
        require(c >= 0 && h >= 0 && w >= 0, "dpac_encode: bad shape");
        require(mode == 0 || mode == 1, "dpac_encode: unknown mode");
        CtxWork& cw = work_of(ctx);
        cw.amax.reserve(sizeof(unsigned) * std::max(c, 1));
        dpac_encode(reinterpret_cast<const float2*>(d_field), c, h, w, mode, cw.amax.as<unsigned>(), d_phase,
                    ctx->stream);
    });
}

extern "C" hs_status hs_poh_field(hs_ctx* ctx, const float* d_phase, int64_t count, float* d_field) {
    return guard([&] { phase_to_field(d_phase, count, reinterpret_cast<float2*>(d_field), ctx->stream); });
}

extern "C" hs_status hs_convert_random_poh_field(hs_ctx* ctx, const hs_poh_config* cfg, const float* d_guide_field,
                                                 float* d_phase, double* h_loss) {
    return guard([&] {
        require(cfg != nullptr, "convert_random_poh: null config");
        require(cfg->planes >= 1, "convert_random_poh: no depth planes");          // convert.cpp:80-81
        require(cfg->steps >= 1, "convert_random_poh: steps must be >= 1");        // :84
        check_spec(&cfg->spec, cfg->c);
        const int c = cfg->c, h = cfg->height, w = cfg->width, L = cfg->planes;
        CtxWork& cw = work_of(ctx);
        cudaStream_t st = ctx->stream;
        const size_t chw = static_cast<size_t>(c) * h * w, hw = static_cast<size_t>(h) * w;
        cw.poh_target.reserve(sizeof(float) * chw);
        cw.poh_masks.reserve(hw * L);
        cw.poh_loss.reserve(sizeof(double) * cfg->steps);
        HS_CUDA(cudaMemcpyAsync(cw.poh_target.p, cfg->h_target, sizeof(float) * chw, cudaMemcpyHostToDevice, st));
        HS_CUDA(cudaMemcpyAsync(cw.poh_masks.p, cfg->h_masks, hw * L, cudaMemcpyHostToDevice, st));
        PohProblem p;
        p.C = c;
        p.H = h;
        p.W = w;
        p.L = L;
        p.pad = cfg->spec.pad_factor;
        p.target = cw.poh_target.as<float>();
        p.masks = cw.poh_masks.as<uint8_t>();
        PohWork& pw = cw.poh;
        pw.prepare(p);
        pw.aw.L = L;
        pw.aw.set_transfer(cfg->spec, cfg->distances, cfg->distances, st);
        random_poh_run(pw, reinterpret_cast<const float2*>(d_guide_field), d_phase, cfg->steps, cfg->lambda_comp,
                       cfg->lambda_field, cfg->lr, cw.poh_loss.as<double>(), st);
        uint32_t flag = 0;
        HS_CUDA(cudaMemcpyAsync(&flag, pw.flag.p, sizeof(flag), cudaMemcpyDeviceToHost, st));
        if (h_loss)
            HS_CUDA(cudaMemcpyAsync(h_loss, cw.poh_loss.p, sizeof(double) * cfg->steps, cudaMemcpyDeviceToHost, st));
        HS_CUDA(cudaStreamSynchronize(st));
        if (flag) throw Error(HS_ENONFINITE, "Adan: non-finite gradient in group phase");
    });
}

// ---- loss -------------------------------------------------------------------------------------
extern "C" hs_status hs_intensity(hs_ctx* ctx, const float* d_field, int64_t count, float* d_out) {
    return guard([&] { intensity_launch(reinterpret_cast<const float2*>(d_field), count, d_out, ctx->stream); });
}

extern "C" hs_status hs_loss(hs_ctx* ctx, int kind, int L, int c, int h, int w, const float* d_recon,
                  const float* d_target, const uint8_t* d_masks, float* d_grads, double* loss) {
    return guard([&] {
        require(L >= 1, "loss: no reconstruction planes");  // loss.cpp:12
        require(kind >= 0 && kind <= 3, "loss: unknown kind");
        CtxWork& cw = work_of(ctx);
        const int slots = loss_partial_slots(kind, L, c, h, w);
        cw.partials.reserve(sizeof(double) * 2 * std::max(slots, 1));
        cw.out3.reserve(sizeof(double) * 3);
        cw.tstats.reserve(sizeof(float2) * ssim_target_stats_elems(c, h, w));
        if (kind == kLossTraining || kind == kLossSsim) {
            require(h >= 11 && w >= 11, "ssim: image smaller than the 11x11 window");
            ssim_target_stats(d_target, c, h, w, cw.tstats.as<float2>(), ctx->stream);
        }
        LossArgs a{kind, L, L, 0, c, h, w, d_recon, nullptr, d_target, cw.tstats.as<float2>(), d_masks, d_grads,
                   nullptr, cw.partials.as<double>()};
        const int used = loss_launch(a, ctx->stream);
        loss_finalize(a, used, cw.out3.as<double>(), ctx->stream);
        double out[3];
        HS_CUDA(cudaMemcpyAsync(out, cw.out3.p, sizeof(out), cudaMemcpyDeviceToHost, ctx->stream));
        HS_CUDA(cudaStreamSynchronize(ctx->stream));
        *loss = out[0];
    });
}

extern "C" hs_status hs_build_masks(const double* h_depth, int h, int w, int L, int near_is_high, uint8_t* h_masks) {
    return guard([&] {
        require(L >= 1, "build_masks: plane count must be >= 1");  // loss.cpp:167
        const size_t n = static_cast<size_t>(h) * w;
        std::memset(h_masks, 0, n * L);
        for (size_t i = 0; i < n; ++i) {  // loss.cpp:172-178
            int bin = static_cast<int>(std::floor(h_depth[i] * L));
            bin = std::min(std::max(bin, 0), L - 1);
            const int plane = near_is_high ? L - 1 - bin : bin;
            h_masks[static_cast<size_t>(plane) * n + i] = 1;
        }
    });
}

// ---- optimizer ------------------------------------------------------------------------------------
extern "C" hs_status hs_cosine_lr(int step, int total_steps, double lr_max, double lr_min, double* out) {
    return guard([&] {
        require(!(total_steps <= 0 || step < 0 || step > total_steps),
                "cosine_lr: step outside [0, total_steps]");  // optimizer.cpp:9-10
        *out = lr_min + 0.5 * (lr_max - lr_min) *
                            (1.0 + std::cos(3.14159265358979323846 * static_cast<double>(step) / total_steps));
    });
}

extern "C" hs_status hs_adan_step(hs_ctx* ctx, const hs_adan_config* cfg, const char* group_name, float* d_params,
                       const float* d_grads, float* d_state, int64_t size, int step_t, double lr) {
    return guard([&] {
        hs_adan_config k = cfg ? *cfg : hs_adan_config{0.98, 0.92, 0.99, 1e-8};
        CtxWork& cw = work_of(ctx);
        cw.flags.reserve(sizeof(uint32_t));
        HS_CUDA(cudaMemsetAsync(cw.flags.p, 0, sizeof(uint32_t), ctx->stream));
        nonfinite_launch(d_grads, size, cw.flags.as<uint32_t>(), ctx->stream);
        uint32_t bad = 0;
        HS_CUDA(cudaMemcpyAsync(&bad, cw.flags.p, sizeof(bad), cudaMemcpyDeviceToHost, ctx->stream));
        HS_CUDA(cudaStreamSynchronize(ctx->stream));
        if (bad)  // optimizer.cpp:52-54
            throw Error(HS_ENONFINITE, std::string("Adan: non-finite gradient in group ") +
                                           (group_name ? group_name : ""));
        adan_group_launch(d_params, d_grads, d_state, size, step_t, lr, k.beta1, k.beta2, k.beta3, k.eps,
                          ctx->stream);
    });
}

// ---- trainer ----------------------------------------------------------------------------------------
// Profiling slots (kernel boundaries): 0 start, 1 binning, 2 raster_fwd,
// 3 rows_fwd, 4 cols_fwd, 5 rows_inv, 6 loss, 7 rows_fwd(bwd), 8 cols_bwd,
// 9 rows_inv(bwd), 10 raster_bwd, 11 adan.
void hs::trainer_enqueue_fwd_bwd(hs_trainer* t, cudaStream_t st, cudaEvent_t shading_ready) {
    const bool prof = t->mark_events;
    auto mark = [&](int i) {
        if (prof) HS_CUDA(cudaEventRecordWithFlags(t->ev[i], st, cudaEventRecordExternal));  // external: kept as a graph node
    };
    mark(0);
    HS_CUDA(cudaMemsetAsync(t->flags.p, 0, sizeof(uint32_t), st));
    {
        NvtxRange r("binning");
        t->rw.project_and_bin(t->params.as<float>(), st, shading_ready);
    }
    mark(1);
    {
        NvtxRange r("raster_fwd");
        raster_forward(t->rw, t->field.as<float2>(), st);
    }
    mark(2);
    {
        NvtxRange r("asm_forward");
        asm_forward(t->aw, t->field.as<float2>(), t->planes.as<float2>(), st, prof ? t->ev + 3 : nullptr);
    }
    {
        NvtxRange r("loss");
        LossArgs a{kLossTraining, t->L, t->L_total, t->plane0, t->c, t->h, t->w, nullptr, t->planes.as<float2>(),
                   t->target.as<float>(), t->tstats.as<float2>(), t->masks.as<uint8_t>(), nullptr,
                   t->dplanes.as<float2>(), t->partials.as<double>(), t->C_total};
        const int used = loss_launch(a, st);
        loss_finalize(a, used, t->out3.as<double>(), st);
    }
    mark(6);
    {
        NvtxRange r("asm_backward");
        asm_backward(t->aw, t->dplanes.as<float2>(), t->back.as<float2>(), st, prof ? t->ev + 7 : nullptr);
    }
    {
        NvtxRange r("raster_bwd");
        raster_backward(t->rw, t->params.as<float>(), t->back.as<float2>(), t->grads.as<float>(),
                        t->flags.as<uint32_t>(), st);
    }
    mark(10);
}

void hs::trainer_enqueue_update(hs_trainer* t, cudaStream_t st) {
    NvtxRange r("adan");
    adan_fused_launch(t->params.as<float>(), t->grads.as<float>(), t->state.as<float>(), t->P, t->groups,
                      t->total_steps, 0.98, 0.92, 0.99, 1e-8, t->step.as<int>(), t->flags.as<uint32_t>(), st);
    if (t->mark_events) HS_CUDA(cudaEventRecordWithFlags(t->ev[11], st, cudaEventRecordExternal));
}

static void trainer_raise(hs_trainer* t, uint32_t flags, const uint32_t* stat);

void hs::trainer_check_after(hs_trainer* t) {
    uint32_t flags = 0, stat[4];
    cudaStream_t st = t->ctx->stream;
    HS_CUDA(cudaMemcpyAsync(&flags, t->flags.p, sizeof(flags), cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaMemcpyAsync(stat, t->rw.status.p, sizeof(stat), cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));
    trainer_raise(t, flags, stat);
}

static void trainer_raise(hs_trainer* t, uint32_t flags, const uint32_t* stat) {
    (void)t;
    if (stat[1]) throw Error(HS_EOVERFLOW, "trainer: tile-pair capacity exceeded; call hs_trainer_reserve_pairs");
    if (stat[2]) throw Error(HS_EINVAL, "activate: non-finite input");
    if (flags) {
        const int g = __builtin_ctz(flags);
        throw Error(HS_ENONFINITE, std::string("Adan: non-finite gradient in group ") + kGroupNames[g]);
    }
}

extern "C" {

hs_status hs_trainer_create(hs_ctx* ctx, const hs_trainer_config* cfg, hs_trainer** out) {
    return guard([&] {
        require(cfg && cfg->n >= 1 && cfg->c >= 1 && cfg->width > 0 && cfg->height > 0,
                "trainer: invalid configuration");
        require(cfg->planes >= 1 && cfg->distances, "trainer: plane count must be >= 1");
        require(cfg->total_steps > 0, "cosine_lr: step outside [0, total_steps]");
        check_spec(&cfg->spec, cfg->c);
        auto t = std::make_unique<hs_trainer>();
        t->ctx = ctx;
        t->n = cfg->n;
        t->c = cfg->c;
        t->w = cfg->width;
        t->h = cfg->height;
        t->L_total = cfg->planes;
        require(cfg->channels_total == 0 || cfg->channels_total >= cfg->c,
                "trainer: channels_total must be 0 or >= the shard's channel count");
        t->C_total = cfg->channels_total > 0 ? cfg->channels_total : cfg->c;
        const int pb = (cfg->plane_end > cfg->plane_begin) ? cfg->plane_begin : 0;
        const int pe = (cfg->plane_end > cfg->plane_begin) ? cfg->plane_end : cfg->planes;
        require(pb >= 0 && pe <= cfg->planes, "trainer: plane shard out of range");
        t->plane0 = pb;
        t->L = pe - pb;
        t->total_steps = cfg->total_steps;
        t->distances.assign(cfg->distances + pb, cfg->distances + pe);
        t->wavelengths.assign(cfg->spec.wavelengths, cfg->spec.wavelengths + cfg->spec.n_wavelengths);
        t->spec = cfg->spec;
        t->spec.wavelengths = t->wavelengths.data();
        const int64_t N = t->n, C = t->c;
        t->P = (6 + 2 * C) * N;
        // group boundaries in the flat buffer (gaussian_set.hpp:14-19; pipeline.cpp:243-249)
        const int64_t b[7] = {0, 2 * N, 4 * N, 5 * N, 5 * N + N * C, 5 * N + 2 * N * C, 6 * N + 2 * N * C};
        const float lrs[6] = {1e-2f, 5e-3f, 1e-3f, 2.5e-3f, 2.5e-3f, 2.5e-2f};
        for (int i = 0; i < 6; ++i) {
            t->groups.begin[i] = b[i];
            t->groups.end[i] = b[i + 1];
            t->groups.base_lr[i] = lrs[i];
        }
        const size_t hw = static_cast<size_t>(t->h) * t->w, chw = hw * C;
        cudaStream_t st = ctx->stream;
        t->params.reserve(sizeof(float) * t->P);
        t->grads.reserve(sizeof(float) * t->P);
        t->state.reserve(sizeof(float) * 4 * t->P);
        HS_CUDA(cudaMemsetAsync(t->state.p, 0, sizeof(float) * 4 * t->P, st));
        HS_CUDA(cudaMemsetAsync(t->grads.p, 0, sizeof(float) * t->P, st));
        t->field.reserve(sizeof(float2) * chw);
        t->planes.reserve(sizeof(float2) * chw * t->L);
        t->dplanes.reserve(sizeof(float2) * chw * t->L);
        t->back.reserve(sizeof(float2) * chw);
        t->target.reserve(sizeof(float) * chw);
        t->masks.reserve(hw * t->L_total);
        HS_CUDA(cudaMemcpyAsync(t->target.p, cfg->h_target, sizeof(float) * chw, cudaMemcpyHostToDevice, st));
        HS_CUDA(cudaMemcpyAsync(t->masks.p, cfg->h_masks, hw * t->L_total, cudaMemcpyHostToDevice, st));
        require(t->h >= 11 && t->w >= 11, "ssim: image smaller than the 11x11 window");
        t->tstats.reserve(sizeof(float2) * ssim_target_stats_elems(t->c, t->h, t->w));
        ssim_target_stats(t->target.as<float>(), t->c, t->h, t->w, t->tstats.as<float2>(), st);
        t->loss_slots = loss_partial_slots(kLossTraining, t->L, t->c, t->h, t->w);
        t->partials.reserve(sizeof(double) * 2 * t->loss_slots);
        t->out3.reserve(sizeof(double) * 3);
        t->flags.reserve(sizeof(uint32_t));
        t->step.reserve(kAdanStepBytes);  // step counters + the fused Adan's precomputed group constants
        HS_CUDA(cudaMemsetAsync(t->step.p, 0, kAdanStepBytes, st));
        adan_init_consts(t->groups, t->total_steps, 0.98, 0.92, 0.99, t->step.as<int>(), st);
        HS_CUDA(cudaMemsetAsync(t->flags.p, 0, sizeof(uint32_t), st));
        t->rw.prepare(t->n, t->c, t->w, t->h);
        t->aw.prepare(t->c, t->h, t->w, t->spec.pad_factor, t->L);
        t->aw.L = t->L;
        t->aw.set_transfer(t->spec, t->distances.data(), t->distances.data(), st);
        for (auto& e : t->ev) HS_CUDA(cudaEventCreate(&e));
        HS_CUDA(cudaStreamSynchronize(st));
        *out = t.release();
    });
}

void hs_trainer_destroy(hs_trainer* tr) { delete tr; }

hs_status hs_trainer_set_params(hs_trainer* t, const float* params, int from_device) {
    return guard([&] {
        HS_CUDA(cudaMemcpyAsync(t->params.p, params, sizeof(float) * t->P,
                                from_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, t->ctx->stream));
        if (!from_device) HS_CUDA(cudaStreamSynchronize(t->ctx->stream));
    });
}

hs_status hs_trainer_get_params(hs_trainer* t, float* params, int to_device) {
    return guard([&] {
        HS_CUDA(cudaMemcpyAsync(params, t->params.p, sizeof(float) * t->P,
                                to_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, t->ctx->stream));
        if (!to_device) HS_CUDA(cudaStreamSynchronize(t->ctx->stream));
    });
}

float* hs_trainer_params_ptr(hs_trainer* t) { return t->params.as<float>(); }
float* hs_trainer_grads_ptr(hs_trainer* t) { return t->grads.as<float>(); }
uint32_t* hs_trainer_flags_ptr(hs_trainer* t) { return t->flags.as<uint32_t>(); }
int64_t hs_trainer_param_count(hs_trainer* t) { return t->P; }
int hs_trainer_step_count(hs_trainer* t) { return t->host_step; }

// Every captured graph of the trainer (they bake in buffer addresses and the
// backward form): dropped when either changes, re-captured on next use.
static void drop_graphs(hs_trainer* t) {
    for (cudaGraphExec_t* g : {&t->graph, &t->prof_graph, &t->host_graph, &t->slab_graph, &t->run_graph0,
                               &t->run_graph}) {
        if (*g) cudaGraphExecDestroy(*g);
        *g = nullptr;
    }
}

hs_status hs_trainer_reserve_pairs(hs_trainer* t, int64_t cap) {
    return guard([&] {
        t->rw.reserve_pairs(cap);
        drop_graphs(t);
    });
}

hs_status hs_trainer_use_graph(hs_trainer* t, int enable) {
    t->use_graph = enable != 0;
    if (!t->use_graph) drop_graphs(t);
    return HS_OK;
}

hs_status hs_trainer_set_deterministic(hs_trainer* t, int enable) {
    const bool tile = enable == 0;
    if (t->rw.tile_bwd != tile) {
        t->rw.tile_bwd = tile;
        drop_graphs(t);
    }
    return HS_OK;
}

hs_status hs_ctx_set_deterministic(hs_ctx* ctx, int enable) {
    return guard([&] { work_of(ctx).rw.tile_bwd = enable == 0; });
}

hs_status hs_trainer_set_profiling(hs_trainer* t, int enable) {
    t->profiling = enable != 0;
    return HS_OK;
}

hs_status hs_trainer_forward_backward(hs_trainer* t) {
    return guard([&] {
        NvtxRange nvtx("hs_trainer_forward_backward");
        require(t->host_step <= t->total_steps, "cosine_lr: step outside [0, total_steps]");
        t->mark_events = t->profiling;  // eager split step: stage events as the plain step
        try {
            trainer_enqueue_fwd_bwd(t, t->ctx->stream);
        } catch (...) {
            t->mark_events = false;
            throw;
        }
        t->mark_events = false;
    });
}

// After a cross-rank gradient all-reduce: re-derive the non-finite group bits
// from the summed buffer, so every rank takes the same decision (a rank's own
// partial may be finite while the sum is not).
hs_status hs_trainer_check_grads(hs_trainer* t) {
    return guard([&] {
        group_nonfinite_launch(t->grads.as<float>(), t->P, t->groups, t->flags.as<uint32_t>(), t->ctx->stream);
    });
}

hs_status hs_trainer_apply_update(hs_trainer* t) {
    return guard([&] {
        NvtxRange nvtx("hs_trainer_apply_update");
        t->mark_events = t->profiling;
        trainer_enqueue_update(t, t->ctx->stream);
        t->mark_events = false;
        t->host_step += 1;
    });
}

hs_status hs_trainer_check_grads_range(hs_trainer* t, int64_t begin, int64_t end) {
    return guard([&] {
        group_nonfinite_launch(t->grads.as<float>(), t->P, t->groups, t->flags.as<uint32_t>(), t->ctx->stream, begin,
                               end);
    });
}

hs_status hs_trainer_apply_update_range(hs_trainer* t, int64_t begin, int64_t end) {
    return guard([&] {
        require(t->host_step <= t->total_steps, "cosine_lr: step outside [0, total_steps]");
        adan_fused_launch(t->params.as<float>(), t->grads.as<float>(), t->state.as<float>(), t->P, t->groups,
                          t->total_steps, 0.98, 0.92, 0.99, 1e-8, t->step.as<int>(), t->flags.as<uint32_t>(),
                          t->ctx->stream, begin, end);
        t->host_step += 1;
    });
}

static void trainer_launch_step(hs_trainer* t) {
    {
        // cosine_lr(step, steps, ...) throws past the horizon (optimizer.cpp:9-10)
        require(t->host_step <= t->total_steps, "cosine_lr: step outside [0, total_steps]");
        cudaStream_t st = t->ctx->stream;
        // profiling: the stage events are recorded by this step only (eagerly,
        // or as event-record nodes of a separate step graph, so that the
        // stage times carry no host enqueue gaps)
        struct Marks {
            hs_trainer* t;
            ~Marks() { t->mark_events = false; }
        } marks{t};
        t->mark_events = t->profiling;
        if (t->use_graph) {
            cudaGraphExec_t& ge = t->profiling ? t->prof_graph : t->graph;
            if (!ge) {
                cudaStream_t cap_st = st;
                bool own = false;
                if (cap_st == nullptr) {  // legacy stream cannot be captured
                    HS_CUDA(cudaStreamCreateWithFlags(&cap_st, cudaStreamNonBlocking));
                    own = true;
                }
                cudaGraph_t g = nullptr;
                HS_CUDA(cudaStreamBeginCapture(cap_st, cudaStreamCaptureModeThreadLocal));
                try {
                    trainer_enqueue_fwd_bwd(t, cap_st);
                    trainer_enqueue_update(t, cap_st);
                } catch (...) {
                    cudaStreamEndCapture(cap_st, &g);
                    if (g) cudaGraphDestroy(g);
                    if (own) cudaStreamDestroy(cap_st);
                    throw;
                }
                HS_CUDA(cudaStreamEndCapture(cap_st, &g));
                HS_CUDA(cudaGraphInstantiate(&ge, g, 0));
                HS_CUDA(cudaGraphDestroy(g));
                if (own) HS_CUDA(cudaStreamDestroy(cap_st));
            }
            HS_CUDA(cudaGraphLaunch(ge, st));
            note_launch(0);
        } else {
            trainer_enqueue_fwd_bwd(t, st);
            trainer_enqueue_update(t, st);
        }
        t->host_step += 1;
    }
}

hs_status hs_trainer_step(hs_trainer* t, double* loss_out) {
    return guard([&] {
        NvtxRange nvtx("hs_trainer_step");
        trainer_launch_step(t);
        if (loss_out) {
            trainer_check_after(t);
            double o3[3];
            HS_CUDA(cudaMemcpy(o3, t->out3.p, sizeof(o3), cudaMemcpyDeviceToHost));
            *loss_out = o3[0];
        }
    });
}

// One step with host-resident parameters (the reference's GaussianSet lives on
// the host, pipeline.cpp:253-297).  The geometry groups are uploaded first on
// the trainer stream; the amplitude/phase groups then go up on a copy stream
// while the geometry is projected and binned, and only the shading kernel
// waits for them.  Then the step, the D2H of the updated parameters and of the loss /
// error words, and ONE synchronisation.  With graphs on, the whole sequence
// (copies included) is one CUDA graph, re-captured when the host buffers change.
static void enqueue_host_step(hs_trainer* t, cudaStream_t st, const float* in, float* out) {
    const size_t N = t->n, geo0 = 5 * N, ap = 2 * N * t->c;  // [pos 2N | scale 2N | rot N | amp | phase | opa N]
    float* d = t->params.as<float>();
    // geometry first (the copy engines would otherwise split the link between
    // the two uploads and delay the binning), then amplitude/phase alongside it
    if (in) {
        HS_CUDA(cudaMemcpyAsync(d, in, sizeof(float) * geo0, cudaMemcpyHostToDevice, st));
        HS_CUDA(cudaMemcpyAsync(d + geo0 + ap, in + geo0 + ap, sizeof(float) * N, cudaMemcpyHostToDevice, st));
    }
    HS_CUDA(cudaEventRecord(t->ev_fork, st));
    HS_CUDA(cudaStreamWaitEvent(t->copy_st, t->ev_fork, 0));
    if (in) HS_CUDA(cudaMemcpyAsync(d + geo0, in + geo0, sizeof(float) * ap, cudaMemcpyHostToDevice, t->copy_st));
    HS_CUDA(cudaEventRecord(t->ev_ap, t->copy_st));
    trainer_enqueue_fwd_bwd(t, st, t->ev_ap);
    trainer_enqueue_update(t, st);
    if (out) HS_CUDA(cudaMemcpyAsync(out, d, sizeof(float) * t->P, cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaMemcpyAsync(t->h_words, t->flags.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaMemcpyAsync(t->h_words + 1, t->rw.status.p, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaMemcpyAsync(t->h_o3, t->out3.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
}

hs_status hs_trainer_step_host(hs_trainer* t, const float* h_params_in, float* h_params_out, double* loss_out) {
    return guard([&] {
        NvtxRange nvtx("hs_trainer_step_host");
        require(t->host_step <= t->total_steps, "cosine_lr: step outside [0, total_steps]");
        cudaStream_t st = t->ctx->stream;
        if (!t->copy_st) {
            HS_CUDA(cudaStreamCreateWithFlags(&t->copy_st, cudaStreamNonBlocking));
            HS_CUDA(cudaEventCreateWithFlags(&t->ev_fork, cudaEventDisableTiming));
            HS_CUDA(cudaEventCreateWithFlags(&t->ev_ap, cudaEventDisableTiming));
            HS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&t->h_words), 5 * sizeof(uint32_t), cudaHostAllocDefault));
            HS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&t->h_o3), 3 * sizeof(double), cudaHostAllocDefault));
        }
        bool done = false;
        if (t->use_graph && st != nullptr) {
            if (t->host_graph && (t->host_in != h_params_in || t->host_out != h_params_out)) {
                HS_CUDA(cudaGraphExecDestroy(t->host_graph));
                t->host_graph = nullptr;
            }
            if (!t->host_graph) {
                cudaGraph_t g = nullptr;
                HS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
                try {
                    enqueue_host_step(t, st, h_params_in, h_params_out);
                } catch (...) {
                    cudaStreamEndCapture(st, &g);
                    if (g) cudaGraphDestroy(g);
                    throw;
                }
                HS_CUDA(cudaStreamEndCapture(st, &g));
                HS_CUDA(cudaGraphInstantiate(&t->host_graph, g, 0));
                HS_CUDA(cudaGraphDestroy(g));
                t->host_in = h_params_in;
                t->host_out = h_params_out;
            }
            HS_CUDA(cudaGraphLaunch(t->host_graph, st));
            note_launch(0);
            done = true;
        }
        if (!done) enqueue_host_step(t, st, h_params_in, h_params_out);
        t->host_step += 1;
        HS_CUDA(cudaStreamSynchronize(st));
        trainer_raise(t, t->h_words[0], t->h_words + 1);
        if (loss_out) *loss_out = t->h_o3[0];
    });
}

// ---- pipelined multi-step run with host-resident parameters ----
// Per-step gate between the raster backward and Adan: logs the step's
// non-finite group bits and rasterizer status (overflow, non-finite input) and
// its loss; after a failed step every later step of the run applies no update
// (flags = group 0: Adan skips all groups and keeps its step counter), so the
// parameters stay as the reference leaves them when Adan::step throws.
}  // extern "C"
namespace hs {
namespace {
__global__ void run_gate_kernel(uint32_t* flags, const uint32_t* stat, const double* o3, uint32_t* words,
                                uint32_t* flog, double* llog) {
    const uint32_t f = *flags;
    const uint32_t s = (stat[1] ? 0x100u : 0u) | (stat[2] ? 0x200u : 0u);
    const uint32_t k = words[1]++;
    flog[k] = f | s;
    llog[k] = o3[0];
    if (words[0]) *flags = 1u;
    else if (f | s) words[0] = 1u;
}
constexpr int kRunBatch = 1024;  // steps per device log (one host check per batch)
}  // namespace
}  // namespace hs
extern "C" {

// One step of the run.  Steady state (tail = true) overlaps the previous
// step's amplitude/phase download (copy stream 2) with this step's geometry
// upload and projection; the graph ends with the download of the geometry
// groups, so the next step's upload reads the values this step wrote.
static void enqueue_run_step(hs_trainer* t, cudaStream_t st, float* h, bool tail) {
    const size_t N = t->n, geo0 = 5 * N, ap = 2 * N * t->c;  // [pos 2N | scale 2N | rot N | amp | phase | opa N]
    float* d = t->params.as<float>();
    if (tail) {  // D2H of step k-1's amplitude/phase groups, alongside this step's start
        HS_CUDA(cudaEventRecord(t->ev_fork, st));
        HS_CUDA(cudaStreamWaitEvent(t->copy_st2, t->ev_fork, 0));
        HS_CUDA(cudaMemcpyAsync(h + geo0, d + geo0, sizeof(float) * ap, cudaMemcpyDeviceToHost, t->copy_st2));
        HS_CUDA(cudaEventRecord(t->ev_apdown, t->copy_st2));
    }
    HS_CUDA(cudaMemcpyAsync(d, h, sizeof(float) * geo0, cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(d + geo0 + ap, h + geo0 + ap, sizeof(float) * N, cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaEventRecord(t->ev_fork, st));
    HS_CUDA(cudaStreamWaitEvent(t->copy_st, t->ev_fork, 0));
    if (tail) HS_CUDA(cudaStreamWaitEvent(t->copy_st, t->ev_apdown, 0));
    HS_CUDA(cudaMemcpyAsync(d + geo0, h + geo0, sizeof(float) * ap, cudaMemcpyHostToDevice, t->copy_st));
    HS_CUDA(cudaEventRecord(t->ev_ap, t->copy_st));
    trainer_enqueue_fwd_bwd(t, st, t->ev_ap);
    run_gate_kernel<<<1, 1, 0, st>>>(t->flags.as<uint32_t>(), t->rw.status.as<uint32_t>(), t->out3.as<double>(),
                                     t->run_words.as<uint32_t>(), t->run_flog.as<uint32_t>(),
                                     t->run_llog.as<double>());
    launch_check("run_gate");
    trainer_enqueue_update(t, st);
    HS_CUDA(cudaMemcpyAsync(h, d, sizeof(float) * geo0, cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaMemcpyAsync(h + geo0 + ap, d + geo0 + ap, sizeof(float) * N, cudaMemcpyDeviceToHost, st));
}

hs_status hs_trainer_run_host(hs_trainer* t, float* h_params, int steps, double* losses_out) {
    return guard([&] {
        NvtxRange nvtx("hs_trainer_run_host");
        require(steps >= 0 && h_params != nullptr, "run_host: bad arguments");
        require(t->R == 0, "run_host: not for row-slab shards (use the slab stages)");
        if (steps == 0) return;
        // cosine_lr(step, steps, ...) throws past the horizon (optimizer.cpp:9-10)
        require(t->host_step + steps - 1 <= t->total_steps, "cosine_lr: step outside [0, total_steps]");
        cudaStream_t st = t->ctx->stream;
        if (!t->copy_st) {
            HS_CUDA(cudaStreamCreateWithFlags(&t->copy_st, cudaStreamNonBlocking));
            HS_CUDA(cudaEventCreateWithFlags(&t->ev_fork, cudaEventDisableTiming));
            HS_CUDA(cudaEventCreateWithFlags(&t->ev_ap, cudaEventDisableTiming));
            HS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&t->h_words), 5 * sizeof(uint32_t), cudaHostAllocDefault));
            HS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&t->h_o3), 3 * sizeof(double), cudaHostAllocDefault));
        }
        if (!t->copy_st2) {
            HS_CUDA(cudaStreamCreateWithFlags(&t->copy_st2, cudaStreamNonBlocking));
            HS_CUDA(cudaEventCreateWithFlags(&t->ev_apdown, cudaEventDisableTiming));
            t->run_words.reserve(2 * sizeof(uint32_t));
            t->run_flog.reserve(kRunBatch * sizeof(uint32_t));
            t->run_llog.reserve(kRunBatch * sizeof(double));
        }
        if (t->run_host != h_params) {
            for (cudaGraphExec_t* g : {&t->run_graph0, &t->run_graph})
                if (*g) {
                    HS_CUDA(cudaGraphExecDestroy(*g));
                    *g = nullptr;
                }
            t->run_host = h_params;
        }
        auto capture = [&](bool tail) {
            cudaGraph_t g = nullptr;
            cudaGraphExec_t ge = nullptr;
            HS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            try {
                enqueue_run_step(t, st, h_params, tail);
            } catch (...) {
                cudaStreamEndCapture(st, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            HS_CUDA(cudaStreamEndCapture(st, &g));
            HS_CUDA(cudaGraphInstantiate(&ge, g, 0));
            HS_CUDA(cudaGraphDestroy(g));
            return ge;
        };
        std::vector<uint32_t> flog(kRunBatch);
        std::vector<double> llog(kRunBatch);
        const size_t N = t->n, geo0 = 5 * N, ap = 2 * N * t->c;
        for (int b0 = 0; b0 < steps; b0 += kRunBatch) {
            const int nb = std::min(kRunBatch, steps - b0);
            HS_CUDA(cudaMemsetAsync(t->run_words.p, 0, 2 * sizeof(uint32_t), st));
            for (int i = 0; i < nb; ++i) {
                if (t->use_graph && st != nullptr) {  // (no capture on the legacy stream)
                    cudaGraphExec_t& ge = i == 0 ? t->run_graph0 : t->run_graph;
                    if (!ge) ge = capture(i != 0);
                    HS_CUDA(cudaGraphLaunch(ge, st));
                    note_launch(0);
                } else {
                    enqueue_run_step(t, st, h_params, i != 0);
                }
            }
            // the last step's amplitude/phase download, the logs, one synchronisation
            float* d = t->params.as<float>();
            HS_CUDA(cudaMemcpyAsync(h_params + geo0, d + geo0, sizeof(float) * ap, cudaMemcpyDeviceToHost, st));
            HS_CUDA(cudaMemcpyAsync(flog.data(), t->run_flog.p, nb * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            HS_CUDA(cudaMemcpyAsync(llog.data(), t->run_llog.p, nb * sizeof(double), cudaMemcpyDeviceToHost, st));
            HS_CUDA(cudaStreamSynchronize(st));
            for (int i = 0; i < nb; ++i) {
                t->host_step += 1;
                if (losses_out) losses_out[b0 + i] = llog[i];
                if (flog[i]) {
                    const uint32_t stat[4] = {0u, (flog[i] & 0x100u) ? 1u : 0u, (flog[i] & 0x200u) ? 1u : 0u, 0u};
                    trainer_raise(t, flog[i] & 0xffu, stat);
                }
            }
        }
    });
}

hs_status hs_trainer_last_loss(hs_trainer* t, double* loss_out, int64_t* npairs_out) {
    return guard([&] {
        trainer_check_after(t);
        double o3[3];
        uint32_t stat[4];
        HS_CUDA(cudaMemcpy(o3, t->out3.p, sizeof(o3), cudaMemcpyDeviceToHost));
        HS_CUDA(cudaMemcpy(stat, t->rw.status.p, sizeof(stat), cudaMemcpyDeviceToHost));
        if (loss_out) *loss_out = o3[0];
        if (npairs_out) *npairs_out = stat[0];
    });
}

hs_status hs_trainer_loss_partials(hs_trainer* t, double* out2) {
    return guard([&] {
        double o3[3];
        HS_CUDA(cudaMemcpyAsync(o3, t->out3.p, sizeof(o3), cudaMemcpyDeviceToHost, t->ctx->stream));
        HS_CUDA(cudaStreamSynchronize(t->ctx->stream));
        out2[0] = o3[1];
        out2[1] = o3[2];
    });
}

hs_status hs_trainer_stage_ms(hs_trainer* t, double* out12) {
    return guard([&] {
        require(t->profiling, "trainer: stage timing needs profiling on");
        HS_CUDA(cudaEventSynchronize(t->ev[11]));
        for (int i = 0; i < 11; ++i) {
            float ms = 0.f;
            HS_CUDA(cudaEventElapsedTime(&ms, t->ev[i], t->ev[i + 1]));
            out12[i] = ms;
        }
        float tot = 0.f;
        HS_CUDA(cudaEventElapsedTime(&tot, t->ev[0], t->ev[11]));
        out12[11] = tot;
    });
}

}  // extern "C"

// ---- row-slab sharding (cfg4: distributed 2D FFT with all-to-all transposes) ----------------
// Layouts (float2 units, CC = column tile width, nt = tiles, ts = nt / R):
//   T1r [C][nt][hr][CC]   row side: this rank's rows of every tile
//   T1c [C][ts][H][CC]    column side: all rows of this rank's tiles
//   exchange buffers are peer-major: [peer][planes][ts][rows][CC]
// Exchange 0: T1r -> T1c (forward rows -> columns), 1: T2c -> T2r with the
// loss-band rows (columns -> rows), 2: T3r own rows -> T3c (backward rows ->
// columns), 3: T4c -> T4r (columns -> rows).
static void slab_build_maps(hs_trainer* t) {
    const int R = t->R, C = t->c, LC = t->L * t->c, H = t->h, hr = t->hr, ts = t->ts, He = t->He;
    const int64_t CC = t->aw.CC, nt = t->aw.ntiles;
    auto fill = [&](ChunkMap& m, int B, auto f) {
        m.A = R;
        m.B = B;
        m.T = ts;
        for (int a = 0; a < R; ++a) f(a, m);
    };
    // 0 pack T1r -> send [s][C][ts][hr][CC]
    fill(t->m_pack[0], C, [&](int a, ChunkMap& m) {
        m.len[a] = hr * CC; m.sA[a] = a * ts * hr * CC; m.sB[a] = nt * hr * CC; m.sT[a] = hr * CC;
        m.dA[a] = int64_t(a) * C * ts * hr * CC; m.dB[a] = ts * hr * CC; m.dT[a] = hr * CC;
    });
    // 0 unpack recv [r][C][ts][hr][CC] -> T1c
    auto unpack_cols = [&](int B) {
        return [=](int a, ChunkMap& m) {
            m.len[a] = hr * CC; m.sA[a] = int64_t(a) * B * ts * hr * CC; m.sB[a] = ts * hr * CC; m.sT[a] = hr * CC;
            m.dA[a] = a * hr * CC; m.dB[a] = int64_t(ts) * H * CC; m.dT[a] = H * CC;
        };
    };
    fill(t->m_unpack[0], C, unpack_cols(C));
    // 1 pack T2c [LC][ts][H][CC] -> send [d][LC][ts][He_d][CC] (loss-band rows of d)
    int64_t off = 0;
    fill(t->m_pack[1], LC, [&](int a, ChunkMap& m) {
        const int64_t he = t->He_of[a];
        m.len[a] = he * CC; m.sA[a] = t->g0_of[a] * CC; m.sB[a] = int64_t(ts) * H * CC; m.sT[a] = H * CC;
        m.dA[a] = off; m.dB[a] = ts * he * CC; m.dT[a] = he * CC;
        off += LC * ts * he * CC;
    });
    // 1 unpack recv [s][LC][ts][He][CC] -> T2r [LC][nt][He][CC]
    fill(t->m_unpack[1], LC, [&](int a, ChunkMap& m) {
        m.len[a] = He * CC; m.sA[a] = int64_t(a) * LC * ts * He * CC; m.sB[a] = int64_t(ts) * He * CC;
        m.sT[a] = He * CC; m.dA[a] = int64_t(a) * ts * He * CC; m.dB[a] = nt * He * CC; m.dT[a] = He * CC;
    });
    // 2 pack T3r own rows -> send [s][LC][ts][hr][CC]
    fill(t->m_pack[2], LC, [&](int a, ChunkMap& m) {
        m.len[a] = hr * CC; m.sA[a] = int64_t(a) * ts * He * CC + t->top * CC; m.sB[a] = nt * He * CC;
        m.sT[a] = He * CC; m.dA[a] = int64_t(a) * LC * ts * hr * CC; m.dB[a] = ts * hr * CC; m.dT[a] = hr * CC;
    });
    fill(t->m_unpack[2], LC, unpack_cols(LC));
    // 3 pack T4c [C][ts][H][CC] -> send [d][C][ts][hr][CC]
    fill(t->m_pack[3], C, [&](int a, ChunkMap& m) {
        m.len[a] = hr * CC; m.sA[a] = a * hr * CC; m.sB[a] = int64_t(ts) * H * CC; m.sT[a] = H * CC;
        m.dA[a] = int64_t(a) * C * ts * hr * CC; m.dB[a] = ts * hr * CC; m.dT[a] = hr * CC;
    });
    // 3 unpack recv [s][C][ts][hr][CC] -> T4r [C][nt][hr][CC]
    fill(t->m_unpack[3], C, [&](int a, ChunkMap& m) {
        m.len[a] = hr * CC; m.sA[a] = int64_t(a) * C * ts * hr * CC; m.sB[a] = ts * hr * CC; m.sT[a] = hr * CC;
        m.dA[a] = int64_t(a) * ts * hr * CC; m.dB[a] = nt * hr * CC; m.dT[a] = hr * CC;
    });
    // element counts (floats) per peer: send, recv
    for (int a = 0; a < R; ++a) {
        const int64_t f = 2 * CC * ts;
        t->s_counts[0][a] = t->s_counts[0][R + a] = f * C * hr;
        t->s_counts[1][a] = f * LC * t->He_of[a];
        t->s_counts[1][R + a] = f * LC * He;
        t->s_counts[2][a] = t->s_counts[2][R + a] = f * LC * hr;
        t->s_counts[3][a] = t->s_counts[3][R + a] = f * C * hr;
    }
}

extern "C" hs_status hs_trainer_set_row_slab(hs_trainer* t, int rank, int ranks) {
    return guard([&] {
        require(ranks >= 1 && ranks <= kMaxPeers && rank >= 0 && rank < ranks, "row slab: bad rank / rank count");
        require(t->L == t->L_total && t->C_total == t->c, "row slab: not combinable with plane or channel shards");
        require(t->h % ranks == 0, "row slab: canvas height must divide into equal slabs");
        AsmWork& aw = t->aw;
        require(static_cast<int64_t>(aw.ntiles) * aw.CC == aw.Px && aw.ntiles % ranks == 0,
                "row slab: padded width must divide into equal column-tile slabs");
        t->R = ranks;
        t->rank = rank;
        t->hr = t->h / ranks;
        t->ts = aw.ntiles / ranks;
        t->He_of.assign(ranks, 0);
        t->g0_of.assign(ranks, 0);
        for (int r = 0; r < ranks; ++r) {
            const int a = std::max(0, r * t->hr - 10), b = std::min(t->h, (r + 1) * t->hr + 10);
            t->g0_of[r] = a;
            t->He_of[r] = b - a;
        }
        t->h0 = rank * t->hr;
        t->rw.band_ty0 = t->h0 / kTile;  // the raster forward reads only the band's tiles
        t->rw.band_ty1 = (t->h0 + t->hr - 1) / kTile;
        t->rw.band_y0 = t->h0;
        t->rw.band_y1 = t->h0 + t->hr - 1;
        t->rw.band_list.reserve(sizeof(uint32_t) * std::max(t->n, 1));  // no allocation inside a captured step
        t->rw.band_n.reserve(sizeof(uint32_t));
        t->g0 = t->g0_of[rank];
        t->He = t->He_of[rank];
        t->top = t->h0 - t->g0;
        require(t->He >= 11, "ssim: image smaller than the 11x11 window");
        const int C = t->c, LC = t->L * t->c, W = t->w, Hm = t->hr + 20;
        const size_t band = static_cast<size_t>(t->He) * W;
        cudaStream_t st = t->ctx->stream;
        t->s_planes.reserve(sizeof(float2) * LC * band);
        t->s_dplanes.reserve(sizeof(float2) * LC * band);
        t->s_target.reserve(sizeof(float) * C * band);
        t->s_masks.reserve(static_cast<size_t>(t->L) * band);
        t->s_tstats.reserve(sizeof(float2) * ssim_target_stats_elems(C, t->He, W));
        const size_t tiled = static_cast<size_t>(aw.ntiles) * Hm * aw.CC;
        t->s_T.reserve(sizeof(float2) * LC * tiled);
        t->s_send.reserve(sizeof(float2) * LC * tiled);
        t->s_recv.reserve(sizeof(float2) * LC * tiled);
        t->s_recv2.reserve(sizeof(float2) * LC * tiled);
        t->s_flags.reserve(sizeof(uint32_t) * (kMaxPeers + 2));
        HS_CUDA(cudaMemsetAsync(t->s_flags.p, 0, sizeof(uint32_t) * (kMaxPeers + 2), st));
        t->s_put = false;
        if (t->slab_graph) {
            HS_CUDA(cudaGraphExecDestroy(t->slab_graph));
            t->slab_graph = nullptr;
        }
        // loss-band slices of the target and the masks, and the band's target window stats
        HS_CUDA(cudaMemcpy2DAsync(t->s_target.p, band * sizeof(float), t->target.as<float>() + static_cast<size_t>(t->g0) * W,
                                  static_cast<size_t>(t->h) * W * sizeof(float), band * sizeof(float), C,
                                  cudaMemcpyDeviceToDevice, st));
        HS_CUDA(cudaMemcpy2DAsync(t->s_masks.p, band, t->masks.as<uint8_t>() + static_cast<size_t>(t->g0) * W,
                                  static_cast<size_t>(t->h) * W, band, t->L, cudaMemcpyDeviceToDevice, st));
        ssim_target_stats(t->s_target.as<float>(), C, t->He, W, t->s_tstats.as<float2>(), st);
        t->s_loss_slots = loss_partial_slots(kLossTraining, t->L, C, t->He, W);
        if (t->s_loss_slots > t->loss_slots) t->partials.reserve(sizeof(double) * 2 * t->s_loss_slots);
        slab_build_maps(t);
        HS_CUDA(cudaStreamSynchronize(st));
    });
}

extern "C" hs_status hs_trainer_slab_counts(hs_trainer* t, int exchange, int64_t* out) {
    return guard([&] {
        require(t->R >= 1, "row slab: trainer is not row-slab sharded");
        require(exchange >= 0 && exchange < 4, "row slab: exchange index outside 0..3");
        for (int i = 0; i < 2 * t->R; ++i) out[i] = t->s_counts[exchange][i];
    });
}

extern "C" float* hs_trainer_slab_send_ptr(hs_trainer* t) { return t->s_send.as<float>(); }
extern "C" float* hs_trainer_slab_recv_ptr(hs_trainer* t) { return t->s_recv.as<float>(); }
extern "C" float* hs_trainer_slab_recv2_ptr(hs_trainer* t) { return t->s_recv2.as<float>(); }
extern "C" uint32_t* hs_trainer_slab_flags_ptr(hs_trainer* t) { return t->s_flags.as<uint32_t>(); }

extern "C" hs_status hs_trainer_slab_set_peers(hs_trainer* t, float* const* recv0, float* const* recv1,
                                               uint32_t* const* flags) {
    return guard([&] {
        require(t->R >= 1, "row slab: trainer is not row-slab sharded");
        require(recv0 && recv1 && flags, "row slab: peer pointer arrays missing");
        for (int a = 0; a < t->R; ++a) {
            require(recv0[a] && recv1[a] && flags[a], "row slab: null peer pointer");
            t->s_peer_recv[0][a] = reinterpret_cast<float2*>(recv0[a]);
            t->s_peer_recv[1][a] = reinterpret_cast<float2*>(recv1[a]);
            t->s_peer_flags[a] = flags[a];
        }
        t->s_put = true;
        if (t->slab_graph) {  // the captured step holds the previous peer addresses
            HS_CUDA(cudaGraphExecDestroy(t->slab_graph));
            t->slab_graph = nullptr;
        }
    });
}

extern "C" uint32_t* hs_trainer_slab_error_ptr(hs_trainer* t) {
    return t->R >= 1 ? t->s_flags.as<uint32_t>() + kMaxPeers : nullptr;
}

extern "C" hs_status hs_trainer_slab_status(hs_trainer* t, uint32_t* error) {
    return guard([&] {
        require(t->R >= 1, "row slab: trainer is not row-slab sharded");
        HS_CUDA(cudaMemcpyAsync(error, t->s_flags.as<uint32_t>() + kMaxPeers, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                t->ctx->stream));
        HS_CUDA(cudaStreamSynchronize(t->ctx->stream));
    });
}

// holo::Rng(seed).uniform(lo, hi) x n (rng.hpp: std::mt19937_64, 53-bit
// mapping), on the host: the initial random-POH phase raster of the reference
// (convert.cpp:88) without a Python-speed generator.
extern "C" hs_status hs_random_uniform(uint64_t seed, int64_t n, double lo, double hi, double* h_out) {
    return guard([&] {
        require(n >= 0 && h_out != nullptr, "random_uniform: bad arguments");
        std::mt19937_64 eng(seed);
        for (int64_t i = 0; i < n; ++i)
            h_out[i] = lo + (hi - lo) * (static_cast<double>(eng() >> 11) * 0x1.0p-53);
    });
}

extern "C" hs_status hs_ipc_get_handle(const void* d_ptr, void* handle64) {
    return guard([&] {
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        cudaIpcMemHandle_t h;
        HS_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
        std::memcpy(handle64, &h, sizeof(h));
    });
}

extern "C" hs_status hs_ipc_open_handle(const void* handle64, void** d_ptr) {
    return guard([&] {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, sizeof(h));
        HS_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

extern "C" hs_status hs_ipc_close(void* d_ptr) {
    return guard([&] { HS_CUDA(cudaIpcCloseMemHandle(d_ptr)); });
}

// Stage k (0..4) of a row-slab step; between stage k and k+1 the caller runs
// all-to-all exchange k (send buffer -> peers' receive buffers, counts from
// hs_trainer_slab_counts).  After stage 4 the gradient buffer holds this
// rank's partial gradient (sum over its rows): all-reduce it, then
// hs_trainer_apply_update.  Loss partial sums: hs_trainer_loss_partials.
void hs::slab_enqueue(hs_trainer* t, int stage, cudaStream_t st) {
    AsmWork& aw = t->aw;
    const int C = t->c, LC = t->L * t->c;
    float2* send = t->s_send.as<float2>();
    // exchange k = stage - 1 arrives in the receive buffer of its parity (put
    // mode; the NCCL path always receives into the first buffer)
    const float2* recv = (t->s_put && ((stage - 1) & 1)) ? t->s_recv2.as<float2>() : t->s_recv.as<float2>();
    uint32_t* epoch = t->s_flags.as<uint32_t>() + kMaxPeers + 1;
    if (t->s_put && stage >= 1 && stage <= 4)
        slab_wait(t->s_flags.as<uint32_t>(), t->R, epoch, t->s_flags.as<uint32_t>() + kMaxPeers, st);
    // pack of exchange k: into the send buffer (NCCL), or straight into the
    // peers' receive buffers at this rank's slot followed by the flag signal
    auto pack = [&](int k, const float2* src) {
        if (!t->s_put) {
            chunk_copy(src, send, t->m_pack[k], st);
            return;
        }
        ChunkMap m = t->m_pack[k];
        for (int a = 0; a < t->R; ++a) {
            m.dptr[a] = t->s_peer_recv[k & 1][a];
            m.dA[a] = static_cast<int64_t>(t->rank) * (t->s_counts[k][a] / 2);
        }
        chunk_copy(src, nullptr, m, st);
        slab_signal(t->s_peer_flags, t->R, t->rank, epoch, st);
    };
    // row FFTs whose last stage stores straight into the peers (put mode,
    // planned grids): the compute kernel IS the exchange; else rows + pack
    auto rows_put = [&](int k, const float2* in, int planes, int h, int row0) {
        if (!t->s_put) return false;
        SlabPut sp{};
        for (int a = 0; a < t->R; ++a) {
            sp.peer[a] = t->s_peer_recv[k & 1][a];
            sp.slot[a] = static_cast<int64_t>(t->rank) * (t->s_counts[k][a] / 2);
        }
        sp.ts = t->ts;
        sp.row0 = row0;
        sp.hout = t->hr;
        sp.ts_magic = static_cast<unsigned>((0x100000000ull + t->ts - 1) / t->ts);
        if (!asm_rows_fwd_put(aw, in, planes, h, sp, st)) return false;
        slab_signal(t->s_peer_flags, t->R, t->rank, epoch, st);
        return true;
    };
    // inverse row FFTs gathering straight from the peer-major receive
    // buffer (the unpack fused into the loads; planned grids)
    auto rows_get = [&](int k, float2* out, int planes, int h) {
        SlabGet sg{};
        sg.ts = t->ts;
        sg.ts_magic = static_cast<unsigned>((0x100000000ull + t->ts - 1) / t->ts);
        sg.per_src = t->s_counts[k][t->R] / 2;  // receive count from source 0 (all sources equal)
        return asm_rows_inv_get(aw, recv, out, planes, h, sg, st);
    };
    // column pass gathering its tiles from the receive buffer of exchange
    // ki (R bulk copies) and putting its rows into the peers for exchange
    // ko (put mode) or into the local T layout (then packed)
    auto cols_slab = [&](bool backward, int ki, int ko, float2* local_out) {
        SlabCol sc{};
        sc.in = recv;
        sc.per_src = t->s_counts[ki][t->R] / 2;
        sc.R = t->R;
        sc.hr = t->hr;
        sc.inv_hr = 1.f / static_cast<float>(t->hr);
        sc.put = t->s_put ? 1 : 0;
        for (int a = 0; a < t->R; ++a) {
            sc.peer[a] = t->s_peer_recv[ko & 1][a];
            sc.slot[a] = static_cast<int64_t>(t->rank) * (t->s_counts[ko][a] / 2);
            sc.g0[a] = ko == 1 ? t->g0_of[a] : a * t->hr;
            sc.he[a] = ko == 1 ? t->He_of[a] : t->hr;
        }
        if (!asm_cols_slab(aw, backward, sc, local_out, t->rank * t->ts, t->ts, st)) return false;
        if (t->s_put) {
            slab_signal(t->s_peer_flags, t->R, t->rank, epoch, st);
        } else {
            chunk_copy(local_out, send, t->m_pack[ko], st);
        }
        return true;
    };
    switch (stage) {
        case 0:  // binning (replicated), raster forward of the own rows, row FFTs, pack
            HS_CUDA(cudaMemsetAsync(t->flags.p, 0, sizeof(uint32_t), st));
            t->rw.project_and_bin(t->params.as<float>(), st);
            raster_forward(t->rw, t->field.as<float2>(), st, t->h0, t->hr);
            if (!rows_put(0, t->field.as<float2>(), C, t->hr, 0)) {
                asm_rows_pass(aw, false, t->field.as<float2>(), aw.T1.as<float2>(), C, t->hr, st);
                pack(0, aw.T1.as<float2>());
            }
            break;
        case 1:  // column FFT x H_l + column IFFT on the own tiles, pack loss bands
            if (!cols_slab(false, 0, 1, aw.T2.as<float2>())) {
                chunk_copy(recv, aw.T1.as<float2>(), t->m_unpack[0], st);
                asm_cols_pass(aw, false, aw.T1.as<float2>(), aw.T2.as<float2>(), t->rank * t->ts, t->ts, st);
                pack(1, aw.T2.as<float2>());
            }
            break;
        case 2: {  // row IFFTs of the loss band, loss + dU, backward row FFTs, pack own rows
            if (!rows_get(1, t->s_planes.as<float2>(), LC, t->He)) {
                chunk_copy(recv, t->s_T.as<float2>(), t->m_unpack[1], st);
                asm_rows_pass(aw, true, t->s_T.as<float2>(), t->s_planes.as<float2>(), LC, t->He, st);
            }
            LossArgs a{kLossTraining, t->L, t->L_total, 0, C, t->He, t->w, nullptr, t->s_planes.as<float2>(),
                       t->s_target.as<float>(), t->s_tstats.as<float2>(), t->s_masks.as<uint8_t>(), nullptr,
                       t->s_dplanes.as<float2>(), t->partials.as<double>(), t->C_total};
            a.H_norm = t->h;
            a.own0 = t->top;
            a.own1 = t->top + t->hr;
            const int used = loss_launch(a, st);
            loss_finalize(a, used, t->out3.as<double>(), st);
            if (!rows_put(2, t->s_dplanes.as<float2>(), LC, t->He, t->top)) {
                asm_rows_pass(aw, false, t->s_dplanes.as<float2>(), t->s_T.as<float2>(), LC, t->He, st);
                pack(2, t->s_T.as<float2>());
            }
            break;
        }
        case 3:  // adjoint column pass on the own tiles, pack
            if (!cols_slab(true, 2, 3, aw.T1.as<float2>())) {
                chunk_copy(recv, aw.T2.as<float2>(), t->m_unpack[2], st);
                asm_cols_pass(aw, true, aw.T2.as<float2>(), aw.T1.as<float2>(), t->rank * t->ts, t->ts, st);
                pack(3, aw.T1.as<float2>());
            }
            break;
        case 4:  // row IFFTs of the own rows, raster backward over the own rows
            if (!rows_get(3, t->back.as<float2>(), C, t->hr)) {
                chunk_copy(recv, aw.T2.as<float2>(), t->m_unpack[3], st);
                asm_rows_pass(aw, true, aw.T2.as<float2>(), t->back.as<float2>(), C, t->hr, st);
            }
            raster_backward(t->rw, t->params.as<float>(), t->back.as<float2>(), t->grads.as<float>(),
                            t->flags.as<uint32_t>(), st, t->h0, t->hr);
            break;
        default: throw Error(HS_EINVAL, "row slab: stage outside 0..4");
    }
}

extern "C" hs_status hs_trainer_slab_stage(hs_trainer* t, int stage) {
    return guard([&] {
        require(t->R >= 1, "row slab: trainer is not row-slab sharded");
        require(t->host_step <= t->total_steps, "cosine_lr: step outside [0, total_steps]");
        slab_enqueue(t, stage, t->ctx->stream);
    });
}

// All five stages of a peer-put rank (no host step between them), captured
// into one CUDA graph on the first call when graphs are on.
extern "C" hs_status hs_trainer_slab_forward_backward(hs_trainer* t) {
    return guard([&] {
        require(t->R >= 1, "row slab: trainer is not row-slab sharded");
        require(t->s_put, "row slab: the one-call step needs the peer-put exchange (hs_trainer_slab_set_peers)");
        require(t->host_step <= t->total_steps, "cosine_lr: step outside [0, total_steps]");
        cudaStream_t st = t->ctx->stream;
        if (!t->use_graph || st == nullptr) {
            for (int k = 0; k < 5; ++k) slab_enqueue(t, k, st);
            return;
        }
        if (!t->slab_graph) {
            cudaGraph_t g = nullptr;
            HS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            try {
                for (int k = 0; k < 5; ++k) slab_enqueue(t, k, st);
            } catch (...) {
                cudaStreamEndCapture(st, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            HS_CUDA(cudaStreamEndCapture(st, &g));
            HS_CUDA(cudaGraphInstantiate(&t->slab_graph, g, 0));
            HS_CUDA(cudaGraphDestroy(g));
        }
        HS_CUDA(cudaGraphLaunch(t->slab_graph, st));
        note_launch(0);
    });
}
