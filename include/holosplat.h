/* holosplat-b200 C ABI -- the drop-in boundary for the reference's optimisation
 * hot path (arxiv 2511.15022 "holosplat", /root/reference/proj).
 *
 * The reference exposes its hot path as the C++ API in namespace holo
 * (proj/core/include/holo/{rasterizer,propagation,loss,optimizer}.hpp) and its
 * only product caller is the step loop proj/core/src/pipeline.cpp:253-297.
 * This header is the thin extern "C" layer underneath the C++ drop-in
 * (include/holo/ headers, libholo_b200.so) and the Python host mirror
 * (paper_2511_15022_b200.holo).  Plain pointers and sizes only.
 *
 * Conventions
 *  - Every function returns hs_status; HS_OK == 0.  On failure the message is
 *    available from hs_last_error() (thread-local), in the reference's words
 *    where the reference raises the same condition.
 *  - "d_" pointers are device pointers on the context's device, "h_" host.
 *  - Gaussian parameters are ONE fp32 buffer of (6 + 2C) * N floats holding
 *    the reference's six groups back to back, in declaration order
 *    (gaussian_set.hpp:14-19):
 *        [pre_position 2N | pre_scale 2N | rotation N | amplitude N*C |
 *         phase N*C | pre_opacity N]
 *    Gradients use the same layout (GaussianSetGrads = GaussianSet).
 *  - Complex fields are interleaved complex64 (float2 re,im), C x H x W
 *    row-major (same element order as holo::ComplexField's planar arrays,
 *    complex_field.hpp:11-35); multi-plane stacks are L x C x H x W.
 *  - Work is issued on the context's stream (hs_ctx_set_stream); functions
 *    that return host scalars synchronise that stream.
 */
#ifndef HOLOSPLAT_H
#define HOLOSPLAT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HS_OK = 0,
    HS_EINVAL = 1,      /* std::invalid_argument in the reference */
    HS_ENONFINITE = 2,  /* std::runtime_error "Adan: non-finite gradient in group <g>" */
    HS_ECUDA = 3,
    HS_ENOMEM = 4,
    HS_EOVERFLOW = 5    /* tile-pair capacity exceeded (grow with hs_trainer_reserve_pairs) */
} hs_status;

typedef struct hs_ctx hs_ctx;
typedef struct hs_trainer hs_trainer;

/* ---- context ---------------------------------------------------------------- */
hs_status hs_ctx_create(int device, hs_ctx** out);
void hs_ctx_destroy(hs_ctx* ctx);
/* cudaStream_t passed as void*; NULL = legacy default stream. */
hs_status hs_ctx_set_stream(hs_ctx* ctx, void* stream);
/* Backward form of the stand-alone hs_rasterize_backward: 1 (default)
 * deterministic per-Gaussian gather, 0 the per-tile backward with atomics. */
hs_status hs_ctx_set_deterministic(hs_ctx* ctx, int enable);
hs_status hs_ctx_synchronize(hs_ctx* ctx);
const char* hs_last_error(void);
/* Number of kernels this library has launched in this process (for the bench's
 * gpu_launches claim). */
uint64_t hs_kernel_launch_count(void);
/* Device-memory helpers so hosts without a CUDA toolchain (the C++ drop-in,
 * ctypes) can stage buffers. */
hs_status hs_device_alloc(hs_ctx* ctx, size_t bytes, void** d_out);
hs_status hs_device_free(hs_ctx* ctx, void* d_ptr);
hs_status hs_copy_h2d(hs_ctx* ctx, void* d_dst, const void* h_src, size_t bytes);
hs_status hs_copy_d2h(hs_ctx* ctx, void* h_dst, const void* d_src, size_t bytes);

/* ---- rasterizer (rasterizer.hpp:12-36, rasterizer.cpp:33-286) --------------- */
/* build_tile_index: pairs sorted by (tile, id); ranges[2t], ranges[2t+1] =
 * [begin,end) of tile t, {0,0} when empty.  Two-call protocol: with cap <
 * needed nothing but *npairs and tiles_xy is written.  Bit-exact with
 * holo::build_tile_index on the same (fp32-valued) parameters. */
/* Binning of the standalone raster entry points (default 1 = tight): keep only
 * the (tile, Gaussian) pairs whose tile the Gaussian's ellipse can reach; the
 * rasterized field is bit-identical to binning with the reference's box lists
 * (0).  hs_build_tile_index always exports the reference's exact lists. */
hs_status hs_ctx_set_tight_binning(hs_ctx* ctx, int tight);
hs_status hs_build_tile_index(hs_ctx* ctx, const float* d_params, int n, int c, int width,
                              int height, uint32_t* d_tiles, uint32_t* d_ids,
                              uint64_t* d_ranges, int64_t cap, int64_t* npairs, int* tiles_xy);
/* rasterize_forward: d_field receives C x H x W complex64. */
hs_status hs_rasterize_forward(hs_ctx* ctx, const float* d_params, int n, int c, int width,
                               int height, float* d_field);
/* rasterize_backward: d_grad_field = dL/d(re,im) interleaved C x H x W; d_grads
 * receives dL/d(params) in the parameter layout. */
hs_status hs_rasterize_backward(hs_ctx* ctx, const float* d_params, int n, int c, int width,
                                int height, const float* d_grad_field, float* d_grads);

/* ---- propagation (propagation.hpp:9-49, propagation.cpp:54-243) -------------- */
typedef struct {
    const double* wavelengths; /* one per channel, metres */
    int n_wavelengths;
    double pixel_pitch;        /* metres */
    int pad_factor;
    double aperture_radius;    /* padded-frequency-grid pixels; 0 disables */
} hs_prop_spec;

/* mode 0: propagate(distance)            (propagation.cpp:174-177)
 * mode 1: propagate_with_mask_distance    (:179-182)
 * mode 2: propagate_backward(distance)    (:184-187) */
hs_status hs_propagate(hs_ctx* ctx, const hs_prop_spec* spec, int mode, double distance,
                       double mask_distance, const float* d_in, int c, int h, int w,
                       float* d_out);
/* propagate_multi: d_out is L x C x H x W. */
hs_status hs_propagate_multi(hs_ctx* ctx, const hs_prop_spec* spec, const double* h_distances,
                             int L, const float* d_in, int c, int h, int w, float* d_out);
/* propagate_multi_backward: d_grads is L x C x H x W, d_out C x H x W. */
hs_status hs_propagate_multi_backward(hs_ctx* ctx, const hs_prop_spec* spec,
                                      const double* h_distances, int L, const float* d_grads,
                                      int c, int h, int w, float* d_out);

/* ---- loss (loss.hpp:10-67, loss.cpp:154-369) ----------------------------------- */
/* intensity_of: |u|^2 (field_core.cpp:88-93); count complex elements. */
hs_status hs_intensity(hs_ctx* ctx, const float* d_field, int64_t count, float* d_out);
/* kind 0 training_loss_grad, 1 loss_recon_grad, 2 loss_ssim_grad, 3 loss_mse_grad.
 * d_recon: L x C x H x W intensities, d_target C x H x W, d_masks L x H x W
 * bytes (build_masks).  d_grads (nullable) receives dL/dI; *loss the value. */
hs_status hs_loss(hs_ctx* ctx, int kind, int L, int c, int h, int w, const float* d_recon,
                  const float* d_target, const uint8_t* d_masks, float* d_grads, double* loss);
/* compute_metrics (pipeline.cpp:135-163): recon and target clipped to [0, 1],
 * per plane PSNR (dB, +inf when identical) and ssim_value (loss.cpp:356-369).
 * d_recon L x C x H x W intensities, d_target C x H x W; h_psnr, h_ssim L doubles. */
hs_status hs_compute_metrics(hs_ctx* ctx, int L, int c, int h, int w, const float* d_recon,
                             const float* d_target, double* h_psnr, double* h_ssim);
/* build_masks (loss.cpp:166-180) on the host, bit-exact. */
hs_status hs_build_masks(const double* h_depth, int h, int w, int L, int near_is_high,
                         uint8_t* h_masks);

/* ---- optimizer (optimizer.hpp:10-49, optimizer.cpp:8-72) --------------------- */
typedef struct {
    double beta1, beta2, beta3, eps;
} hs_adan_config;

/* One Adan step for one group: d_state holds 4*size floats [m | v | n | g_prev].
 * step_t is the group's 1-based step after increment.  The non-finite check
 * happens before any update (optimizer.cpp:52-54): on a non-finite gradient
 * nothing is modified and HS_ENONFINITE is returned with group_name in the
 * message. */
hs_status hs_adan_step(hs_ctx* ctx, const hs_adan_config* cfg, const char* group_name,
                       float* d_params, const float* d_grads, float* d_state, int64_t size,
                       int step_t, double lr);
/* cosine_lr (optimizer.cpp:8-13). */
hs_status hs_cosine_lr(int step, int total_steps, double lr_max, double lr_min, double* out);

/* ---- phase-only hologram conversion (convert.hpp, convert.cpp:20-184) ------------ */
/* dpac_encode (convert.cpp:31-60) BEFORE canonicalize_phase -- the hosts
 * canonicalise in fp64 like the reference: mode 0 DpacMode::direct,
 * 1 DpacMode::classical.  d_field C x H x W complex64 -> d_phase C x H x W. */
hs_status hs_dpac_encode(hs_ctx* ctx, const float* d_field, int c, int h, int w, int mode, float* d_phase);
/* poh_field (convert.cpp:62-69): d_field = e^{i d_phase}, count elements. */
hs_status hs_poh_field(hs_ctx* ctx, const float* d_phase, int64_t count, float* d_field);
typedef struct {
    int c, height, width, planes;  /* guide / target shape, L */
    const double* distances;       /* L plane distances */
    hs_prop_spec spec;
    const float* h_target;         /* C x H x W target intensity */
    const uint8_t* h_masks;        /* L x H x W (TargetStack::masks) */
    int steps;
    double lambda_comp, lambda_field, lr;  /* RandomPohOptions (convert.hpp) */
} hs_poh_config;
/* convert_random_poh_field (convert.cpp:71-174), device resident.  d_phase
 * holds the initial raster (Rng(seed).uniform(-pi, pi) in element order) and
 * receives the optimised phase, not yet canonicalised; h_loss (steps doubles,
 * nullable) receives every step's loss.  Errors: HS_EINVAL for no planes or
 * steps < 1 (the reference's messages), HS_ENONFINITE "Adan: non-finite
 * gradient in group phase". */
hs_status hs_convert_random_poh_field(hs_ctx* ctx, const hs_poh_config* cfg, const float* d_guide_field,
                                      float* d_phase, double* h_loss);

/* ---- trainer: the fused step loop body (pipeline.cpp:253-297) ------------------ */
typedef struct {
    int n, c, width, height;
    int planes;                 /* L */
    const double* distances;    /* L plane distances (make_depth_planes) */
    hs_prop_spec spec;
    int total_steps;            /* cosine schedule horizon (config.steps) */
    const float* h_target;      /* C x H x W linear intensity in [0,1] */
    const uint8_t* h_masks;     /* L x H x W (build_masks) */
    /* Optional plane shard for multi-GPU (owned planes [plane_begin,
     * plane_end)); loss normalisers always use the global L.  0,0 = all. */
    int plane_begin, plane_end;
    /* Optional wavelength (channel) shard: this trainer holds c of the
     * channels_total channels of the scene (its spec, target and amplitude /
     * phase columns are that slice); the loss normalisers use channels_total.
     * 0 = c (no channel sharding). */
    int channels_total;
} hs_trainer_config;

hs_status hs_trainer_create(hs_ctx* ctx, const hs_trainer_config* cfg, hs_trainer** out);
void hs_trainer_destroy(hs_trainer* tr);
/* Parameters in the layout above; from host (fp32) or device. */
hs_status hs_trainer_set_params(hs_trainer* tr, const float* params, int from_device);
hs_status hs_trainer_get_params(hs_trainer* tr, float* params, int to_device);
/* Device pointers owned by the trainer (params, grads), for zero-copy use
 * (e.g. a torch.distributed all_reduce of the gradient buffer). */
float* hs_trainer_params_ptr(hs_trainer* tr);
float* hs_trainer_grads_ptr(hs_trainer* tr);
int64_t hs_trainer_param_count(hs_trainer* tr);
/* One full iteration: raster fwd -> ASM fwd -> loss -> ASM bwd -> raster bwd
 * -> Adan x6.  *loss_out (nullable) receives the loss of this iteration (that
 * synchronises); pass NULL to stay asynchronous and fetch it later with
 * hs_trainer_last_loss. */
hs_status hs_trainer_step(hs_trainer* tr, double* loss_out);
/* One iteration with HOST-resident parameters, like the reference loop where the
 * GaussianSet lives on the host: H2D of h_params_in (nullable), the step, D2H
 * of the updated parameters into h_params_out (nullable) and of the loss --
 * queued on the trainer stream with a single synchronisation.  Use pinned host
 * memory for full copy bandwidth. */
hs_status hs_trainer_step_host(hs_trainer* tr, const float* h_params_in, float* h_params_out, double* loss_out);
/* `steps` steps with host-resident parameters: h_params (pinned, the flat
 * [pos | scale | rot | amp | phase | opa] fp32 layout) is uploaded before and
 * overwritten with the updated parameters after EVERY step, as `steps` calls
 * of hs_trainer_step_host(tr, h, h, ...) would do; the copies are pipelined
 * across steps (step k's amplitude/phase download overlaps step k+1's geometry
 * upload and projection).  losses_out (nullable) receives each step's loss.
 * A non-finite gradient / rasterizer error at step j raises as
 * hs_trainer_step_host would at step j; later steps of the call leave the
 * parameters untouched (the reference's loop stops at the throw). */
hs_status hs_trainer_run_host(hs_trainer* tr, float* h_params, int steps, double* losses_out);
/* Split form for multi-GPU: forward+backward into the gradient buffer, then
 * (after the caller all-reduced hs_trainer_grads_ptr) the optimizer update. */
hs_status hs_trainer_forward_backward(hs_trainer* tr);
hs_status hs_trainer_apply_update(hs_trainer* tr);
/* After the caller summed the gradient buffer over ranks: re-derive the
 * per-group non-finite bits from the sum, so every rank skips the same groups
 * (Adan::step throws on the first non-finite group, optimizer.cpp:52-54). */
hs_status hs_trainer_check_grads(hs_trainer* tr);
/* Device word of the step's non-finite gradient groups (bit g = group g, in
 * the order of pipeline.cpp:244-249).  hs_trainer_apply_update skips every
 * group from the lowest set bit on, as the reference's Adan::step throw does
 * (optimizer.cpp:52-54).  Sharded callers make the ranks agree on it (keep
 * only the lowest bit, min-reduce across ranks) before the update. */
uint32_t* hs_trainer_flags_ptr(hs_trainer* tr);
hs_status hs_trainer_last_loss(hs_trainer* tr, double* loss_out, int64_t* npairs_out);
/* Loss partial sums of this rank (recon sum, ssim sum) for cross-rank loss. */
hs_status hs_trainer_loss_partials(hs_trainer* tr, double* out2);
hs_status hs_trainer_reserve_pairs(hs_trainer* tr, int64_t cap);
/* Capture one step into a CUDA graph and replay it (0/1). */
hs_status hs_trainer_use_graph(hs_trainer* tr, int enable);
/* Raster backward form.  Default (0): the per-tile backward with vector
 * atomics into per-Gaussian rows (fastest; the last bits of the gradients
 * depend on the atomic order).  1: the per-Gaussian gather, bit-reproducible
 * run to run (row-slab shards: over their band list). */
hs_status hs_trainer_set_deterministic(hs_trainer* tr, int enable);
/* Device event timing of the last step, ms per kernel slot:
 * [binning, raster_fwd, rows_fwd, cols_fwd, rows_inv, loss, rows_fwd(bwd),
 *  cols_bwd, rows_inv(bwd), raster_bwd, adan, total].  Needs profiling on.
 * With graphs on, profiled steps replay a separate step graph that holds the
 * stage event records (no host enqueue gaps in the stage times); with graphs
 * off the events are recorded eagerly (also by forward_backward +
 * apply_update). */
hs_status hs_trainer_set_profiling(hs_trainer* tr, int enable);
hs_status hs_trainer_stage_ms(hs_trainer* tr, double* out12);
int hs_trainer_step_count(hs_trainer* tr);

/* ---- row-slab sharding: the 4K step over R GPUs -------------
 * No reference interface: the reference is single-process (propagation.cpp:
 * 186-294 runs one 2D FFT per channel on the host).  Rank `rank` of `ranks`
 * owns canvas rows [rank H/R, (rank+1) H/R) and padded-spectrum column tiles
 * [rank nt/R, (rank+1) nt/R).  A step is five stages with an all-to-all between
 * consecutive stages (the 2D-FFT transposes):
 *   stage 0  binning, raster forward of the own rows, row FFTs        -> exchange 0
 *   stage 1  column FFT x H_l, column IFFT of the own tiles            -> exchange 1
 *   stage 2  row IFFTs of the loss band (own rows + 10-row halos),
 *            loss + dL/dU, backward row FFTs                           -> exchange 2
 *   stage 3  adjoint column pass of the own tiles                      -> exchange 3
 *   stage 4  row IFFTs of the own rows, raster backward over them
 * then an all-reduce (sum) of hs_trainer_grads_ptr, hs_trainer_apply_update,
 * and an all-reduce of hs_trainer_loss_partials.  Exchange e sends
 * counts[p] floats from the send buffer (peer-major, in peer order) to peer p
 * and receives recv[p] floats from peer p into the receive buffer (peer-major):
 * all_to_all_single(recv, send, recv_counts, send_counts).
 * Requires H % ranks == 0, (padded width / tile width) % ranks == 0, ranks <= 16,
 * no plane or channel sharding. */
hs_status hs_trainer_set_row_slab(hs_trainer* tr, int rank, int ranks);
/* out[2*ranks]: send counts per peer, then receive counts per peer (floats). */
hs_status hs_trainer_slab_counts(hs_trainer* tr, int exchange, int64_t* out);
float* hs_trainer_slab_send_ptr(hs_trainer* tr);
float* hs_trainer_slab_recv_ptr(hs_trainer* tr);
hs_status hs_trainer_slab_stage(hs_trainer* tr, int stage);
/* Peer-put exchange (instead of an all-to-all between the stages): the pack
 * at the end of stage k stores straight into every peer's receive buffer of
 * parity k & 1 (at this rank's slot) and signals the peers' flag arrays; stage
 * k + 1 begins by waiting on this rank's flags (bounded: ~2 s, then
 * hs_trainer_slab_status reports 1).  recv0 / recv1 / flags hold, per rank,
 * device addresses valid in this context -- the peers' hs_trainer_slab_recv_ptr,
 * hs_trainer_slab_recv2_ptr and hs_trainer_slab_flags_ptr mapped with CUDA IPC
 * (hs_ipc_*) or P2P; the own entries are the own buffers. */
float* hs_trainer_slab_recv2_ptr(hs_trainer* tr);
uint32_t* hs_trainer_slab_flags_ptr(hs_trainer* tr);
hs_status hs_trainer_slab_set_peers(hs_trainer* tr, float* const* recv0, float* const* recv1,
                                    uint32_t* const* flags);
hs_status hs_trainer_slab_status(hs_trainer* tr, uint32_t* error);
/* Device address of the peer-put timeout word hs_trainer_slab_status reads
 * (sticky until hs_trainer_set_row_slab; NULL without row slabs). */
uint32_t* hs_trainer_slab_error_ptr(hs_trainer* tr);
/* Peer-put mode: stages 0..4 in one call (no host step between them; the
 * exchange epochs are device counters), replayed as one CUDA graph when
 * hs_trainer_use_graph is on.  Follow with the gradient all-reduce and
 * hs_trainer_apply_update. */
hs_status hs_trainer_slab_forward_backward(hs_trainer* tr);
/* ---- NCCL communicator in the context + one-call sharded step ----
 * No reference interface: the reference is single-process.  One rank per GPU.
 * hs_comm_unique_id (on one rank; ship the 128 bytes to the others out of band),
 * then hs_ctx_comm_init on every rank; or hs_ctx_comm_adopt a caller-owned
 * ncclComm_t.  hs_ctx_destroy releases an owned communicator. */
hs_status hs_comm_unique_id(void* id128);
hs_status hs_ctx_comm_init(hs_ctx* ctx, const void* id128, int nranks, int rank);
hs_status hs_ctx_comm_adopt(hs_ctx* ctx, void* nccl_comm);
hs_status hs_ctx_comm_info(hs_ctx* ctx, int* nranks, int* rank);
hs_status hs_ctx_comm_destroy(hs_ctx* ctx);
/* One sharded optimisation step of this rank over the ctx communicator, on the
 * ctx stream: plane shards (plane_begin/end) and row slabs all-reduce the
 * gradient buffer, wavelength shards (channels_total > c) its 6N geometry
 * groups; row slabs exchange by grouped ncclSend/ncclRecv between the stages
 * (or by the peer-put stores when hs_trainer_slab_set_peers was called).  The
 * ranks then agree on the first non-finite gradient group (min-reduce of the
 * lowest flag bit), apply Adan and all-reduce the loss sums.  loss_out
 * (nullable) syncs and receives the global loss; errors as hs_trainer_step. */
hs_status hs_trainer_sharded_step(hs_trainer* tr, double* loss_out);
/* Sharded optimizer update (ZeRO-1 style, after a reduce-scatter of the
 * gradient): the non-finite group bits of grads[begin, end) only (agree on
 * them across ranks, then), and Adan over params[begin, end) with the
 * matching moments -- then all-gather the parameters.  Both ranges must
 * start on a multiple of 4 floats for the vectorised update; the device
 * step counter and the cosine schedule advance as in hs_trainer_apply_update. */
hs_status hs_trainer_check_grads_range(hs_trainer* tr, int64_t begin, int64_t end);
hs_status hs_trainer_apply_update_range(hs_trainer* tr, int64_t begin, int64_t end);

/* holo::Rng(seed).uniform(lo, hi) drawn n times into h_out (rng.hpp; host). */
hs_status hs_random_uniform(uint64_t seed, int64_t n, double lo, double hi, double* h_out);
/* CUDA IPC of a device allocation: 64-byte handle out; open maps a peer
 * process's allocation into this context (lazy peer access); close unmaps. */
hs_status hs_ipc_get_handle(const void* d_ptr, void* handle64);
hs_status hs_ipc_open_handle(const void* handle64, void** d_ptr);
hs_status hs_ipc_close(void* d_ptr);

#ifdef __cplusplus
}
#endif

#endif /* HOLOSPLAT_H */
