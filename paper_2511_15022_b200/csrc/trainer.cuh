// The device-resident trainer (hs_trainer of include/holosplat.h) shared by
// capi.cu (step loop, row slabs) and comm.cu (NCCL-sharded steps), and the
// C-ABI error guard.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "asm.cuh"
#include "loss.cuh"
#include "raster.cuh"

namespace hs {

hs_status fail(hs_status s, const std::string& m);  // sets hs_last_error()

// Runs f, mapping exceptions to hs_status + hs_last_error().
template <class F>
hs_status guard(F&& f) {
    try {
        f();
        return HS_OK;
    } catch (const Error& e) {
        return fail(e.status, e.what());
    } catch (const std::bad_alloc&) {
        return fail(HS_ENOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(HS_ECUDA, e.what());
    }
}

}  // namespace hs

struct hs_trainer {
    using DevBuf = hs::DevBuf;
    using RasterWork = hs::RasterWork;
    using AsmWork = hs::AsmWork;
    using AdanGroups = hs::AdanGroups;
    using ChunkMap = hs::ChunkMap;
    static constexpr int kMaxPeers = hs::kMaxPeers;
    hs_ctx* ctx = nullptr;
    int n = 0, c = 0, w = 0, h = 0, L = 0, L_total = 0, plane0 = 0, total_steps = 0, C_total = 0;
    std::vector<double> distances;
    std::vector<double> wavelengths;
    hs_prop_spec spec{};
    int64_t P = 0;
    DevBuf params, grads, state, field, planes, dplanes, back, target, tstats, masks, partials, out3,
        flags, step;
    RasterWork rw;
    AsmWork aw;
    AdanGroups groups{};
    int host_step = 0;
    int loss_slots = 0;
    bool use_graph = false;
    cudaGraphExec_t graph = nullptr;
    cudaGraphExec_t prof_graph = nullptr;  // the step graph with the stage-timing event records
    bool mark_events = false;              // record the stage events while enqueuing (profiled step)
    bool profiling = false;
    cudaEvent_t ev[12] = {};  // profiling: start + after each of the 11 kernel slots
    // host-resident step (hs_trainer_step_host): copy stream, fork/join events,
    // pinned result words, and its own graph keyed by the host buffers
    cudaStream_t copy_st = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_ap = nullptr;
    uint32_t* h_words = nullptr;  // pinned: flags, status[4]
    double* h_o3 = nullptr;       // pinned: loss, recon sum, ssim sum
    cudaGraphExec_t host_graph = nullptr;
    const float* host_in = nullptr;
    float* host_out = nullptr;
    // pipelined multi-step host run (hs_trainer_run_host): a second copy
    // stream for the deferred amplitude/phase download, the first-step and
    // steady-state graphs keyed by the host buffer, and the per-run device
    // words {halt, step index} + per-step flag / loss logs
    cudaStream_t copy_st2 = nullptr;
    cudaEvent_t ev_apdown = nullptr;
    cudaGraphExec_t run_graph0 = nullptr, run_graph = nullptr;
    float* run_host = nullptr;
    DevBuf run_words, run_flog, run_llog;
    // row-slab sharding (hs_trainer_set_row_slab): rank `rank` of R owns canvas
    // rows [h0, h0 + hr) and column tiles [rank ts, rank ts + ts); its loss band
    // is rows [g0, g0 + He) (own rows + up to 10 halo rows each side)
    int R = 0, rank = 0, hr = 0, ts = 0, h0 = 0, g0 = 0, He = 0, top = 0;
    std::vector<int> He_of, g0_of;
    DevBuf s_planes, s_dplanes, s_target, s_tstats, s_masks, s_T, s_send, s_recv;
    ChunkMap m_pack[4], m_unpack[4];
    int64_t s_counts[4][2 * kMaxPeers] = {};
    // peer-put exchange (hs_trainer_slab_set_peers): the pack kernels store
    // straight into the peers' receive buffers (double-buffered by exchange
    // parity), then signal the peers' flag arrays; the next stage waits on
    // this rank's flags.  No NCCL call on the data path.
    bool s_put = false;
    float2* s_peer_recv[2][kMaxPeers] = {};
    uint32_t* s_peer_flags[kMaxPeers] = {};
    DevBuf s_recv2, s_flags;  // flags: [0, R) per-source epochs, [kMaxPeers] error word, [kMaxPeers + 1] own epoch
    cudaGraphExec_t slab_graph = nullptr;  // stages 0..4 of the put exchange, captured
    int s_loss_slots = 0;
    ~hs_trainer() {
        if (graph) cudaGraphExecDestroy(graph);
        if (prof_graph) cudaGraphExecDestroy(prof_graph);
        if (host_graph) cudaGraphExecDestroy(host_graph);
        if (run_graph0) cudaGraphExecDestroy(run_graph0);
        if (run_graph) cudaGraphExecDestroy(run_graph);
        if (ev_apdown) cudaEventDestroy(ev_apdown);
        if (copy_st2) cudaStreamDestroy(copy_st2);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_ap) cudaEventDestroy(ev_ap);
        if (copy_st) cudaStreamDestroy(copy_st);
        if (slab_graph) cudaGraphExecDestroy(slab_graph);
        if (h_words) cudaFreeHost(h_words);
        if (h_o3) cudaFreeHost(h_o3);
    }
};

namespace hs {

// capi.cu: the step's halves and the row-slab stages (enqueued on st)
void trainer_enqueue_fwd_bwd(hs_trainer* t, cudaStream_t st, cudaEvent_t shading_ready = nullptr);
void trainer_enqueue_update(hs_trainer* t, cudaStream_t st);
void trainer_check_after(hs_trainer* t);  // syncs; throws HS_ENONFINITE / HS_EOVERFLOW / HS_EINVAL
void slab_enqueue(hs_trainer* t, int stage, cudaStream_t st);

}  // namespace hs
