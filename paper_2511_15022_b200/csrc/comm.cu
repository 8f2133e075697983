// NCCL inside the library: the communicator lives in the hs_ctx (SURVEY
// §8(b): "NCCL comm handles live in the ctx") and hs_trainer_sharded_step runs
// one sharded optimisation step end to end -- forward/backward of this rank's
// share, the exchanges, the gradient all-reduce, the cross-rank agreement on
// non-finite gradient groups, Adan and the loss sums -- on the ctx stream, so
// a C or C++ host (the reference's own callers) can shard without torch.
//
// The reference is single-process; the decompositions are the
// ones of SURVEY §8(e):
//   * planes   (hs_trainer_config.plane_begin/end): all-reduce of the whole
//              (6+2C)N gradient buffer (the adjoint is a sum over planes,
//              propagate_multi_backward propagation.cpp:229-240);
//   * channels (channels_total > c): all-reduce of the 6N geometry gradients,
//              amplitude/phase stay rank-local;
//   * row slabs (hs_trainer_set_row_slab): four transposes per step, as
//              grouped ncclSend/ncclRecv all-to-alls between the stages, or the
//              peer-put stores of hs_trainer_slab_set_peers; then the gradient
//              all-reduce.
//
// libnccl is opened lazily (dlopen on the first hs_comm_* / sharded call), not
// linked: loading libholosplat.so must not pull a libnccl.so.2 into a process
// before torch brings its own (same soname, newer symbols).  An already
// loaded libnccl.so.2 (torch's) is reused; else the system one is opened.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "trainer.cuh"

using namespace hs;

namespace {

constexpr uint32_t kNoGroup = 1u << 30;

struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*CommCount)(const ncclComm_t, int*);
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    const char* (*GetErrorString)(ncclResult_t);
};

const Nccl& nccl() {
    static Nccl api{};
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("NCCL unavailable: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) {
            void* f = dlsym(h, name);
            if (!f && err.empty()) err = std::string("NCCL symbol missing: ") + name;
            return f;
        };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.CommCount = reinterpret_cast<decltype(api.CommCount)>(sym("ncclCommCount"));
        api.CommUserRank = reinterpret_cast<decltype(api.CommUserRank)>(sym("ncclCommUserRank"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.ReduceScatter = reinterpret_cast<decltype(api.ReduceScatter)>(sym("ncclReduceScatter"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    });
    if (!err.empty()) throw Error(HS_ECUDA, err);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(HS_ECUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

ncclComm_t comm_of(hs_ctx* ctx) {
    require(ctx->comm != nullptr, "sharded step: no NCCL communicator in the context (hs_ctx_comm_init)");
    return static_cast<ncclComm_t>(ctx->comm);
}

// flags -> lowest set bit (the first non-finite group), kNoGroup when clean
__global__ void lowest_group_kernel(const uint32_t* __restrict__ flags, uint32_t* __restrict__ word) {
    const uint32_t f = *flags;
    *word = f ? (f & (~f + 1u)) : kNoGroup;
}

__global__ void apply_group_kernel(const uint32_t* __restrict__ word, uint32_t* __restrict__ flags) {
    const uint32_t w = *word;
    *flags = w == kNoGroup ? 0u : w;
}

// The training loss from the all-reduced (recon, ssim) sums, as loss_finalize.
__global__ void loss_combine_kernel(double* __restrict__ out3, double n_el, int L_norm, double count) {
    out3[0] = out3[1] / (n_el * L_norm) + 0.005 * (1.0 - out3[2] / count);  // kSsimWeight, loss.hpp:14
}

void all_to_all(hs_trainer* t, int e, ncclComm_t comm, cudaStream_t st) {
    const int R = t->R;
    const int64_t* sc = t->s_counts[e];
    const int64_t* rc = t->s_counts[e] + R;
    const float* send = t->s_send.as<float>();
    float* recv = t->s_recv.as<float>();
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    int64_t so = 0, ro = 0;
    for (int p = 0; p < R; ++p) {
        if (sc[p]) nccl_check(nccl().Send(send + so, static_cast<size_t>(sc[p]), ncclFloat, p, comm, st), "ncclSend");
        if (rc[p]) nccl_check(nccl().Recv(recv + ro, static_cast<size_t>(rc[p]), ncclFloat, p, comm, st), "ncclRecv");
        so += sc[p];
        ro += rc[p];
    }
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
}

}  // namespace

extern "C" {

hs_status hs_comm_unique_id(void* id128) {
    return guard([&] {
        require(id128 != nullptr, "hs_comm_unique_id: null output");
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
        ncclUniqueId id;
        nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id128, &id, sizeof(id));
    });
}

hs_status hs_ctx_comm_init(hs_ctx* ctx, const void* id128, int nranks, int rank) {
    return guard([&] {
        require(ctx && id128, "hs_ctx_comm_init: null argument");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "hs_ctx_comm_init: rank outside [0, nranks)");
        require(ctx->comm == nullptr, "hs_ctx_comm_init: the context already has a communicator");
        HS_CUDA(cudaSetDevice(ctx->device));
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        ncclComm_t c = nullptr;
        nccl_check(nccl().CommInitRank(&c, nranks, id, rank), "ncclCommInitRank");
        ctx->comm = c;
        ctx->comm_size = nranks;
        ctx->comm_rank = rank;
        ctx->comm_owned = true;
    });
}

hs_status hs_ctx_comm_adopt(hs_ctx* ctx, void* nccl_comm) {
    return guard([&] {
        require(ctx && nccl_comm, "hs_ctx_comm_adopt: null argument");
        require(ctx->comm == nullptr, "hs_ctx_comm_adopt: the context already has a communicator");
        ncclComm_t c = static_cast<ncclComm_t>(nccl_comm);
        int n = 0, r = 0;
        nccl_check(nccl().CommCount(c, &n), "ncclCommCount");
        nccl_check(nccl().CommUserRank(c, &r), "ncclCommUserRank");
        ctx->comm = c;
        ctx->comm_size = n;
        ctx->comm_rank = r;
        ctx->comm_owned = false;
    });
}

hs_status hs_ctx_comm_info(hs_ctx* ctx, int* nranks, int* rank) {
    return guard([&] {
        require(ctx->comm != nullptr, "hs_ctx_comm_info: no communicator");
        if (nranks) *nranks = ctx->comm_size;
        if (rank) *rank = ctx->comm_rank;
    });
}

hs_status hs_ctx_comm_destroy(hs_ctx* ctx) {
    return guard([&] {
        if (!ctx || !ctx->comm) return;
        if (ctx->comm_owned) nccl_check(nccl().CommDestroy(static_cast<ncclComm_t>(ctx->comm)), "ncclCommDestroy");
        if (ctx->comm_scratch) cudaFree(ctx->comm_scratch);
        ctx->comm = nullptr;
        ctx->comm_scratch = nullptr;
        ctx->comm_size = 1;
        ctx->comm_rank = 0;
    });
}

// One sharded step; see the file comment.  loss_out (nullable): the global
// training loss, read back with one synchronisation, which also raises the
// step's errors (HS_ENONFINITE naming the reference's first non-finite group,
// HS_ECUDA for a peer-put exchange timeout).
hs_status hs_trainer_sharded_step(hs_trainer* t, double* loss_out) {
    return guard([&] {
        hs_ctx* ctx = t->ctx;
        ncclComm_t comm = comm_of(ctx);
        const int world = ctx->comm_size;
        cudaStream_t st = ctx->stream;
        require(t->host_step <= t->total_steps, "cosine_lr: step outside [0, total_steps]");
        const bool slabs = t->R >= 1;
        const bool channels = t->C_total > t->c;
        const bool planes = t->L < t->L_total;
        require(!slabs || t->R == world, "sharded step: row slabs need ranks == communicator size");
        require(!slabs || t->rank == ctx->comm_rank, "sharded step: slab rank != communicator rank");
        if (!ctx->comm_scratch) HS_CUDA(cudaMalloc(&ctx->comm_scratch, 64));
        uint32_t* word = static_cast<uint32_t*>(ctx->comm_scratch);

        // forward + backward of this rank's share
        if (slabs && t->s_put) {
            for (int k = 0; k < 5; ++k) slab_enqueue(t, k, st);  // stores into the peers, device-flag sync
        } else if (slabs) {
            for (int k = 0; k < 4; ++k) {
                slab_enqueue(t, k, st);
                all_to_all(t, k, comm, st);
            }
            slab_enqueue(t, 4, st);
        } else {
            trainer_enqueue_fwd_bwd(t, st);
        }
        // gradient sum: everything (planes, slabs) or the geometry groups (channels)
        // (also at world 1, where the collectives are copies: one code path).
        // Planes and slabs shard the update ZeRO-1 style when the buffer splits
        // into equal multiples of 4 floats: reduce-scatter (in place), the
        // non-finite check and Adan on the own shard, all-gather (in place).
        float* g = t->grads.as<float>();
        const int64_t shard = t->P / world;
        const bool sharded = !(channels && !planes && !slabs) && world > 1 && t->P % world == 0 && shard % 4 == 0;
        const int64_t sb = sharded ? shard * ctx->comm_rank : 0, se = sharded ? sb + shard : t->P;
        {
            if (sharded) {
                nccl_check(nccl().ReduceScatter(g, g + sb, static_cast<size_t>(shard), ncclFloat, ncclSum, comm, st),
                           "ncclReduceScatter");
            } else if (channels && !planes && !slabs) {
                const size_t N = t->n;
                nccl_check(nccl().AllReduce(g, g, 5 * N, ncclFloat, ncclSum, comm, st), "ncclAllReduce");
                float* opa = g + 5 * N + 2 * N * t->c;
                nccl_check(nccl().AllReduce(opa, opa, N, ncclFloat, ncclSum, comm, st), "ncclAllReduce");
            } else {
                nccl_check(nccl().AllReduce(g, g, static_cast<size_t>(t->P), ncclFloat, ncclSum, comm, st),
                           "ncclAllReduce");
            }
            // the non-finite groups of the SUMMED gradient, then every rank keeps
            // the lowest group any rank saw (channel shards hold rank-local groups)
            group_nonfinite_launch(g, t->P, t->groups, t->flags.as<uint32_t>(), st, sb, se);
            lowest_group_kernel<<<1, 1, 0, st>>>(t->flags.as<uint32_t>(), word);
            nccl_check(nccl().AllReduce(word, word, 1, ncclUint32, ncclMin, comm, st), "ncclAllReduce");
            apply_group_kernel<<<1, 1, 0, st>>>(word, t->flags.as<uint32_t>());
            launch_check("sharded_step agreement");
            // loss sums (recon, ssim) -> the global loss
            double* o3 = t->out3.as<double>();
            nccl_check(nccl().AllReduce(o3 + 1, o3 + 1, 2, ncclDouble, ncclSum, comm, st), "ncclAllReduce");
            const int Cn = t->C_total > 0 ? t->C_total : t->c;
            const double n_el = static_cast<double>(Cn) * t->h * t->w;
            const double count = static_cast<double>(t->L_total) * Cn * (t->h - 10) * (t->w - 10);
            loss_combine_kernel<<<1, 1, 0, st>>>(o3, n_el, t->L_total, count);
            launch_check("sharded_step loss");
        }
        if (sharded) {
            float* prm = t->params.as<float>();
            adan_fused_launch(prm, g, t->state.as<float>(), t->P, t->groups, t->total_steps, 0.98, 0.92, 0.99, 1e-8,
                              t->step.as<int>(), t->flags.as<uint32_t>(), st, sb, se);
            nccl_check(nccl().AllGather(prm + sb, prm, static_cast<size_t>(shard), ncclFloat, comm, st),
                       "ncclAllGather");
        } else {
            trainer_enqueue_update(t, st);
        }
        t->host_step += 1;
        if (loss_out) {
            if (slabs && t->s_put) {
                uint32_t err = 0;
                HS_CUDA(cudaMemcpyAsync(&err, t->s_flags.as<uint32_t>() + kMaxPeers, sizeof(err),
                                        cudaMemcpyDeviceToHost, st));
                HS_CUDA(cudaStreamSynchronize(st));
                if (err) throw Error(HS_ECUDA, "row slab: a peer-put exchange timed out waiting for a peer");
            }
            trainer_check_after(t);
            double o3[3];
            HS_CUDA(cudaMemcpy(o3, t->out3.p, sizeof(o3), cudaMemcpyDeviceToHost));
            *loss_out = o3[0];
        }
    });
}

}  // extern "C"
