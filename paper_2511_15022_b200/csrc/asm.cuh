// Band-limited angular spectrum propagation (K4-K6, K8-K10 of SURVEY §2.1).
#pragma once

#include "common.cuh"
#include "fft.cuh"

namespace hs {

// Per (channel, plane) transfer-function constants, built on the host in fp64
// exactly like make_band_limit (propagation.cpp:54-70).
struct TfConst {
    float kd_mod;   // fmod(k * phase_distance, 2 pi)
    float kd;       // k * phase_distance
    float bx, by;   // (2 pi / (nx pitch k))^2, (2 pi / (ny pitch k))^2
    int mx_max, my_max;  // largest |m| inside the band limit (strict <, propagation.cpp:89)
    double a4;      // 4 * aperture^2, <= 0 disables the aperture (:149-159)
};

struct AsmWork {
    int C = 0, H = 0, W = 0, pad = 0, L = 0;
    int Px = 0, Py = 0, ox = 0, oy = 0, CC = 4, ntiles = 0;
    fft::Plan plan_x, plan_y;
    const float2* twx_ptr = nullptr;  // W_n tables (cached per device)
    const float2* twy_ptr = nullptr;
    DevBuf T1, T2;    // column-tiled intermediates
    DevBuf tf;        // TfConst [L][C]
    std::vector<TfConst> tf_host;
    size_t smem_rows = 0, smem_cols = 0;
    // compile-time planned path (asm_static.cu), when (Px, Py) has a plan
    bool use_static = false;
    const float2* stw_x = nullptr;  // stage twiddle tables of the static plans
    const float2* stw_y = nullptr;

    void prepare(int C, int H, int W, int pad, int L);
    // phase/mask distances per plane (propagate: both = d; backward: phase -d).
    void set_transfer(const hs_prop_spec& spec, const double* phase_d, const double* mask_d,
                      cudaStream_t st);
};

// forward: in C x H x W -> out L x C x H x W  (propagate_multi, propagation.cpp:189-212)
// ev (nullable): 3 events recorded after each of the three kernels.
void asm_forward(AsmWork& w, const float2* d_in, float2* d_out, cudaStream_t st,
                 cudaEvent_t* ev = nullptr);
// backward: grads L x C x H x W -> out C x H x W (propagate_multi_backward, propagation.cpp:214-243)
// conj = true applies conj(H) (the adjoint); the transfer constants must be
// those of the forward planes.
void asm_backward(AsmWork& w, const float2* d_grads, float2* d_out, cudaStream_t st,
                  cudaEvent_t* ev = nullptr);

fft::Plan make_plan(int n);

// ---- shared device helpers (asm.cu generic kernels, asm_static.cu planned kernels) ----
__device__ __forceinline__ int wrapped(int k, int n) { return k < n - n / 2 ? k : k - n; }

// H(kx, ky) for one (channel, plane); CONJ applies the adjoint.
template <bool CONJ>
__device__ __forceinline__ float2 transfer(const TfConst& t, int mx, int my) {
    if (abs(mx) > t.mx_max || abs(my) > t.my_max) return make_float2(0.f, 0.f);
    if (t.a4 > 0.0) {
        const long long ax = 2LL * mx + 1, ay = 2LL * my + 1;
        if (static_cast<double>(ax * ax + ay * ay) >= t.a4) return make_float2(0.f, 0.f);
    }
    const float fmx = static_cast<float>(mx), fmy = static_cast<float>(my);
    const float q = t.bx * fmx * fmx + t.by * fmy * fmy;  // (2 pi f / k)^2
    float ph = 0.f;
    if (q < 1.f) ph = t.kd_mod - t.kd * q / (1.f + sqrtf(1.f - q));  // kz d = kd - kd q/(1+sqrt(1-q))
    float s, c;
    sincosf(ph, &s, &c);
    return make_float2(c, CONJ ? -s : s);
}

struct RowArgs {
    const float2* in;
    float2* out;
    int W, H, Px, ox, ntiles;
    float scale;
    fft::Plan plan;
    const float2* tw;
};

struct ColArgs {
    const float2* in;   // fwd: T1 [C][tiles][H][CC]; bwd: T3 [L][C][tiles][H][CC]
    float2* out;        // fwd: T2 [L][C][tiles][H][CC]; bwd: T4 [C][tiles][H][CC]
    int C, H, Py, Px, oy, ntiles, L;
    fft::Plan plan;
    const float2* tw;
    const TfConst* tf;  // [L][C]
    int tile0 = 0;      // global index of tile 0 of this call (column-slab shard)
};

// ---- row-slab sharding (cfg4 distributed FFT) ------------------------
// The three passes of asm_forward / asm_backward on explicit buffers.
// Row pass over `planes` stacked fields of h rows each: forward
// in [planes][h][W] -> T [planes][ntiles][h][CC]; inverse T -> [planes][h][W]
// (cropped, x 1/(Px Py)).
void asm_rows_pass(AsmWork& w, bool inverse, const float2* in, float2* out, int planes, int h, cudaStream_t st);
// Column pass over the column tiles [tile0, tile0 + ntiles_local) of all H
// rows: forward T [C][nt][H][CC] -> [L][C][nt][H][CC] (x H_l), backward
// [L][C][nt][H][CC] -> [C][nt][H][CC] (sum_l x conj H_l).
void asm_cols_pass(AsmWork& w, bool backward, const float2* in, float2* out, int tile0, int ntiles_local,
                   cudaStream_t st);

// Block copy for the all-to-all layouts: chunk (a, b, t), a < A (peer),
// b < B (plane), t < T (tile), copies len[a] float2 from
// src[sA[a] + b sB[a] + t sT[a]] to dst[dA[a] + b dB[a] + t dT[a]].
constexpr int kMaxPeers = 16;
// dptr[a] (optional): destination base for peer a (a peer's receive buffer
// mapped into this context: same device, P2P or CUDA IPC), else dst.
struct ChunkMap {
    int A = 0, B = 0, T = 0;
    int64_t len[kMaxPeers], sA[kMaxPeers], sB[kMaxPeers], sT[kMaxPeers], dA[kMaxPeers], dB[kMaxPeers],
        dT[kMaxPeers];
    float2* dptr[kMaxPeers] = {};
};
void chunk_copy(const float2* src, float2* dst, const ChunkMap& m, cudaStream_t st);
// Exchange flags of the peer-put transposes.  The exchange epoch lives on the
// device (*epoch, this rank's counter), so a captured step replays correctly:
// signal increments it and writes the new value into slot `me` of every
// peer's flag array (system-scope release after a fence); wait spins
// (acquire) until every slot of this rank's flags reaches *epoch, and gives
// up after ~2 s with error[0] = 1 (no hang when a peer died).
void slab_signal(uint32_t* const* peer_flags, int ranks, int me, uint32_t* epoch, cudaStream_t st);
void slab_wait(const uint32_t* flags, int ranks, const uint32_t* epoch, uint32_t* error, cudaStream_t st);

// Row FFT whose last stage stores straight into the peers' receive buffers
// (row-slab peer-put exchange fused into the compute kernel): the output
// column tile T belongs to rank s = T / ts; only rows [row0, row0 + hout) of
// each plane are sent, to peer[s] + slot[s] + ((plane ts + T - s ts) hout +
// y - row0) CC + cc.  Returns false when the grid has no planned row kernel
// (the caller then runs asm_rows_pass + a pack).
struct SlabPut {
    float2* peer[kMaxPeers];
    int64_t slot[kMaxPeers];
    int ts, row0, hout;
    unsigned ts_magic;  // ceil(2^32 / ts)
};
bool asm_rows_fwd_put(AsmWork& w, const float2* in, int planes, int h, const SlabPut& sp, cudaStream_t st);
// Inverse row pass reading its column tiles straight from a peer-major
// receive buffer [src s][planes][ts][h][CC] (tile T = s ts + tl), i.e. the
// exchange's unpack fused into the load; false without a planned row kernel.
struct SlabGet {
    int ts;
    unsigned ts_magic;  // ceil(2^32 / ts)
    int64_t per_src;    // float2 per source segment = planes ts h CC
};
bool asm_rows_inv_get(AsmWork& w, const float2* recv, float2* out, int planes, int h, const SlabGet& sg,
                      cudaStream_t st);
// Column pass of a row-slab rank (single plane, planned grids): each tile's
// H rows are gathered from the R source segments of the peer-major receive
// buffer by R TMA bulk copies (the unpack fused into the load), and the
// cropped output rows are either stored to the local T layout (out) or put
// straight into every peer whose row band [g0[d], g0[d] + he[d]) holds them
// (peer[d] + slot[d] + ((plane ts + tl) he[d] + y - g0[d]) CC + cc).
struct SlabCol {
    const float2* in;
    int64_t per_src;
    int R, hr;
    float inv_hr;
    int put;
    float2* peer[kMaxPeers];
    int64_t slot[kMaxPeers];
    int g0[kMaxPeers], he[kMaxPeers];
};
bool asm_cols_slab(AsmWork& w, bool backward, const SlabCol& sc, float2* out, int tile0, int ntiles_local,
                   cudaStream_t st);

// Static (compile-time planned) propagation path; false when (Px, Py) has no plan.
bool static_plan_cc(int Px, int Py, int pad, int L, int* cc);
bool static_forward(AsmWork& w, const float2* d_in, float2* d_out, cudaStream_t st, cudaEvent_t* ev);
bool static_backward(AsmWork& w, const float2* d_grads, float2* d_out, cudaStream_t st, cudaEvent_t* ev);
void static_prepare(AsmWork& w);
bool static_rows_pass(AsmWork& w, bool inverse, const float2* in, float2* out, int planes, int h, cudaStream_t st);
bool static_cols_pass(AsmWork& w, bool backward, const float2* in, float2* out, int tile0, int ntiles_local,
                      cudaStream_t st);

}  // namespace hs
