// Rasterizer work buffers and launchers (K0 projection, K1 binning, K2 forward,
// K3 backward).  See raster.cu for the kernels and the reference mapping.
#pragma once

#include "common.cuh"

namespace hs {

// Device-resident projection + tile index for one (set, canvas).  Buffers are
// reused across calls and only grow.
#ifndef HS_TILE_BWD_DEFAULT
#define HS_TILE_BWD_DEFAULT true
#endif

struct RasterWork {
    int n = 0, c = 0, width = 0, height = 0;
    int tiles_x = 0, tiles_y = 0, tile_bits = 0;
    DevBuf rec;      // 3 x N float4, SoA (fp32 shading record)
    DevBuf shade;    // C x N float4, SoA: amp*cos, amp*sin, cos, sin
    DevBuf p64;      // 8 x N doubles, SoA (exact fp64 record for boundary rechecks)
    DevBuf pbox;     // int4 pixel bbox (x0,x1,y0,y1) clamped to the canvas
    DevBuf tbox;     // int4 tile bbox
    DevBuf trows;    // uint4 per Gaussian: touched tile columns of the first box rows (tight binning)
    DevBuf tcount;   // uint32 Gaussians per tile
    DevBuf toffset;  // uint32 exclusive scan of tcount
    DevBuf raw;      // backward partial sums, (7+2C) x N floats (SoA)
    DevBuf ids;      // uint32 Gaussian ids grouped by tile, ascending within a tile
    DevBuf scratch;  // 2 x cap uint32: global bitonic fallback for huge tiles
    DevBuf ranges;   // uint2 [begin,end) per tile
    DevBuf status;   // uint32[4]: [0] K (pairs), [1] overflow, [2] non-finite param, [3] unused
    DevBuf work;     // uint32 work counter of the persistent backward
    DevBuf raw16;    // per-tile backward: [N][16] float partial sums (AoS, vector atomics)
    // Backward form: per-tile with atomics (fast, last bits depend on the
    // atomic order) or the deterministic per-Gaussian gather (K3).
    bool tile_bwd = HS_TILE_BWD_DEFAULT;
    int sms = 0;     // SM count of the device (persistent grids)
    int64_t cap = 0; // pair capacity
    int band_ty0 = 0, band_ty1 = 1 << 30;  // tile rows binned (a row-slab rank: its band)
    // row-slab rank: the Gaussians whose pixel box meets rows [band_y0, band_y1]
    // (compacted after the projection; binning and the backward walk only them)
    int band_y0 = -1, band_y1 = -1;
    DevBuf band_list, band_n;
    bool banded() const { return band_y0 >= 0; }
    // Tight binning (default): keep only the (tile, Gaussian) pairs whose tile the
    // ellipse can reach; the forward field is bit-identical.  false: the
    // reference's exact box list (build_tile_index export).
    bool tight = true;

    void prepare(int n_, int c_, int w_, int h_);
    void reserve_pairs(int64_t cap_);
    // K0 + K1 + shading on stream; leaves per-tile sorted ids + ranges on device
    // (K in status[0]).  shading_ready (nullable): event the shading kernel waits
    // for -- the amplitude/phase groups may still be uploading while the
    // geometry is projected and binned.
    void project_and_bin(const float* d_params, cudaStream_t st, cudaEvent_t shading_ready = nullptr);
};

// Row band [y0, y0 + hs) (hs < 0: to the bottom): the forward writes only
// those rows (field = C x hs x W), the backward reads only those rows of the
// gradient field (C x hs x W) and sums each Gaussian over its footprint inside
// the band -- the partial gradient of a row-slab shard.
void raster_forward(const RasterWork& rw, float2* d_field, cudaStream_t st, int y0 = 0, int hs = -1);
void raster_backward(const RasterWork& rw, const float* d_params, const float2* d_grad_field,
                     float* d_grads, uint32_t* d_flags, cudaStream_t st, int y0 = 0, int hs = -1);
// tiles/ids (uint32) + ranges (uint64 pairs) export for build_tile_index.
void export_tile_index(const RasterWork& rw, int64_t k, uint32_t* d_tiles, uint32_t* d_ids,
                       uint64_t* d_ranges, cudaStream_t st);

}  // namespace hs
