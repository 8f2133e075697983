// holosplat-b200 drop-in: the complex Gaussian rasterizer
// (proj/core/include/holo/rasterizer.hpp:12-36) on the B200:
// hs_build_tile_index / hs_rasterize_forward / hs_rasterize_backward.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "holo/complex_field.hpp"
#include "holo/gaussian_set.hpp"

namespace holo {

inline constexpr int kTileSize = 16;

struct TileIndex {
    int tiles_x = 0, tiles_y = 0;
    std::vector<std::pair<uint32_t, uint32_t>> pairs;  // (tile, id), sorted
    std::vector<std::pair<size_t, size_t>> ranges;     // [begin, end) per tile
};

TileIndex build_tile_index(const GaussianSet& set, int width, int height);
ComplexField rasterize_forward(const GaussianSet& set, int width, int height);
GaussianSetGrads rasterize_backward(const GaussianSet& set, const RealField& grad_real,
                                    const RealField& grad_imag);

}  // namespace holo
