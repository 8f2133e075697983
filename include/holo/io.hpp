// holosplat-b200 drop-in: the binary artifact formats of the reference
// (proj/core/include/holo/io.hpp, io.cpp:237-335) -- CGHF complex fields and
// CGGS Gaussian sets, little-endian, written through a temp file + rename.
// The PNG ingest/egress of that header (libpng) is run orchestration around the
// hot path and is out of scope.
#pragma once

#include <string>

#include "holo/complex_field.hpp"
#include "holo/gaussian_set.hpp"

namespace holo {

// "CGHF": magic, u16 version 1, u32 C, H, W, u8 dtype (0 f32, 1 f64), all real
// values then all imaginary values (planar).
void write_field(const std::string& path, const ComplexField& field, bool as_f64 = true);
ComplexField read_field(const std::string& path);

// "CGGS": magic, u16 version 1, u32 N, u32 C, the six parameter groups in
// declaration order as f32.
void write_gaussians(const std::string& path, const GaussianSet& set);
GaussianSet read_gaussians(const std::string& path);

// temp file in the same directory, then rename
void atomic_write(const std::string& path, const std::string& bytes);

}  // namespace holo
