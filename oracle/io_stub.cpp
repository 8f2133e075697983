// Test infrastructure (oracle) -- NOT part of the product path.
//
// Throwing stand-ins for the reference's disk/PNG layer (holo/io.hpp, backed by
// libpng in proj/core/src/io.cpp, which is absent from this image).  They exist
// only so the reference's pipeline.cpp (init_gaussians, resolve_gaussian_count)
// links into oracle/_ref; nothing on the hot path touches io.
#include <stdexcept>
#include <string>

#include "holo/io.hpp"

namespace holo {
namespace {
[[noreturn]] void unavailable(const char* what) {
    throw std::runtime_error(std::string("oracle build has no io: ") + what);
}
}  // namespace

void write_field(const std::string&, const ComplexField&, bool) { unavailable("write_field"); }
ComplexField read_field(const std::string&) { unavailable("read_field"); }
void write_gaussians(const std::string&, const GaussianSet&) { unavailable("write_gaussians"); }
GaussianSet read_gaussians(const std::string&) { unavailable("read_gaussians"); }
RealField read_image_linear(const std::string&) { unavailable("read_image_linear"); }
void write_image_srgb(const std::string&, const RealField&) { unavailable("write_image_srgb"); }
RealField read_depth(const std::string&) { unavailable("read_depth"); }
void write_depth_png(const std::string&, const RealField&, int) { unavailable("write_depth_png"); }
void write_phase_png(const std::string&, const RealField&, int) { unavailable("write_phase_png"); }
RealField read_phase_png(const std::string&) { unavailable("read_phase_png"); }
double srgb_to_linear(double) { unavailable("srgb_to_linear"); }
double linear_to_srgb(double) { unavailable("linear_to_srgb"); }
void atomic_write(const std::string&, const std::string&) { unavailable("atomic_write"); }

}  // namespace holo
