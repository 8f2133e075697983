// holosplat-b200 drop-in: the end-of-run metrics of the reference's pipeline
// (proj/core/include/holo/pipeline.hpp:47-57, pipeline.cpp:135-163).  The rest
// of that header (RunConfig, train, artifacts) is the run orchestration around
// the hot path and is out of scope for this library.
#pragma once

#include <vector>

#include "holo/complex_field.hpp"

namespace holo {

struct Metrics {
    std::vector<double> psnr;  // dB per plane; +inf for identical images
    std::vector<double> ssim;
    double mean_psnr = 0.0;
    double mean_ssim = 0.0;
};

// PSNR of [0,1]-clamped images (host fp64, pipeline.cpp:135-147)
double psnr_value(const RealField& recon, const RealField& target);

// per-plane PSNR and ssim_value of clipped reconstructions, on the B200
Metrics compute_metrics(const std::vector<RealField>& recon, const RealField& target);

}  // namespace holo
