// pstereo/depth_variance.hpp -- drop-in for the caller-facing part of
// proj/include/pstereo/depth_variance.hpp:10-29: the constants, CameraParams
// and DepthResult. The confidence filter, depth conversion and the per-patch
// variance fit (filter_validity, disparity_to_depth, estimate_patch_variance)
// run inside run_pipeline on the device and are not separate entry points.
#pragma once

#include "fields.hpp"

namespace pstereo {

inline constexpr double kMinDisparity = 0.1;    // px; smaller => no depth
inline constexpr double kSigmaFallback = 2.0;   // px; rejected variance fits
inline constexpr int kVarianceFitIterations = 10;
inline constexpr double kVarianceFitMaxResidual = 0.1;

struct CameraParams {
  double focal_px = 0.0;
  double baseline = 0.0;  // the unit of the output depth
};

struct DepthResult {
  ScalarField depth;  // focal_px * baseline / disparity
  ScalarField sigma;  // depth std (has_sigma)
  bool has_sigma = false;
};

}  // namespace pstereo
