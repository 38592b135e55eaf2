// pstereo/config.hpp -- drop-in for proj/include/pstereo/config.hpp:12-37.
// PipelineConfig keeps the reference's fields and published defaults (a
// caller fills it exactly as before); validate() runs the library's checks
// (src/coarse_to_fine.cpp:18-49 plus the device path's patch-size cap) and
// throws ConfigError with the same message.
#pragma once

#include <cstdint>
#include <cstring>
#include <vector>

#include "errors.hpp"
#include "../pstereo_gpu.h"

namespace pstereo {

struct PipelineConfig {
  int coarsest_exp = 5;   // level n = image downsampled by 2^n
  int finest_exp = 1;
  int patch_size = 10;    // px
  double overlap = 0.55;  // shared fraction of the patch side
  int min_iterations = 12;
  int max_iterations = 12;
  double early_stop_good = 0.05;
  double early_stop_bad = 0.95;
  double early_stop_improve = 0.10;
  std::vector<double> window_offsets = {0.5, 1.0};  // window {-1,-.5,0,.5,1}
  double sigma_s = 4.0;
  double pixel_threshold = 0.15;
  double gamma = 0.75;
  double valid_patch_ratio = 0.75;
  bool estimate_variance = false;
  int threads = 1;         // validated; the device schedules on its own
  std::uint64_t seed = 1;  // synthetic scenes only
};

namespace gpu {
namespace detail {

// PipelineConfig -> the C ABI's POD (zeroed first: the struct's bytes key the
// context cache, padding included)
inline pstereo_params to_c(const PipelineConfig& c) {
  pstereo_params p;
  std::memset(&p, 0, sizeof p);
  pstereo_default_params(&p);
  p.coarsest_exp = c.coarsest_exp;
  p.finest_exp = c.finest_exp;
  p.patch_size = c.patch_size;
  p.overlap = c.overlap;
  p.min_iterations = c.min_iterations;
  p.max_iterations = c.max_iterations;
  p.early_stop_good = c.early_stop_good;
  p.early_stop_bad = c.early_stop_bad;
  p.early_stop_improve = c.early_stop_improve;
  p.n_window_offsets = int(c.window_offsets.size());
  for (int i = 0; i < PSTEREO_MAX_OFFSETS; ++i)
    p.window_offsets[i] = i < p.n_window_offsets ? c.window_offsets[std::size_t(i)] : 0.0;
  p.sigma_s = c.sigma_s;
  p.pixel_threshold = c.pixel_threshold;
  p.gamma = c.gamma;
  p.valid_patch_ratio = c.valid_patch_ratio;
  p.estimate_variance = c.estimate_variance ? 1 : 0;
  p.threads = c.threads;
  return p;
}

}  // namespace detail
}  // namespace gpu

inline void validate(const PipelineConfig& cfg) {
  const pstereo_params p = gpu::detail::to_c(cfg);
  char msg[256] = {0};
  if (pstereo_validate(&p, msg, sizeof msg) != PSTEREO_OK) throw ConfigError(msg);
}

}  // namespace pstereo
