// pstereo/coarse_to_fine.hpp -- drop-in for the caller-facing part of
// proj/include/pstereo/coarse_to_fine.hpp:39-103: PatchEstimate,
// LevelEstimate, MatchStats, MatchResult (with `finest`, the finest level's
// fused fields and its accepted patches) and match_stereo, which runs on the
// device through pstereo_gpu_match_f32. The per-level internals the reference
// also declares there (PatchGrid, fuse_level, init_next_level, ...) are
// kernels here and are not separate entry points.
#pragma once

#include <cmath>
#include <cstddef>
#include <string>
#include <vector>

#include "config.hpp"
#include "fields.hpp"
#include "gpu_runtime.hpp"
#include "image.hpp"

namespace pstereo {

struct PatchEstimate {
  double cx = 0.0;
  double cy = 0.0;
  double u = 0.0;          // disparity, level px
  double prob = 0.0;       // propagated probability (fusion weight)
  double posterior = 0.0;  // this level's window posterior
  double sigma_k = 0.0;    // variance-fit std, level px
  bool has_sigma = false;
};

struct LevelEstimate {
  int level_exp = 0;
  int width = 0;
  int height = 0;
  ScalarField disparity;
  ScalarField probability;
  ScalarField var_disp;
  bool has_variance = false;
  std::vector<PatchEstimate> patches;  // accepted patches, patch-index order
};

struct MatchStats {
  struct Level {
    int exp = 0;
    int grid_patches = 0;
    int extracted = 0;
    int converged = 0;
    int accepted = 0;
  };
  std::vector<Level> levels;  // coarsest first
};

struct MatchResult {
  ScalarField disparity;  // full resolution, before the confidence filter
  ScalarField probability;
  ScalarField var_disp;  // px^2 (estimate_variance)
  bool has_variance = false;
  LevelEstimate finest;
  MatchStats stats;
};

namespace gpu {
namespace detail {

[[noreturn]] inline void size_mismatch(const GrayImage& l, const GrayImage& r) {
  throw DegenerateInputError("build_pyramid: left is " + std::to_string(l.width) + "x" +
                             std::to_string(l.height) + " but right is " +
                             std::to_string(r.width) + "x" + std::to_string(r.height));
}

// nullptr when every pixel of every image is valid (the mask-free kernels)
inline bool all_valid(const std::vector<const GrayImage*>& imgs) {
  for (const GrayImage* g : imgs)
    for (std::uint8_t v : g->valid)
      if (!v) return false;
  return true;
}

struct LevelDims {
  int n = 0;
  int w[PSTEREO_MAX_LEVELS], h[PSTEREO_MAX_LEVELS], e[PSTEREO_MAX_LEVELS];
};

inline LevelDims level_dims(const pstereo_params& p, int width, int height) {
  LevelDims d;
  const int rc = pstereo_level_dims(&p, width, height, &d.n, d.w, d.h, d.e);
  if (rc != PSTEREO_OK) {
    if (rc == PSTEREO_EDEGENERATE)
      throw DegenerateInputError("build_pyramid: coarsest level of " + std::to_string(width) +
                                 "x" + std::to_string(height) + " is smaller than one patch (" +
                                 std::to_string(p.patch_size) + ")");
    raise(rc, "level geometry");
  }
  return d;
}

// patches on one axis of a level, an upper bound: make_patch_grid
// (src/coarse_to_fine.cpp:51-88) places ceil((L - s) / stride) + 1 centres,
// stride = max(1, lrint(s * (1 - overlap))) (ties to even)
inline std::size_t grid_cap(int extent, const pstereo_params& p) {
  long st = std::lrint(p.patch_size * (1.0 - p.overlap));
  if (st < 1) st = 1;
  return extent < p.patch_size ? 1 : std::size_t((extent - p.patch_size) / st + 2);
}

inline MatchStats to_stats(const pstereo_level_stats* s, int n) {
  MatchStats m;
  for (int l = 0; l < n; ++l)
    m.levels.push_back({s[l].exp, s[l].grid_patches, s[l].extracted, s[l].converged,
                        s[l].accepted});
  return m;
}

}  // namespace detail
}  // namespace gpu

inline MatchResult match_stereo(const GrayImage& left, const GrayImage& right,
                                const PipelineConfig& cfg) {
  validate(cfg);
  if (left.width != right.width || left.height != right.height)
    gpu::detail::size_mismatch(left, right);
  const int w = left.width, h = left.height;
  const std::size_t px = std::size_t(w) * std::size_t(h);
  const pstereo_params p = gpu::detail::to_c(cfg);
  const gpu::detail::LevelDims dims = gpu::detail::level_dims(p, w, h);
  const int fi = dims.n - 1;  // finest level (coarsest first)
  const int lw = dims.w[fi], lh = dims.h[fi], fe = dims.e[fi];
  pstereo_ctx* ctx = gpu::detail::context_for(p, w, h, 1);

  MatchResult m;
  m.disparity = ScalarField::sized(w, h);
  m.probability = ScalarField::sized(w, h);
  m.has_variance = cfg.estimate_variance;
  if (m.has_variance) m.var_disp = ScalarField::sized(w, h);
  std::vector<double> prob(px);
  std::vector<pstereo_level_stats> stats(std::size_t(dims.n));
  const std::size_t cap = gpu::detail::grid_cap(lw, p) * gpu::detail::grid_cap(lh, p);
  std::vector<pstereo_patch_estimate> recs(cap);
  int n_recs = 0;
  pstereo_outputs o{};
  o.dtype = PSTEREO_F64;
  o.match_disparity = m.disparity.values.data();
  o.match_valid = m.disparity.valid.data();
  o.probability = prob.data();
  if (m.has_variance) o.var_disp = m.var_disp.values.data();
  o.stats = stats.data();
  o.finest = recs.data();
  o.finest_count = &n_recs;
  o.finest_cap = int(cap);
  const bool mask = !gpu::detail::all_valid({&left, &right});
  const int rc = pstereo_gpu_match_f32(
      ctx, 1, w, h, left.data.data(), mask && !left.valid.empty() ? left.valid.data() : nullptr,
      right.data.data(), mask && !right.valid.empty() ? right.valid.data() : nullptr, 0, 1.0, 1.0,
      &o, nullptr);
  if (rc != PSTEREO_OK) gpu::detail::raise(rc, pstereo_gpu_last_error(ctx));
  // probability and variance share the disparity's validity (fuse_level)
  for (std::size_t i = 0; i < px; ++i) {
    if (!m.disparity.valid[i]) continue;
    m.probability.values[i] = prob[i];
    m.probability.valid[i] = 1;
    if (m.has_variance) m.var_disp.valid[i] = 1;
  }
  m.stats = gpu::detail::to_stats(stats.data(), dims.n);

  // the finest level: the full-resolution fields are its nearest-neighbour
  // upsampling scaled by 2^fe (disparity), 1 (probability) and 4^fe
  // (variance), exactly (src/coarse_to_fine.cpp:166-180, :328-337), so level
  // pixel (x, y) is full pixel (x << fe, y << fe) divided back -- a power of
  // two, no rounding
  LevelEstimate& f = m.finest;
  f.level_exp = fe;
  f.width = lw;
  f.height = lh;
  f.has_variance = m.has_variance;
  f.disparity = ScalarField::sized(lw, lh);
  f.probability = ScalarField::sized(lw, lh);
  if (f.has_variance) f.var_disp = ScalarField::sized(lw, lh);
  const double s1 = double(1LL << fe), s2 = s1 * s1;
  for (int y = 0; y < lh; ++y)
    for (int x = 0; x < lw; ++x) {
      const std::size_t src = std::size_t(y << fe) * std::size_t(w) + std::size_t(x << fe);
      const std::size_t dst = f.disparity.index(x, y);
      const std::uint8_t ok = m.disparity.valid[src];
      f.disparity.values[dst] = m.disparity.values[src] / s1;
      f.disparity.valid[dst] = ok;
      f.probability.values[dst] = m.probability.values[src];
      f.probability.valid[dst] = ok;
      if (f.has_variance) {
        f.var_disp.values[dst] = m.var_disp.values[src] / s2;
        f.var_disp.valid[dst] = ok;
      }
    }
  if (n_recs > int(cap)) throw gpu::GpuError("match_stereo: finest-level records truncated");
  f.patches.reserve(std::size_t(n_recs));
  for (int k = 0; k < n_recs; ++k) {
    const pstereo_patch_estimate& r = recs[std::size_t(k)];
    f.patches.push_back({r.cx, r.cy, r.u, r.prob, r.posterior, r.sigma_k, m.has_variance});
  }
  return m;
}

}  // namespace pstereo
