// pstereo/pipeline.hpp -- drop-in for proj/include/pstereo/pipeline.hpp:10-22:
// PipelineOutput and run_pipeline (match -> confidence filter -> depth,
// src/pipeline.cpp:9-37), one device call through pstereo_gpu_match_f32.
// Also pstereo::gpu::run_pipeline_batch, the same over equally sized pairs in
// one batched call (the throughput entry point).
#pragma once

#include <algorithm>
#include <chrono>
#include <string>
#include <cstddef>
#include <vector>

#include "coarse_to_fine.hpp"
#include "depth_variance.hpp"

namespace pstereo {

struct PipelineOutput {
  ScalarField disparity;  // filtered
  ScalarField probability;
  DepthResult depth;
  MatchStats stats;
  double runtime_ms = 0.0;  // wall time of the device call (per pair in a batch)
};

namespace gpu {

inline std::vector<PipelineOutput> run_pipeline_batch(const std::vector<GrayImage>& lefts,
                                                      const std::vector<GrayImage>& rights,
                                                      const PipelineConfig& cfg,
                                                      const CameraParams& cam) {
  validate(cfg);
  std::vector<PipelineOutput> res;
  if (lefts.size() != rights.size())
    throw DegenerateInputError("run_pipeline_batch: " + std::to_string(lefts.size()) +
                               " left but " + std::to_string(rights.size()) + " right images");
  if (lefts.empty()) return res;
  const int w = lefts[0].width, h = lefts[0].height, n = int(lefts.size());
  std::vector<const GrayImage*> all;
  for (int k = 0; k < n; ++k) {
    const GrayImage &l = lefts[std::size_t(k)], &r = rights[std::size_t(k)];
    if (l.width != r.width || l.height != r.height) detail::size_mismatch(l, r);
    if (l.width != w || l.height != h)
      throw DegenerateInputError("run_pipeline_batch: pair " + std::to_string(k) +
                                 " differs in size from pair 0");
    all.push_back(&l);
    all.push_back(&r);
  }
  const pstereo_params p = detail::to_c(cfg);
  const detail::LevelDims dims = detail::level_dims(p, w, h);
  const std::size_t px = std::size_t(w) * std::size_t(h);
  const bool mask = !detail::all_valid(all);
  std::vector<float> L(px * n), R(px * n);
  std::vector<std::uint8_t> LV, RV;
  if (mask) {
    LV.assign(px * n, 1);
    RV.assign(px * n, 1);
  }
  for (int k = 0; k < n; ++k) {
    const GrayImage &l = lefts[std::size_t(k)], &r = rights[std::size_t(k)];
    std::copy(l.data.begin(), l.data.end(), L.begin() + std::ptrdiff_t(px * k));
    std::copy(r.data.begin(), r.data.end(), R.begin() + std::ptrdiff_t(px * k));
    if (mask && !l.valid.empty())
      std::copy(l.valid.begin(), l.valid.end(), LV.begin() + std::ptrdiff_t(px * k));
    if (mask && !r.valid.empty())
      std::copy(r.valid.begin(), r.valid.end(), RV.begin() + std::ptrdiff_t(px * k));
  }
  pstereo_ctx* ctx = detail::context_for(p, w, h, n);
  std::vector<double> disp(px * n), prob(px * n), depth(px * n), sigma;
  std::vector<std::uint8_t> dvalid(px * n), depth_valid(px * n), sigma_valid;
  std::vector<pstereo_level_stats> stats(std::size_t(dims.n) * n);
  pstereo_outputs o{};
  o.dtype = PSTEREO_F64;
  o.disparity = disp.data();
  o.disparity_valid = dvalid.data();
  o.probability = prob.data();
  o.depth = depth.data();
  o.depth_valid = depth_valid.data();
  if (cfg.estimate_variance) {
    sigma.resize(px * n);
    sigma_valid.resize(px * n);
    o.depth_sigma = sigma.data();
    o.sigma_valid = sigma_valid.data();
  }
  o.stats = stats.data();
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = pstereo_gpu_match_f32(ctx, n, w, h, L.data(), mask ? LV.data() : nullptr,
                                       R.data(), mask ? RV.data() : nullptr, 0, cam.focal_px,
                                       cam.baseline, &o, nullptr);
  const auto t1 = std::chrono::steady_clock::now();
  if (rc != PSTEREO_OK) detail::raise(rc, pstereo_gpu_last_error(ctx));
  const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count() / n;
  res.resize(std::size_t(n));
  auto fill = [&](ScalarField& f, const std::vector<double>& v,
                  const std::vector<std::uint8_t>& ok, int k) {
    f = ScalarField::sized(w, h);
    std::copy(v.begin() + std::ptrdiff_t(px * k), v.begin() + std::ptrdiff_t(px * (k + 1)),
              f.values.begin());
    std::copy(ok.begin() + std::ptrdiff_t(px * k), ok.begin() + std::ptrdiff_t(px * (k + 1)),
              f.valid.begin());
  };
  for (int k = 0; k < n; ++k) {
    PipelineOutput& out = res[std::size_t(k)];
    fill(out.disparity, disp, dvalid, k);
    fill(out.probability, prob, dvalid, k);  // prob.valid := filtered.valid (:31)
    fill(out.depth.depth, depth, depth_valid, k);
    out.depth.has_sigma = cfg.estimate_variance;
    if (cfg.estimate_variance) fill(out.depth.sigma, sigma, sigma_valid, k);
    out.stats = detail::to_stats(stats.data() + std::size_t(dims.n) * k, dims.n);
    out.runtime_ms = ms;
  }
  return res;
}

}  // namespace gpu

inline PipelineOutput run_pipeline(const GrayImage& left, const GrayImage& right,
                                   const PipelineConfig& cfg, const CameraParams& cam) {
  if (left.width != right.width || left.height != right.height)
    gpu::detail::size_mismatch(left, right);
  return gpu::run_pipeline_batch({left}, {right}, cfg, cam).front();
}

}  // namespace pstereo
