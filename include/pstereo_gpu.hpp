// pstereo_gpu.hpp -- the reference's C++ entry points, re-exposed on the B200
// C ABI (include/pstereo_gpu.h). Header-only; link libpstereo_gpu.so.
//
// Mirrors (names, argument meaning, error behaviour):
//   PipelineConfig, validate       proj/include/pstereo/config.hpp:12-37
//   ConfigError, DegenerateInputError  proj/include/pstereo/errors.hpp:9-31
//   GrayImage, Raster              proj/include/pstereo/image.hpp:12-26
//   ScalarField                    proj/include/pstereo/fields.hpp:10-39
//   MatchStats, MatchResult,
//   match_stereo                   proj/include/pstereo/coarse_to_fine.hpp:80-103
//   CameraParams, DepthResult      proj/include/pstereo/depth_variance.hpp:20-29
//   PipelineOutput, run_pipeline   proj/include/pstereo/pipeline.hpp:10-22
//   IoError, load_image, load_calibration, write_pfm, read_pfm, metrics CSV
//                                  proj/include/pstereo/io.hpp, src/io.cpp
//   SceneSpec, load_scene_spec, RenderedScene, render_scene
//                                  proj/include/pstereo/synth.hpp, src/synth.cpp
//   BenchResult, run_benchmark     proj/include/pstereo/bench.hpp, src/bench.cpp
// A caller such as the reference's run_benchmark (src/bench.cpp:24) or
// run_match (src/runner.cpp:140) switches by including this header instead of
// pipeline.hpp and defining PSTEREO_GPU_AS_DEFAULT (which makes pstereo::X
// resolve to pstereo::gpu::X). Results are bit-identical to the reference
// (var_disp / depth sigma within 1e-3 relative); see DESIGN.md.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "pstereo_gpu.h"

namespace pstereo {
namespace gpu {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DegenerateInputError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct GpuError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct PipelineConfig {
  int coarsest_exp = 5;
  int finest_exp = 1;
  int patch_size = 10;
  double overlap = 0.55;
  int min_iterations = 12;
  int max_iterations = 12;
  double early_stop_good = 0.05;
  double early_stop_bad = 0.95;
  double early_stop_improve = 0.10;
  std::vector<double> window_offsets = {0.5, 1.0};
  double sigma_s = 4.0;
  double pixel_threshold = 0.15;
  double gamma = 0.75;
  double valid_patch_ratio = 0.75;
  bool estimate_variance = false;
  int threads = 1;
  std::uint64_t seed = 1;
};

struct Raster {
  int width = 0;
  int height = 0;
  int channels = 0;
  std::vector<std::uint8_t> pixels;
};

struct GrayImage {
  int width = 0;
  int height = 0;
  std::vector<float> data;
  std::vector<std::uint8_t> valid;
};

struct ScalarField {
  int width = 0;
  int height = 0;
  std::vector<double> values;
  std::vector<std::uint8_t> valid;
  static ScalarField sized(int w, int h) {
    ScalarField f;
    f.width = w;
    f.height = h;
    f.values.assign(std::size_t(w) * h, 0.0);
    f.valid.assign(std::size_t(w) * h, 0);
    return f;
  }
};

struct MatchStats {
  struct Level {
    int exp = 0;
    int grid_patches = 0;
    int extracted = 0;
    int converged = 0;
    int accepted = 0;
  };
  std::vector<Level> levels;
};

struct MatchResult {
  ScalarField disparity;
  ScalarField probability;
  ScalarField var_disp;
  bool has_variance = false;
  MatchStats stats;
};

struct CameraParams {
  double focal_px = 0.0;
  double baseline = 0.0;
};

struct DepthResult {
  ScalarField depth;
  ScalarField sigma;
  bool has_sigma = false;
};

struct PipelineOutput {
  ScalarField disparity;
  ScalarField probability;
  DepthResult depth;
  MatchStats stats;
  double runtime_ms = 0.0;
};

namespace detail {

inline pstereo_params to_c(const PipelineConfig& c) {
  pstereo_params p;
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
  for (std::size_t i = 0; i < c.window_offsets.size() && i < PSTEREO_MAX_OFFSETS; ++i)
    p.window_offsets[i] = c.window_offsets[i];
  p.sigma_s = c.sigma_s;
  p.pixel_threshold = c.pixel_threshold;
  p.gamma = c.gamma;
  p.valid_patch_ratio = c.valid_patch_ratio;
  p.estimate_variance = c.estimate_variance ? 1 : 0;
  p.threads = c.threads;
  return p;
}

[[noreturn]] inline void raise(int code, const std::string& msg) {
  if (code == PSTEREO_ECONFIG) throw ConfigError(msg);
  if (code == PSTEREO_EDEGENERATE) throw DegenerateInputError(msg);
  throw GpuError(msg);
}

// One device context per (config, size) per thread: contexts are not
// re-entrant (include/pstereo_gpu.h).
struct CtxDeleter {
  void operator()(pstereo_ctx* c) const { pstereo_gpu_destroy(c); }
};
using CtxPtr = std::unique_ptr<pstereo_ctx, CtxDeleter>;

inline pstereo_ctx* context_for(const pstereo_params& p, int w, int h, int n) {
  thread_local std::map<std::tuple<std::string, int, int, int>, CtxPtr> cache;
  const std::string key(reinterpret_cast<const char*>(&p), sizeof p);
  auto& slot = cache[std::make_tuple(key, w, h, n)];
  if (!slot) {
    pstereo_ctx* c = nullptr;
    const int rc = pstereo_gpu_create(0, &p, w, h, n, &c);
    if (rc) raise(rc, rc == PSTEREO_ECONFIG ? "config: invalid" : "pstereo_gpu_create failed");
    slot.reset(c);
  }
  return slot.get();
}

}  // namespace detail

// validate (src/coarse_to_fine.cpp:18-49)
inline void validate(const PipelineConfig& cfg) {
  const pstereo_params p = detail::to_c(cfg);
  char msg[256] = {0};
  const int rc = pstereo_validate(&p, msg, sizeof msg);
  if (rc) detail::raise(rc, msg);
}

// Batched run_pipeline over equally sized GrayImage pairs (the throughput API).
inline std::vector<PipelineOutput> run_pipeline_batch(const std::vector<GrayImage>& lefts,
                                                      const std::vector<GrayImage>& rights,
                                                      const PipelineConfig& cfg,
                                                      const CameraParams& cam) {
  validate(cfg);
  std::vector<PipelineOutput> res;
  if (lefts.empty()) return res;
  if (lefts.size() != rights.size()) throw DegenerateInputError("batch size mismatch");
  const int w = lefts[0].width, h = lefts[0].height, n = int(lefts.size());
  for (int k = 0; k < n; ++k)
    if (lefts[k].width != w || lefts[k].height != h || rights[k].width != w ||
        rights[k].height != h)
      throw DegenerateInputError("build_pyramid: left and right differ in size");
  const std::size_t px = std::size_t(w) * h;
  std::vector<float> L(px * n), R(px * n);
  std::vector<std::uint8_t> LV(px * n, 1), RV(px * n, 1);
  for (int k = 0; k < n; ++k) {
    std::copy(lefts[k].data.begin(), lefts[k].data.end(), L.begin() + px * k);
    std::copy(rights[k].data.begin(), rights[k].data.end(), R.begin() + px * k);
    if (!lefts[k].valid.empty())
      std::copy(lefts[k].valid.begin(), lefts[k].valid.end(), LV.begin() + px * k);
    if (!rights[k].valid.empty())
      std::copy(rights[k].valid.begin(), rights[k].valid.end(), RV.begin() + px * k);
  }
  const pstereo_params p = detail::to_c(cfg);
  pstereo_ctx* ctx = detail::context_for(p, w, h, n);
  const int nl = cfg.coarsest_exp - cfg.finest_exp + 1;
  std::vector<double> disp(px * n), prob(px * n), depth(px * n), sigma(px * n);
  std::vector<std::uint8_t> dvalid(px * n), depth_valid(px * n), sigma_valid(px * n);
  std::vector<pstereo_level_stats> stats(std::size_t(nl) * n);
  pstereo_outputs o{};
  o.dtype = PSTEREO_F64;
  o.on_device = 0;
  o.disparity = disp.data();
  o.disparity_valid = dvalid.data();
  o.probability = prob.data();
  o.depth = depth.data();
  o.depth_valid = depth_valid.data();
  if (cfg.estimate_variance) {
    o.depth_sigma = sigma.data();
    o.sigma_valid = sigma_valid.data();
  }
  o.stats = stats.data();
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = pstereo_gpu_match_f32(ctx, n, w, h, L.data(), LV.data(), R.data(), RV.data(), 0,
                                       cam.focal_px, cam.baseline, &o, nullptr);
  const auto t1 = std::chrono::steady_clock::now();
  if (rc) detail::raise(rc, pstereo_gpu_last_error(ctx));
  res.resize(std::size_t(n));
  for (int k = 0; k < n; ++k) {
    PipelineOutput& out = res[std::size_t(k)];
    auto fill = [&](ScalarField& f, const std::vector<double>& v, const std::vector<std::uint8_t>& ok) {
      f = ScalarField::sized(w, h);
      std::copy(v.begin() + px * k, v.begin() + px * (k + 1), f.values.begin());
      std::copy(ok.begin() + px * k, ok.begin() + px * (k + 1), f.valid.begin());
    };
    fill(out.disparity, disp, dvalid);
    fill(out.probability, prob, dvalid);
    fill(out.depth.depth, depth, depth_valid);
    out.depth.has_sigma = cfg.estimate_variance;
    if (cfg.estimate_variance) fill(out.depth.sigma, sigma, sigma_valid);
    for (int l = 0; l < nl; ++l) {
      const pstereo_level_stats& s = stats[std::size_t(k) * nl + l];
      out.stats.levels.push_back({s.exp, s.grid_patches, s.extracted, s.converged, s.accepted});
    }
    out.runtime_ms = std::chrono::duration<double, std::milli>(t1 - t0).count() / n;
  }
  return res;
}

// run_pipeline (inc/pipeline.hpp:20-22)
inline PipelineOutput run_pipeline(const GrayImage& left, const GrayImage& right,
                                   const PipelineConfig& cfg, const CameraParams& cam) {
  if (left.width != right.width || left.height != right.height)
    throw DegenerateInputError("build_pyramid: left and right differ in size");
  return run_pipeline_batch({left}, {right}, cfg, cam).front();
}

// match_stereo (inc/coarse_to_fine.hpp:102-103): pre-filter fields.
inline MatchResult match_stereo(const GrayImage& left, const GrayImage& right,
                                const PipelineConfig& cfg) {
  validate(cfg);
  if (left.width != right.width || left.height != right.height)
    throw DegenerateInputError("build_pyramid: left and right differ in size");
  const int w = left.width, h = left.height;
  const std::size_t px = std::size_t(w) * h;
  const pstereo_params p = detail::to_c(cfg);
  pstereo_ctx* ctx = detail::context_for(p, w, h, 1);
  MatchResult m;
  m.disparity = ScalarField::sized(w, h);
  m.probability = ScalarField::sized(w, h);
  m.has_variance = cfg.estimate_variance;
  if (m.has_variance) m.var_disp = ScalarField::sized(w, h);
  const int nl = cfg.coarsest_exp - cfg.finest_exp + 1;
  std::vector<pstereo_level_stats> stats(static_cast<std::size_t>(nl));
  std::vector<double> prob(px);
  pstereo_outputs o{};
  o.dtype = PSTEREO_F64;
  o.match_disparity = m.disparity.values.data();
  o.match_valid = m.disparity.valid.data();
  o.probability = prob.data();
  if (m.has_variance) o.var_disp = m.var_disp.values.data();
  o.stats = stats.data();
  const int rc = pstereo_gpu_match_f32(ctx, 1, w, h, left.data.data(),
                                       left.valid.empty() ? nullptr : left.valid.data(),
                                       right.data.data(),
                                       right.valid.empty() ? nullptr : right.valid.data(), 0, 1.0,
                                       1.0, &o, nullptr);
  if (rc) detail::raise(rc, pstereo_gpu_last_error(ctx));
  for (std::size_t i = 0; i < px; ++i) {
    if (!m.disparity.valid[i]) continue;
    m.probability.values[i] = prob[i];
    m.probability.valid[i] = 1;
    if (m.has_variance) m.var_disp.valid[i] = 1;
  }
  for (const auto& s : stats)
    m.stats.levels.push_back({s.exp, s.grid_patches, s.extracted, s.converged, s.accepted});
  return m;
}

// FrameMetrics / compute_metrics (inc/metrics.hpp:14-32, src/metrics.cpp:10-52)
struct FrameMetrics {
  std::string frame;
  double mean_err = std::numeric_limits<double>::quiet_NaN();
  double median_err = std::numeric_limits<double>::quiet_NaN();
  long long valid_px = 0;
  double runtime_ms = 0.0;
  double coverage_rate = std::numeric_limits<double>::quiet_NaN();
  bool has_errors = false;
};

inline FrameMetrics compute_metrics(const ScalarField& estimate, const ScalarField& reference,
                                    const ScalarField* sigma, double runtime_ms,
                                    const std::string& frame) {
  const int w = estimate.width, h = estimate.height;
  pstereo_params p;
  pstereo_default_params(&p);
  p.coarsest_exp = 0;
  p.finest_exp = 0;
  p.patch_size = 2;
  pstereo_ctx* ctx = detail::context_for(p, w, h, 1);
  pstereo_frame_metrics m{};
  const int rc = pstereo_gpu_metrics(
      ctx, 1, w, h, estimate.values.data(), estimate.valid.data(), reference.values.data(),
      reference.valid.data(), sigma ? sigma->values.data() : nullptr,
      sigma ? sigma->valid.data() : nullptr, 0, &m, nullptr);
  if (rc) detail::raise(rc, pstereo_gpu_last_error(ctx));
  FrameMetrics f;
  f.frame = frame;
  f.runtime_ms = runtime_ms;
  f.valid_px = m.valid_px;
  f.has_errors = m.has_errors != 0;
  f.mean_err = m.mean_err;
  f.median_err = m.median_err;
  f.coverage_rate = m.coverage_rate;
  return f;
}

// ---- caller side: I/O formats, scenes, benchmark ----

enum class IoErrorKind { missing_file, decode_failure, write_failure, dimension_mismatch };
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void raise_io(int rc, const char* msg) {
  if (rc == PSTEREO_EIO) throw IoError(msg);
  if (rc) raise(rc, msg);
}
}  // namespace detail

// load_image (src/io.cpp:253-263): PGM/PPM/PNG -> Raster
inline Raster load_image(const std::string& path) {
  char msg[512];
  Raster r;
  detail::raise_io(pstereo_load_image(path.c_str(), &r.width, &r.height, &r.channels, nullptr, 0,
                                      msg, sizeof msg),
                   msg);
  r.pixels.resize(std::size_t(r.width) * r.height * r.channels);
  detail::raise_io(pstereo_load_image(path.c_str(), &r.width, &r.height, &r.channels,
                                      r.pixels.data(), r.pixels.size(), msg, sizeof msg),
                   msg);
  return r;
}

struct CalibrationFile {
  double focal_px = 0.0;
  double baseline_mm = 0.0;
  int width = 0;
  int height = 0;
};

// load_calibration (src/io.cpp:266-281)
inline CalibrationFile load_calibration(const std::string& path) {
  char msg[512];
  CalibrationFile c;
  detail::raise_io(pstereo_load_calibration(path.c_str(), &c.focal_px, &c.baseline_mm, &c.width,
                                            &c.height, msg, sizeof msg),
                   msg);
  return c;
}

// write_pfm (src/io.cpp:297-310): -1 at invalid pixels, rows bottom to top
inline void write_pfm(const ScalarField& field, const std::string& path) {
  std::vector<float> v(field.values.size());
  for (std::size_t i = 0; i < v.size(); ++i) v[i] = float(field.values[i]);
  char msg[512];
  detail::raise_io(pstereo_write_pfm(path.c_str(), field.width, field.height, v.data(),
                                     field.valid.data(), 0, msg, sizeof msg),
                   msg);
}

struct PfmImage {
  int width = 0;
  int height = 0;
  std::vector<float> values;  // row-major, top to bottom
};

// read_pfm (src/io.cpp:312-341)
inline PfmImage read_pfm(const std::string& path) {
  char msg[512];
  PfmImage img;
  detail::raise_io(pstereo_read_pfm(path.c_str(), &img.width, &img.height, nullptr, 0, msg,
                                    sizeof msg),
                   msg);
  img.values.resize(std::size_t(img.width) * img.height);
  detail::raise_io(pstereo_read_pfm(path.c_str(), &img.width, &img.height, img.values.data(),
                                    img.values.size(), msg, sizeof msg),
                   msg);
  return img;
}

inline pstereo_metrics_row to_row(const FrameMetrics& m) {
  pstereo_metrics_row r{};
  std::snprintf(r.frame, sizeof r.frame, "%s", m.frame.c_str());
  r.mean_err = m.mean_err;
  r.median_err = m.median_err;
  r.valid_px = m.valid_px;
  r.runtime_ms = m.runtime_ms;
  r.coverage_rate = m.coverage_rate;
  r.has_errors = m.has_errors ? 1 : 0;
  return r;
}

// metrics CSV (src/io.cpp:346-439)
inline std::string metrics_csv_header() { return pstereo_metrics_csv_header(); }
inline std::string format_metrics_row(const FrameMetrics& m) {
  const pstereo_metrics_row r = to_row(m);
  char buf[1024];
  if (pstereo_format_metrics_row(&r, buf, sizeof buf) < 0) throw GpuError("metrics row too long");
  return buf;
}
inline void write_metrics_csv(const std::vector<FrameMetrics>& rows, const std::string& path) {
  std::vector<pstereo_metrics_row> r;
  for (const FrameMetrics& m : rows) r.push_back(to_row(m));
  char msg[512];
  detail::raise_io(
      pstereo_write_metrics_csv(path.c_str(), r.data(), int(r.size()), msg, sizeof msg), msg);
}
inline std::vector<FrameMetrics> read_metrics_csv(const std::string& path) {
  char msg[512];
  int n = 0;
  detail::raise_io(pstereo_read_metrics_csv(path.c_str(), nullptr, 0, &n, msg, sizeof msg), msg);
  std::vector<pstereo_metrics_row> r(static_cast<std::size_t>(n > 0 ? n : 1));
  detail::raise_io(pstereo_read_metrics_csv(path.c_str(), r.data(), n, &n, msg, sizeof msg), msg);
  std::vector<FrameMetrics> out;
  for (int i = 0; i < n; ++i) {
    FrameMetrics m;
    m.frame = r[i].frame;
    m.mean_err = r[i].mean_err;
    m.median_err = r[i].median_err;
    m.valid_px = r[i].valid_px;
    m.runtime_ms = r[i].runtime_ms;
    m.coverage_rate = r[i].coverage_rate;
    m.has_errors = r[i].has_errors != 0;
    out.push_back(m);
  }
  return out;
}

// SceneSpec (inc/pstereo/synth.hpp:20-50) is the C POD; load_scene_spec
// (src/synth.cpp:301-393)
using SceneSpec = pstereo_scene_spec;
inline SceneSpec default_scene() {
  SceneSpec s;
  pstereo_scene_default(&s);
  return s;
}
inline SceneSpec load_scene_spec(const std::string& path) {
  char msg[512];
  SceneSpec s;
  detail::raise_io(pstereo_load_scene_spec(path.c_str(), &s, msg, sizeof msg), msg);
  return s;
}

struct RenderedScene {
  GrayImage left;
  GrayImage right;
  ScalarField ref_disparity;
  ScalarField ref_depth;
  CameraParams cam;
  SceneSpec spec;
};

// render_scene (src/synth.cpp:209-284) on the device; host results
inline RenderedScene render_scene(const SceneSpec& spec, int device = 0) {
  const int w = spec.width, h = spec.height;
  const std::size_t px = std::size_t(w) * h;
  RenderedScene out;
  out.spec = spec;
  out.cam = CameraParams{spec.focal_px, spec.baseline};
  out.left = GrayImage{w, h, std::vector<float>(px), std::vector<std::uint8_t>(px, 1)};
  out.right = GrayImage{w, h, std::vector<float>(px), std::vector<std::uint8_t>(px, 1)};
  out.ref_disparity = ScalarField::sized(w, h);
  out.ref_depth = ScalarField::sized(w, h);
  std::fill(out.ref_disparity.valid.begin(), out.ref_disparity.valid.end(), 1);
  std::fill(out.ref_depth.valid.begin(), out.ref_depth.valid.end(), 1);
  const int rc = pstereo_render_host(device, &spec, 1, out.left.data.data(),
                                     out.right.data.data(), out.ref_disparity.values.data(),
                                     out.ref_depth.values.data());
  if (rc) detail::raise(rc, pstereo_render_last_error());
  return out;
}

struct BenchResult {
  std::vector<FrameMetrics> frames;
  FrameMetrics aggregate;  // arithmetic means across frames, frame = "average"
};

// run_benchmark (src/bench.cpp:11-67): render, run_pipeline `repetitions`
// times (mean runtime), depth-error metrics against the scene's reference
inline BenchResult run_benchmark(const std::vector<SceneSpec>& scenes, const PipelineConfig& cfg,
                                 int repetitions) {
  if (repetitions < 1) throw ConfigError("benchmark repetitions must be >= 1");
  if (scenes.empty()) throw ConfigError("benchmark needs at least one scene");
  BenchResult result;
  for (const SceneSpec& spec : scenes) {
    const RenderedScene scene = render_scene(spec);
    double total_ms = 0.0;
    PipelineOutput output;
    for (int rep = 0; rep < repetitions; ++rep) {
      output = run_pipeline(scene.left, scene.right, cfg, scene.cam);
      total_ms += output.runtime_ms;
    }
    result.frames.push_back(compute_metrics(output.depth.depth, scene.ref_depth,
                                            output.depth.has_sigma ? &output.depth.sigma : nullptr,
                                            total_ms / repetitions, spec.name));
  }
  FrameMetrics agg;
  agg.frame = "average";
  double mean_sum = 0.0, median_sum = 0.0, cover_sum = 0.0, px_sum = 0.0, ms_sum = 0.0;
  std::size_t err_n = 0, cover_n = 0;
  for (const FrameMetrics& m : result.frames) {
    if (m.has_errors) {
      mean_sum += m.mean_err;
      median_sum += m.median_err;
      ++err_n;
    }
    if (!std::isnan(m.coverage_rate)) {
      cover_sum += m.coverage_rate;
      ++cover_n;
    }
    px_sum += double(m.valid_px);
    ms_sum += m.runtime_ms;
  }
  if (err_n > 0) {
    agg.mean_err = mean_sum / double(err_n);
    agg.median_err = median_sum / double(err_n);
    agg.has_errors = true;
  }
  if (cover_n > 0) agg.coverage_rate = cover_sum / double(cover_n);
  agg.valid_px = (long long)(std::size_t(px_sum / double(result.frames.size()) + 0.5));
  agg.runtime_ms = ms_sum / double(result.frames.size());
  result.aggregate = agg;
  return result;
}

}  // namespace gpu

#ifdef PSTEREO_GPU_AS_DEFAULT
using namespace gpu;
#endif

}  // namespace pstereo
