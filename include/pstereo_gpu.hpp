// pstereo_gpu.hpp -- the library's C++ API beyond the reference's own
// headers. Header-only over the C ABI (include/pstereo_gpu.h); link
// libpstereo_gpu.so.
//
// The drop-in for the reference's matching core is the header tree
// include/pstereo/ (config, errors, fields, image, coarse_to_fine,
// depth_variance, pipeline .hpp): same file names, namespace, types and
// signatures as proj/include/pstereo/, so a reference caller switches by
// putting include/ ahead of the reference's include directory and linking
// libpstereo_gpu.so instead of the matcher's sources.
//
// This header adds, in namespace pstereo::gpu:
//   run_pipeline_batch             batched run_pipeline (include/pstereo/pipeline.hpp)
//   set_device / device / clear_contexts  (include/pstereo/gpu_runtime.hpp)
//   FrameMetrics, compute_metrics  inc/metrics.hpp:14-32, src/metrics.cpp:10-52 (device)
//   load_image, load_calibration, write_pfm, read_pfm, metrics CSV
//                                  proj/include/pstereo/io.hpp, src/io.cpp
//   SceneSpec, load_scene_spec, RenderedScene, render_scene (device)
//                                  proj/include/pstereo/synth.hpp, src/synth.cpp
//   BenchResult, run_benchmark     proj/include/pstereo/bench.hpp, src/bench.cpp
// and aliases the boundary types (pstereo::gpu::GrayImage = pstereo::GrayImage,
// ...). Results are bit-identical to the reference (var_disp / depth sigma
// within 1e-3 relative); see DESIGN.md.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <limits>
#include <string>
#include <vector>

#include "pstereo/pipeline.hpp"
#include "pstereo_gpu.h"

namespace pstereo {
namespace gpu {

using pstereo::CameraParams;
using pstereo::ConfigError;
using pstereo::DegenerateInputError;
using pstereo::DepthResult;
using pstereo::GrayImage;
using pstereo::IoError;
using pstereo::IoErrorKind;
using pstereo::LevelEstimate;
using pstereo::MatchResult;
using pstereo::MatchStats;
using pstereo::PatchEstimate;
using pstereo::PipelineConfig;
using pstereo::PipelineOutput;
using pstereo::Raster;
using pstereo::ScalarField;
using pstereo::match_stereo;
using pstereo::run_pipeline;
using pstereo::validate;

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

namespace detail {
inline void raise_io(int rc, const char* msg) {
  if (rc) raise(rc, msg);  // PSTEREO_EIO -> IoError with its kind
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
inline RenderedScene render_scene(const SceneSpec& spec, int dev = -1) {
  if (dev < 0) dev = device();
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
  const int rc = pstereo_render_host(dev, &spec, 1, out.left.data.data(),
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
}  // namespace pstereo
