// ref_glue.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Implements oracle/bdis_oracle.h by calling the UNMODIFIED reference
// library (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libbdis_ref.so). Nothing here re-implements the algorithm:
// every entry point marshals plain C buffers into the reference's own types
// (GrayImage, PipelineConfig, WindowSamples, ScalarField, ...) and calls the
// reference function named in its comment. Exceptions map to the exit-code
// convention of src/runner.cpp:107-124 (ConfigError 2, DegenerateInput 4,
// anything else 1).

#include <cstring>
#include <exception>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "bdis_oracle.h"
#include "pstereo/coarse_to_fine.hpp"
#include "pstereo/config.hpp"
#include "pstereo/depth_variance.hpp"
#include "pstereo/errors.hpp"
#include "pstereo/fast_exp.hpp"
#include "pstereo/image.hpp"
#include "pstereo/lk_solver.hpp"
#include "pstereo/patch.hpp"
#include "pstereo/pipeline.hpp"
#include "pstereo/metrics.hpp"
#include "pstereo/pyramid.hpp"
#include "pstereo/spatial_mask.hpp"
#include "pstereo/synth.hpp"
#include "pstereo/kv.hpp"
#include "pstereo/window_posterior.hpp"

using namespace pstereo;

namespace {

PipelineConfig to_cfg(const bo_config* c) {
  PipelineConfig cfg;
  cfg.coarsest_exp = c->coarsest_exp;
  cfg.finest_exp = c->finest_exp;
  cfg.patch_size = c->patch_size;
  cfg.overlap = c->overlap;
  cfg.min_iterations = c->min_iterations;
  cfg.max_iterations = c->max_iterations;
  cfg.early_stop_good = c->early_stop_good;
  cfg.early_stop_bad = c->early_stop_bad;
  cfg.early_stop_improve = c->early_stop_improve;
  cfg.window_offsets.assign(c->window_offsets,
                            c->window_offsets + c->n_window_offsets);
  cfg.sigma_s = c->sigma_s;
  cfg.pixel_threshold = c->pixel_threshold;
  cfg.gamma = c->gamma;
  cfg.valid_patch_ratio = c->valid_patch_ratio;
  cfg.estimate_variance = c->estimate_variance != 0;
  cfg.threads = c->threads;
  return cfg;
}

GrayImage to_gray(const bo_image* img) {
  GrayImage g = make_gray(img->width, img->height);
  const std::size_t n = std::size_t(img->width) * img->height;
  std::memcpy(g.data.data(), img->data, n * sizeof(float));
  if (img->valid) std::memcpy(g.valid.data(), img->valid, n);
  return g;
}

std::vector<float> grad_vec(const bo_image* img, const float* grad) {
  return std::vector<float>(grad, grad + std::size_t(img->width) * img->height);
}

void put_msg(char* msg, int cap, const char* what) {
  if (!msg || cap <= 0) return;
  std::strncpy(msg, what, std::size_t(cap) - 1);
  msg[cap - 1] = 0;
}

template <typename Fn>
int guarded(char* msg, int cap, Fn&& fn) {
  try {
    fn();
    return BO_OK;
  } catch (const ConfigError& e) {
    put_msg(msg, cap, e.what());
    return BO_ECONFIG;
  } catch (const DegenerateInputError& e) {
    put_msg(msg, cap, e.what());
    return BO_EDEGENERATE;
  } catch (const std::exception& e) {
    put_msg(msg, cap, e.what());
    return BO_EINTERNAL;
  }
}

std::optional<PatchSystem> system_of(const bo_image* left, const float* grad,
                                     double cx, double cy, int size) {
  const GrayImage l = to_gray(left);
  auto patch = extract_patch(l, cx, cy, size);  // src/patch.cpp:5-38
  if (!patch) return std::nullopt;
  return precompute_patch_system(std::move(*patch), grad_vec(left, grad),
                                 left->width, left->height, 0);  // src/lk_solver.cpp:7-36
}

void fill_info(const PatchSystem& sys, bo_patch_info* info) {
  if (!info) return;
  info->mean = sys.patch.mean;
  info->valid_fraction = sys.patch.valid_fraction;
  info->valid_count = sys.patch.valid_count;
  info->hessian = sys.hessian;
  info->template_msq = sys.template_msq;
  info->degenerate = sys.degenerate ? 1 : 0;
}

void copy_field(const ScalarField& f, double* v, uint8_t* ok) {
  if (v) std::memcpy(v, f.values.data(), f.values.size() * sizeof(double));
  if (ok) std::memcpy(ok, f.valid.data(), f.valid.size());
}

void copy_stats(const MatchStats& s, int* out, int* n_levels) {
  *n_levels = int(s.levels.size());
  if (!out) return;
  for (std::size_t i = 0; i < s.levels.size(); ++i) {
    out[5 * i + 0] = s.levels[i].exp;
    out[5 * i + 1] = s.levels[i].grid_patches;
    out[5 * i + 2] = s.levels[i].extracted;
    out[5 * i + 3] = s.levels[i].converged;
    out[5 * i + 4] = s.levels[i].accepted;
  }
}

WindowSamples window_of(int n, const double* offsets, const double* residuals,
                        const uint8_t* valid, int center) {
  WindowSamples w;
  if (offsets) w.offsets.assign(offsets, offsets + n);
  else w.offsets.assign(std::size_t(n), 0.0);
  if (residuals) w.residuals.assign(residuals, residuals + n);
  else w.residuals.assign(std::size_t(n), 0.0);
  w.valid.assign(valid, valid + n);
  w.center_index = center;
  return w;
}

}  // namespace

extern "C" {

void bo_default_config(bo_config* c) {
  const PipelineConfig d;  // inc/config.hpp:12-33 defaults
  c->coarsest_exp = d.coarsest_exp;
  c->finest_exp = d.finest_exp;
  c->patch_size = d.patch_size;
  c->overlap = d.overlap;
  c->min_iterations = d.min_iterations;
  c->max_iterations = d.max_iterations;
  c->early_stop_good = d.early_stop_good;
  c->early_stop_bad = d.early_stop_bad;
  c->early_stop_improve = d.early_stop_improve;
  c->n_window_offsets = int(d.window_offsets.size());
  for (std::size_t i = 0; i < d.window_offsets.size(); ++i)
    c->window_offsets[i] = d.window_offsets[i];
  c->sigma_s = d.sigma_s;
  c->pixel_threshold = d.pixel_threshold;
  c->gamma = d.gamma;
  c->valid_patch_ratio = d.valid_patch_ratio;
  c->estimate_variance = d.estimate_variance ? 1 : 0;
  c->threads = d.threads;
}

int bo_validate(const bo_config* c, char* msg, int cap) {
  return guarded(msg, cap, [&] { validate(to_cfg(c)); });  // src/coarse_to_fine.cpp:18-49
}

double bo_fast_exp(double x) { return fast_exp(x); }  // inc/fast_exp.hpp:16-28

void bo_spatial_mask(int size, double sigma_s, double* out) {
  const SpatialMask m = build_spatial_mask(size, sigma_s);  // src/spatial_mask.cpp:7-23
  std::memcpy(out, m.weights.data(), m.weights.size() * sizeof(double));
}

void bo_to_grayscale(int w, int h, int channels, const uint8_t* px, float* out,
                     uint8_t* valid) {
  Raster r;
  r.width = w;
  r.height = h;
  r.channels = channels;
  r.pixels.assign(px, px + std::size_t(w) * h * channels);
  const GrayImage g = to_grayscale(r);  // src/image.cpp:16-43
  std::memcpy(out, g.data.data(), g.data.size() * sizeof(float));
  std::memcpy(valid, g.valid.data(), g.valid.size());
}

int bo_sample_bilinear(const bo_image* img, double x, double y, double* value) {
  const GrayImage g = to_gray(img);
  const BilinearSample s = sample_bilinear(g, x, y);  // inc/image.hpp:53-71
  *value = s.value;
  return s.valid ? 1 : 0;
}

void bo_downsample_half(int w, int h, const float* data, const uint8_t* valid,
                        float* out, uint8_t* out_valid) {
  const bo_image im{w, h, data, valid};
  const GrayImage d = downsample_half(to_gray(&im));  // src/pyramid.cpp:9-28
  std::memcpy(out, d.data.data(), d.data.size() * sizeof(float));
  std::memcpy(out_valid, d.valid.data(), d.valid.size());
}

void bo_gradient_x(int w, int h, const float* data, float* out) {
  const bo_image im{w, h, data, nullptr};
  const std::vector<float> g = gradient_x(to_gray(&im));  // src/pyramid.cpp:30-42
  std::memcpy(out, g.data(), g.size() * sizeof(float));
}

int bo_extract_patch(const bo_image* img, double cx, double cy, int size,
                     double* values, uint8_t* valid, bo_patch_info* info) {
  const auto p = extract_patch(to_gray(img), cx, cy, size);  // src/patch.cpp:5-38
  if (!p) return 0;
  if (values) std::memcpy(values, p->values.data(), p->values.size() * sizeof(double));
  if (valid) std::memcpy(valid, p->valid.data(), p->valid.size());
  if (info) {
    info->mean = p->mean;
    info->valid_fraction = p->valid_fraction;
    info->valid_count = p->valid_count;
  }
  return 1;
}

int bo_patch_system(const bo_image* left, const float* grad, double cx,
                    double cy, int size, double* jacobian, bo_patch_info* info) {
  const auto sys = system_of(left, grad, cx, cy, size);
  if (!sys) return 0;
  if (jacobian)
    std::memcpy(jacobian, sys->jacobian.data(), sys->jacobian.size() * sizeof(double));
  fill_info(*sys, info);
  return 1;
}

int bo_eval_residual(const bo_image* left, const float* grad,
                     const bo_image* right, double cx, double cy, int size,
                     double u, double* msq, double* jr, int* n) {
  const auto sys = system_of(left, grad, cx, cy, size);
  if (!sys) return 0;
  LkScratch scratch;
  const ResidualEval ev = eval_patch_residual(*sys, to_gray(right), u, scratch);  // src/lk_solver.cpp:38-81
  *msq = ev.msq;
  *jr = ev.jr;
  *n = ev.n;
  return 1;
}

int bo_solve_patch(const bo_image* left, const float* grad,
                   const bo_image* right, double cx, double cy, int size,
                   double u_init, const bo_lk_params* p, double* u,
                   int* converged, int* iterations, double* final_residual) {
  const auto sys = system_of(left, grad, cx, cy, size);
  if (!sys) return 0;
  LkParams lp;
  lp.min_iterations = p->min_iterations;
  lp.max_iterations = p->max_iterations;
  lp.update_epsilon = p->update_epsilon;
  lp.stop_good = p->stop_good;
  lp.stop_bad = p->stop_bad;
  lp.stop_improve = p->stop_improve;
  LkScratch scratch;
  const LkResult r = solve_patch_disparity(*sys, to_gray(right), u_init, lp, scratch);  // src/lk_solver.cpp:83-132
  *u = r.u;
  *converged = r.converged ? 1 : 0;
  *iterations = r.iterations;
  *final_residual = r.final_residual;
  return 1;
}

int bo_sample_window(const bo_image* left, const float* grad,
                     const bo_image* right, double cx, double cy, int size,
                     double u_k, int n_mags, const double* mags,
                     double* offsets, double* residuals, uint8_t* valid,
                     int* center_index) {
  const auto sys = system_of(left, grad, cx, cy, size);
  if (!sys) return -1;
  LkScratch scratch;
  const std::vector<double> m(mags, mags + n_mags);
  const auto w = sample_window(*sys, to_gray(right), u_k, m, scratch);  // src/window_posterior.cpp:10-40
  if (!w) return 0;
  std::memcpy(offsets, w->offsets.data(), w->offsets.size() * sizeof(double));
  std::memcpy(residuals, w->residuals.data(), w->residuals.size() * sizeof(double));
  std::memcpy(valid, w->valid.data(), w->valid.size());
  *center_index = w->center_index;
  return 1;
}

double bo_dynamic_sigma(int n, const double* residuals, const uint8_t* valid,
                        double sigma_floor) {
  return dynamic_sigma(window_of(n, nullptr, residuals, valid, n / 2),
                       sigma_floor);  // src/window_posterior.cpp:42-59
}

void bo_window_priors(int n, const double* residuals, const uint8_t* valid,
                      double sigma_r, int patch_size, int use_fast_exp,
                      double* priors) {
  const auto p = window_priors(window_of(n, nullptr, residuals, valid, n / 2),
                               sigma_r, patch_size, use_fast_exp != 0);  // src/window_posterior.cpp:61-72
  std::memcpy(priors, p.data(), p.size() * sizeof(double));
}

int bo_patch_posterior(int n, const double* residuals, const uint8_t* valid,
                       int center_index, double sigma_r, int patch_size,
                       int use_fast_exp, double* probability, int* is_min) {
  const auto post =
      patch_posterior(window_of(n, nullptr, residuals, valid, center_index),
                      sigma_r, patch_size, use_fast_exp != 0);  // src/window_posterior.cpp:74-96
  if (!post) return 0;
  *probability = post->probability;
  *is_min = post->is_local_minimum ? 1 : 0;
  return 1;
}

void bo_estimate_variance(int n, const double* offsets, const uint8_t* valid,
                          int center_index, const double* priors,
                          double sigma_fallback, double* sigma_k, double* c_k,
                          int* accepted, int* reason, double* fit_residual) {
  const WindowSamples w = window_of(n, offsets, nullptr, valid, center_index);
  const PatchVariance pv = estimate_patch_variance(
      w, std::span<const double>(priors, std::size_t(n)), sigma_fallback);  // src/depth_variance.cpp:94-170
  *sigma_k = pv.sigma_k;
  *c_k = pv.c_k;
  *accepted = pv.accepted ? 1 : 0;
  *reason = int(pv.reason);
  *fit_residual = pv.fit_residual;
}

int bo_make_patch_grid(int w, int h, int patch_size, double overlap,
                       int* stride, int* nx, int* ny, double* xs, double* ys,
                       int cap) {
  int rc = BO_OK;
  rc = guarded(nullptr, 0, [&] {
    const PatchGrid g = make_patch_grid(w, h, 0, patch_size, overlap);  // src/coarse_to_fine.cpp:51-88
    *stride = g.stride;
    *nx = int(g.xs.size());
    *ny = int(g.ys.size());
    for (int i = 0; i < *nx && i < cap; ++i) xs[i] = g.xs[std::size_t(i)];
    for (int i = 0; i < *ny && i < cap; ++i) ys[i] = g.ys[std::size_t(i)];
  });
  return rc;
}

double bo_level_weight(int n, int n_levels, const int* levels) {
  return level_weight(n, std::span<const int>(levels, std::size_t(n_levels)));  // src/coarse_to_fine.cpp:90-94
}

double bo_propagate_probability(double posterior, double inherited, int n,
                                int n_levels, const int* levels) {
  return propagate_probability(posterior, inherited, n,
                               std::span<const int>(levels, std::size_t(n_levels)));  // :96-99
}

void bo_fuse_level(int n_patches, const double* cx, const double* cy,
                   const double* u, const double* prob, const double* sigma_k,
                   int size, double sigma_s, int w, int h, int with_variance,
                   double* disp, uint8_t* disp_valid, double* prob_out,
                   uint8_t* prob_valid, double* var, uint8_t* var_valid) {
  std::vector<PatchEstimate> pes(static_cast<std::size_t>(n_patches));
  for (int i = 0; i < n_patches; ++i) {
    pes[std::size_t(i)].cx = cx[i];
    pes[std::size_t(i)].cy = cy[i];
    pes[std::size_t(i)].u = u[i];
    pes[std::size_t(i)].prob = prob[i];
    pes[std::size_t(i)].posterior = prob[i];
    pes[std::size_t(i)].sigma_k = sigma_k ? sigma_k[i] : 0.0;
    pes[std::size_t(i)].has_sigma = sigma_k != nullptr;
  }
  const SpatialMask mask = build_spatial_mask(size, sigma_s);
  const LevelEstimate est =
      fuse_level(std::move(pes), mask, w, h, 1, with_variance != 0);  // src/coarse_to_fine.cpp:101-150
  copy_field(est.disparity, disp, disp_valid);
  copy_field(est.probability, prob_out, prob_valid);
  if (with_variance) copy_field(est.var_disp, var, var_valid);
}

void bo_init_next_level(int cw, int ch, const double* values,
                        const uint8_t* valid, int fw, int fh, double* out) {
  ScalarField c = ScalarField::sized(cw, ch);
  std::memcpy(c.values.data(), values, c.values.size() * sizeof(double));
  std::memcpy(c.valid.data(), valid, c.valid.size());
  const ScalarField f = init_next_level(c, fw, fh);  // src/coarse_to_fine.cpp:152-164
  std::memcpy(out, f.values.data(), f.values.size() * sizeof(double));
}

void bo_upsample_to_full(int w, int h, const double* values,
                         const uint8_t* valid, int fw, int fh, int exp,
                         double scale_per_level, double* out,
                         uint8_t* out_valid) {
  ScalarField c = ScalarField::sized(w, h);
  std::memcpy(c.values.data(), values, c.values.size() * sizeof(double));
  std::memcpy(c.valid.data(), valid, c.valid.size());
  const ScalarField f = upsample_to_full(c, fw, fh, exp, scale_per_level);  // :166-180
  copy_field(f, out, out_valid);
}

void bo_remove_small_components(const uint8_t* valid, int w, int h,
                                long long min_px, uint8_t* out) {
  const std::vector<uint8_t> v(valid, valid + std::size_t(w) * h);
  const auto r = remove_small_components(v, w, h, min_px);  // src/depth_variance.cpp:43-76
  std::memcpy(out, r.data(), r.size());
}

void bo_filter_validity(int w, int h, const uint8_t* disp_valid,
                        const double* prob, const uint8_t* prob_valid,
                        double gamma, double pixel_threshold, int patch_size,
                        uint8_t* out_valid) {
  ScalarField d = ScalarField::sized(w, h);
  std::memcpy(d.valid.data(), disp_valid, d.valid.size());
  ScalarField p = ScalarField::sized(w, h);
  std::memcpy(p.values.data(), prob, p.values.size() * sizeof(double));
  std::memcpy(p.valid.data(), prob_valid, p.valid.size());
  const ScalarField f = filter_validity(d, p, gamma, pixel_threshold, patch_size);  // :78-92
  std::memcpy(out_valid, f.valid.data(), f.valid.size());
}

void bo_disparity_to_depth(int w, int h, const double* disp,
                           const uint8_t* disp_valid, const double* var,
                           const uint8_t* var_valid, double focal_px,
                           double baseline, double min_disparity,
                           double* depth, uint8_t* depth_valid, double* sigma,
                           uint8_t* sigma_valid) {
  ScalarField d = ScalarField::sized(w, h);
  std::memcpy(d.values.data(), disp, d.values.size() * sizeof(double));
  std::memcpy(d.valid.data(), disp_valid, d.valid.size());
  const CameraParams cam{focal_px, baseline};
  if (var) {
    ScalarField v = ScalarField::sized(w, h);
    std::memcpy(v.values.data(), var, v.values.size() * sizeof(double));
    std::memcpy(v.valid.data(), var_valid, v.valid.size());
    const DepthResult r = disparity_to_depth(d, v, cam, min_disparity);  // :25-41
    copy_field(r.depth, depth, depth_valid);
    copy_field(r.sigma, sigma, sigma_valid);
  } else {
    const DepthResult r = disparity_to_depth(d, cam, min_disparity);  // :9-23
    copy_field(r.depth, depth, depth_valid);
  }
}

int bo_match_stereo(const bo_image* left, const bo_image* right,
                    const bo_config* cfg, bo_match_outputs* out, char* msg,
                    int cap) {
  return guarded(msg, cap, [&] {
    const MatchResult m = match_stereo(to_gray(left), to_gray(right), to_cfg(cfg));  // src/coarse_to_fine.cpp:211-341
    copy_field(m.disparity, out->disparity, out->disparity_valid);
    copy_field(m.probability, out->probability, out->probability_valid);
    out->has_variance = m.has_variance ? 1 : 0;
    if (m.has_variance) copy_field(m.var_disp, out->var_disp, out->var_valid);
    copy_stats(m.stats, out->stats, &out->n_levels);
    out->finest_count = int(m.finest.patches.size());
    if (out->finest) {
      for (int i = 0; i < out->finest_count && i < out->finest_cap; ++i) {
        const PatchEstimate& p = m.finest.patches[std::size_t(i)];
        double* row = out->finest + 7 * i;
        row[0] = p.cx;
        row[1] = p.cy;
        row[2] = p.u;
        row[3] = p.prob;
        row[4] = p.posterior;
        row[5] = p.sigma_k;
        row[6] = p.has_sigma ? 1.0 : 0.0;
      }
    }
  });
}

int bo_run_pipeline(const bo_image* left, const bo_image* right,
                    const bo_config* cfg, double focal_px, double baseline,
                    bo_outputs* out, char* msg, int cap) {
  const GrayImage l = to_gray(left);
  const GrayImage r = to_gray(right);
  const PipelineConfig c = to_cfg(cfg);
  return guarded(msg, cap, [&] {
    const PipelineOutput o = run_pipeline(l, r, c, CameraParams{focal_px, baseline});  // src/pipeline.cpp:9-37
    copy_field(o.disparity, out->disparity, out->disparity_valid);
    copy_field(o.probability, out->probability, out->probability_valid);
    copy_field(o.depth.depth, out->depth, out->depth_valid);
    out->has_sigma = o.depth.has_sigma ? 1 : 0;
    if (o.depth.has_sigma) copy_field(o.depth.sigma, out->depth_sigma, out->sigma_valid);
    copy_stats(o.stats, out->stats, &out->n_levels);
    out->runtime_ms = o.runtime_ms;
  });
}

void bo_compute_metrics(int w, int h, const double* est, const uint8_t* est_valid,
                        const double* ref, const uint8_t* ref_valid, const double* sigma,
                        const uint8_t* sigma_valid, bo_frame_metrics* out) {
  auto field = [&](const double* v, const uint8_t* ok) {
    ScalarField f = ScalarField::sized(w, h);
    std::memcpy(f.values.data(), v, f.values.size() * sizeof(double));
    std::memcpy(f.valid.data(), ok, f.valid.size());
    return f;
  };
  const ScalarField e = field(est, est_valid), r = field(ref, ref_valid);
  ScalarField sg;
  if (sigma) sg = field(sigma, sigma_valid);
  const FrameMetrics m = compute_metrics(e, r, sigma ? &sg : nullptr, 0.0, "");  // src/metrics.cpp:10-52
  out->valid_px = m.valid_px;
  long long compared = 0;
  for (std::size_t i = 0; i < e.valid.size(); ++i) compared += (e.valid[i] && r.valid[i]) ? 1 : 0;
  out->compared = compared;
  out->has_errors = m.has_errors ? 1 : 0;
  out->mean_err = m.mean_err;
  out->median_err = m.median_err;
  out->coverage_rate = m.coverage_rate;
}


// ---- analytic scene renderer (src/synth.cpp) ----

static SceneSpec to_scene(const bo_scene* b) {
  SceneSpec s;
  s.name = b->name;
  s.surface = b->surface == 1 ? SurfaceKind::slanted_plane
              : b->surface == 2 ? SurfaceKind::sphere : SurfaceKind::plane;
  s.disparity = b->disparity;
  s.disparity0 = b->disparity0;
  s.disparity_gradient = b->disparity_gradient;
  s.sphere_depth = b->sphere_depth;
  s.sphere_radius = b->sphere_radius;
  s.background_depth = b->background_depth;
  s.texture = b->texture == 1 ? TextureKind::checker
              : b->texture == 2 ? TextureKind::constant : TextureKind::perlin;
  s.texture_scale = b->texture_scale;
  s.texture_octaves = b->texture_octaves;
  s.shading = b->shading == 1 ? ShadingKind::nonlambertian : ShadingKind::diffuse;
  s.ambient = b->ambient;
  s.highlight_strength = b->highlight_strength;
  s.highlight_falloff = b->highlight_falloff;
  s.noise_std = b->noise_std;
  s.seed = b->seed;
  s.seed_explicit = b->seed_explicit != 0;
  s.focal_px = b->focal_px;
  s.baseline = b->baseline;
  s.width = b->width;
  s.height = b->height;
  return s;
}

double bo_scene_disparity_at(const bo_scene* s, double x, double y) {
  return scene_disparity_at(to_scene(s), x, y);  // src/synth.cpp:131-133
}

double bo_scene_intensity_at(const bo_scene* s, double x, double y) {
  return scene_intensity_at(to_scene(s), x, y);  // src/synth.cpp:192-207
}

double bo_value_noise(double x, double y, uint64_t seed, int octaves, double base_scale) {
  return value_noise(x, y, seed, octaves, base_scale);  // src/synth.cpp:43-72
}

double bo_gaussian_noise(uint64_t seed, uint64_t stream, uint64_t index) {
  return gaussian_noise(seed, stream, index);  // src/synth.cpp:33-41
}

int bo_render_scene(const bo_scene* b, float* left, float* right, double* ref_disparity,
                    double* ref_depth) {
  const RenderedScene r = render_scene(to_scene(b));  // src/synth.cpp:209-284
  std::memcpy(left, r.left.data.data(), r.left.data.size() * sizeof(float));
  std::memcpy(right, r.right.data.data(), r.right.data.size() * sizeof(float));
  std::memcpy(ref_disparity, r.ref_disparity.values.data(),
              r.ref_disparity.values.size() * sizeof(double));
  std::memcpy(ref_depth, r.ref_depth.values.data(), r.ref_depth.values.size() * sizeof(double));
  return 0;
}

}  // extern "C"

// synth.cpp links against the kv parser of io.cpp (libpng, not built here);
// the oracle never parses scene files through the reference, so these are
// link-time stubs only.
namespace pstereo {
const std::string* KvFile::find(const std::string&) const { return nullptr; }
KvFile load_kv_file(const std::string& path) { throw ConfigError(path + ": kv parser not built"); }
double kv_double_or(const KvFile&, const std::string&, double f) { return f; }
long long kv_int_or(const KvFile&, const std::string&, long long f) { return f; }
std::string kv_string_or(const KvFile&, const std::string&, const std::string& f) { return f; }
}  // namespace pstereo
