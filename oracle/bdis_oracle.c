/*
 * bdis_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU checker for the GPU
 * product, never shipped and never on the product path.
 *
 * A plain-C restatement of the reference's per-frame BDIS path
 * (run_pipeline, src/pipeline.cpp:9-37). Every function cites the reference
 * file:line it restates. Arithmetic is IEEE double / float with no FMA
 * contraction (built with -ffp-contract=off), sums run in the reference's
 * sequential order, and rounding uses the same primitives (lround = half away
 * from zero, lrint = ties-to-even, C casts truncate), so results are meant to
 * be bit-identical to the reference build. That claim is pinned by
 * tests/test_oracle_pins.py against oracle/_ref/libbdis_ref.so (the reference
 * itself) and the tests/golden fixtures (fixtures the reference generated).
 *
 * Single-threaded: the reference's cfg.threads only changes scheduling, never
 * results (src/coarse_to_fine.cpp:184-186), so it is validated and ignored.
 */
#include "bdis_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ */
/* small helpers                                                       */

static double clampd(double x, double lo, double hi) {
  /* std::clamp(v, lo, hi): (v < lo) ? lo : (hi < v) ? hi : v */
  return (x < lo) ? lo : ((hi < x) ? hi : x);
}
static int clampi(int x, int lo, int hi) {
  return (x < lo) ? lo : ((hi < x) ? hi : x);
}
static int mini(int a, int b) { return b < a ? b : a; }
static double maxd(double a, double b) { return (a < b) ? b : a; } /* std::max */

static void set_msg(char* msg, int cap, const char* text) {
  if (!msg || cap <= 0) return;
  snprintf(msg, (size_t)cap, "%s", text);
}

/* ------------------------------------------------------------------ */
/* config: inc/config.hpp:12-33, validate src/coarse_to_fine.cpp:18-49 */

void bo_default_config(bo_config* c) {
  memset(c, 0, sizeof *c);
  c->coarsest_exp = 5;
  c->finest_exp = 1;
  c->patch_size = 10;
  c->overlap = 0.55;
  c->min_iterations = 12;
  c->max_iterations = 12;
  c->early_stop_good = 0.05;
  c->early_stop_bad = 0.95;
  c->early_stop_improve = 0.10;
  c->n_window_offsets = 2;
  c->window_offsets[0] = 0.5;
  c->window_offsets[1] = 1.0;
  c->sigma_s = 4.0;
  c->pixel_threshold = 0.15;
  c->gamma = 0.75;
  c->valid_patch_ratio = 0.75;
  c->estimate_variance = 0;
  c->threads = 1;
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x < y) ? -1 : (y < x) ? 1 : 0;
}

int bo_validate(const bo_config* c, char* msg, int cap) {
#define FAIL(text)                       \
  do {                                   \
    set_msg(msg, cap, "config: " text); \
    return BO_ECONFIG;                   \
  } while (0)
  if (c->patch_size < 2) FAIL("patch_size must be >= 2");
  if (c->finest_exp < 0) FAIL("finest_exp must be >= 0");
  if (c->coarsest_exp < c->finest_exp) FAIL("coarsest_exp must be >= finest_exp");
  if (c->coarsest_exp > 16) FAIL("coarsest_exp is unreasonably large");
  if (!(c->overlap >= 0.0 && c->overlap < 1.0)) FAIL("overlap must lie in [0, 1)");
  if (c->min_iterations < 1) FAIL("min_iterations must be >= 1");
  if (c->max_iterations < c->min_iterations)
    FAIL("max_iterations must be >= min_iterations");
  if (!(c->early_stop_good > 0.0)) FAIL("early_stop_good must be > 0");
  if (!(c->early_stop_bad > 0.0)) FAIL("early_stop_bad must be > 0");
  if (!(c->early_stop_improve >= 0.0)) FAIL("early_stop_improve must be >= 0");
  if (c->n_window_offsets <= 0) FAIL("window_offsets must not be empty");
  if (c->n_window_offsets > BO_MAX_OFFSETS) FAIL("too many window offsets");
  for (int i = 0; i < c->n_window_offsets; ++i)
    if (!(c->window_offsets[i] > 0.0)) FAIL("window offsets must be positive magnitudes");
  {
    double s[BO_MAX_OFFSETS];
    memcpy(s, c->window_offsets, sizeof(double) * (size_t)c->n_window_offsets);
    qsort(s, (size_t)c->n_window_offsets, sizeof(double), cmp_double);
    for (int i = 1; i < c->n_window_offsets; ++i)
      if (s[i] == s[i - 1]) FAIL("window offsets must be distinct");
  }
  if (!(c->sigma_s > 0.0)) FAIL("sigma_s must be > 0");
  if (!(c->pixel_threshold >= 0.0 && c->pixel_threshold <= 1.0))
    FAIL("pixel_threshold must lie in [0, 1]");
  if (!(c->gamma >= 0.0)) FAIL("gamma must be >= 0");
  if (!(c->valid_patch_ratio > 0.0 && c->valid_patch_ratio <= 1.0))
    FAIL("valid_patch_ratio must lie in (0, 1]");
  if (c->threads < 1) FAIL("threads must be >= 1");
#undef FAIL
  return BO_OK;
}

/* ------------------------------------------------------------------ */
/* inc/fast_exp.hpp:10-28 (Schraudolph, double layout)                */

double bo_fast_exp(double x) {
  if (x < -30.0) return 0.0;
  const double scale = 4503599627370496.0 / 0.6931471805599453;
  const int64_t bias = ((int64_t)1023 << 52) - ((int64_t)60801 << 32);
  const int64_t bits = (int64_t)(x * scale) + bias;
  double out;
  memcpy(&out, &bits, sizeof out);
  return out;
}

/* src/spatial_mask.cpp:7-23 */
void bo_spatial_mask(int size, double sigma_s, double* out) {
  const double half = (size - 1) * 0.5;
  const double denom = 2.0 * sigma_s * sigma_s;
  for (int j = 0; j < size; ++j) {
    const double dy = j - half;
    for (int i = 0; i < size; ++i) {
      const double dx = i - half;
      out[j * size + i] = bo_fast_exp(-(dx * dx + dy * dy) / denom);
    }
  }
}

/* ------------------------------------------------------------------ */
/* images: src/image.cpp:16-43, inc/image.hpp:53-90, src/pyramid.cpp   */

void bo_to_grayscale(int w, int h, int channels, const uint8_t* px, float* out,
                     uint8_t* valid) {
  const double inv255 = 1.0 / 255.0;
  const size_t n = (size_t)w * (size_t)h;
  for (size_t i = 0; i < n; ++i) {
    const uint8_t* p = px + i * (size_t)channels;
    double v;
    int ok = 1;
    if (channels == 1) {
      v = p[0] * inv255;
    } else {
      if (channels == 4) ok = p[3] != 0;
      v = (0.299 * p[0] + 0.587 * p[1] + 0.114 * p[2]) * inv255;
    }
    out[i] = (float)v;
    valid[i] = (uint8_t)(ok ? 1 : 0);
  }
}

static int in_bounds(const bo_image* img, double x, double y) {
  return x >= 0.0 && x <= img->width - 1.0 && y >= 0.0 && y <= img->height - 1.0;
}

static int img_valid(const bo_image* img, int x, int y) {
  return img->valid ? img->valid[(size_t)y * (size_t)img->width + (size_t)x] != 0 : 1;
}

/* inc/image.hpp:53-71 */
int bo_sample_bilinear(const bo_image* img, double x, double y, double* value) {
  const int inside = in_bounds(img, x, y);
  const double cx = clampd(x, 0.0, (double)(img->width - 1));
  const double cy = clampd(y, 0.0, (double)(img->height - 1));
  const int x0 = (int)cx;
  const int y0 = (int)cy;
  const int x1 = mini(x0 + 1, img->width - 1);
  const int y1 = mini(y0 + 1, img->height - 1);
  const double fx = cx - x0;
  const double fy = cy - y0;
  const float* d = img->data;
  const size_t W = (size_t)img->width;
  const double top = (1.0 - fx) * d[(size_t)y0 * W + x0] + fx * d[(size_t)y0 * W + x1];
  const double bot = (1.0 - fx) * d[(size_t)y1 * W + x0] + fx * d[(size_t)y1 * W + x1];
  *value = (1.0 - fy) * top + fy * bot;
  return inside && img_valid(img, x0, y0) && img_valid(img, x1, y0) &&
         img_valid(img, x0, y1) && img_valid(img, x1, y1);
}

/* inc/image.hpp:75-90 */
static double sample_plane(const float* plane, int width, int height, double x,
                           double y) {
  const double cx = clampd(x, 0.0, (double)(width - 1));
  const double cy = clampd(y, 0.0, (double)(height - 1));
  const int x0 = (int)cx;
  const int y0 = (int)cy;
  const int x1 = mini(x0 + 1, width - 1);
  const int y1 = mini(y0 + 1, height - 1);
  const double fx = cx - x0;
  const double fy = cy - y0;
  const size_t W = (size_t)width;
  const double top = (1.0 - fx) * plane[(size_t)y0 * W + x0] + fx * plane[(size_t)y0 * W + x1];
  const double bot = (1.0 - fx) * plane[(size_t)y1 * W + x0] + fx * plane[(size_t)y1 * W + x1];
  return (1.0 - fy) * top + fy * bot;
}

/* src/pyramid.cpp:9-28 */
void bo_downsample_half(int w, int h, const float* data, const uint8_t* valid,
                        float* out, uint8_t* out_valid) {
  const int ow = (w + 1) / 2;
  const int oh = (h + 1) / 2;
  for (int y = 0; y < oh; ++y) {
    const int y0 = 2 * y;
    const int y1 = mini(2 * y + 1, h - 1);
    for (int x = 0; x < ow; ++x) {
      const int x0 = 2 * x;
      const int x1 = mini(2 * x + 1, w - 1);
      const float a = data[(size_t)y0 * w + x0], b = data[(size_t)y0 * w + x1];
      const float c = data[(size_t)y1 * w + x0], d = data[(size_t)y1 * w + x1];
      out[(size_t)y * ow + x] = 0.25f * (a + b + c + d);
      int ok = 1;
      if (valid)
        ok = valid[(size_t)y0 * w + x0] && valid[(size_t)y0 * w + x1] &&
             valid[(size_t)y1 * w + x0] && valid[(size_t)y1 * w + x1];
      out_valid[(size_t)y * ow + x] = (uint8_t)(ok ? 1 : 0);
    }
  }
}

/* src/pyramid.cpp:30-42 */
void bo_gradient_x(int w, int h, const float* data, float* out) {
  memset(out, 0, sizeof(float) * (size_t)w * (size_t)h);
  if (w < 2) return;
  for (int y = 0; y < h; ++y) {
    const float* r = data + (size_t)y * w;
    float* g = out + (size_t)y * w;
    g[0] = r[1] - r[0];
    for (int x = 1; x < w - 1; ++x) g[x] = 0.5f * (r[x + 1] - r[x - 1]);
    g[w - 1] = r[w - 1] - r[w - 2];
  }
}

/* ------------------------------------------------------------------ */
/* patch system: src/patch.cpp:5-38, src/lk_solver.cpp:7-36            */

typedef struct patch_sys {
  double cx, cy;
  int size;
  double* values;   /* mean removed; 0 where invalid */
  uint8_t* valid;
  double mean, valid_fraction;
  int valid_count;
  double* jacobian;
  double hessian, template_msq;
  int degenerate;
} patch_sys;

static double poff(int size, int i) { return i - (size - 1) * 0.5; } /* inc/patch.hpp:24 */

/* src/patch.cpp:5-38; returns 0 when no sample is valid */
static int extract(const bo_image* img, double cx, double cy, int size, patch_sys* p) {
  p->cx = cx;
  p->cy = cy;
  p->size = size;
  const int n = size * size;
  double sum = 0.0;
  int count = 0;
  for (int j = 0; j < size; ++j) {
    const double y = cy + poff(size, j);
    for (int i = 0; i < size; ++i) {
      double v;
      const int ok = bo_sample_bilinear(img, cx + poff(size, i), y, &v);
      p->values[j * size + i] = v;
      p->valid[j * size + i] = (uint8_t)ok;
      if (ok) {
        sum += v;
        ++count;
      }
    }
  }
  if (count == 0) return 0;
  p->mean = sum / count;
  p->valid_count = count;
  p->valid_fraction = (double)count / (double)n;
  for (int i = 0; i < n; ++i) p->values[i] = p->valid[i] ? p->values[i] - p->mean : 0.0;
  return 1;
}

/* src/lk_solver.cpp:7-36 */
static void precompute(patch_sys* p, const float* grad, int w, int h) {
  const int size = p->size;
  double hess = 0.0, tsq = 0.0;
  for (int k = 0; k < size * size; ++k) p->jacobian[k] = 0.0;
  for (int j = 0; j < size; ++j) {
    const double y = p->cy + poff(size, j);
    for (int i = 0; i < size; ++i) {
      const int idx = j * size + i;
      if (!p->valid[idx]) continue;
      const double g = sample_plane(grad, w, h, p->cx + poff(size, i), y);
      p->jacobian[idx] = g;
      hess += g * g;
      tsq += p->values[idx] * p->values[idx];
    }
  }
  p->hessian = hess;
  p->template_msq = p->valid_count > 0 ? tsq / p->valid_count : 0.0;
  p->degenerate = !(hess >= 1e-8) || !isfinite(hess);
}

typedef struct scratch {
  double* samples;
  uint8_t* ok;
} scratch;

typedef struct resid {
  double msq, jr;
  int n;
} resid;

/* src/lk_solver.cpp:38-81 */
static resid eval_residual(const patch_sys* p, const bo_image* right, double u,
                           scratch* s) {
  const int size = p->size;
  const int n = size * size;
  memset(s->ok, 0, (size_t)n);
  double sum = 0.0;
  int count = 0;
  for (int j = 0; j < size; ++j) {
    const double y = p->cy + poff(size, j);
    for (int i = 0; i < size; ++i) {
      const int idx = j * size + i;
      if (!p->valid[idx]) continue;
      double v;
      if (!bo_sample_bilinear(right, p->cx + poff(size, i) - u, y, &v)) continue;
      s->samples[idx] = v;
      s->ok[idx] = 1;
      sum += v;
      ++count;
    }
  }
  resid ev;
  ev.msq = INFINITY;
  ev.jr = 0.0;
  ev.n = count;
  if (count == 0) return ev;
  const double mean = sum / count;
  double ssr = 0.0, jr = 0.0;
  for (int idx = 0; idx < n; ++idx) {
    if (!s->ok[idx]) continue;
    const double r = (s->samples[idx] - mean) - p->values[idx];
    ssr += r * r;
    jr += p->jacobian[idx] * r;
  }
  ev.msq = ssr / count;
  ev.jr = jr;
  return ev;
}

typedef struct lk_out {
  double u;
  int converged, iterations;
  double final_residual;
} lk_out;

/* src/lk_solver.cpp:83-132 */
static lk_out solve(const patch_sys* p, const bo_image* right, double u_init,
                    const bo_lk_params* prm, scratch* s, int want_final) {
  lk_out res;
  res.u = u_init;
  res.converged = 0;
  res.iterations = 0;
  res.final_residual = INFINITY;
  if (p->degenerate) return res;
  if (!in_bounds(right, p->cx - u_init, p->cy)) return res;
  double u = u_init, prev = INFINITY, last_delta = 0.0;
  int updated = 0, it = 1;
  for (; it <= prm->max_iterations; ++it) {
    const resid ev = eval_residual(p, right, u, s);
    if (ev.n == 0) {
      res.u = u;
      res.iterations = it;
      return res;
    }
    const double r = ev.msq;
    if (it >= prm->min_iterations) {
      if (r < prm->stop_good) {
        res.converged = 1;
        break;
      }
      if (r > prm->stop_bad * p->template_msq) break;
      if (isfinite(prev) && (prev - r) < prm->stop_improve * prev) {
        res.converged = updated && fabs(last_delta) < prm->update_epsilon;
        break;
      }
    }
    const double delta = ev.jr / p->hessian;
    u += delta;
    last_delta = delta;
    updated = 1;
    prev = r;
    if (fabs(delta) < prm->update_epsilon) {
      res.converged = 1;
      break;
    }
  }
  res.iterations = mini(it, prm->max_iterations);
  res.u = u;
  /* final_residual is never read on the pipeline path; computed on demand. */
  if (want_final) res.final_residual = eval_residual(p, right, u, s).msq;
  return res;
}

/* ------------------------------------------------------------------ */
/* window posterior: src/window_posterior.cpp:10-96                     */

typedef struct window {
  int n, center;
  double offsets[2 * BO_MAX_OFFSETS + 1];
  double residuals[2 * BO_MAX_OFFSETS + 1];
  uint8_t valid[2 * BO_MAX_OFFSETS + 1];
} window;

/* offsets: sorted symmetric closure with 0 (src/window_posterior.cpp:13-22) */
static void window_offsets(int n_mags, const double* mags, window* w) {
  double m[BO_MAX_OFFSETS];
  memcpy(m, mags, sizeof(double) * (size_t)n_mags);
  qsort(m, (size_t)n_mags, sizeof(double), cmp_double);
  int k = 0;
  for (int i = n_mags - 1; i >= 0; --i) w->offsets[k++] = -m[i];
  w->center = k;
  w->offsets[k++] = 0.0;
  for (int i = 0; i < n_mags; ++i) w->offsets[k++] = m[i];
  w->n = k;
}

/* src/window_posterior.cpp:10-40; returns 0 when the window is dropped */
static int sample_window(const patch_sys* p, const bo_image* right, double u_k,
                         window* w, scratch* s) {
  int invalid = 0;
  for (int i = 0; i < w->n; ++i) {
    const resid ev = eval_residual(p, right, u_k + w->offsets[i], s);
    const int ok = ev.n == p->valid_count;
    w->residuals[i] = ev.msq;
    w->valid[i] = (uint8_t)ok;
    if (!ok) ++invalid;
  }
  if (invalid > 1 || !w->valid[w->center]) return 0;
  return 1;
}

/* src/window_posterior.cpp:42-59 */
double bo_dynamic_sigma(int n, const double* residuals, const uint8_t* valid,
                        double sigma_floor) {
  double sum = 0.0;
  int count = 0;
  for (int i = 0; i < n; ++i) {
    if (!valid[i]) continue;
    sum += residuals[i];
    ++count;
  }
  if (count == 0) return sigma_floor;
  const double mean = sum / count;
  double ss = 0.0;
  for (int i = 0; i < n; ++i) {
    if (!valid[i]) continue;
    const double d = residuals[i] - mean;
    ss += d * d;
  }
  return maxd(sqrt(ss / count), sigma_floor);
}

/* src/window_posterior.cpp:61-72 */
void bo_window_priors(int n, const double* residuals, const uint8_t* valid,
                      double sigma_r, int patch_size, int use_fast_exp,
                      double* priors) {
  const double denom = 2.0 * sigma_r * sigma_r * (double)patch_size * (double)patch_size;
  for (int i = 0; i < n; ++i) {
    priors[i] = 0.0;
    if (!valid[i]) continue;
    const double e = -residuals[i] / denom;
    priors[i] = use_fast_exp ? bo_fast_exp(e) : exp(e);
  }
}

/* src/window_posterior.cpp:74-96; returns 0 when every weight underflowed */
int bo_patch_posterior(int n, const double* residuals, const uint8_t* valid,
                       int center_index, double sigma_r, int patch_size,
                       int use_fast_exp, double* probability, int* is_min) {
  double priors[2 * BO_MAX_OFFSETS + 1];
  bo_window_priors(n, residuals, valid, sigma_r, patch_size, use_fast_exp, priors);
  double denom = 0.0;
  for (int i = 0; i < n; ++i) denom += priors[i];
  if (denom <= 0.0) return 0;
  *probability = priors[center_index] / denom;
  *is_min = 1;
  const double c = residuals[center_index];
  for (int i = 0; i < n; ++i) {
    if (i == center_index || !valid[i]) continue;
    if (!(c < residuals[i])) {
      *is_min = 0;
      break;
    }
  }
  return 1;
}

/* src/depth_variance.cpp:94-170 */
void bo_estimate_variance(int nw, const double* offsets, const uint8_t* valid,
                          int center_index, const double* priors,
                          double sigma_fallback, double* sigma_k, double* c_k,
                          int* accepted, int* reason, double* fit_residual) {
  enum { NONE = 0, TOO_LARGE = 1, NOT_GAUSSIAN = 2 };
  *sigma_k = sigma_fallback;
  *c_k = 0.0;
  *accepted = 0;
  *reason = NOT_GAUSSIAN;
  *fit_residual = 0.0;
  double delta[2 * BO_MAX_OFFSETS + 1], p[2 * BO_MAX_OFFSETS + 1];
  double center_prior = 0.0;
  int n = 0;
  for (int i = 0; i < nw; ++i) {
    if (!valid[i]) continue;
    delta[n] = offsets[i];
    p[n] = priors[i];
    ++n;
    if (i == center_index) center_prior = priors[i];
  }
  if (n < 3) return;
  for (int i = 0; i < n; ++i) {
    if (delta[i] == 0.0) continue;
    if (!(center_prior > p[i])) return;
  }
  double c = 1.0;
  double sigma = sqrt(0.1);
  for (int iter = 0; iter < 10; ++iter) {
    double a00 = 0.0, a01 = 0.0, a11 = 0.0, b0 = 0.0, b1 = 0.0;
    for (int i = 0; i < n; ++i) {
      const double d2 = delta[i] * delta[i];
      const double g = exp(-d2 / (2.0 * sigma * sigma));
      const double r = c * g - p[i];
      const double jc = g;
      const double js = c * g * d2 / (sigma * sigma * sigma);
      a00 += jc * jc;
      a01 += jc * js;
      a11 += js * js;
      b0 -= jc * r;
      b1 -= js * r;
    }
    if (!(a00 > 0.0)) return;
    const double l00 = sqrt(a00);
    const double l01 = a01 / l00;
    const double d11 = a11 - l01 * l01;
    if (!(d11 > 1e-300)) return;
    const double l11 = sqrt(d11);
    const double y0 = b0 / l00;
    const double y1 = (b1 - l01 * y0) / l11;
    const double xs = y1 / l11;
    const double xc = (y0 - l01 * xs) / l00;
    c += xc;
    sigma += xs;
    if (!isfinite(c) || !isfinite(sigma) || sigma <= 0.0) return;
  }
  double ssr = 0.0;
  for (int i = 0; i < n; ++i) {
    const double g = exp(-delta[i] * delta[i] / (2.0 * sigma * sigma));
    const double r = c * g - p[i];
    ssr += r * r;
  }
  *fit_residual = sqrt(ssr / (double)n);
  if (!isfinite(*fit_residual)) return;
  if (*fit_residual > 0.1) {
    *reason = TOO_LARGE;
    return;
  }
  *sigma_k = sigma;
  *c_k = c;
  *accepted = 1;
  *reason = NONE;
}

/* ------------------------------------------------------------------ */
/* per-stage entry points on caller images                              */

typedef struct sys_buf {
  patch_sys p;
  scratch s;
  double mem[4 * 64 * 64];
  uint8_t vmem[2 * 64 * 64];
} sys_buf;

static sys_buf* sys_alloc(int size) {
  if (size > 64 || size < 1) return NULL;
  sys_buf* b = (sys_buf*)calloc(1, sizeof(sys_buf));
  const int n = size * size;
  b->p.values = b->mem;
  b->p.jacobian = b->mem + n;
  b->s.samples = b->mem + 2 * n;
  b->p.valid = b->vmem;
  b->s.ok = b->vmem + n;
  return b;
}

static sys_buf* build_sys(const bo_image* left, const float* grad, double cx,
                          double cy, int size) {
  sys_buf* b = sys_alloc(size);
  if (!b) return NULL;
  if (!extract(left, cx, cy, size, &b->p)) {
    free(b);
    return NULL;
  }
  precompute(&b->p, grad, left->width, left->height);
  return b;
}

int bo_extract_patch(const bo_image* img, double cx, double cy, int size,
                     double* values, uint8_t* valid, bo_patch_info* info) {
  sys_buf* b = sys_alloc(size);
  if (!b) return 0;
  const int ok = extract(img, cx, cy, size, &b->p);
  if (ok) {
    if (values) memcpy(values, b->p.values, sizeof(double) * (size_t)(size * size));
    if (valid) memcpy(valid, b->p.valid, (size_t)(size * size));
    if (info) {
      info->mean = b->p.mean;
      info->valid_fraction = b->p.valid_fraction;
      info->valid_count = b->p.valid_count;
    }
  }
  free(b);
  return ok;
}

int bo_patch_system(const bo_image* left, const float* grad, double cx,
                    double cy, int size, double* jacobian, bo_patch_info* info) {
  sys_buf* b = build_sys(left, grad, cx, cy, size);
  if (!b) return 0;
  if (jacobian) memcpy(jacobian, b->p.jacobian, sizeof(double) * (size_t)(size * size));
  if (info) {
    info->mean = b->p.mean;
    info->valid_fraction = b->p.valid_fraction;
    info->valid_count = b->p.valid_count;
    info->hessian = b->p.hessian;
    info->template_msq = b->p.template_msq;
    info->degenerate = b->p.degenerate;
  }
  free(b);
  return 1;
}

int bo_eval_residual(const bo_image* left, const float* grad,
                     const bo_image* right, double cx, double cy, int size,
                     double u, double* msq, double* jr, int* n) {
  sys_buf* b = build_sys(left, grad, cx, cy, size);
  if (!b) return 0;
  const resid ev = eval_residual(&b->p, right, u, &b->s);
  *msq = ev.msq;
  *jr = ev.jr;
  *n = ev.n;
  free(b);
  return 1;
}

int bo_solve_patch(const bo_image* left, const float* grad,
                   const bo_image* right, double cx, double cy, int size,
                   double u_init, const bo_lk_params* prm, double* u,
                   int* converged, int* iterations, double* final_residual) {
  sys_buf* b = build_sys(left, grad, cx, cy, size);
  if (!b) return 0;
  const lk_out r = solve(&b->p, right, u_init, prm, &b->s, 1);
  *u = r.u;
  *converged = r.converged;
  *iterations = r.iterations;
  *final_residual = r.final_residual;
  free(b);
  return 1;
}

int bo_sample_window(const bo_image* left, const float* grad,
                     const bo_image* right, double cx, double cy, int size,
                     double u_k, int n_mags, const double* mags,
                     double* offsets, double* residuals, uint8_t* valid,
                     int* center_index) {
  sys_buf* b = build_sys(left, grad, cx, cy, size);
  if (!b) return -1;
  window w;
  window_offsets(n_mags, mags, &w);
  const int ok = sample_window(&b->p, right, u_k, &w, &b->s);
  if (ok) {
    memcpy(offsets, w.offsets, sizeof(double) * (size_t)w.n);
    memcpy(residuals, w.residuals, sizeof(double) * (size_t)w.n);
    memcpy(valid, w.valid, (size_t)w.n);
    *center_index = w.center;
  }
  free(b);
  return ok;
}

/* ------------------------------------------------------------------ */
/* grid and level bookkeeping: src/coarse_to_fine.cpp:51-99             */

typedef struct grid {
  int stride, nx, ny;
  double* xs;
  double* ys;
} grid;

static int grid_axis(double c0, double cmax, int stride, double* out, int cap) {
  int n = 0;
  for (int k = 0;; ++k) {
    const double c = c0 + (double)k * stride;
    if (c >= cmax - 1e-9) {
      if (out && n < cap) out[n] = cmax;
      ++n;
      break;
    }
    if (out && n < cap) out[n] = c;
    ++n;
  }
  return n;
}

/* src/coarse_to_fine.cpp:51-88; returns BO_EDEGENERATE if smaller than a patch */
static int make_grid(int w, int h, int size, double overlap, grid* g) {
  const double c0 = (size - 1) * 0.5;
  const double cmax_x = (w - 1) - c0;
  const double cmax_y = (h - 1) - c0;
  if (cmax_x < c0 || cmax_y < c0) return BO_EDEGENERATE;
  long st = lrint(size * (1.0 - overlap));
  g->stride = st > 1 ? (int)st : 1;
  g->nx = grid_axis(c0, cmax_x, g->stride, NULL, 0);
  g->ny = grid_axis(c0, cmax_y, g->stride, NULL, 0);
  g->xs = (double*)malloc(sizeof(double) * (size_t)g->nx);
  g->ys = (double*)malloc(sizeof(double) * (size_t)g->ny);
  grid_axis(c0, cmax_x, g->stride, g->xs, g->nx);
  grid_axis(c0, cmax_y, g->stride, g->ys, g->ny);
  return BO_OK;
}

int bo_make_patch_grid(int w, int h, int patch_size, double overlap,
                       int* stride, int* nx, int* ny, double* xs, double* ys,
                       int cap) {
  grid g;
  const int rc = make_grid(w, h, patch_size, overlap, &g);
  if (rc != BO_OK) return rc;
  *stride = g.stride;
  *nx = g.nx;
  *ny = g.ny;
  for (int i = 0; i < g.nx && i < cap; ++i) xs[i] = g.xs[i];
  for (int i = 0; i < g.ny && i < cap; ++i) ys[i] = g.ys[i];
  free(g.xs);
  free(g.ys);
  return BO_OK;
}

/* src/coarse_to_fine.cpp:90-94 */
double bo_level_weight(int n, int n_levels, const int* levels) {
  double denom = 0.0;
  for (int i = 0; i < n_levels; ++i) denom += exp2((double)levels[i]);
  return exp2((double)n) / denom;
}

/* src/coarse_to_fine.cpp:96-99 */
double bo_propagate_probability(double posterior, double inherited, int n,
                                int n_levels, const int* levels) {
  return clampd(inherited + bo_level_weight(n, n_levels, levels) * posterior, 0.0, 1.0);
}

/* ------------------------------------------------------------------ */
/* fusion and resampling: src/coarse_to_fine.cpp:101-180                */

typedef struct field {
  int w, h;
  double* v;
  uint8_t* ok;
} field;

static field field_new(int w, int h) {
  field f;
  f.w = w;
  f.h = h;
  f.v = (double*)calloc((size_t)w * (size_t)h, sizeof(double));
  f.ok = (uint8_t*)calloc((size_t)w * (size_t)h, 1);
  return f;
}
static void field_free(field* f) {
  free(f->v);
  free(f->ok);
  f->v = NULL;
  f->ok = NULL;
}

typedef struct estimate {
  double cx, cy, u, prob, posterior, sigma_k;
  int has_sigma;
} estimate;

/* src/coarse_to_fine.cpp:101-150 */
static void fuse(const estimate* pes, int n_pes, const double* mask, int size,
                 int w, int h, int with_var, field* disp, field* prob,
                 field* var) {
  const size_t n = (size_t)w * (size_t)h;
  double* sw = (double*)calloc(n, sizeof(double));
  double* swu = (double*)calloc(n, sizeof(double));
  double* swp = (double*)calloc(n, sizeof(double));
  double* sw2s = with_var ? (double*)calloc(n, sizeof(double)) : NULL;
  const double half = (size - 1) * 0.5;
  for (int k = 0; k < n_pes; ++k) {
    const estimate* pe = &pes[k];
    for (int j = 0; j < size; ++j) {
      const int y = (int)lround(pe->cy + (j - half));
      if (y < 0 || y >= h) continue;
      for (int i = 0; i < size; ++i) {
        const int x = (int)lround(pe->cx + (i - half));
        if (x < 0 || x >= w) continue;
        const double wt = pe->prob * mask[j * size + i];
        const size_t idx = (size_t)y * (size_t)w + (size_t)x;
        sw[idx] += wt;
        swu[idx] += wt * pe->u;
        swp[idx] += wt * pe->prob;
        if (with_var) sw2s[idx] += wt * wt * pe->sigma_k * pe->sigma_k;
      }
    }
  }
  for (size_t i = 0; i < n; ++i) {
    if (sw[i] <= 0.0) continue;
    disp->v[i] = swu[i] / sw[i];
    disp->ok[i] = 1;
    prob->v[i] = swp[i] / sw[i];
    prob->ok[i] = 1;
    if (with_var) {
      var->v[i] = sw2s[i] / (sw[i] * sw[i]);
      var->ok[i] = 1;
    }
  }
  free(sw);
  free(swu);
  free(swp);
  free(sw2s);
}

void bo_fuse_level(int n_patches, const double* cx, const double* cy,
                   const double* u, const double* prob, const double* sigma_k,
                   int size, double sigma_s, int w, int h, int with_variance,
                   double* disp_out, uint8_t* disp_valid, double* prob_out,
                   uint8_t* prob_valid, double* var_out, uint8_t* var_valid) {
  estimate* pes = (estimate*)calloc((size_t)(n_patches > 0 ? n_patches : 1), sizeof(estimate));
  for (int i = 0; i < n_patches; ++i) {
    pes[i].cx = cx[i];
    pes[i].cy = cy[i];
    pes[i].u = u[i];
    pes[i].prob = prob[i];
    pes[i].sigma_k = sigma_k ? sigma_k[i] : 0.0;
  }
  double* mask = (double*)malloc(sizeof(double) * (size_t)(size * size));
  bo_spatial_mask(size, sigma_s, mask);
  field d = field_new(w, h), p = field_new(w, h), v = field_new(w, h);
  fuse(pes, n_patches, mask, size, w, h, with_variance, &d, &p, &v);
  const size_t n = (size_t)w * (size_t)h;
  memcpy(disp_out, d.v, n * sizeof(double));
  memcpy(disp_valid, d.ok, n);
  memcpy(prob_out, p.v, n * sizeof(double));
  memcpy(prob_valid, p.ok, n);
  if (with_variance) {
    memcpy(var_out, v.v, n * sizeof(double));
    memcpy(var_valid, v.ok, n);
  }
  field_free(&d);
  field_free(&p);
  field_free(&v);
  free(mask);
  free(pes);
}

/* src/coarse_to_fine.cpp:152-164 */
static void init_next(const field* coarse, int fw, int fh, double* out) {
  for (int y = 0; y < fh; ++y) {
    const int cy = mini(y / 2, coarse->h - 1);
    for (int x = 0; x < fw; ++x) {
      const int cx = mini(x / 2, coarse->w - 1);
      const size_t ci = (size_t)cy * (size_t)coarse->w + (size_t)cx;
      out[(size_t)y * fw + x] = coarse->ok[ci] ? 2.0 * coarse->v[ci] : 0.0;
    }
  }
}

void bo_init_next_level(int cw, int ch, const double* values,
                        const uint8_t* valid, int fw, int fh, double* out) {
  field c;
  c.w = cw;
  c.h = ch;
  c.v = (double*)values;
  c.ok = (uint8_t*)valid;
  init_next(&c, fw, fh, out);
}

/* src/coarse_to_fine.cpp:166-180 */
static void upsample(const field* f, int fw, int fh, int e, double scale_per_level,
                     double* out, uint8_t* out_ok) {
  if (e == 0) {
    memcpy(out, f->v, sizeof(double) * (size_t)f->w * (size_t)f->h);
    memcpy(out_ok, f->ok, (size_t)f->w * (size_t)f->h);
    return;
  }
  const double scale = pow(scale_per_level, e);
  for (int y = 0; y < fh; ++y) {
    const int sy = mini(y >> e, f->h - 1);
    for (int x = 0; x < fw; ++x) {
      const int sx = mini(x >> e, f->w - 1);
      const size_t si = (size_t)sy * (size_t)f->w + (size_t)sx;
      const size_t o = (size_t)y * (size_t)fw + (size_t)x;
      if (!f->ok[si]) {
        out[o] = 0.0;
        out_ok[o] = 0;
        continue;
      }
      out[o] = scale * f->v[si];
      out_ok[o] = 1;
    }
  }
}

void bo_upsample_to_full(int w, int h, const double* values,
                         const uint8_t* valid, int fw, int fh, int e,
                         double scale_per_level, double* out,
                         uint8_t* out_valid) {
  field f;
  f.w = w;
  f.h = h;
  f.v = (double*)values;
  f.ok = (uint8_t*)valid;
  upsample(&f, fw, fh, e, scale_per_level, out, out_valid);
}

/* ------------------------------------------------------------------ */
/* confidence filter and depth: src/depth_variance.cpp:9-92              */

/* src/depth_variance.cpp:43-76 (component membership is order-free, so a
 * breadth-first fill yields the same mask as the reference's DFS) */
void bo_remove_small_components(const uint8_t* valid, int w, int h,
                                long long min_px, uint8_t* out) {
  const size_t n = (size_t)w * (size_t)h;
  uint8_t* seen = (uint8_t*)calloc(n, 1);
  size_t* queue = (size_t*)malloc(sizeof(size_t) * (n ? n : 1));
  memset(out, 0, n);
  for (size_t start = 0; start < n; ++start) {
    if (!valid[start] || seen[start]) continue;
    size_t head = 0, tail = 0;
    queue[tail++] = start;
    seen[start] = 1;
    while (head < tail) {
      const size_t idx = queue[head++];
      const int x = (int)(idx % (size_t)w), y = (int)(idx / (size_t)w);
      const int nx[4] = {x - 1, x + 1, x, x};
      const int ny[4] = {y, y, y - 1, y + 1};
      for (int k = 0; k < 4; ++k) {
        if (nx[k] < 0 || nx[k] >= w || ny[k] < 0 || ny[k] >= h) continue;
        const size_t ni = (size_t)ny[k] * (size_t)w + (size_t)nx[k];
        if (!valid[ni] || seen[ni]) continue;
        seen[ni] = 1;
        queue[tail++] = ni;
      }
    }
    if ((long long)tail >= min_px)
      for (size_t k = 0; k < tail; ++k) out[queue[k]] = 1;
  }
  free(seen);
  free(queue);
}

/* src/depth_variance.cpp:78-92 */
void bo_filter_validity(int w, int h, const uint8_t* disp_valid,
                        const double* prob, const uint8_t* prob_valid,
                        double gamma, double pixel_threshold, int patch_size,
                        uint8_t* out_valid) {
  const size_t n = (size_t)w * (size_t)h;
  uint8_t* m = (uint8_t*)malloc(n ? n : 1);
  for (size_t i = 0; i < n; ++i) {
    m[i] = disp_valid[i];
    if (!m[i]) continue;
    if (!prob_valid[i] || prob[i] < pixel_threshold) m[i] = 0;
  }
  long long min_px = llround(ceil(gamma * (double)patch_size * (double)patch_size - 1e-9));
  if (min_px < 1) min_px = 1;
  bo_remove_small_components(m, w, h, min_px, out_valid);
  free(m);
}

/* src/depth_variance.cpp:9-41 */
void bo_disparity_to_depth(int w, int h, const double* disp,
                           const uint8_t* disp_valid, const double* var,
                           const uint8_t* var_valid, double focal_px,
                           double baseline, double min_disparity,
                           double* depth, uint8_t* depth_valid, double* sigma,
                           uint8_t* sigma_valid) {
  const size_t n = (size_t)w * (size_t)h;
  const double fb = focal_px * baseline;
  for (size_t i = 0; i < n; ++i) {
    depth[i] = 0.0;
    depth_valid[i] = 0;
    if (!disp_valid[i]) continue;
    const double u = disp[i];
    if (!(u >= min_disparity)) continue;
    depth[i] = fb / u;
    depth_valid[i] = 1;
  }
  if (!var) return;
  for (size_t i = 0; i < n; ++i) {
    sigma[i] = 0.0;
    sigma_valid[i] = 0;
    if (!depth_valid[i] || !var_valid[i]) continue;
    const double u = disp[i];
    const double su = sqrt(maxd(var[i], 0.0));
    sigma[i] = fb / (u * u) * su;
    sigma_valid[i] = 1;
  }
}

/* ------------------------------------------------------------------ */
/* the matcher: src/coarse_to_fine.cpp:211-341                          */

typedef struct level_img {
  int e, w, h;
  float* l;
  uint8_t* lv;
  float* r;
  uint8_t* rv;
  float* g;
} level_img;

typedef struct match_state {
  int n_levels;
  level_img* lv;  /* coarsest first */
  int* stats;     /* n_levels * 5 */
  field disp, prob, var;
  int has_var;
  int fw, fh;
  estimate* finest;
  int n_finest;
} match_state;

/* src/pyramid.cpp:44-96. Level images are owned by the pyramid except the
 * caller's full-resolution planes (stored when finest_exp == 0). */
static void free_level_images(level_img* lv, int n, const bo_image* left,
                              const bo_image* right) {
  for (int i = 0; i < n; ++i) {
    if (lv[i].l != left->data) free(lv[i].l);
    if (lv[i].lv != left->valid) free(lv[i].lv);
    if (lv[i].r != right->data) free(lv[i].r);
    if (lv[i].rv != right->valid) free(lv[i].rv);
    free(lv[i].g);
  }
  free(lv);
}

static int build_pyramid(const bo_image* left, const bo_image* right, int ce,
                         int fe, int min_patch, level_img** out, char* msg, int cap) {
  *out = NULL;
  if (left->width != right->width || left->height != right->height) {
    set_msg(msg, cap, "build_pyramid: left and right differ in size");
    return BO_EDEGENERATE;
  }
  if (fe < 0 || ce < fe) {
    set_msg(msg, cap, "build_pyramid: bad level range");
    return BO_EDEGENERATE;
  }
  const int n = ce - fe + 1;
  level_img* all = (level_img*)calloc((size_t)ce + 1, sizeof(level_img));
  all[0].e = 0;
  all[0].w = left->width;
  all[0].h = left->height;
  all[0].l = (float*)left->data;
  all[0].r = (float*)right->data;
  const size_t n0 = (size_t)left->width * (size_t)left->height;
  all[0].lv = (uint8_t*)left->valid;
  all[0].rv = (uint8_t*)right->valid;
  if (!left->valid) {
    all[0].lv = (uint8_t*)malloc(n0 ? n0 : 1);
    memset(all[0].lv, 1, n0);
  }
  if (!right->valid) {
    all[0].rv = (uint8_t*)malloc(n0 ? n0 : 1);
    memset(all[0].rv, 1, n0);
  }
  for (int e = 1; e <= ce; ++e) {
    const level_img* P = &all[e - 1];
    level_img* L = &all[e];
    L->e = e;
    L->w = (P->w + 1) / 2;
    L->h = (P->h + 1) / 2;
    const size_t nn = (size_t)L->w * (size_t)L->h;
    L->l = (float*)malloc(sizeof(float) * (nn ? nn : 1));
    L->lv = (uint8_t*)malloc(nn ? nn : 1);
    L->r = (float*)malloc(sizeof(float) * (nn ? nn : 1));
    L->rv = (uint8_t*)malloc(nn ? nn : 1);
    bo_downsample_half(P->w, P->h, P->l, P->lv, L->l, L->lv);
    bo_downsample_half(P->w, P->h, P->r, P->rv, L->r, L->rv);
  }
  level_img* lv = (level_img*)calloc((size_t)n, sizeof(level_img));
  for (int e = 0; e <= ce; ++e) {
    if (e >= fe) {
      lv[ce - e] = all[e];
    } else if (e > 0) {
      free(all[e].l);
      free(all[e].lv);
      free(all[e].r);
      free(all[e].rv);
    } else {
      if (all[0].lv != left->valid) free(all[0].lv);
      if (all[0].rv != right->valid) free(all[0].rv);
    }
  }
  free(all);
  for (int i = 0; i < n; ++i) {
    lv[i].g = (float*)malloc(sizeof(float) * ((size_t)lv[i].w * (size_t)lv[i].h + 1));
    bo_gradient_x(lv[i].w, lv[i].h, lv[i].l, lv[i].g);
  }
  *out = lv;
  if (lv[0].w < min_patch || lv[0].h < min_patch) {
    set_msg(msg, cap, "build_pyramid: coarsest level is smaller than one patch");
    return BO_EDEGENERATE;
  }
  return BO_OK;
}

static int match_core(const bo_image* left, const bo_image* right,
                      const bo_config* cfg, match_state* st, char* msg, int cap) {
  int rc = bo_validate(cfg, msg, cap);
  if (rc != BO_OK) return rc;
  const int ce = cfg->coarsest_exp, fe = cfg->finest_exp, size = cfg->patch_size;
  level_img* lv = NULL;
  rc = build_pyramid(left, right, ce, fe, size, &lv, msg, cap);
  const int n_levels = ce - fe + 1;
  if (rc != BO_OK) {
    if (lv) free_level_images(lv, n_levels, left, right);
    return rc;
  }
  double* mask = (double*)malloc(sizeof(double) * (size_t)(size * size));
  bo_spatial_mask(size, cfg->sigma_s, mask);
  int level_set[32];
  for (int e = ce, k = 0; e >= fe; --e) level_set[k++] = e;

  bo_lk_params lk;
  lk.min_iterations = cfg->min_iterations;
  lk.max_iterations = cfg->max_iterations;
  lk.update_epsilon = 1e-2; /* kUpdateEpsilon, inc/lk_solver.hpp:12 */
  lk.stop_good = cfg->early_stop_good;
  lk.stop_bad = cfg->early_stop_bad;
  lk.stop_improve = cfg->early_stop_improve;

  window wtemplate;
  window_offsets(cfg->n_window_offsets, cfg->window_offsets, &wtemplate);

  st->n_levels = n_levels;
  st->stats = (int*)calloc((size_t)n_levels * 5, sizeof(int));
  sys_buf* sb = sys_alloc(size);
  double* init = NULL;
  int have_init = 0, have_prev = 0;
  field prev_disp = {0, 0, NULL, NULL}, prev_prob = {0, 0, NULL, NULL},
        prev_var = {0, 0, NULL, NULL};
  estimate* prev_pes = NULL;
  int prev_n = 0;

  for (int li = 0; li < n_levels; ++li) {
    const level_img* L = &lv[li];
    const int w = L->w, h = L->h;
    const int want_var = cfg->estimate_variance && L->e == fe;
    grid g;
    rc = make_grid(w, h, size, cfg->overlap, &g);
    if (rc != BO_OK) {
      set_msg(msg, cap, "make_patch_grid: level is smaller than one patch");
      break;
    }
    const bo_image limg = {w, h, L->l, L->lv};
    const bo_image rimg = {w, h, L->r, L->rv};
    const int count = g.nx * g.ny;
    estimate* slots = (estimate*)calloc((size_t)count, sizeof(estimate));
    uint8_t* stage = (uint8_t*)calloc((size_t)count, 1); /* 0 skipped 1 solved 2 converged 3 accepted */
    for (int i = 0; i < count; ++i) {
      /* per-patch body, src/coarse_to_fine.cpp:247-300 */
      const double cx = g.xs[i % g.nx], cy = g.ys[i / g.nx];
      patch_sys* p = &sb->p;
      if (!extract(&limg, cx, cy, size, p)) continue;
      if (p->valid_fraction < cfg->valid_patch_ratio) continue;
      precompute(p, L->g, w, h);
      if (p->degenerate) continue;
      stage[i] = 1;
      double u0 = 0.0;
      if (have_init) {
        const int ix = clampi((int)lround(cx), 0, w - 1);
        const int iy = clampi((int)lround(cy), 0, h - 1);
        u0 = init[(size_t)iy * (size_t)w + (size_t)ix];
      }
      const lk_out r = solve(p, &rimg, u0, &lk, &sb->s, 0);
      if (!r.converged) continue;
      stage[i] = 2;
      window win = wtemplate;
      if (!sample_window(p, &rimg, r.u, &win, &sb->s)) continue;
      const double sigma_r = bo_dynamic_sigma(win.n, win.residuals, win.valid, 1e-4);
      double post;
      int is_min;
      if (!bo_patch_posterior(win.n, win.residuals, win.valid, win.center, sigma_r,
                              size, 1, &post, &is_min) ||
          !is_min)
        continue;
      double inherited = 0.0;
      if (have_prev) {
        const int px = clampi((int)lround(cx / 2.0), 0, prev_prob.w - 1);
        const int py = clampi((int)lround(cy / 2.0), 0, prev_prob.h - 1);
        const size_t pi = (size_t)py * (size_t)prev_prob.w + (size_t)px;
        if (prev_prob.ok[pi]) inherited = prev_prob.v[pi];
      }
      estimate* pe = &slots[i];
      pe->cx = cx;
      pe->cy = cy;
      pe->u = r.u;
      pe->posterior = post;
      pe->prob = bo_propagate_probability(post, inherited, L->e, n_levels, level_set);
      if (want_var) {
        double priors[2 * BO_MAX_OFFSETS + 1];
        bo_window_priors(win.n, win.residuals, win.valid, sigma_r, size, 1, priors);
        double sk, ck, fr;
        int acc, reason;
        bo_estimate_variance(win.n, win.offsets, win.valid, win.center, priors, 2.0,
                             &sk, &ck, &acc, &reason, &fr);
        pe->sigma_k = sk;
        pe->has_sigma = 1;
      }
      stage[i] = 3;
    }
    /* compaction + MatchStats, src/coarse_to_fine.cpp:302-314 */
    estimate* kept = (estimate*)calloc((size_t)(count > 0 ? count : 1), sizeof(estimate));
    int nk = 0;
    int* s5 = st->stats + 5 * li;
    s5[0] = L->e;
    s5[1] = count;
    for (int i = 0; i < count; ++i) {
      if (stage[i] >= 1) ++s5[2];
      if (stage[i] >= 2) ++s5[3];
      if (stage[i] == 3) {
        ++s5[4];
        kept[nk++] = slots[i];
      }
    }
    field d = field_new(w, h), pr = field_new(w, h);
    field va = want_var ? field_new(w, h) : (field){0, 0, NULL, NULL};
    fuse(kept, nk, mask, size, w, h, want_var, &d, &pr, &va);
    if (L->e != fe) {
      const level_img* nx = &lv[li + 1];
      free(init);
      init = (double*)malloc(sizeof(double) * (size_t)nx->w * (size_t)nx->h);
      init_next(&d, nx->w, nx->h, init);
      have_init = 1;
    }
    field_free(&prev_disp);
    field_free(&prev_prob);
    field_free(&prev_var);
    free(prev_pes);
    prev_disp = d;
    prev_prob = pr;
    prev_var = va;
    prev_pes = kept;
    prev_n = nk;
    have_prev = 1;
    free(slots);
    free(stage);
    free(g.xs);
    free(g.ys);
  }
  free(init);
  free(sb);
  free(mask);
  free_level_images(lv, n_levels, left, right);
  if (rc != BO_OK) {
    field_free(&prev_disp);
    field_free(&prev_prob);
    field_free(&prev_var);
    free(prev_pes);
    return rc;
  }
  st->disp = prev_disp;
  st->prob = prev_prob;
  st->var = prev_var;
  st->has_var = cfg->estimate_variance;
  st->finest = prev_pes;
  st->n_finest = prev_n;
  return BO_OK;
}

static void match_free(match_state* st) {
  field_free(&st->disp);
  field_free(&st->prob);
  field_free(&st->var);
  free(st->finest);
  free(st->stats);
}

int bo_match_stereo(const bo_image* left, const bo_image* right,
                    const bo_config* cfg, bo_match_outputs* out, char* msg,
                    int cap) {
  match_state st;
  memset(&st, 0, sizeof st);
  const int rc = match_core(left, right, cfg, &st, msg, cap);
  if (rc != BO_OK) return rc;
  const int W = left->width, H = left->height, fe = cfg->finest_exp;
  /* match tail, src/coarse_to_fine.cpp:328-337 */
  upsample(&st.disp, W, H, fe, 2.0, out->disparity, out->disparity_valid);
  upsample(&st.prob, W, H, fe, 1.0, out->probability, out->probability_valid);
  out->has_variance = st.has_var;
  if (st.has_var && out->var_disp) upsample(&st.var, W, H, fe, 4.0, out->var_disp, out->var_valid);
  out->n_levels = st.n_levels;
  if (out->stats) memcpy(out->stats, st.stats, sizeof(int) * 5 * (size_t)st.n_levels);
  out->finest_count = st.n_finest;
  if (out->finest) {
    for (int i = 0; i < st.n_finest && i < out->finest_cap; ++i) {
      double* row = out->finest + 7 * i;
      row[0] = st.finest[i].cx;
      row[1] = st.finest[i].cy;
      row[2] = st.finest[i].u;
      row[3] = st.finest[i].prob;
      row[4] = st.finest[i].posterior;
      row[5] = st.finest[i].sigma_k;
      row[6] = st.finest[i].has_sigma ? 1.0 : 0.0;
    }
  }
  match_free(&st);
  return BO_OK;
}

/* src/pipeline.cpp:9-37 */
int bo_run_pipeline(const bo_image* left, const bo_image* right,
                    const bo_config* cfg, double focal_px, double baseline,
                    bo_outputs* out, char* msg, int cap) {
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  const int W = left->width, H = left->height;
  const size_t n = (size_t)W * (size_t)H;
  double* md = (double*)malloc(sizeof(double) * (n ? n : 1));
  uint8_t* mdv = (uint8_t*)malloc(n ? n : 1);
  double* mp = (double*)malloc(sizeof(double) * (n ? n : 1));
  uint8_t* mpv = (uint8_t*)malloc(n ? n : 1);
  double* mv = cfg->estimate_variance ? (double*)malloc(sizeof(double) * (n ? n : 1)) : NULL;
  uint8_t* mvv = cfg->estimate_variance ? (uint8_t*)malloc(n ? n : 1) : NULL;
  bo_match_outputs mo;
  memset(&mo, 0, sizeof mo);
  mo.disparity = md;
  mo.disparity_valid = mdv;
  mo.probability = mp;
  mo.probability_valid = mpv;
  mo.var_disp = mv;
  mo.var_valid = mvv;
  mo.stats = out->stats;
  const int rc = bo_match_stereo(left, right, cfg, &mo, msg, cap);
  if (rc == BO_OK) {
    out->n_levels = mo.n_levels;
    uint8_t* fv = (uint8_t*)malloc(n ? n : 1);
    bo_filter_validity(W, H, mdv, mp, mpv, cfg->gamma, cfg->pixel_threshold,
                       cfg->patch_size, fv);
    memcpy(out->disparity, md, n * sizeof(double));
    memcpy(out->disparity_valid, fv, n);
    memcpy(out->probability, mp, n * sizeof(double));
    memcpy(out->probability_valid, fv, n);
    out->has_sigma = mo.has_variance;
    double* sig = out->depth_sigma;
    uint8_t* sigv = out->sigma_valid;
    double* tmp_s = NULL;
    uint8_t* tmp_sv = NULL;
    if (mo.has_variance && (!sig || !sigv)) {
      tmp_s = (double*)malloc(sizeof(double) * (n ? n : 1));
      tmp_sv = (uint8_t*)malloc(n ? n : 1);
      sig = tmp_s;
      sigv = tmp_sv;
    }
    bo_disparity_to_depth(W, H, md, fv, mo.has_variance ? mv : NULL, mvv, focal_px,
                          baseline, 0.1, out->depth, out->depth_valid, sig, sigv);
    free(tmp_s);
    free(tmp_sv);
    free(fv);
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  out->runtime_ms = (double)(t1.tv_sec - t0.tv_sec) * 1e3 + (double)(t1.tv_nsec - t0.tv_nsec) * 1e-6;
  free(md);
  free(mdv);
  free(mp);
  free(mpv);
  free(mv);
  free(mvv);
  return rc;
}

/* ------------------------------------------------------------------------
 * compute_metrics (src/metrics.cpp:10-52): errors |est - ref| over pixels
 * valid on both sides, in index order; mean = sequential sum / count; median
 * = the middle order statistic (mean of the two middle ones for an even
 * count: nth_element twice, :40-48 -- order statistics do not depend on the
 * selection algorithm, so a sort gives the same values); coverage = share of
 * compared pixels with a valid sigma and |e| <= 1.96 sigma (:33).
 * ------------------------------------------------------------------------ */

void bo_compute_metrics(int w, int h, const double* est, const uint8_t* est_valid,
                        const double* ref, const uint8_t* ref_valid, const double* sigma,
                        const uint8_t* sigma_valid, bo_frame_metrics* out) {
  const size_t n = (size_t)w * (size_t)h;
  out->mean_err = NAN;
  out->median_err = NAN;
  out->coverage_rate = NAN;
  out->has_errors = 0;
  out->valid_px = 0;
  for (size_t i = 0; i < n; ++i) out->valid_px += est_valid[i] != 0; /* fields.hpp valid_count */
  double* errs = (double*)malloc((n ? n : 1) * sizeof(double));
  size_t m = 0;
  long long covered = 0;
  for (size_t i = 0; i < n; ++i) {
    if (!est_valid[i] || !ref_valid[i]) continue;
    const double e = fabs(est[i] - ref[i]);
    errs[m++] = e;
    if (sigma && sigma_valid[i] && e <= 1.96 * sigma[i]) ++covered;
  }
  out->compared = (long long)m;
  if (m == 0) {
    free(errs);
    return;
  }
  out->has_errors = 1;
  double sum = 0.0;
  for (size_t i = 0; i < m; ++i) sum += errs[i];
  out->mean_err = sum / (double)m;
  qsort(errs, m, sizeof(double), cmp_double);
  const size_t mid = m / 2;
  out->median_err = (m % 2 == 1) ? errs[mid] : 0.5 * (errs[mid - 1] + errs[mid]);
  if (sigma) out->coverage_rate = (double)covered / (double)m;
  free(errs);
}

/* ========================================================================
 * Analytic scene renderer, SURVEY.md 8f row 4 (src/synth.cpp). Plain-C
 * restatement of scene_depth_at / scene_intensity_at / render_scene; pinned
 * against the reference's own render_scene (oracle/_ref) bit for bit in
 * tests/test_oracle_kats.py.
 * ======================================================================== */

/* splitmix (src/synth.cpp:16-21) */
static uint64_t sc_splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* hash_unit (src/synth.cpp:24-27) */
static double sc_hash_unit(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t h = sc_splitmix(a ^ sc_splitmix(b ^ sc_splitmix(c)));
  return (double)(h >> 11) * 0x1.0p-53;
}

/* gaussian_noise (src/synth.cpp:33-41) */
double bo_gaussian_noise(uint64_t seed, uint64_t stream, uint64_t index) {
  const double u1 = 1.0 - sc_hash_unit(seed, stream * 2 + 1, index);
  const double u2 = sc_hash_unit(seed, stream * 2 + 2, index);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* value_noise (src/synth.cpp:43-72) */
double bo_value_noise(double x, double y, uint64_t seed, int octaves, double base_scale) {
  double sum = 0.0, norm = 0.0, amp = 1.0, wavelength = base_scale;
  for (int o = 0; o < octaves; ++o) {
    const double gx = x / wavelength, gy = y / wavelength;
    const double fx = floor(gx), fy = floor(gy);
    const int64_t ix = (int64_t)fx, iy = (int64_t)fy;
    const double tx = (gx - fx) * (gx - fx) * (3.0 - 2.0 * (gx - fx));
    const double ty = (gy - fy) * (gy - fy) * (3.0 - 2.0 * (gy - fy));
    const uint64_t os = sc_splitmix(seed + (uint64_t)o);
    const double v00 = sc_hash_unit(os, (uint64_t)ix, (uint64_t)iy);
    const double v10 = sc_hash_unit(os, (uint64_t)(ix + 1), (uint64_t)iy);
    const double v01 = sc_hash_unit(os, (uint64_t)ix, (uint64_t)(iy + 1));
    const double v11 = sc_hash_unit(os, (uint64_t)(ix + 1), (uint64_t)(iy + 1));
    const double v = (1.0 - ty) * ((1.0 - tx) * v00 + tx * v10) + ty * ((1.0 - tx) * v01 + tx * v11);
    sum += amp * v;
    norm += amp;
    amp *= 0.5;
    wavelength *= 0.5;
  }
  return sum / norm;
}

/* reference_depth (src/synth.cpp:84-95) */
static double sc_reference_depth(const bo_scene* s) {
  const double fb = s->focal_px * s->baseline;
  if (s->surface == 1) return fb / s->disparity0;
  if (s->surface == 2) return s->background_depth;
  return fb / s->disparity;
}

/* sphere_hit (src/synth.cpp:104-113) on the ray (rx, ry, 1) */
static double sc_sphere_hit(const bo_scene* s, double rx, double ry, double rz) {
  const double zc = s->sphere_depth + s->sphere_radius;
  const double dd = rx * rx + ry * ry + rz * rz;
  const double dc = rz * zc;
  const double disc = dc * dc - dd * (zc * zc - s->sphere_radius * s->sphere_radius);
  if (disc < 0.0) return -1.0;
  const double t = (dc - sqrt(disc)) / dd;
  if (t <= 0.0) return -1.0;
  return t * rz;
}

/* scene_depth_at (src/synth.cpp:117-129); pixel_ray :98-101 */
static double sc_depth_at(const bo_scene* s, double x, double y) {
  const double fb = s->focal_px * s->baseline;
  if (s->surface == 1) return fb / (s->disparity0 + s->disparity_gradient * x);
  if (s->surface == 2) {
    const double rx = (x - 0.5 * (s->width - 1)) / s->focal_px;
    const double ry = (y - 0.5 * (s->height - 1)) / s->focal_px;
    const double z = sc_sphere_hit(s, rx, ry, 1.0);
    return z > 0.0 ? z : s->background_depth;
  }
  return fb / s->disparity;
}

/* scene_disparity_at (src/synth.cpp:131-133) */
double bo_scene_disparity_at(const bo_scene* s, double x, double y) {
  return s->focal_px * s->baseline / sc_depth_at(s, x, y);
}

/* texture_at (src/synth.cpp:137-158) */
static double sc_texture_at(const bo_scene* s, double wx, double wy) {
  const double wavelength = s->texture_scale * sc_reference_depth(s) / s->focal_px;
  if (s->texture == 0) {
    const double t = bo_value_noise(wx / wavelength * s->texture_scale,
                                    wy / wavelength * s->texture_scale, s->seed,
                                    s->texture_octaves, s->texture_scale);
    return 0.1 + 0.8 * t;
  }
  if (s->texture == 1) {
    const int64_t cx = (int64_t)floor(wx / wavelength);
    const int64_t cy = (int64_t)floor(wy / wavelength);
    return ((cx + cy) & 1) ? 0.8 : 0.2;
  }
  return 0.5;
}

/* facing_cos (src/synth.cpp:161-188) */
static double sc_facing_cos(const bo_scene* s, double x, double y, double z) {
  if (s->surface == 1) {
    const double d = s->disparity0 + s->disparity_gradient * x;
    const double fb = s->focal_px * s->baseline;
    const double dzdx = -fb * s->disparity_gradient / (d * d);
    const double xc = x - 0.5 * (s->width - 1);
    const double a = z / s->focal_px + xc / s->focal_px * dzdx;
    const double c = a / sqrt(a * a + dzdx * dzdx);
    return c > 0.0 ? c : 0.0; /* std::max(0.0, c) */
  }
  if (s->surface == 2) {
    const double rx = (x - 0.5 * (s->width - 1)) / s->focal_px;
    const double ry = (y - 0.5 * (s->height - 1)) / s->focal_px;
    const double zhit = sc_sphere_hit(s, rx, ry, 1.0);
    if (zhit <= 0.0) return 1.0;
    const double zc = s->sphere_depth + s->sphere_radius;
    const double nz = (zhit - zc) / s->sphere_radius;
    return -nz > 0.0 ? -nz : 0.0;
  }
  return 1.0;
}

static double sc_clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

/* scene_intensity_at (src/synth.cpp:192-207) */
double bo_scene_intensity_at(const bo_scene* s, double x, double y) {
  const double z = sc_depth_at(s, x, y);
  const double rx = (x - 0.5 * (s->width - 1)) / s->focal_px;
  const double ry = (y - 0.5 * (s->height - 1)) / s->focal_px;
  double v = sc_texture_at(s, rx * z, ry * z);
  const double cosa = sc_facing_cos(s, x, y, z);
  v *= s->ambient + (1.0 - s->ambient) * cosa;
  if (s->shading == 1) {
    const double hl = s->highlight_strength * pow(cosa, s->highlight_falloff);
    v = v * (1.0 - hl) + hl * 0.95;
  }
  return sc_clamp01(v);
}

/* render_scene (src/synth.cpp:209-284) */
int bo_render_scene(const bo_scene* s, float* left, float* right, double* ref_disparity,
                    double* ref_depth) {
  const int w = s->width, h = s->height;
  const double fb = s->focal_px * s->baseline;
  double dmax = 0.0;
  if (s->surface == 0) {
    dmax = s->disparity + 1.0;
  } else if (s->surface == 1) {
    const double g = s->disparity_gradient;
    dmax = g > 0.0 ? (s->disparity0 + g * (w - 1) + 1.0) / (1.0 - g) : s->disparity0 + 1.0;
  } else {
    dmax = fb / s->sphere_depth + 1.0;
  }
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t idx = (size_t)y * w + x;
      const double d_ref = bo_scene_disparity_at(s, x, y);
      ref_disparity[idx] = d_ref;
      ref_depth[idx] = fb / d_ref;
      double v = bo_scene_intensity_at(s, x, y);
      if (s->noise_std > 0.0) v += s->noise_std * bo_gaussian_noise(s->seed, 0, idx);
      left[idx] = (float)sc_clamp01(v);
      double hi = dmax, lo = 0.0;
      const double step = 0.25;
      for (double d = dmax - step; d > 0.0; d -= step) {
        if (d - bo_scene_disparity_at(s, x + d, y) <= 0.0) {
          lo = d;
          break;
        }
        hi = d;
      }
      for (int it = 0; it < 50; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid - bo_scene_disparity_at(s, x + mid, y) <= 0.0) lo = mid;
        else hi = mid;
      }
      const double d_star = 0.5 * (lo + hi);
      double rv = bo_scene_intensity_at(s, x + d_star, y);
      if (s->noise_std > 0.0) rv += s->noise_std * bo_gaussian_noise(s->seed, 1, idx);
      right[idx] = (float)sc_clamp01(rv);
    }
  return 0;
}
