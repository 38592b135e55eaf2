/*
 * synth.c -- deterministic synthetic rectified stereo pairs for the
 * BASELINE.json configs (host C; no GPU needed).
 *
 * Stand-in for the paper's datasets (synthetic colon / SCARED / SERV-CT /
 * Hamlyn), which are not available here. Follows the
 * recipe in BASELINE.json configs[0..4]:
 *   (1) left view: multi-octave value noise (seeded hash lattice, smoothstep
 *       interpolation -- the same construction idea as the reference's
 *       value_noise, src/synth.cpp:43-72), scaled to [0,255], rounded;
 *   (2) disparity: d = d_min + d_range * s, s = min-max normalised Gaussian
 *       blur (sigma px, kernel truncated at 3 sigma, edge-clamped) of seeded
 *       uniform white noise;
 *   (3) right view: the left view bilinearly sampled at x + d (reference
 *       convention x_right = x_left - d, proj/README.md:186-189), plus
 *       N(0, noise_sigma) DN, clamped and rounded to uint8;
 *   (4) optional photometric stress (config 1): textureless discs covering
 *       ~30% of the scene, per-view gain U(0.8,1.2), saturated specular blobs
 *       placed independently per view, x0.4 darkening of a random half-plane.
 * 3-channel variants draw independent octaves per channel.
 * Everything is integer-hash driven, so a (spec, seed) pair always produces
 * the same bytes on every host.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/pstereo_gpu.h"

static uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* uniform [0,1) keyed by (a, b, c) */
static double unit3(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t h = mix64(a ^ mix64(b ^ mix64(c ^ 0x5851F42D4C957F2Dull)));
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

static double gauss3(uint64_t a, uint64_t b, uint64_t c) {
  const double u1 = 1.0 - unit3(a, b * 2 + 1, c);
  const double u2 = unit3(a, b * 2 + 2, c);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

static double smooth(double t) { return t * t * (3.0 - 2.0 * t); }

static double value_noise(double x, double y, uint64_t key, int octaves,
                          double wavelength) {
  double sum = 0.0, norm = 0.0, amp = 1.0;
  for (int o = 0; o < octaves; ++o) {
    const double gx = x / wavelength, gy = y / wavelength;
    const double fx = floor(gx), fy = floor(gy);
    const int64_t ix = (int64_t)fx, iy = (int64_t)fy;
    const double tx = smooth(gx - fx), ty = smooth(gy - fy);
    const uint64_t ok = mix64(key + (uint64_t)o * 0x1000193ull);
    const double v00 = unit3(ok, (uint64_t)ix, (uint64_t)iy);
    const double v10 = unit3(ok, (uint64_t)(ix + 1), (uint64_t)iy);
    const double v01 = unit3(ok, (uint64_t)ix, (uint64_t)(iy + 1));
    const double v11 = unit3(ok, (uint64_t)(ix + 1), (uint64_t)(iy + 1));
    const double v = (1.0 - ty) * ((1.0 - tx) * v00 + tx * v10) +
                     ty * ((1.0 - tx) * v01 + tx * v11);
    sum += amp * v;
    norm += amp;
    amp *= 0.5;
    wavelength *= 0.5;
  }
  return sum / norm;
}

/* separable Gaussian blur, kernel truncated at ceil(3 sigma), edge clamp */
static void blur(float* img, int w, int h, double sigma) {
  const int r = (int)ceil(3.0 * sigma);
  float* k = (float*)malloc(sizeof(float) * (size_t)(2 * r + 1));
  double ks = 0.0;
  for (int i = -r; i <= r; ++i) ks += exp(-(double)i * i / (2.0 * sigma * sigma));
  for (int i = -r; i <= r; ++i)
    k[i + r] = (float)(exp(-(double)i * i / (2.0 * sigma * sigma)) / ks);
  const int n = w > h ? w : h;
  float* line = (float*)malloc(sizeof(float) * (size_t)(n + 2 * r));
  float* tmp = (float*)malloc(sizeof(float) * (size_t)n);
  for (int y = 0; y < h; ++y) {
    float* row = img + (size_t)y * w;
    for (int i = -r; i < w + r; ++i) line[i + r] = row[i < 0 ? 0 : (i >= w ? w - 1 : i)];
    for (int x = 0; x < w; ++x) {
      float acc = 0.0f;
      const float* src = line + x;
      for (int i = 0; i <= 2 * r; ++i) acc += k[i] * src[i];
      tmp[x] = acc;
    }
    memcpy(row, tmp, sizeof(float) * (size_t)w);
  }
  for (int x = 0; x < w; ++x) {
    for (int i = -r; i < h + r; ++i)
      line[i + r] = img[(size_t)(i < 0 ? 0 : (i >= h ? h - 1 : i)) * w + x];
    for (int y = 0; y < h; ++y) {
      float acc = 0.0f;
      const float* src = line + y;
      for (int i = 0; i <= 2 * r; ++i) acc += k[i] * src[i];
      tmp[y] = acc;
    }
    for (int y = 0; y < h; ++y) img[(size_t)y * w + x] = tmp[y];
  }
  free(k);
  free(line);
  free(tmp);
}

static double clamp255(double v) { return v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v); }

void pstereo_synth_default(pstereo_synth_spec* s, int config) {
  memset(s, 0, sizeof *s);
  s->width = 640;
  s->height = 480;
  s->channels = 1;
  s->seed = 0;
  s->octaves = 4;
  s->base_wavelength = 32.0;
  s->d_min = 5.0;
  s->d_range = 35.0;
  s->blur_sigma = 40.0;
  s->noise_sigma = 2.0;
  s->stress = 0;
  if (config == 1) {
    s->seed = 1;
    s->stress = 1;
  } else if (config == 3) {
    s->width = 1280;
    s->height = 1024;
    s->octaves = 5;
    s->base_wavelength = 64.0;
    s->d_min = 8.0;
    s->d_range = 120.0;
    s->blur_sigma = 80.0;
  }
}

int pstereo_synth_pair(const pstereo_synth_spec* s, uint64_t seed, uint8_t* left,
                       uint8_t* right, float* disparity) {
  const int w = s->width, h = s->height, C = s->channels;
  if (w <= 0 || h <= 0 || (C != 1 && C != 3)) return PSTEREO_ECONFIG;
  const size_t n = (size_t)w * (size_t)h;
  const uint64_t key = mix64(seed * 0x9E3779B97F4A7C15ull + 0xB5AD4ECEDA1CE2A9ull);
  /* (2) disparity field */
  float* d = (float*)malloc(sizeof(float) * n);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) d[(size_t)y * w + x] = (float)unit3(key ^ 0xD15Full, (uint64_t)x, (uint64_t)y);
  blur(d, w, h, s->blur_sigma);
  float lo = d[0], hi = d[0];
  for (size_t i = 0; i < n; ++i) {
    lo = d[i] < lo ? d[i] : lo;
    hi = d[i] > hi ? d[i] : hi;
  }
  const float span = hi > lo ? hi - lo : 1.0f;
  for (size_t i = 0; i < n; ++i) d[i] = (float)(s->d_min + s->d_range * (double)((d[i] - lo) / span));
  /* stress layout, shared by both views' scene texture */
  enum { MAXD = 256 };
  double dcx[MAXD], dcy[MAXD], dr[MAXD], dval[MAXD];
  int nd = 0;
  double hp_nx = 0.0, hp_ny = 0.0, hp_c = 0.0;
  if (s->stress) {
    /* textureless discs until ~30% of the area is covered */
    uint8_t* cov = (uint8_t*)calloc(n, 1);
    size_t covered = 0;
    for (int k = 0; k < MAXD && covered < (size_t)(0.30 * (double)n); ++k) {
      const double cx = unit3(key, 101, (uint64_t)k) * w;
      const double cy = unit3(key, 102, (uint64_t)k) * h;
      const double r = 20.0 + 40.0 * unit3(key, 103, (uint64_t)k);
      dcx[nd] = cx;
      dcy[nd] = cy;
      dr[nd] = r;
      dval[nd] = 40.0 + 175.0 * unit3(key, 104, (uint64_t)k);
      ++nd;
      const int x0 = (int)fmax(0.0, cx - r), x1 = (int)fmin(w - 1.0, cx + r);
      const int y0 = (int)fmax(0.0, cy - r), y1 = (int)fmin(h - 1.0, cy + r);
      for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) {
          const double dx = x - cx, dy = y - cy;
          if (dx * dx + dy * dy <= r * r && !cov[(size_t)y * w + x]) {
            cov[(size_t)y * w + x] = 1;
            ++covered;
          }
        }
    }
    free(cov);
    const double ang = 6.283185307179586 * unit3(key, 201, 0);
    hp_nx = cos(ang);
    hp_ny = sin(ang);
    hp_c = hp_nx * (unit3(key, 202, 0) * w) + hp_ny * (unit3(key, 203, 0) * h);
  }
  /* (1) scene texture in scene (left) coordinates, per channel */
  double* tex = (double*)malloc(sizeof(double) * n * (size_t)C);
  for (int c = 0; c < C; ++c) {
    const uint64_t ck = mix64(key + 0x7E57ull + (uint64_t)c * 0x51ED27ull);
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        double v = 255.0 * value_noise(x + 0.5, y + 0.5, ck, s->octaves, s->base_wavelength);
        for (int k = 0; k < nd; ++k) {
          const double dx = x - dcx[k], dy = y - dcy[k];
          if (dx * dx + dy * dy <= dr[k] * dr[k]) v = dval[k];
        }
        tex[((size_t)y * w + x) * (size_t)C + (size_t)c] = v;
      }
  }
  /* views */
  for (int view = 0; view < 2; ++view) {
    uint8_t* out = view == 0 ? left : right;
    const double gain = s->stress ? 0.8 + 0.4 * unit3(key, 301, (uint64_t)view) : 1.0;
    double bx[10], by[10], bs[10];
    if (s->stress)
      for (int b = 0; b < 10; ++b) {
        bx[b] = unit3(key, 400 + (uint64_t)view, (uint64_t)b) * w;
        by[b] = unit3(key, 410 + (uint64_t)view, (uint64_t)b) * h;
        bs[b] = 5.0 + 10.0 * unit3(key, 420 + (uint64_t)view, (uint64_t)b);
      }
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        const size_t i = (size_t)y * w + x;
        double spec = 0.0, dark = 1.0;
        if (s->stress) {
          for (int b = 0; b < 10; ++b) {
            const double dx = x - bx[b], dy = y - by[b];
            spec += 400.0 * exp(-(dx * dx + dy * dy) / (2.0 * bs[b] * bs[b]));
          }
          if (hp_nx * x + hp_ny * y > hp_c) dark = 0.4;
        }
        for (int c = 0; c < C; ++c) {
          double v;
          if (view == 0) {
            v = tex[i * (size_t)C + (size_t)c];
          } else {
            /* right(x) = left(x + d), bilinear, edge clamp */
            double sx = x + (double)d[i];
            if (sx > w - 1.0) sx = w - 1.0;
            const int x0 = (int)sx;
            const int x1 = x0 + 1 < w ? x0 + 1 : w - 1;
            const double f = sx - x0;
            const double* row = tex + (size_t)y * w * (size_t)C;
            v = (1.0 - f) * row[(size_t)x0 * C + c] + f * row[(size_t)x1 * C + c];
            v += s->noise_sigma * gauss3(key ^ 0xA015Eull, (uint64_t)c, i);
          }
          v = (v * gain) * dark + spec;
          out[i * (size_t)C + (size_t)c] = (uint8_t)lrint(clamp255(v));
        }
      }
  }
  if (disparity) memcpy(disparity, d, sizeof(float) * n);
  free(d);
  free(tex);
  return PSTEREO_OK;
}

typedef struct synth_job {
  const pstereo_synth_spec* s;
  uint64_t seed0;
  int n, next_lock_dummy;
  uint8_t* left;
  uint8_t* right;
  int* counter;
  pthread_mutex_t* mu;
  int rc;
} synth_job;

static void* synth_worker(void* arg) {
  synth_job* j = (synth_job*)arg;
  const size_t stride = (size_t)j->s->width * (size_t)j->s->height * (size_t)j->s->channels;
  for (;;) {
    pthread_mutex_lock(j->mu);
    const int k = (*j->counter)++;
    pthread_mutex_unlock(j->mu);
    if (k >= j->n) break;
    const int rc = pstereo_synth_pair(j->s, j->seed0 + (uint64_t)k, j->left + stride * (size_t)k,
                                      j->right + stride * (size_t)k, NULL);
    if (rc) j->rc = rc;
  }
  return NULL;
}

int pstereo_synth_batch(const pstereo_synth_spec* s, int n_pairs, uint64_t seed0,
                        uint8_t* left, uint8_t* right, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  pthread_t th[64];
  synth_job jobs[64];
  int counter = 0;
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  for (int t = 0; t < threads; ++t) {
    jobs[t].s = s;
    jobs[t].seed0 = seed0;
    jobs[t].n = n_pairs;
    jobs[t].left = left;
    jobs[t].right = right;
    jobs[t].counter = &counter;
    jobs[t].mu = &mu;
    jobs[t].rc = 0;
    pthread_create(&th[t], NULL, synth_worker, &jobs[t]);
  }
  int rc = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    if (jobs[t].rc) rc = jobs[t].rc;
  }
  return rc;
}
