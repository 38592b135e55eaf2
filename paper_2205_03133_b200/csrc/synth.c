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
#include "synth_core.h"

int pstereo_synth_blur_weights(double sigma, float* k, int cap) {
  const int r = (int)ceil(3.0 * sigma);
  if (!k || cap < 2 * r + 1) return r;
  double ks = 0.0;
  for (int i = -r; i <= r; ++i) ks += syn_exp(-(double)i * i / (2.0 * sigma * sigma));
  for (int i = -r; i <= r; ++i)
    k[i + r] = (float)(syn_exp(-(double)i * i / (2.0 * sigma * sigma)) / ks);
  return r;
}

/* separable Gaussian blur, kernel truncated at ceil(3 sigma), edge clamp;
 * float accumulation in tap order (bdis_synth.cu repeats it exactly) */
static void blur(float* img, int w, int h, double sigma) {
  const int r = pstereo_synth_blur_weights(sigma, NULL, 0);
  float* k = (float*)malloc(sizeof(float) * (size_t)(2 * r + 1));
  pstereo_synth_blur_weights(sigma, k, 2 * r + 1);
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

int pstereo_synth_check(const pstereo_synth_spec* s) {
  if (!s || s->width <= 0 || s->height <= 0 || (s->channels != 1 && s->channels != 3))
    return PSTEREO_ECONFIG;
  if (s->octaves < 1 || s->octaves > 16 || !(s->base_wavelength > 0.0) ||
      !(s->blur_sigma > 0.0) || !(s->blur_sigma <= 1024.0) || !(s->noise_sigma >= 0.0))
    return PSTEREO_ECONFIG;
  return PSTEREO_OK;
}

/* textureless discs until ~30% of the area is covered (config-1 stress) */
int pstereo_synth_discs(const pstereo_synth_spec* s, uint64_t key, double* dcx, double* dcy,
                        double* dr, double* dval) {
  const int w = s->width, h = s->height;
  const size_t n = (size_t)w * (size_t)h;
  uint8_t* cov = (uint8_t*)calloc(n, 1);
  size_t covered = 0;
  int nd = 0;
  for (int k = 0; k < SYN_MAX_DISCS && covered < (size_t)(0.30 * (double)n); ++k) {
    double cx, cy, r, val;
    syn_disc(key, k, w, h, &cx, &cy, &r, &val);
    dcx[nd] = cx;
    dcy[nd] = cy;
    dr[nd] = r;
    dval[nd] = val;
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
  return nd;
}

int pstereo_synth_pair(const pstereo_synth_spec* s, uint64_t seed, uint8_t* left,
                       uint8_t* right, float* disparity) {
  if (pstereo_synth_check(s)) return PSTEREO_ECONFIG;
  const int w = s->width, h = s->height, C = s->channels;
  const size_t n = (size_t)w * (size_t)h;
  const uint64_t key = syn_pair_key(seed);
  /* (2) disparity field */
  float* d = (float*)malloc(sizeof(float) * n);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) d[(size_t)y * w + x] = syn_white(key, x, y);
  blur(d, w, h, s->blur_sigma);
  float lo = d[0], hi = d[0];
  for (size_t i = 0; i < n; ++i) {
    lo = d[i] < lo ? d[i] : lo;
    hi = d[i] > hi ? d[i] : hi;
  }
  const float span = hi > lo ? hi - lo : 1.0f;
  for (size_t i = 0; i < n; ++i) d[i] = syn_normalise(d[i], lo, span, s->d_min, s->d_range);
  /* stress layout, shared by both views' scene texture */
  double dcx[SYN_MAX_DISCS], dcy[SYN_MAX_DISCS], dr[SYN_MAX_DISCS], dval[SYN_MAX_DISCS];
  int nd = 0;
  double hp_nx = 0.0, hp_ny = 0.0, hp_c = 0.0;
  if (s->stress) {
    nd = pstereo_synth_discs(s, key, dcx, dcy, dr, dval);
    syn_half_plane(key, w, h, &hp_nx, &hp_ny, &hp_c);
  }
  /* (1) scene texture in scene (left) coordinates, per channel */
  double* tex = (double*)malloc(sizeof(double) * n * (size_t)C);
  for (int c = 0; c < C; ++c) {
    const uint64_t ck = syn_channel_key(key, c);
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x)
        tex[((size_t)y * w + x) * (size_t)C + (size_t)c] =
            syn_texture(x, y, ck, s->octaves, s->base_wavelength, nd, dcx, dcy, dr, dval);
  }
  /* views */
  for (int view = 0; view < 2; ++view) {
    uint8_t* out = view == 0 ? left : right;
    const double gain = syn_gain(key, s->stress, view);
    double bx[SYN_BLOBS], by[SYN_BLOBS], bs[SYN_BLOBS];
    if (s->stress)
      for (int b = 0; b < SYN_BLOBS; ++b) syn_blob(key, view, b, w, h, &bx[b], &by[b], &bs[b]);
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        const size_t i = (size_t)y * w + x;
        double spec = 0.0, dark = 1.0;
        if (s->stress) {
          spec = syn_specular(bx, by, bs, x, y);
          if (hp_nx * x + hp_ny * y > hp_c) dark = 0.4;
        }
        for (int c = 0; c < C; ++c) {
          double v;
          if (view == 0) {
            v = tex[i * (size_t)C + (size_t)c];
          } else {
            v = syn_right_tex(tex + (size_t)y * w * (size_t)C, w, C, c, x, d[i]);
            v += s->noise_sigma * syn_gauss3(key ^ 0xA015Eull, (uint64_t)c, i);
          }
          out[i * (size_t)C + (size_t)c] = syn_finish(v, gain, dark, spec);
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
