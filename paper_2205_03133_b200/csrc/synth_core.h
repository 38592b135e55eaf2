/*
 * synth_core.h -- the per-element arithmetic of the synthetic pair generator,
 * shared verbatim by the host generator (synth.c, plain C) and the device
 * generator (bdis_synth.cu). Both sides compile it without FMA contraction
 * (gcc -ffp-contract=off, nvcc --fmad=false) and use only IEEE-exact
 * operations (+ - * / sqrt floor, integer hashing), so the two generators
 * produce the same bytes.
 *
 * libm's exp/log/cos are not part of that set (glibc and CUDA differ by an
 * ulp here and there), so the three transcendentals the recipe needs -- the
 * Box-Muller draw (log, cos) and the Gaussian blur / specular weights (exp) --
 * are evaluated here with fixed polynomials: accurate to a few ulp, and above
 * all the same on every host and device. The hash is the splitmix64
 * finaliser, the same construction as the reference's keyed noise
 * (src/synth.cpp:16-27).
 */
#ifndef PSTEREO_SYNTH_CORE_H
#define PSTEREO_SYNTH_CORE_H

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define SYN_FN static __host__ __device__ __forceinline__
#define SYN_FLOOR(x) floor(x)
#define SYN_SQRT(x) sqrt(x)
#else
#include <math.h>
#define SYN_FN static inline
#define SYN_FLOOR(x) floor(x)
#define SYN_SQRT(x) sqrt(x)
#endif

SYN_FN uint64_t syn_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* uniform [0,1) keyed by (a, b, c) */
SYN_FN double syn_unit3(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t h = syn_mix64(a ^ syn_mix64(b ^ syn_mix64(c ^ 0x5851F42D4C957F2Dull)));
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

SYN_FN double syn_from_bits(uint64_t b) {
  double d;
  memcpy(&d, &b, sizeof d);
  return d;
}

SYN_FN uint64_t syn_to_bits(double d) {
  uint64_t b;
  memcpy(&b, &d, sizeof b);
  return b;
}

/* exp(x) for x <= ~700: x = k ln2 + r, |r| <= ln2/2, Taylor to r^13, times 2^k.
 * Returns 0 below -700 (the generator's weights there are far below any
 * contribution that survives rounding to uint8 / float). */
SYN_FN double syn_exp(double x) {
  if (!(x > -700.0)) return 0.0;
  if (x > 700.0) x = 700.0;
  const double k = SYN_FLOOR(x * 1.4426950408889634 + 0.5);
  const double r = (x - k * 6.93147180369123816490e-01) - k * 1.90821492927058770002e-10;
  double p = 1.6059043836821613e-10;             /* 1/13! */
  p = p * r + 2.0876756987868099e-09;            /* 1/12! */
  p = p * r + 2.5052108385441720e-08;            /* 1/11! */
  p = p * r + 2.7557319223985893e-07;            /* 1/10! */
  p = p * r + 2.7557319223985888e-06;            /* 1/9!  */
  p = p * r + 2.4801587301587302e-05;            /* 1/8!  */
  p = p * r + 1.9841269841269841e-04;            /* 1/7!  */
  p = p * r + 1.3888888888888889e-03;            /* 1/6!  */
  p = p * r + 8.3333333333333332e-03;            /* 1/5!  */
  p = p * r + 4.1666666666666664e-02;            /* 1/4!  */
  p = p * r + 1.6666666666666666e-01;            /* 1/3!  */
  p = p * r + 0.5;
  p = p * r + 1.0;
  p = p * r + 1.0;
  const int64_t e = (int64_t)k + 1023;           /* k in [-1010, 1010] */
  return p * syn_from_bits((uint64_t)e << 52);
}

/* log(u) for normal u > 0: u = m 2^e with m in [sqrt(1/2), sqrt(2)],
 * log m = 2 atanh((m-1)/(m+1)) as a series in s = f^2 (|f| <= 0.1716). */
SYN_FN double syn_log(double u) {
  const uint64_t b = syn_to_bits(u);
  int64_t e = (int64_t)((b >> 52) & 0x7FF) - 1023;
  double m = syn_from_bits((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull);
  if (m > 1.4142135623730951) {
    m *= 0.5;
    e += 1;
  }
  const double f = (m - 1.0) / (m + 1.0);
  const double s = f * f;
  double p = 1.0 / 23.0;
  p = p * s + 1.0 / 21.0;
  p = p * s + 1.0 / 19.0;
  p = p * s + 1.0 / 17.0;
  p = p * s + 1.0 / 15.0;
  p = p * s + 1.0 / 13.0;
  p = p * s + 1.0 / 11.0;
  p = p * s + 1.0 / 9.0;
  p = p * s + 1.0 / 7.0;
  p = p * s + 1.0 / 5.0;
  p = p * s + 1.0 / 3.0;
  p = p * s + 1.0;
  const double de = (double)e;
  return de * 6.93147180369123816490e-01 + ((2.0 * f) * p + de * 1.90821492927058770002e-10);
}

/* cos(x) and sin(x) for |x| <= pi/4, Taylor to x^18 / x^17. */
SYN_FN double syn_cos_small(double x) {
  const double z = x * x;
  double p = 1.5619206968586225e-16;             /* 1/18! */
  p = p * -z + 4.7794773323873853e-14;           /* 1/16! */
  p = p * -z + 1.1470745597729725e-11;           /* 1/14! */
  p = p * -z + 2.0876756987868099e-09;           /* 1/12! */
  p = p * -z + 2.7557319223985893e-07;           /* 1/10! */
  p = p * -z + 2.4801587301587302e-05;           /* 1/8!  */
  p = p * -z + 1.3888888888888889e-03;           /* 1/6!  */
  p = p * -z + 4.1666666666666664e-02;           /* 1/4!  */
  p = p * -z + 0.5;
  p = p * -z + 1.0;
  return p;
}

SYN_FN double syn_sin_small(double x) {
  const double z = x * x;
  double p = 2.8114572543455206e-15;             /* 1/17! */
  p = p * -z + 7.6471637318198164e-13;           /* 1/15! */
  p = p * -z + 1.6059043836821613e-10;           /* 1/13! */
  p = p * -z + 2.5052108385441720e-08;           /* 1/11! */
  p = p * -z + 2.7557319223985888e-06;           /* 1/9!  */
  p = p * -z + 1.9841269841269841e-04;           /* 1/7!  */
  p = p * -z + 8.3333333333333332e-03;           /* 1/5!  */
  p = p * -z + 1.6666666666666666e-01;           /* 1/3!  */
  p = p * -z + 1.0;
  return p * x;
}

/* cos(2 pi t) for t in [0, 1): quadrant q = floor(4t) and r = t - q/4 are
 * exact; r > 1/8 is folded to the complementary angle. */
SYN_FN double syn_cos2pi(double t) {
  const double q = SYN_FLOOR(t * 4.0);
  double r = t - q * 0.25;
  const int quad = (int)q & 3;
  const int fold = r > 0.125;
  if (fold) r = 0.25 - r;
  const double x = r * 6.283185307179586;
  /* want cos(2 pi r0) for quadrants 0/2, sin(2 pi r0) for 1/3 (r0 = unfolded) */
  const int use_cos = ((quad & 1) == 0) != fold;
  const double v = use_cos ? syn_cos_small(x) : syn_sin_small(x);
  return (quad == 1 || quad == 2) ? -v : v;
}

/* standard normal draw keyed by (a, b, c): Box-Muller on two keyed uniforms
 * (the reference's gaussian_noise construction, src/synth.cpp:33-40). */
SYN_FN double syn_gauss3(uint64_t a, uint64_t b, uint64_t c) {
  const double u1 = 1.0 - syn_unit3(a, b * 2 + 1, c); /* (0, 1] */
  const double u2 = syn_unit3(a, b * 2 + 2, c);
  return SYN_SQRT(-2.0 * syn_log(u1)) * syn_cos2pi(u2);
}

SYN_FN double syn_smooth(double t) { return t * t * (3.0 - 2.0 * t); }

/* multi-octave value noise in [0,1] (the construction of the reference's
 * value_noise, src/synth.cpp:43-72). */
SYN_FN double syn_value_noise(double x, double y, uint64_t key, int octaves, double wavelength) {
  double sum = 0.0, norm = 0.0, amp = 1.0;
  for (int o = 0; o < octaves; ++o) {
    const double gx = x / wavelength, gy = y / wavelength;
    const double fx = SYN_FLOOR(gx), fy = SYN_FLOOR(gy);
    const int64_t ix = (int64_t)fx, iy = (int64_t)fy;
    const double tx = syn_smooth(gx - fx), ty = syn_smooth(gy - fy);
    const uint64_t ok = syn_mix64(key + (uint64_t)o * 0x1000193ull);
    const double v00 = syn_unit3(ok, (uint64_t)ix, (uint64_t)iy);
    const double v10 = syn_unit3(ok, (uint64_t)(ix + 1), (uint64_t)iy);
    const double v01 = syn_unit3(ok, (uint64_t)ix, (uint64_t)(iy + 1));
    const double v11 = syn_unit3(ok, (uint64_t)(ix + 1), (uint64_t)(iy + 1));
    const double v = (1.0 - ty) * ((1.0 - tx) * v00 + tx * v10) +
                     ty * ((1.0 - tx) * v01 + tx * v11);
    sum += amp * v;
    norm += amp;
    amp *= 0.5;
    wavelength *= 0.5;
  }
  return sum / norm;
}

/* ---- keys and per-pair constants ---- */

SYN_FN uint64_t syn_pair_key(uint64_t seed) {
  return syn_mix64(seed * 0x9E3779B97F4A7C15ull + 0xB5AD4ECEDA1CE2A9ull);
}

/* white noise of the disparity field at (x, y) */
SYN_FN float syn_white(uint64_t key, int x, int y) {
  return (float)syn_unit3(key ^ 0xD15Full, (uint64_t)x, (uint64_t)y);
}

SYN_FN uint64_t syn_channel_key(uint64_t key, int c) {
  return syn_mix64(key + 0x7E57ull + (uint64_t)c * 0x51ED27ull);
}

#define SYN_MAX_DISCS 256
#define SYN_BLOBS 10

/* textureless disc k (config-1 stress): centre, radius, intensity */
SYN_FN void syn_disc(uint64_t key, int k, int w, int h, double* cx, double* cy, double* r,
                     double* val) {
  *cx = syn_unit3(key, 101, (uint64_t)k) * w;
  *cy = syn_unit3(key, 102, (uint64_t)k) * h;
  *r = 20.0 + 40.0 * syn_unit3(key, 103, (uint64_t)k);
  *val = 40.0 + 175.0 * syn_unit3(key, 104, (uint64_t)k);
}

/* darkened half-plane: n.x > c */
SYN_FN void syn_half_plane(uint64_t key, int w, int h, double* nx, double* ny, double* c) {
  const double t = syn_unit3(key, 201, 0);
  *nx = syn_cos2pi(t);
  *ny = syn_cos2pi(t < 0.75 ? t + 0.25 : t - 0.75); /* sin(2 pi t) = cos(2 pi (t - 1/4)) */
  *c = *nx * (syn_unit3(key, 202, 0) * w) + *ny * (syn_unit3(key, 203, 0) * h);
}

SYN_FN double syn_gain(uint64_t key, int stress, int view) {
  return stress ? 0.8 + 0.4 * syn_unit3(key, 301, (uint64_t)view) : 1.0;
}

/* specular blob b of a view: centre and sigma */
SYN_FN void syn_blob(uint64_t key, int view, int b, int w, int h, double* bx, double* by,
                     double* bs) {
  *bx = syn_unit3(key, 400 + (uint64_t)view, (uint64_t)b) * w;
  *by = syn_unit3(key, 410 + (uint64_t)view, (uint64_t)b) * h;
  *bs = 5.0 + 10.0 * syn_unit3(key, 420 + (uint64_t)view, (uint64_t)b);
}

SYN_FN double syn_clamp255(double v) { return v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v); }

/* round half to even (lrint under the default mode) of a value in [0, 255] */
SYN_FN uint8_t syn_round_u8(double v) {
  const double c = syn_clamp255(v);
  const double f = SYN_FLOOR(c);
  const double d = c - f;
  double r = f;
  if (d > 0.5 || (d == 0.5 && ((int64_t)f & 1))) r = f + 1.0;
  return (uint8_t)(int)r;
}

/* final photometric model of one sample: v -> (v * gain) * dark + spec */
SYN_FN uint8_t syn_finish(double v, double gain, double dark, double spec) {
  return syn_round_u8((v * gain) * dark + spec);
}

/* disparity normalisation d = d_min + d_range * (b - lo) / span */
SYN_FN float syn_normalise(float b, float lo, float span, double d_min, double d_range) {
  return (float)(d_min + d_range * (double)((b - lo) / span));
}

/* right-view texture sample at x + d (bilinear, edge clamp), reference
 * convention x_right = x_left - d (proj/README.md:186-189); `row` is the
 * texture row, C channels interleaved. */
SYN_FN double syn_right_tex(const double* row, int w, int C, int c, int x, float d) {
  double sx = x + (double)d;
  if (sx > w - 1.0) sx = w - 1.0;
  if (sx < 0.0) sx = 0.0;
  const int x0 = (int)sx;
  const int x1 = x0 + 1 < w ? x0 + 1 : w - 1;
  const double f = sx - x0;
  return (1.0 - f) * row[(size_t)x0 * C + c] + f * row[(size_t)x1 * C + c];
}

/* scene texture of channel key ck at pixel (x, y); the last textureless disc
 * containing the pixel overrides the noise */
SYN_FN double syn_texture(int x, int y, uint64_t ck, int octaves, double wavelength, int nd,
                          const double* dcx, const double* dcy, const double* dr,
                          const double* dval) {
  double v = 255.0 * syn_value_noise(x + 0.5, y + 0.5, ck, octaves, wavelength);
  for (int k = 0; k < nd; ++k) {
    const double dx = x - dcx[k], dy = y - dcy[k];
    if (dx * dx + dy * dy <= dr[k] * dr[k]) v = dval[k];
  }
  return v;
}

/* saturating specular term of a view at (x, y) */
SYN_FN double syn_specular(const double* bx, const double* by, const double* bs, int x, int y) {
  double spec = 0.0;
  for (int b = 0; b < SYN_BLOBS; ++b) {
    const double dx = x - bx[b], dy = y - by[b];
    spec += 400.0 * syn_exp(-(dx * dx + dy * dy) / (2.0 * bs[b] * bs[b]));
  }
  return spec;
}

/* Gaussian weights of the disparity blur (kernel truncated at ceil(3 sigma)),
 * computed on the host only (synth.c) and handed to the device generator.
 * Returns the radius r; k receives 2r+1 weights when cap allows. */
#if !defined(__CUDACC__)
int pstereo_synth_blur_weights(double sigma, float* k, int cap);
#else
extern "C" int pstereo_synth_blur_weights(double sigma, float* k, int cap);
#endif

#endif /* PSTEREO_SYNTH_CORE_H */
