// bdis_device.cuh -- device-side numerics shared by the BDIS kernels.
//
// Everything here mirrors the reference's double/float arithmetic operation
// for operation (the TU is compiled with --fmad=false and the critical spots
// use explicit _rn intrinsics), so the GPU produces the same bits as the x86-64
// SSE2 reference build. Citations: src/ = proj/src/, inc/ = proj/include/pstereo/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bdis {

constexpr int kMaxPatch = 32;
constexpr int kMaxWin = 33;  // 2 * PSTEREO_MAX_OFFSETS + 1

enum Stage : uint8_t { kSkipped = 0, kSolved = 1, kConverged = 2, kAccepted = 3 };

// Patch lattice of one level (src/coarse_to_fine.cpp:51-88). Centre k < n-1 is
// c0 + k*stride, the last one is clamped to cmax, so the footprint of patch k
// starts at k*stride (k < n-1) or at L - size (k = n-1): all integers.
struct Grid {
  int nx, ny, stride, size;
  double c0, cmax_x, cmax_y;
  int lastx0, lasty0;
};

// Row pitch (floats) of the padded right view: w + 1 values (the duplicated
// last column) rounded up to a multiple of four, so rows start 16-byte aligned
// and the pyramid stores them as float4.
__host__ __device__ __forceinline__ int rpad_pitch(int w) { return (w + 4) & ~3; }

// One pyramid level of a batch of pairs: planes are [pair][h][w].
struct Level {
  int e, w, h;
  long long plane;
  const float* left;
  const uint8_t* lvalid;
  const float* right;
  const uint8_t* rvalid;
  float* grad;     // gradient_x of left (src/pyramid.cpp:30-42)
  uint8_t* lq;     // 4-tap validity of left at (x,y) (inc/image.hpp:68-69)
  uint8_t* rq;     // 4-tap validity of right at (x,y)
  float* rpad;     // right view, rows of rpad_pitch(w) (rpad[w] = rpad[w-1]: the
                   // x1 = min(x0+1, w-1) clamp of inc/image.hpp:60)
  Grid g;
  // per-patch records [pair][ny][nx] (PatchEstimate, inc/coarse_to_fine.hpp:39-47)
  double* u;
  double* prob;
  double* post;
  double* sigma;
  uint8_t* stage;
  double level_w;  // level_weight(e, levels), src/coarse_to_fine.cpp:90-94
};

// inc/fast_exp.hpp:16-28 -- Schraudolph's exponent-field trick, double layout.
__device__ __forceinline__ double fast_exp(double x) {
  if (x < -30.0) return 0.0;
  const double scale = 4503599627370496.0 / 0.6931471805599453;
  const long long bias = (1023LL << 52) - (60801LL << 32);
  const long long bits = __double2ll_rz(__dmul_rn(x, scale)) + bias;
  return __longlong_as_double(bits);
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}

// std::lround: half away from zero.
__device__ __forceinline__ int lround_i(double v) { return (int)llround(v); }

// Weighted gather of the accepted patches of level P that cover pixel (x, y),
// in ascending patch index -- the exact accumulation order of fuse_level's
// scatter (src/coarse_to_fine.cpp:120-135), so the sums are bit-identical.
struct Fused {
  double sw, swu, swp, sw2s;
};

// Global-memory records of one level (the default accessor of gather_with).
struct GlobalRecords {
  const Level& P;
  long long base;
  __device__ __forceinline__ uint8_t stage(int ky, int kx) const {
    return P.stage[base + (long long)ky * P.g.nx + kx];
  }
  __device__ __forceinline__ double prob(int ky, int kx) const {
    return P.prob[base + (long long)ky * P.g.nx + kx];
  }
  __device__ __forceinline__ double u(int ky, int kx) const {
    return P.u[base + (long long)ky * P.g.nx + kx];
  }
  __device__ __forceinline__ double sigma(int ky, int kx) const {
    return P.sigma[base + (long long)ky * P.g.nx + kx];
  }
};

// Covering patches of one pixel coordinate along an axis: regular patches
// [lo, hi] (starts k*stride) plus the clamped last patch when `last`.
struct Cover {
  int lo, hi;
  bool last;
};

__device__ __forceinline__ Cover cover_of(int x, int n, int s, int st, int last0) {
  Cover c;
  c.lo = (x - s + 1 <= 0) ? 0 : (x - s + 1 + st - 1) / st;
  c.hi = min(n - 2, x / st);
  c.last = x >= last0;
  return c;
}

template <bool kProb, bool kVar, typename Rec>
__device__ __forceinline__ Fused gather_cover(const Grid& g, const Rec& rec, int x, int y,
                                              Cover cx, Cover cy,
                                              const double* __restrict__ mask) {
  const int s = g.size, st = g.stride;
  Fused f{0.0, 0.0, 0.0, 0.0};
  // fuse_level visits accepted patches only (src/coarse_to_fine.cpp:120-135);
  // the records of the others hold prob = u = sigma = 0 (k_patches phase 3),
  // so they add w = +0.0, which leaves every sum bit-identical (the sums start
  // at +0.0 and never become -0.0) -- no dependent stage load
  auto add = [&](int ky, int kx, double m) {
    const double pr = rec.prob(ky, kx);
    const double w = __dmul_rn(pr, m);
    f.sw = __dadd_rn(f.sw, w);
    f.swu = __dadd_rn(f.swu, __dmul_rn(w, rec.u(ky, kx)));
    if (kProb) f.swp = __dadd_rn(f.swp, __dmul_rn(w, pr));
    if (kVar) {
      const double sk = rec.sigma(ky, kx);
      f.sw2s = __dadd_rn(f.sw2s, __dmul_rn(__dmul_rn(__dmul_rn(w, w), sk), sk));
    }
  };
  auto row = [&](int ky, int y0) {
    const double* mrow = mask + (y - y0) * s;
    for (int kx = cx.lo; kx <= cx.hi; ++kx) add(ky, kx, mrow[x - kx * st]);
    if (cx.last) add(ky, g.nx - 1, mrow[x - g.lastx0]);
  };
  // ascending patch index: rows ky ascending, columns kx ascending
  for (int ky = cy.lo; ky <= cy.hi; ++ky) row(ky, ky * st);
  if (cy.last) row(g.ny - 1, g.lasty0);
  return f;
}

template <bool kProb, bool kVar, typename Rec>
__device__ __forceinline__ Fused gather_with(const Grid& g, const Rec& rec, int x, int y,
                                             const double* __restrict__ mask) {
  return gather_cover<kProb, kVar>(g, rec, x, y,
                                   cover_of(x, g.nx, g.size, g.stride, g.lastx0),
                                   cover_of(y, g.ny, g.size, g.stride, g.lasty0), mask);
}

// Patches of a level covering pixel columns [xa, xb] form one contiguous index
// range (the clamped last patch has the largest start); same for rows.
__device__ __forceinline__ void covering_range(int a, int b, int n, int s, int st, int last0,
                                               int* k0, int* k1) {
  *k0 = (a - s + 1 <= 0) ? 0 : min(n - 1, (a - s + 1 + st - 1) / st);
  *k1 = b >= last0 ? n - 1 : min(n - 2, b / st);
  if (*k1 < *k0) *k1 = *k0;
}

template <bool kProb, bool kVar>
__device__ __forceinline__ Fused gather(const Level& P, long long pair, int x, int y,
                                        const double* __restrict__ mask) {
  const GlobalRecords rec{P, pair * (long long)P.g.nx * P.g.ny};
  return gather_with<kProb, kVar>(P.g, rec, x, y, mask);
}

// The Gauss-Newton loop of variance_fit below for the symmetric five-point
// window (points ordered -a, -b, 0, b, a): same arithmetic, same order of the
// sums, with g and d r / d sigma shared between +-o.
__device__ inline double variance_fit5(const double* delta, const double* p, double fallback) {
  const double d2a = __dmul_rn(delta[0], delta[0]);
  const double d2b = __dmul_rn(delta[1], delta[1]);
  const double d2c = __dmul_rn(delta[2], delta[2]);
  double c = 1.0;
  double sigma = sqrt(0.1);
  for (int iter = 0; iter < 10; ++iter) {  // kVarianceFitIterations
    const double den = __dmul_rn(__dmul_rn(2.0, sigma), sigma);
    const double s3 = __dmul_rn(__dmul_rn(sigma, sigma), sigma);
    const double ga = exp(__ddiv_rn(-d2a, den));
    const double gb = exp(__ddiv_rn(-d2b, den));
    // delta = 0: -0 / den = -0 and exp(-0) = 1 exactly whenever den > 0
    const double gc = den > 0.0 ? 1.0 : exp(__ddiv_rn(-d2c, den));
    const double ja = __ddiv_rn(__dmul_rn(__dmul_rn(c, ga), d2a), s3);
    const double jb = __ddiv_rn(__dmul_rn(__dmul_rn(c, gb), d2b), s3);
    // (c * 1) * 0 / s3 = +-0 with the sign of c, for finite c and s3 > 0
    const double jc = (gc == 1.0 && s3 > 0.0) ? copysign(0.0, c)
                                              : __ddiv_rn(__dmul_rn(__dmul_rn(c, gc), d2c), s3);
    const double gs[5] = {ga, gb, gc, gb, ga};
    const double js5[5] = {ja, jb, jc, jb, ja};
    double a00 = 0.0, a01 = 0.0, a11 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const double g = gs[i], js = js5[i];
      const double r = __dsub_rn(__dmul_rn(c, g), p[i]);
      a00 = __dadd_rn(a00, __dmul_rn(g, g));
      a01 = __dadd_rn(a01, __dmul_rn(g, js));
      a11 = __dadd_rn(a11, __dmul_rn(js, js));
      b0 = __dsub_rn(b0, __dmul_rn(g, r));
      b1 = __dsub_rn(b1, __dmul_rn(js, r));
    }
    if (!(a00 > 0.0)) return fallback;
    const double l00 = __dsqrt_rn(a00);
    const double l01 = __ddiv_rn(a01, l00);
    const double d11 = __dsub_rn(a11, __dmul_rn(l01, l01));
    if (!(d11 > 1e-300)) return fallback;
    const double l11 = __dsqrt_rn(d11);
    const double y0 = __ddiv_rn(b0, l00);
    const double y1 = __ddiv_rn(__dsub_rn(b1, __dmul_rn(l01, y0)), l11);
    const double xs = __ddiv_rn(y1, l11);
    const double xc = __ddiv_rn(__dsub_rn(y0, __dmul_rn(l01, xs)), l00);
    c = __dadd_rn(c, xc);
    sigma = __dadd_rn(sigma, xs);
    if (!isfinite(c) || !isfinite(sigma) || sigma <= 0.0) return fallback;
  }
  const double den = __dmul_rn(__dmul_rn(2.0, sigma), sigma);
  // (-delta) * delta == -(delta * delta) exactly
  const double ga = exp(__ddiv_rn(-d2a, den));
  const double gb = exp(__ddiv_rn(-d2b, den));
  const double gc = den > 0.0 ? 1.0 : exp(__ddiv_rn(-d2c, den));
  const double gs[5] = {ga, gb, gc, gb, ga};
  double ssr = 0.0;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const double r = __dsub_rn(__dmul_rn(c, gs[i]), p[i]);
    ssr = __dadd_rn(ssr, __dmul_rn(r, r));
  }
  const double fit = __dsqrt_rn(__ddiv_rn(ssr, 5.0));
  if (!isfinite(fit)) return fallback;
  if (fit > 0.1) return fallback;  // kVarianceFitMaxResidual
  return sigma;
}

// estimate_patch_variance (src/depth_variance.cpp:94-170) on the window
// priors. CUDA exp() may differ from glibc's by an ulp: sigma_k agrees to
// ~1e-15 relative, which is why var_disp is held to 1e-3 rel, not bits.
__device__ inline double variance_fit(const double* woff, int nwin, int wcenter, const double* res,
                               const uint8_t* ok, double denom) {
  // The common case first -- the default five-point window {-a, -b, 0, b, a}
  // with every sample valid -- with the priors in registers (the general
  // path below compacts the valid samples through a dynamically indexed
  // array, i.e. local memory). Same operations in the same order.
  if (nwin == 5 && wcenter == 2 && ok[0] && ok[1] && ok[2] && ok[3] && ok[4] &&
      woff[2] == 0.0 && woff[0] == -woff[4] && woff[1] == -woff[3]) {
    double d5[5], p5[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      d5[k] = woff[k];
      p5[k] = fast_exp(__ddiv_rn(-res[k], denom));
    }
#pragma unroll
    for (int k = 0; k < 5; ++k)
      if (k != 2 && !(p5[2] > p5[k])) return 2.0;  // kSigmaFallback
    return variance_fit5(d5, p5, 2.0);
  }
  double delta[kMaxWin], p[kMaxWin];
  double center_prior = 0.0;
  int n = 0;
  for (int k = 0; k < nwin; ++k) {
    if (!ok[k]) continue;
    const double pr = fast_exp(__ddiv_rn(-res[k], denom));
    delta[n] = woff[k];
    p[n] = pr;
    ++n;
    if (k == wcenter) center_prior = pr;
  }
  const double fallback = 2.0;  // kSigmaFallback, inc/depth_variance.hpp:15
  if (n < 3) return fallback;
  for (int i = 0; i < n; ++i) {
    if (delta[i] == 0.0) continue;
    if (!(center_prior > p[i])) return fallback;
  }
  // The common window -- five valid samples at {-a, -b, 0, b, a} (the
  // symmetric closure of two offsets) -- has three distinct d2 = delta^2, and
  // g and d r / d sigma depend on the offset only through d2: evaluate them
  // once per distinct d2 (the same operations on the same operands, hence the
  // same bits as per point), in registers.
  if (n == 5 && delta[2] == 0.0 && delta[0] == -delta[4] && delta[1] == -delta[3])
    return variance_fit5(delta, p, fallback);
  double c = 1.0;
  double sigma = sqrt(0.1);
  for (int iter = 0; iter < 10; ++iter) {  // kVarianceFitIterations
    double a00 = 0.0, a01 = 0.0, a11 = 0.0, b0 = 0.0, b1 = 0.0;
    for (int i = 0; i < n; ++i) {
      const double d2 = __dmul_rn(delta[i], delta[i]);
      const double g = exp(__ddiv_rn(-d2, __dmul_rn(__dmul_rn(2.0, sigma), sigma)));
      const double r = __dsub_rn(__dmul_rn(c, g), p[i]);
      const double js = __ddiv_rn(__dmul_rn(__dmul_rn(c, g), d2),
                                  __dmul_rn(__dmul_rn(sigma, sigma), sigma));
      a00 = __dadd_rn(a00, __dmul_rn(g, g));
      a01 = __dadd_rn(a01, __dmul_rn(g, js));
      a11 = __dadd_rn(a11, __dmul_rn(js, js));
      b0 = __dsub_rn(b0, __dmul_rn(g, r));
      b1 = __dsub_rn(b1, __dmul_rn(js, r));
    }
    if (!(a00 > 0.0)) return fallback;
    const double l00 = __dsqrt_rn(a00);
    const double l01 = __ddiv_rn(a01, l00);
    const double d11 = __dsub_rn(a11, __dmul_rn(l01, l01));
    if (!(d11 > 1e-300)) return fallback;
    const double l11 = __dsqrt_rn(d11);
    const double y0 = __ddiv_rn(b0, l00);
    const double y1 = __ddiv_rn(__dsub_rn(b1, __dmul_rn(l01, y0)), l11);
    const double xs = __ddiv_rn(y1, l11);
    const double xc = __ddiv_rn(__dsub_rn(y0, __dmul_rn(l01, xs)), l00);
    c = __dadd_rn(c, xc);
    sigma = __dadd_rn(sigma, xs);
    if (!isfinite(c) || !isfinite(sigma) || sigma <= 0.0) return fallback;
  }
  double ssr = 0.0;
  for (int i = 0; i < n; ++i) {
    const double g = exp(__ddiv_rn(__dmul_rn(-delta[i], delta[i]),
                                   __dmul_rn(__dmul_rn(2.0, sigma), sigma)));
    const double r = __dsub_rn(__dmul_rn(c, g), p[i]);
    ssr = __dadd_rn(ssr, __dmul_rn(r, r));
  }
  const double fit = __dsqrt_rn(__ddiv_rn(ssr, (double)n));
  if (!isfinite(fit)) return fallback;
  if (fit > 0.1) return fallback;  // kVarianceFitMaxResidual
  return sigma;
}

}  // namespace bdis
