// bdis_kernels.cu -- sm_100a kernels of the BDIS per-frame path.
//
// Stage map (reference -> kernel):
//   to_grayscale            src/image.cpp:16-43        k_gray_u8
//   downsample_half         src/pyramid.cpp:9-28       k_downsample
//   gradient_x + tap tables src/pyramid.cpp:30-42,
//                           inc/image.hpp:53-71        k_level_tables
//   per-patch body          src/coarse_to_fine.cpp:247-300
//     extract/precompute/solve/window/posterior/propagate/variance
//                                                      k_patches
//   fuse_level (finest) + filter threshold
//                           src/coarse_to_fine.cpp:101-150,
//                           src/depth_variance.cpp:78-86  k_fuse_finest
//   remove_small_components src/depth_variance.cpp:43-76  k_ccl_*
//   upsample_to_full + disparity_to_depth
//                           src/coarse_to_fine.cpp:166-180,328-337,
//                           src/depth_variance.cpp:9-41   k_output
//   MatchStats              src/coarse_to_fine.cpp:302-314 k_stats
// Coarse levels are never fused densely: the next level gathers the fused
// values it needs (init_next_level / inherited probability, :257-283) at its
// patch centres straight from the coarse patch records (bdis::gather).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <math_constants.h>

#include "bdis_device.cuh"
#include "bdis_kernels.h"

namespace bdis {

// --------------------------------------------------------------------------
// pyramid

// src/image.cpp:16-43: uint8 raster -> fp32 [0,1] + validity (alpha == 0).
__global__ void k_gray_u8(const uint8_t* __restrict__ src, int channels,
                          long long n_px, float* __restrict__ out,
                          uint8_t* __restrict__ valid) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n_px) return;
  const double inv255 = 1.0 / 255.0;
  const uint8_t* p = src + i * channels;
  double v;
  uint8_t ok = 1;
  if (channels == 1) {
    v = __dmul_rn((double)p[0], inv255);
  } else {
    if (channels == 4) ok = p[3] != 0;
    const double s = __dadd_rn(__dadd_rn(__dmul_rn(0.299, (double)p[0]),
                                         __dmul_rn(0.587, (double)p[1])),
                               __dmul_rn(0.114, (double)p[2]));
    v = __dmul_rn(s, inv255);
  }
  out[i] = __double2float_rn(v);
  valid[i] = ok;
}

// src/pyramid.cpp:9-28, both views at once. grid.y = pair.
__global__ void k_downsample(const float* __restrict__ sl,
                             const uint8_t* __restrict__ slv,
                             const float* __restrict__ sr,
                             const uint8_t* __restrict__ srv, int sw, int sh,
                             float* __restrict__ dl, uint8_t* __restrict__ dlv,
                             float* __restrict__ dr, uint8_t* __restrict__ drv,
                             int dw, int dh) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dw * dh) return;
  const long long pair = blockIdx.y;
  const int x = i % dw, y = i / dw;
  const int x0 = 2 * x, x1 = min(2 * x + 1, sw - 1);
  const int y0 = 2 * y, y1 = min(2 * y + 1, sh - 1);
  const long long sb = pair * (long long)sw * sh, db = pair * (long long)dw * dh;
  const long long a = sb + (long long)y0 * sw + x0, b = sb + (long long)y0 * sw + x1;
  const long long c = sb + (long long)y1 * sw + x0, d = sb + (long long)y1 * sw + x1;
  dl[db + i] = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(__fadd_rn(sl[a], sl[b]), sl[c]), sl[d]));
  dr[db + i] = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(__fadd_rn(sr[a], sr[b]), sr[c]), sr[d]));
  dlv[db + i] = (slv[a] && slv[b] && slv[c] && slv[d]) ? 1 : 0;
  drv[db + i] = (srv[a] && srv[b] && srv[c] && srv[d]) ? 1 : 0;
}

// Per level: gradient of the left view (src/pyramid.cpp:30-42), the 4-tap
// validity used by sample_bilinear at integer rows (inc/image.hpp:68-69: taps
// (x0,y0),(x1,y0),(x0,y1),(x1,y1) with x1 = min(x0+1,w-1), y1 = min(y0+1,h-1))
// for both views, and the right view's (x0, x1) tap pair.
__global__ void k_level_tables(Level L) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.w * L.h) return;
  const long long base = blockIdx.y * L.plane;
  const int w = L.w, h = L.h;
  const int x = i % w, y = i / w;
  const int x1 = min(x + 1, w - 1), y1 = min(y + 1, h - 1);
  const float* l = L.left + base + (long long)y * w;
  float g = 0.0f;
  if (w >= 2) {
    if (x == 0) g = __fsub_rn(l[1], l[0]);
    else if (x == w - 1) g = __fsub_rn(l[w - 1], l[w - 2]);
    else g = __fmul_rn(0.5f, __fsub_rn(l[x + 1], l[x - 1]));
  }
  L.grad[base + i] = g;
  const uint8_t* lv = L.lvalid + base;
  const uint8_t* rv = L.rvalid + base;
  const long long p00 = (long long)y * w + x, p10 = (long long)y * w + x1;
  const long long p01 = (long long)y1 * w + x, p11 = (long long)y1 * w + x1;
  L.lq[base + i] = (lv[p00] && lv[p10] && lv[p01] && lv[p11]) ? 1 : 0;
  L.rq[base + i] = (rv[p00] && rv[p10] && rv[p01] && rv[p11]) ? 1 : 0;
  const float* r = L.right + base;
  L.rab[base + i] = make_float2(r[p00], r[p10]);
}

// --------------------------------------------------------------------------
// the per-patch solve

struct ResidualEval {
  double msq, jr;
  int n;
};

// eval_patch_residual (src/lk_solver.cpp:38-81) for a lattice patch whose
// footprint starts at integer (x0, y0): template samples sit on integer
// pixels (fx = fy = 0), right samples on integer rows at x = (x0+i) - u.
__device__ __forceinline__ ResidualEval eval_residual(
    const Level& L, long long base, int x0, int y0, int s, double mean,
    double u) {
  const int w = L.w;
  const double wm1 = (double)(w - 1);
  const uint8_t* __restrict__ lq = L.lq + base;
  const uint8_t* __restrict__ rq = L.rq + base;
  const float2* __restrict__ rab = L.rab + base;
  const float* __restrict__ lf = L.left + base;
  const float* __restrict__ gr = L.grad + base;
  double sum = 0.0;
  int count = 0;
  for (int j = 0; j < s; ++j) {
    const long long row = (long long)(y0 + j) * w;
    for (int i = 0; i < s; ++i) {
      if (!lq[row + x0 + i]) continue;
      const double X = __dsub_rn((double)(x0 + i), u);
      if (!(X >= 0.0 && X <= wm1)) continue;
      const int xi = __double2int_rz(X);
      if (!rq[row + xi]) continue;
      const double fx = __dsub_rn(X, (double)xi);
      const float2 ab = rab[row + xi];
      const double v = __dadd_rn(__dmul_rn(__dsub_rn(1.0, fx), (double)ab.x),
                                 __dmul_rn(fx, (double)ab.y));
      sum = __dadd_rn(sum, v);
      ++count;
    }
  }
  ResidualEval ev;
  ev.msq = CUDART_INF;
  ev.jr = 0.0;
  ev.n = count;
  if (count == 0) return ev;
  const double rmean = __ddiv_rn(sum, (double)count);
  double ssr = 0.0, jr = 0.0;
  for (int j = 0; j < s; ++j) {
    const long long row = (long long)(y0 + j) * w;
    for (int i = 0; i < s; ++i) {
      const long long p = row + x0 + i;
      if (!lq[p]) continue;
      const double X = __dsub_rn((double)(x0 + i), u);
      if (!(X >= 0.0 && X <= wm1)) continue;
      const int xi = __double2int_rz(X);
      if (!rq[row + xi]) continue;
      const double fx = __dsub_rn(X, (double)xi);
      const float2 ab = rab[row + xi];
      const double v = __dadd_rn(__dmul_rn(__dsub_rn(1.0, fx), (double)ab.x),
                                 __dmul_rn(fx, (double)ab.y));
      const double t = __dsub_rn((double)lf[p], mean);
      const double r = __dsub_rn(__dsub_rn(v, rmean), t);
      ssr = __dadd_rn(ssr, __dmul_rn(r, r));
      jr = __dadd_rn(jr, __dmul_rn((double)gr[p], r));
    }
  }
  ev.msq = __ddiv_rn(ssr, (double)count);
  ev.jr = jr;
  return ev;
}

// estimate_patch_variance (src/depth_variance.cpp:94-170). Uses CUDA exp(),
// which can differ from glibc's exp by an ulp: sigma_k agrees to ~1e-15 rel.
__device__ double estimate_variance(const PatchParams& pp, const double* res,
                                    const uint8_t* ok, double sigma_r) {
  const double denom = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, sigma_r), sigma_r),
                                           (double)pp.size),
                                 (double)pp.size);
  double delta[kMaxWin], p[kMaxWin];
  double center_prior = 0.0;
  int n = 0;
  for (int k = 0; k < pp.nwin; ++k) {
    if (!ok[k]) continue;
    const double pr = fast_exp(__ddiv_rn(-res[k], denom));
    delta[n] = pp.woff[k];
    p[n] = pr;
    ++n;
    if (k == pp.wcenter) center_prior = pr;
  }
  const double fallback = 2.0;  // kSigmaFallback, inc/depth_variance.hpp:15
  if (n < 3) return fallback;
  for (int i = 0; i < n; ++i) {
    if (delta[i] == 0.0) continue;
    if (!(center_prior > p[i])) return fallback;
  }
  double c = 1.0;
  double sigma = sqrt(0.1);
  for (int iter = 0; iter < 10; ++iter) {
    double a00 = 0.0, a01 = 0.0, a11 = 0.0, b0 = 0.0, b1 = 0.0;
    for (int i = 0; i < n; ++i) {
      const double d2 = __dmul_rn(delta[i], delta[i]);
      const double g = exp(__ddiv_rn(-d2, __dmul_rn(__dmul_rn(2.0, sigma), sigma)));
      const double r = __dsub_rn(__dmul_rn(c, g), p[i]);
      const double jc = g;
      const double js = __ddiv_rn(__dmul_rn(__dmul_rn(c, g), d2),
                                  __dmul_rn(__dmul_rn(sigma, sigma), sigma));
      a00 = __dadd_rn(a00, __dmul_rn(jc, jc));
      a01 = __dadd_rn(a01, __dmul_rn(jc, js));
      a11 = __dadd_rn(a11, __dmul_rn(js, js));
      b0 = __dsub_rn(b0, __dmul_rn(jc, r));
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

// One thread per patch of one level, all pairs of the batch: the body of the
// reference's parallel_patches lambda (src/coarse_to_fine.cpp:247-300).
__global__ void __launch_bounds__(128) k_patches(Level L, Level P, PatchParams pp) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const Grid& g = L.g;
  const int np = g.nx * g.ny;
  if (tid >= (long long)pp.n_pairs * np) return;
  const long long pair = tid / np;
  const int k = (int)(tid - pair * np);
  const int kx = k % g.nx, ky = k / g.nx;
  const int s = g.size;
  const double cx = (kx == g.nx - 1) ? g.cmax_x : __dadd_rn(g.c0, (double)kx * g.stride);
  const double cy = (ky == g.ny - 1) ? g.cmax_y : __dadd_rn(g.c0, (double)ky * g.stride);
  const int x0 = (kx == g.nx - 1) ? g.lastx0 : kx * g.stride;
  const int y0 = (ky == g.ny - 1) ? g.lasty0 : ky * g.stride;
  const long long base = pair * L.plane;
  const int w = L.w, h = L.h;
  const uint8_t* __restrict__ lq = L.lq + base;
  const float* __restrict__ lf = L.left + base;
  const float* __restrict__ gr = L.grad + base;
  uint8_t stage = kSkipped;
  double u_out = 0.0, prob_out = 0.0, post_out = 0.0, sig_out = 0.0;

  do {
    // extract_patch (src/patch.cpp:5-38): integer sample positions.
    double sum = 0.0;
    int count = 0;
    for (int j = 0; j < s; ++j) {
      const long long row = (long long)(y0 + j) * w + x0;
      for (int i = 0; i < s; ++i) {
        if (!lq[row + i]) continue;
        sum = __dadd_rn(sum, (double)lf[row + i]);
        ++count;
      }
    }
    if (count == 0) break;
    const double mean = __ddiv_rn(sum, (double)count);
    const double vfrac = __ddiv_rn((double)count, (double)(s * s));
    if (vfrac < pp.vpr) break;  // src/coarse_to_fine.cpp:251
    // precompute_patch_system (src/lk_solver.cpp:7-36)
    double hess = 0.0, tsq = 0.0;
    for (int j = 0; j < s; ++j) {
      const long long row = (long long)(y0 + j) * w + x0;
      for (int i = 0; i < s; ++i) {
        if (!lq[row + i]) continue;
        const double gv = (double)gr[row + i];
        hess = __dadd_rn(hess, __dmul_rn(gv, gv));
        const double t = __dsub_rn((double)lf[row + i], mean);
        tsq = __dadd_rn(tsq, __dmul_rn(t, t));
      }
    }
    const double tmsq = __ddiv_rn(tsq, (double)count);
    if (!(hess >= 1e-8) || !isfinite(hess)) break;  // degenerate, :254
    stage = kSolved;

    // u0 = init_next_level(prev fused disparity) at the centre (:257-262,
    // :152-164), gathered from the coarse records.
    double u = 0.0;
    if (pp.have_prev) {
      const int ix = clampi(lround_i(cx), 0, w - 1);
      const int iy = clampi(lround_i(cy), 0, h - 1);
      const int px = min(ix / 2, P.w - 1), py = min(iy / 2, P.h - 1);
      const Fused f = gather<false, false>(P, pair, px, py, pp.prev_mask);
      if (!(f.sw <= 0.0)) u = __dmul_rn(2.0, __ddiv_rn(f.swu, f.sw));
    }

    // solve_patch_disparity (src/lk_solver.cpp:83-132)
    {
      const double xc = __dsub_rn(cx, u);
      if (!(xc >= 0.0 && xc <= (double)(w - 1))) break;
    }
    bool converged = false;
    {
      double prev = CUDART_INF, last_delta = 0.0;
      bool updated = false;
      for (int it = 1; it <= pp.max_it; ++it) {
        const ResidualEval ev = eval_residual(L, base, x0, y0, s, mean, u);
        if (ev.n == 0) break;
        const double r = ev.msq;
        if (it >= pp.min_it) {
          if (r < pp.stop_good) {
            converged = true;
            break;
          }
          if (r > __dmul_rn(pp.stop_bad, tmsq)) break;
          if (isfinite(prev) && __dsub_rn(prev, r) < __dmul_rn(pp.stop_improve, prev)) {
            converged = updated && fabs(last_delta) < 1e-2;
            break;
          }
        }
        const double delta = __ddiv_rn(ev.jr, hess);
        u = __dadd_rn(u, delta);
        last_delta = delta;
        updated = true;
        prev = r;
        if (fabs(delta) < 1e-2) {  // kUpdateEpsilon, inc/lk_solver.hpp:12
          converged = true;
          break;
        }
      }
    }
    if (!converged) break;
    stage = kConverged;

    // sample_window (src/window_posterior.cpp:10-40)
    double res[kMaxWin];
    uint8_t ok[kMaxWin];
    int invalid = 0;
    for (int q = 0; q < pp.nwin; ++q) {
      const ResidualEval ev = eval_residual(L, base, x0, y0, s, mean, __dadd_rn(u, pp.woff[q]));
      ok[q] = ev.n == count;
      res[q] = ev.msq;
      if (!ok[q]) ++invalid;
    }
    if (invalid > 1 || !ok[pp.wcenter]) break;
    // dynamic_sigma (:42-59)
    double sigma_r;
    {
      double ssum = 0.0;
      int cnt = 0;
      for (int q = 0; q < pp.nwin; ++q) {
        if (!ok[q]) continue;
        ssum = __dadd_rn(ssum, res[q]);
        ++cnt;
      }
      const double m = __ddiv_rn(ssum, (double)cnt);
      double ss = 0.0;
      for (int q = 0; q < pp.nwin; ++q) {
        if (!ok[q]) continue;
        const double d = __dsub_rn(res[q], m);
        ss = __dadd_rn(ss, __dmul_rn(d, d));
      }
      const double sd = __dsqrt_rn(__ddiv_rn(ss, (double)cnt));
      sigma_r = (sd < 1e-4) ? 1e-4 : sd;  // std::max(sd, kSigmaFloor)
    }
    // window_priors + patch_posterior (:61-96)
    double posterior;
    {
      const double denom = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, sigma_r), sigma_r),
                                               (double)s),
                                     (double)s);
      double psum = 0.0, pc = 0.0;
      for (int q = 0; q < pp.nwin; ++q) {
        const double pr = ok[q] ? fast_exp(__ddiv_rn(-res[q], denom)) : 0.0;
        psum = __dadd_rn(psum, pr);
        if (q == pp.wcenter) pc = pr;
      }
      if (psum <= 0.0) break;
      posterior = __ddiv_rn(pc, psum);
      const double c = res[pp.wcenter];
      bool is_min = true;
      for (int q = 0; q < pp.nwin; ++q) {
        if (q == pp.wcenter || !ok[q]) continue;
        if (!(c < res[q])) {
          is_min = false;
          break;
        }
      }
      if (!is_min) break;  // :273
    }
    // inherited probability + propagate_probability (:275-291, :96-99)
    double inherited = 0.0;
    if (pp.have_prev) {
      const int px = clampi(lround_i(__ddiv_rn(cx, 2.0)), 0, P.w - 1);
      const int py = clampi(lround_i(__ddiv_rn(cy, 2.0)), 0, P.h - 1);
      const Fused f = gather<true, false>(P, pair, px, py, pp.prev_mask);
      if (!(f.sw <= 0.0)) inherited = __ddiv_rn(f.swp, f.sw);
    }
    double pr = __dadd_rn(inherited, __dmul_rn(L.level_w, posterior));
    pr = (pr < 0.0) ? 0.0 : ((1.0 < pr) ? 1.0 : pr);
    u_out = u;
    prob_out = pr;
    post_out = posterior;
    if (pp.want_var) sig_out = estimate_variance(pp, res, ok, sigma_r);
    stage = kAccepted;
  } while (false);

  const long long rec = pair * (long long)np + k;
  L.stage[rec] = stage;
  L.u[rec] = u_out;
  L.prob[rec] = prob_out;
  L.post[rec] = post_out;
  L.sigma[rec] = sig_out;
}

// --------------------------------------------------------------------------
// finest level: fusion, filter, components, output

// fuse_level at the finest level (src/coarse_to_fine.cpp:101-150) plus the
// probability threshold of filter_validity (src/depth_variance.cpp:81-86).
__global__ void k_fuse_finest(Level L, FinestBufs fb, const double* __restrict__ mask,
                              int want_var, double threshold) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.w * L.h) return;
  const long long pair = blockIdx.y;
  const int x = i % L.w, y = i / L.w;
  Fused f;
  if (want_var) f = gather<true, true>(L, pair, x, y, mask);
  else f = gather<true, false>(L, pair, x, y, mask);
  const long long o = pair * L.plane + i;
  const bool valid = !(f.sw <= 0.0);
  double d = 0.0, p = 0.0, v = 0.0;
  if (valid) {
    d = __ddiv_rn(f.swu, f.sw);
    p = __ddiv_rn(f.swp, f.sw);
    if (want_var) v = __ddiv_rn(f.sw2s, __dmul_rn(f.sw, f.sw));
  }
  fb.disp[o] = d;
  fb.prob[o] = p;
  if (want_var) fb.var[o] = v;
  fb.mvalid[o] = valid ? 1 : 0;
  const bool keep = valid && !(p < threshold);
  fb.mask[o] = keep ? 1 : 0;
  fb.label[o] = keep ? i : -1;
}

// 4-connected components of the thresholded finest mask (the full-resolution
// mask is its block replication, so components and areas carry over with
// per-pixel area weights). Union-find with atomicMin links: the component
// partition -- hence the kept mask -- is independent of scheduling.
__device__ __forceinline__ int uf_find(const int* lab, int p) {
  const volatile int* l = lab;
  int q = l[p];
  while (q != p) {
    p = q;
    q = l[p];
  }
  return p;
}

__device__ __forceinline__ void uf_union(int* lab, int a, int b) {
  for (;;) {
    a = uf_find(lab, a);
    b = uf_find(lab, b);
    if (a == b) return;
    if (a < b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(&lab[a], b);
    if (old == a) return;
    a = old;
  }
}

__global__ void k_ccl_merge(int w, int h, long long plane, const uint8_t* __restrict__ mask,
                            int* lab) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w * h) return;
  const long long base = blockIdx.y * plane;
  if (!mask[base + i]) return;
  int* l = lab + base;
  const int x = i % w;
  if (x > 0 && mask[base + i - 1]) uf_union(l, i, i - 1);
  if (i >= w && mask[base + i - w]) uf_union(l, i, i - w);
}

__global__ void k_ccl_area(int w, int h, long long plane, int full_w, int full_h, int e,
                           const uint8_t* __restrict__ mask, int* lab, int* area) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w * h) return;
  const long long base = blockIdx.y * plane;
  if (!mask[base + i]) return;
  const int root = uf_find(lab + base, i);
  lab[base + i] = root;
  const int x = i % w, y = i / w;
  const int bx = min(1 << e, full_w - (x << e));
  const int by = min(1 << e, full_h - (y << e));
  atomicAdd(&area[base + root], bx * by);
}

// upsample_to_full (src/coarse_to_fine.cpp:166-180, :328-337), the area rule
// of filter_validity (src/depth_variance.cpp:87-90), run_pipeline's mask
// sharing (src/pipeline.cpp:21-22) and disparity_to_depth (:9-41).
template <typename T>
__global__ void k_output(OutputArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.W * a.H) return;
  const long long pair = blockIdx.y;
  const int X = i % a.W, Y = i / a.W;
  const int fx = min(X >> a.e, a.fw - 1), fy = min(Y >> a.e, a.fh - 1);
  const long long f = pair * a.fplane + (long long)fy * a.fw + fx;
  const bool mv = a.mvalid[f] != 0;
  bool keep = false;
  if (a.fmask[f]) keep = a.area[pair * a.fplane + a.label[f]] >= a.min_px;
  const double d = mv ? __dmul_rn(a.scale_d, a.disp[f]) : 0.0;
  const double p = mv ? __dmul_rn(1.0, a.prob[f]) : 0.0;
  const long long o = pair * (long long)a.W * a.H + i;
  T* disp = (T*)a.out_disp;
  if (disp) disp[o] = (T)d;
  if (a.out_dvalid) a.out_dvalid[o] = keep ? 1 : 0;
  if (a.out_prob) ((T*)a.out_prob)[o] = (T)p;
  if (a.out_mdisp) ((T*)a.out_mdisp)[o] = (T)d;
  if (a.out_mvalid) a.out_mvalid[o] = mv ? 1 : 0;
  const bool dv = keep && (d >= 0.1);  // kMinDisparity, inc/depth_variance.hpp:13
  if (a.out_depth) ((T*)a.out_depth)[o] = (T)(dv ? __ddiv_rn(a.fb, d) : 0.0);
  if (a.out_depth_valid) a.out_depth_valid[o] = dv ? 1 : 0;
  if (a.has_var) {
    const double v = mv ? __dmul_rn(a.scale_v, a.var[f]) : 0.0;
    if (a.out_var) ((T*)a.out_var)[o] = (T)v;
    const bool sv = dv && mv;
    if (a.out_sigma) {
      double sg = 0.0;
      if (sv) {
        const double vv = (v < 0.0) ? 0.0 : v;  // std::max(var, 0.0)
        sg = __dmul_rn(__ddiv_rn(a.fb, __dmul_rn(d, d)), __dsqrt_rn(vv));
      }
      ((T*)a.out_sigma)[o] = (T)sg;
    }
    if (a.out_sigma_valid) a.out_sigma_valid[o] = sv ? 1 : 0;
  }
}

// MatchStats per pair and level (src/coarse_to_fine.cpp:302-314).
__global__ void k_stats(StatsArgs a) {
  const int pair = blockIdx.x, lvl = blockIdx.y;
  const uint8_t* st = a.stage[lvl] + (long long)pair * a.np[lvl];
  int c1 = 0, c2 = 0, c3 = 0;
  for (int i = threadIdx.x; i < a.np[lvl]; i += blockDim.x) {
    const uint8_t v = st[i];
    c1 += v >= kSolved;
    c2 += v >= kConverged;
    c3 += v == kAccepted;
  }
  for (int o = 16; o > 0; o >>= 1) {
    c1 += __shfl_xor_sync(0xffffffffu, c1, o);
    c2 += __shfl_xor_sync(0xffffffffu, c2, o);
    c3 += __shfl_xor_sync(0xffffffffu, c3, o);
  }
  __shared__ int red[3][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[0][warp] = c1;
    red[1][warp] = c2;
    red[2][warp] = c3;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int t1 = 0, t2 = 0, t3 = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      t1 += red[0][q];
      t2 += red[1][q];
      t3 += red[2][q];
    }
    int* o = a.out + ((long long)pair * a.n_levels + lvl) * 3;
    o[0] = t1;
    o[1] = t2;
    o[2] = t3;
  }
}

// --------------------------------------------------------------------------
// launchers

static inline unsigned blocks_for(long long n, int t) { return (unsigned)((n + t - 1) / t); }

void launch_gray_u8(const uint8_t* src, int channels, long long n_px, float* out,
                    uint8_t* valid, cudaStream_t s) {
  k_gray_u8<<<blocks_for(n_px, 256), 256, 0, s>>>(src, channels, n_px, out, valid);
}

void launch_downsample(const float* sl, const uint8_t* slv, const float* sr,
                       const uint8_t* srv, int sw, int sh, float* dl, uint8_t* dlv,
                       float* dr, uint8_t* drv, int dw, int dh, int n_pairs,
                       cudaStream_t s) {
  dim3 grid(blocks_for((long long)dw * dh, 256), n_pairs);
  k_downsample<<<grid, 256, 0, s>>>(sl, slv, sr, srv, sw, sh, dl, dlv, dr, drv, dw, dh);
}

void launch_level_tables(const Level& L, int n_pairs, cudaStream_t s) {
  dim3 grid(blocks_for((long long)L.w * L.h, 256), n_pairs);
  k_level_tables<<<grid, 256, 0, s>>>(L);
}

void launch_patches(const Level& L, const Level& P, const PatchParams& pp, cudaStream_t s) {
  const long long n = (long long)pp.n_pairs * L.g.nx * L.g.ny;
  k_patches<<<blocks_for(n, 128), 128, 0, s>>>(L, P, pp);
}

void launch_fuse_finest(const Level& L, const FinestBufs& fb, const double* mask,
                        int want_var, double threshold, int n_pairs, cudaStream_t s) {
  dim3 grid(blocks_for((long long)L.w * L.h, 256), n_pairs);
  k_fuse_finest<<<grid, 256, 0, s>>>(L, fb, mask, want_var, threshold);
}

void launch_ccl(int w, int h, long long plane, int full_w, int full_h, int e,
                const uint8_t* mask, int* lab, int* area, int n_pairs, cudaStream_t s) {
  dim3 grid(blocks_for((long long)w * h, 256), n_pairs);
  k_ccl_merge<<<grid, 256, 0, s>>>(w, h, plane, mask, lab);
  k_ccl_area<<<grid, 256, 0, s>>>(w, h, plane, full_w, full_h, e, mask, lab, area);
}

void launch_output(const OutputArgs& a, int f64, int n_pairs, cudaStream_t s) {
  dim3 grid(blocks_for((long long)a.W * a.H, 256), n_pairs);
  if (f64) k_output<double><<<grid, 256, 0, s>>>(a);
  else k_output<float><<<grid, 256, 0, s>>>(a);
}

void launch_stats(const StatsArgs& a, int n_pairs, cudaStream_t s) {
  dim3 grid(n_pairs, a.n_levels);
  k_stats<<<grid, 256, 0, s>>>(a);
}

}  // namespace bdis
