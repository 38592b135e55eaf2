// bdis_patches_rt.cu -- k_patches_rt: the per-patch body of match_stereo
// (src/coarse_to_fine.cpp:247-300) for small patches (s <= 8) of fully valid
// inputs, with the template held in registers.
//
// Same arithmetic as k_patches (bdis_patches.cu), different resource split:
//   * a lane keeps its patch's template pixels L_i (s*s floats) in registers
//     and forms t_i = L_i - mean (extract_patch, src/patch.cpp:35-36) on use, so the
//     shared-memory band only holds the right view and the gradient (fp32,
//     padded x + x/32) -- about a third of k_patches' footprint per patch;
//   * that buys ~4 patches per lane in the CTA's pool: lanes take patches from
//     the pool as they finish (persistent lanes, no lockstep), and the
//     12-iteration LK stragglers overlap with other lanes' work instead of
//     idling the CTA;
//   * each lane finishes its own patch (window posterior, strict local
//     minimum, inherited probability, propagation, record) right after its
//     last window evaluation; only the Gauss-Newton variance fit, when
//     requested, runs in a balanced final phase.
// Every sum is still one lane's sequential row-major chain, so results are
// bit-identical to the reference (and to k_patches).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <math.h>
#include <math_constants.h>
#include <stdint.h>

#include "bdis_device.cuh"
#include "bdis_kernels.h"

namespace bdis {

namespace {

__device__ __forceinline__ int pad4(int x) { return x + (x >> 5); }
inline int pad4_host(int x) { return x + (x >> 5); }

struct RtLayout {
  size_t oR, oG, oMean, oHess, oTmsq, oU, oWres, oCnt, oPool, oCounters, oStage, oWok, total;
};

__host__ __device__ inline RtLayout rt_layout(int rows, int rpitch, int gpitch, int npb, int nwin,
                                              bool var) {
  RtLayout l;
  size_t o = 0;
  auto take = [&](size_t bytes, size_t align) {
    o = (o + align - 1) / align * align;
    const size_t r = o;
    o += bytes;
    return r;
  };
  l.oR = take(size_t(rows) * rpitch * 4, 16);
  l.oG = take(size_t(rows) * gpitch * 4, 16);
  l.oMean = take(size_t(npb) * 8, 8);
  l.oHess = take(size_t(npb) * 8, 8);
  l.oTmsq = take(size_t(npb) * 8, 8);
  l.oU = take(size_t(npb) * 8, 8);
  l.oWres = take(var ? size_t(npb) * nwin * 8 : 0, 8);
  l.oCnt = take(size_t(npb) * 4, 4);
  l.oPool = take(size_t(npb) * 4, 4);
  l.oCounters = take(16, 4);
  l.oStage = take(size_t(npb), 1);
  l.oWok = take(var ? size_t(npb) * nwin : 0, 1);
  l.total = (o + 15) / 16 * 16;
  return l;
}

}  // namespace

template <int S>
__global__ void __launch_bounds__(128, 2) k_patches_rt(Level L, Level P, PatchParams pp,
                                                        BandPlan bp) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Grid& g = L.g;
  const int w = L.w, h = L.h;
  const long long pair = blockIdx.y;
  const int ky0 = blockIdx.x * bp.rb;
  const int ky1 = min(ky0 + bp.rb, g.ny);
  const int npb = (ky1 - ky0) * g.nx;
  const int nwin = pp.nwin;
  const int tid = threadIdx.x, nt = blockDim.x;
  auto row_start = [&](int ky) { return ky == g.ny - 1 ? g.lasty0 : ky * g.stride; };
  auto col_start = [&](int kx) { return kx == g.nx - 1 ? g.lastx0 : kx * g.stride; };
  const int ylo = row_start(ky0);
  const int nrows = row_start(ky1 - 1) + S - ylo;
  const RtLayout lay = rt_layout(bp.smem_rows, bp.rpitch, bp.fpitch, bp.npb, nwin, pp.want_var);
  float* sR = (float*)(smem + lay.oR);
  float* sG = (float*)(smem + lay.oG);
  double* st_mean = (double*)(smem + lay.oMean);
  double* st_hess = (double*)(smem + lay.oHess);
  double* st_tmsq = (double*)(smem + lay.oTmsq);
  double* st_u = (double*)(smem + lay.oU);
  double* st_wres = (double*)(smem + lay.oWres);
  int* st_cnt = (int*)(smem + lay.oCnt);
  int* pool = (int*)(smem + lay.oPool);
  int* counters = (int*)(smem + lay.oCounters);  // [0] pool size, [1] next
  uint8_t* st_stage = smem + lay.oStage;
  uint8_t* st_wok = smem + lay.oWok;

  const long long pbase = pair * L.plane;
  const float* gL = L.left + pbase;  // template pixels come straight from L2
  {
    const float* gR = L.rpad + pair * (long long)(w + 1) * h + (long long)ylo * (w + 1);
    for (int r = 0; r < nrows; ++r) {
      for (int x = tid; x <= w; x += nt) sR[r * bp.rpitch + pad4(x)] = gR[(long long)r * (w + 1) + x];
      const float* gg = L.grad + pbase + (long long)(ylo + r) * w;
      for (int x = tid; x < w; x += nt) sG[r * bp.fpitch + pad4(x)] = gg[x];
    }
  }
  if (tid < 2) counters[tid] = 0;
  __syncthreads();

  const long long rec0 = pair * (long long)g.nx * g.ny + (long long)ky0 * g.nx;
  // ---- phase 1: extract_patch + precompute_patch_system + u0 (:250-262)
  for (int p = tid; p < npb; p += nt) {
    const int kx = p % g.nx, ky = ky0 + p / g.nx;
    const int x0 = col_start(kx), y0 = row_start(ky);
    const float* lr = gL + (long long)y0 * w + x0;
    double sum = 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j)
#pragma unroll
      for (int i = 0; i < S; ++i) sum = __dadd_rn(sum, (double)lr[j * w + i]);
    const int count = S * S;
    const double mean = __ddiv_rn(sum, (double)count);
    uint8_t stage = kSkipped;
    if (!(__ddiv_rn((double)count, (double)count) < pp.vpr)) {  // valid fraction 1 (:251)
      double hess = 0.0, tsq = 0.0;
      const float* gr = sG + (y0 - ylo) * bp.fpitch;
#pragma unroll
      for (int j = 0; j < S; ++j)
#pragma unroll
        for (int i = 0; i < S; ++i) {
          const double gv = (double)gr[j * bp.fpitch + pad4(x0 + i)];
          hess = __dadd_rn(hess, __dmul_rn(gv, gv));
          const double t = __dsub_rn((double)lr[j * w + i], mean);
          tsq = __dadd_rn(tsq, __dmul_rn(t, t));
        }
      if ((hess >= 1e-8) && isfinite(hess)) {  // degenerate (:254)
        stage = kSolved;
        const double cx = kx == g.nx - 1 ? g.cmax_x : __dadd_rn(g.c0, (double)kx * g.stride);
        const double cy = ky == g.ny - 1 ? g.cmax_y : __dadd_rn(g.c0, (double)ky * g.stride);
        double u = 0.0;
        if (pp.have_prev) {
          const int ix = clampi(lround_i(cx), 0, w - 1);
          const int iy = clampi(lround_i(cy), 0, h - 1);
          const Fused f = gather<false, false>(P, pair, min(ix / 2, P.w - 1),
                                              min(iy / 2, P.h - 1), pp.prev_mask);
          if (!(f.sw <= 0.0)) u = __dmul_rn(2.0, __ddiv_rn(f.swu, f.sw));
        }
        st_mean[p] = mean;
        st_hess[p] = hess;
        st_tmsq[p] = __ddiv_rn(tsq, (double)count);
        st_u[p] = u;
        st_cnt[p] = count;
        const double xc = __dsub_rn(cx, u);  // in_bounds(cx - u0, cy)
        if (xc >= 0.0 && xc <= (double)(w - 1)) pool[atomicAdd(&counters[0], 1)] = p;
      }
    }
    st_stage[p] = stage;
    const long long rec = rec0 + p;
    L.stage[rec] = stage;
    L.u[rec] = 0.0;
    L.prob[rec] = 0.0;
    L.post[rec] = 0.0;
    L.sigma[rec] = 0.0;
  }
  __syncthreads();

  // ---- phase 2: persistent lanes
  const int n_pool = counters[0];
  const double wm1 = (double)(w - 1);
  int p = -1, x0 = 0, k = -1, it = 0;
  double u = 0.0, prev = CUDART_INF, lastd = 0.0, hess = 0.0, tmsq = 0.0;
  float tl[S * S];  // template pixels L_i (t_i = L_i - mean, src/patch.cpp:35-36)
  double mean = 0.0;
  double wres[kMaxWin];
  unsigned wok = 0;
  const float* rbase = sR;  // right rows of the patch
  const float* gbase = sG;  // gradient rows of the patch
  auto take = [&]() {
    const int q = atomicAdd(&counters[1], 1);
    p = q < n_pool ? pool[q] : -1;
    if (p < 0) return;
    const int kx = p % g.nx, ky = ky0 + p / g.nx;
    x0 = col_start(kx);
    const int y0 = row_start(ky);
    rbase = sR + (y0 - ylo) * bp.rpitch;
    gbase = sG + (y0 - ylo) * bp.fpitch;
    mean = st_mean[p];
    const float* lr = gL + (long long)y0 * w + x0;
#pragma unroll
    for (int j = 0; j < S; ++j)
#pragma unroll
      for (int i = 0; i < S; ++i) tl[j * S + i] = lr[j * w + i];
    u = st_u[p];
    hess = st_hess[p];
    tmsq = st_tmsq[p];
    k = -1;
    it = 0;
    prev = CUDART_INF;
    lastd = 0.0;
    wok = 0;
  };
  take();
  while (p >= 0) {
    const double uu = k < 0 ? u : __dadd_rn(u, pp.woff[k]);
    // ---- eval_patch_residual (src/lk_solver.cpp:38-81): column table once
    int cxi[S];
    double cfx[S], comf[S];
    unsigned inb = 0, contig = 0;
    const double xd0 = (double)x0;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const double X = __dsub_rn(__dadd_rn(xd0, (double)i), uu);  // (cx + offset(i)) - u
      const bool in = X >= 0.0 && X <= wm1;
      const int xi = in ? __double2int_rz(X) : 0;
      cxi[i] = xi;
      cfx[i] = in ? __dsub_rn(X, (double)xi) : 0.0;
      comf[i] = __dsub_rn(1.0, cfx[i]);
      inb |= (unsigned)in << i;
      if (i > 0 && xi == cxi[i - 1] + 1) contig |= 1u << i;
    }
    // one predicated path: taps are reused when contiguous (a_i == b_{i-1}),
    // samples of columns outside the image are skipped (invalid, :55-58)
    double msq = CUDART_INF, jrs = 0.0;
    const int n = S * __popc(inb);
    if (n > 0) {
      double sum = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const float* rr = rbase + j * bp.rpitch;
        double b = 0.0;
        asm volatile("" ::: "memory");  // keep the scheduler from hoisting whole rows
#pragma unroll
        for (int i = 0; i < S; ++i) {
          const double a = ((contig >> i) & 1u) ? b : (double)rr[pad4(cxi[i])];
          b = (double)rr[pad4(cxi[i] + 1)];
          const double v = __dadd_rn(__dmul_rn(comf[i], a), __dmul_rn(cfx[i], b));
          if ((inb >> i) & 1u) sum = __dadd_rn(sum, v);
        }
      }
      const double rmean = __ddiv_rn(sum, (double)n);
      double ssr = 0.0, jr = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const float* rr = rbase + j * bp.rpitch;
        const float* gr = gbase + j * bp.fpitch;
        double b = 0.0;
        asm volatile("" ::: "memory");
#pragma unroll
        for (int i = 0; i < S; ++i) {
          const double a = ((contig >> i) & 1u) ? b : (double)rr[pad4(cxi[i])];
          b = (double)rr[pad4(cxi[i] + 1)];
          const double v = __dadd_rn(__dmul_rn(comf[i], a), __dmul_rn(cfx[i], b));
          const double r = __dsub_rn(__dsub_rn(v, rmean), __dsub_rn((double)tl[j * S + i], mean));
          const double g2 = (double)gr[pad4(x0 + i)];
          if ((inb >> i) & 1u) {
            ssr = __dadd_rn(ssr, __dmul_rn(r, r));
            jr = __dadd_rn(jr, __dmul_rn(g2, r));
          }
        }
      }
      msq = __ddiv_rn(ssr, (double)n);
      jrs = jr;
    }
    // ---- state machine
    bool finished = false;
    if (k >= 0) {
      // sample_window (src/window_posterior.cpp:28-37)
      wres[k] = msq;
      if (n == st_cnt[p]) wok |= 1u << k;
      if (++k == nwin) {
        finished = true;
        // dynamic_sigma + window_priors + patch_posterior (:42-96), :273-299
        int invalid = 0;
        for (int q = 0; q < nwin; ++q) invalid += !((wok >> q) & 1u);
        bool accept = !(invalid > 1 || !((wok >> pp.wcenter) & 1u));
        if (accept) {
          double ssum = 0.0;
          int cnt = 0;
          for (int q = 0; q < nwin; ++q) {
            if (!((wok >> q) & 1u)) continue;
            ssum = __dadd_rn(ssum, wres[q]);
            ++cnt;
          }
          const double mm = __ddiv_rn(ssum, (double)cnt);
          double ss = 0.0;
          for (int q = 0; q < nwin; ++q) {
            if (!((wok >> q) & 1u)) continue;
            const double d = __dsub_rn(wres[q], mm);
            ss = __dadd_rn(ss, __dmul_rn(d, d));
          }
          const double sd = __dsqrt_rn(__ddiv_rn(ss, (double)cnt));
          const double sigma_r = (sd < 1e-4) ? 1e-4 : sd;
          const double denom = __dmul_rn(
              __dmul_rn(__dmul_rn(__dmul_rn(2.0, sigma_r), sigma_r), (double)S), (double)S);
          double psum = 0.0, pc = 0.0;
          for (int q = 0; q < nwin; ++q) {
            const double pr = ((wok >> q) & 1u) ? fast_exp(__ddiv_rn(-wres[q], denom)) : 0.0;
            psum = __dadd_rn(psum, pr);
            if (q == pp.wcenter) pc = pr;
          }
          accept = !(psum <= 0.0);
          if (accept) {
            const double c = wres[pp.wcenter];
            for (int q = 0; q < nwin; ++q) {
              if (q == pp.wcenter || !((wok >> q) & 1u)) continue;
              if (!(c < wres[q])) {
                accept = false;
                break;
              }
            }
          }
          if (accept) {
            const double posterior = __ddiv_rn(pc, psum);
            const int kx = p % g.nx, ky = ky0 + p / g.nx;
            const double cx = kx == g.nx - 1 ? g.cmax_x : __dadd_rn(g.c0, (double)kx * g.stride);
            const double cy = ky == g.ny - 1 ? g.cmax_y : __dadd_rn(g.c0, (double)ky * g.stride);
            double inherited = 0.0;
            if (pp.have_prev) {
              const int px = clampi(lround_i(__ddiv_rn(cx, 2.0)), 0, P.w - 1);
              const int py = clampi(lround_i(__ddiv_rn(cy, 2.0)), 0, P.h - 1);
              const Fused f = gather<true, false>(P, pair, px, py, pp.prev_mask);
              if (!(f.sw <= 0.0)) inherited = __ddiv_rn(f.swp, f.sw);
            }
            double pr = __dadd_rn(inherited, __dmul_rn(L.level_w, posterior));
            pr = (pr < 0.0) ? 0.0 : ((1.0 < pr) ? 1.0 : pr);
            const long long rec = rec0 + p;
            L.u[rec] = u;
            L.prob[rec] = pr;
            L.post[rec] = posterior;
            L.stage[rec] = kAccepted;
            st_stage[p] = kAccepted;
            if (pp.want_var) {
              for (int q = 0; q < nwin; ++q) {
                st_wres[p * nwin + q] = wres[q];
                st_wok[p * nwin + q] = (wok >> q) & 1u;
              }
              st_u[p] = denom;  // reused: the prior denominator for the variance fit
            }
          }
        }
        if (!accept) L.stage[rec0 + p] = kConverged;
      }
    } else {
      // one iteration of solve_patch_disparity (src/lk_solver.cpp:96-127)
      ++it;
      bool done = false, conv = false;
      if (n == 0) {
        done = true;
      } else {
        if (it >= pp.min_it) {
          if (msq < pp.stop_good) {
            conv = done = true;
          } else if (msq > __dmul_rn(pp.stop_bad, tmsq)) {
            done = true;
          } else if (isfinite(prev) && __dsub_rn(prev, msq) < __dmul_rn(pp.stop_improve, prev)) {
            conv = it > 1 && fabs(lastd) < 1e-2;
            done = true;
          }
        }
        if (!done) {
          const double delta = __ddiv_rn(jrs, hess);
          u = __dadd_rn(u, delta);
          lastd = delta;
          prev = msq;
          if (fabs(delta) < 1e-2) conv = done = true;
          else if (it >= pp.max_it) done = true;
        }
      }
      if (done) {
        if (conv) {
          k = 0;  // window samples next
        } else {
          finished = true;
        }
      }
    }
    if (finished) take();
  }

  // ---- phase 3: Gauss-Newton variance fit (src/depth_variance.cpp:94-170)
  if (pp.want_var) {
    __syncthreads();
    for (int q = tid; q < npb; q += nt) {
      if (st_stage[q] != kAccepted) continue;
      L.sigma[rec0 + q] =
          variance_fit(pp.woff, nwin, pp.wcenter, st_wres + q * nwin, st_wok + q * nwin, st_u[q]);
    }
  }
}

bool plan_bands_rt(const Level& L, const PatchParams& pp, int max_smem_per_cta, BandPlan* out) {
  const Grid& g = L.g;
  // opt-in (PSTEREO_TUNE_RT=1): at 255 registers it runs 8 warps/SM and measured
  // slower than k_patches on config 2 (see profiles/)
  if (!pp.all_valid || g.size != 8 || !getenv("PSTEREO_TUNE_RT")) return false;
  BandPlan bp{};
  bp.rpitch = pad4_host(L.w) + 1;
  bp.fpitch = pad4_host(L.w - 1) + 1;
  bp.bpitch = 0;
  auto bytes_for = [&](int rb) {
    const int rows = (rb - 1) * g.stride + g.size;
    return rt_layout(rows, bp.rpitch, bp.fpitch, rb * g.nx, pp.nwin, pp.want_var).total;
  };
  auto env = [](const char* k, int d) {
    const char* v = getenv(k);
    return v ? atoi(v) : d;
  };
  const int threads = 128;
  const int ppl10 = env("PSTEREO_TUNE_RT_PPL10", 40);
  const int ctas = env("PSTEREO_TUNE_RT_CTAS", 2);
  const size_t per_sm = size_t(max_smem_per_cta) / ctas - 1024;
  int rb = std::max(1, std::min(g.ny, (ppl10 * threads / 10 + g.nx / 2) / g.nx));
  while (rb > 1 && bytes_for(rb) > per_sm) --rb;
  if (bytes_for(rb) > size_t(max_smem_per_cta)) return false;
  bp.use_smem = 1;
  bp.rb = rb;
  bp.n_bands = (g.ny + rb - 1) / rb;
  bp.npb = rb * g.nx;
  bp.smem_rows = (rb - 1) * g.stride + g.size;
  bp.smem_bytes = bytes_for(rb);
  bp.threads = threads;
  *out = bp;
  return true;
}

cudaError_t launch_patches_rt(const Level& L, const Level& P, const PatchParams& pp,
                              const BandPlan& bp, cudaStream_t s) {
  auto kern = k_patches_rt<8>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)bp.smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grid(bp.n_bands, pp.n_pairs);
  kern<<<grid, bp.threads, bp.smem_bytes, s>>>(L, P, pp, bp);
  return cudaGetLastError();
}

}  // namespace bdis
