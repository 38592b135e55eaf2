// bdis_patches.cu -- k_patches: the per-patch body of match_stereo
// (src/coarse_to_fine.cpp:247-300) for every patch of one pyramid level of a
// batch of pairs: extract_patch + precompute_patch_system (src/patch.cpp:5-38,
// src/lk_solver.cpp:7-36), the 1-D inverse-compositional LK solve
// (src/lk_solver.cpp:83-132), the residual window (src/window_posterior.cpp:
// 10-96), probability propagation (src/coarse_to_fine.cpp:90-99) and the
// optional Gauss-Newton variance fit (src/depth_variance.cpp:94-170).
//
// B200 mapping
//   * one CTA per (pair, band of `rb` patch rows); the band's rows of the
//     right view, left view and gradient (fp32) are staged in shared memory,
//     padded (slot x + x/32) so the stride-`stride` accesses of neighbouring
//     patches hit distinct banks;
//   * a thread owns one patch at a time and sums its samples in the
//     reference's sequential row-major order -- that is what makes every sum
//     bit-identical to the CPU (a warp tree reduction would reorder them);
//   * phases: (1) balanced setup of every band patch (extract, Hessian, u0
//     gather from the coarser level's records); (2) rounds of one residual
//     evaluation per busy lane: running LK solves packed into the lowest slots
//     and refilled from the CTA's pool, the remaining lanes taking window
//     samples of patches that converged in earlier rounds -- a long solve
//     keeps one warp busy, not a quarter of every warp; (3) balanced finish
//     (posterior, local-minimum test, inherited probability, variance fit,
//     records);
//   * the right-sample position x = (cx + offset(i)) - u of column i does not
//     depend on the row, so each evaluation computes the exact per-column
//     truncation x0_i and weight fx_i once (s conversions instead of s*s) and
//     applies them to every row: the literal sample_bilinear arithmetic
//     (inc/image.hpp:53-71) with no per-sample double<->int conversions.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <math.h>
#include <math_constants.h>
#include <stdint.h>

#include "bdis_device.cuh"
#include "bdis_kernels.h"

#ifndef KP_FT_SKIP
#define KP_FT_SKIP 10  // patch size without the interior-warp column table (A/B builds)
#endif

namespace bdis {

namespace {

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gsrc) : "memory");
}
// programmatic dependent launch: wait for the preceding grid's completion /
// let the following grid start launching (sm_90+ griddepcontrol)
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
// a shared-memory load by window address (address = per-thread column + a
// warp-uniform row offset: ptxas folds the sum into LDS [R + UR])
__device__ __forceinline__ float lds_f32(unsigned addr) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
// element index -> byte offset, opaque to the optimiser: otherwise it keeps
// element offsets and re-forms every address with a per-load LEA
__device__ __forceinline__ unsigned byte_ofs(int elem) {
  unsigned b;
  // a rotate (== shift for elem < 2^30): a plain shl is folded back into the LEA
  asm("shf.l.wrap.b32 %0, %1, %1, 2;" : "=r"(b) : "r"(elem));
  return b;
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

struct Ev {
  double msq, jr;
  int n;
};

template <bool kSmem>
struct Rows {
  // fp32 rows in shared memory, padded (slot x + x/32: neighbouring patches
  // read columns 4 apart, which unpadded is a 4-way bank conflict), or the
  // level planes in global memory (right view as rows of rpad_pitch(w)).
  const float* R;    // right view
  const float* Lf;   // left view
  const float* Gf;   // gradient of the left view
  const uint8_t* lq; // 4-tap validity (kValid only)
  const uint8_t* rq;
  int rp, fp, bp;    // row pitches (slots)
  __device__ __forceinline__ static int s4(int x) { return kSmem ? x + (x >> 5) : x; }
  __device__ __forceinline__ static int s8(int x) { return s4(x); }
};

// eval_patch_residual (src/lk_solver.cpp:38-81) of a lattice patch whose
// footprint starts at column x0 and row r0 of `rw`, at disparity u.
template <int S, bool kSmem, bool kValid, bool kJr = true>
__device__ __forceinline__ Ev eval_patch(const Rows<kSmem>& rw, int w, int s_rt, int x0,
                                         int r0, int rpad, double mean, double u) {
  // S > 0: the patch size; S < 0: a runtime size of at most -S; S == 0: up to kMaxPatch
  constexpr int SA = S > 0 ? S : (S < 0 ? -S : kMaxPatch);
  const int s = S > 0 ? S : s_rt;
  const double wm1 = (double)(w - 1);
  const double xd0 = (double)x0;
  Ev ev;
  ev.jr = 0.0;
  ev.msq = CUDART_INF;
  // Fully valid inputs, shared-memory rows: one predicated path. The in-bounds
  // columns form a run [lo, hi] (x grows with i); when their taps are
  // contiguous (x0_i = base + i -- always, unless x sits within rounding of an
  // integer) sample i reads taps base+i, base+i+1 and reuses the left tap of
  // column i+1. Out-of-image columns (invalid samples, inc/image.hpp:55,68)
  // read the zero padding (`rpad` = s slots either side of the row) and are masked
  // out of the sums. Lanes therefore never split between code paths.
  constexpr bool kRun = kSmem && !kValid && S > 0;
  constexpr unsigned kAll = SA >= 32 ? 0xffffffffu : ((1u << SA) - 1u);
  double mo[SA], mf[SA], mk[SA];  // weights (1-fx, fx) and column mask, 0 when masked
  unsigned inb = 0;
  int base = 0;
  bool ctg = false;
  if constexpr (kRun) {
    // Interior warps (every lane's columns inside the image -- x grows with i,
    // so the end columns decide): fx_i = X_i - (base + i) with one truncation
    // per patch; the subtraction is exact and lands in [0, 1) exactly when
    // trunc(X_i) is base + i (tested on the high word), which makes fx_i the
    // value the per-column truncation gives. Any lane failing sends the warp
    // to the general table.
    bool fast = false;
    const double X0 = __dsub_rn(xd0, u);
    const double XL = __dsub_rn(__dadd_rn(xd0, (double)(SA - 1)), u);
    // (not at s = 10: measured 2% slower there, 8% faster at s = 16)
    if (S != KP_FT_SKIP && __all_sync(__activemask(), X0 >= 0.0 && XL <= wm1)) {
      base = __double2int_rz(X0);
      const double bd = (double)base;
      bool okc = true;
#pragma unroll
      for (int i = 0; i < SA; ++i) {
        const double X = __dsub_rn(__dadd_rn(xd0, (double)i), u);
        const double f = __dsub_rn(X, __dadd_rn(bd, (double)i));
        okc = okc && (unsigned)__double2hiint(f) < 0x3ff00000u;
        mf[i] = f;
        mo[i] = __dsub_rn(1.0, f);
        mk[i] = 1.0;
      }
      fast = __all_sync(__activemask(), okc);
      if (fast) {
        inb = kAll;
        ctg = true;
      }
    }
    if (!fast) {
      // sample_bilinear's clamp / truncation / weight per column
      bool have = false;
      ctg = true;
      inb = 0;
#pragma unroll
      for (int i = 0; i < SA; ++i) {
        const double X = __dsub_rn(__dadd_rn(xd0, (double)i), u);  // (cx + offset(i)) - u
        const bool in = X >= 0.0 && X <= wm1;
        const int xi = in ? __double2int_rz(X) : 0;
        const double fx = in ? __dsub_rn(X, (double)xi) : 0.0;
        mf[i] = fx;
        mo[i] = in ? __dsub_rn(1.0, fx) : 0.0;
        mk[i] = in ? 1.0 : 0.0;
        inb |= (unsigned)in << i;
        if (in && !have) base = xi - i, have = true;  // first in-bounds column
        else if (in && xi != base + i) ctg = false;
      }
      ctg = ctg && have;
    }
  }
  if (ctg) {
    int offT[SA];
#pragma unroll
    for (int i = 0; i < SA; ++i) offT[i] = rw.s4(x0 + i);
    const int n = SA * __popc(inb);
    ev.n = n;
    const int xb = base + rpad;  // smem column of tap `base`
    // Per-thread byte addresses of the patch's tap / template columns in its
    // first row; the row offset j * pitch is the same for every lane, so it
    // stays in the uniform datapath and each load is LDS [R + UR] with no
    // per-load address instruction (measured: 19 of the 120 instructions of a
    // window-pass row were IMADs forming these addresses)
    unsigned cR[SA + 1], cL[SA];  // byte offsets of the columns within their arrays
#pragma unroll
    for (int i = 0; i <= SA; ++i) cR[i] = byte_ofs(r0 * rw.rp + rw.s8(xb + i));
#pragma unroll
    for (int i = 0; i < SA; ++i) cL[i] = byte_ofs(r0 * rw.fp + offT[i]);
    // uniform parts: array base (shared window) + row offset
    const unsigned bR = (unsigned)__cvta_generic_to_shared(rw.R);
    const unsigned bL = (unsigned)__cvta_generic_to_shared(rw.Lf);
    const unsigned bG = (unsigned)__cvta_generic_to_shared(rw.Gf);
    const unsigned rp4 = rw.rp * 4, fp4 = rw.fp * 4;
    double sum = 0.0;
    // s = 12 and 8: rows two at a time, the next row's taps loading under this
    // row's chain -- 26-32% faster at s = 12 / stride 4 (configs 3 and 4);
    // at s = 8 -0.5% on config 2 and -1.3% single-pair latency (+1% on the
    // variance config 1); s = 10 / 16 measured slower with it, and so did the
    // residual pass (profiles/r02/k_patches_experiments.md)
#pragma unroll((S == 12 || S == 8) ? 2 : 1)
    for (int j = 0; j < SA; ++j) {
      const unsigned oR = bR + j * rp4;
      double a = (double)lds_f32(cR[0] + oR);
#pragma unroll
      for (int i = 0; i < SA; ++i) {
        const double b = (double)lds_f32(cR[i + 1] + oR);
        // masked columns have cfx = comf = 0: v = +-0 leaves the sum unchanged
        sum = __dadd_rn(sum, __dadd_rn(__dmul_rn(mo[i], a), __dmul_rn(mf[i], b)));
        a = b;
      }
    }
    const double rmean = __ddiv_rn(sum, (double)n);
    double ssr = 0.0, jr = 0.0;
    auto pass2 = [&](auto masked) {
      constexpr bool kMask = decltype(masked)::value;
#pragma unroll 1
      for (int j = 0; j < SA; ++j) {
        const unsigned oR = bR + j * rp4, oL = bL + j * fp4, oG = bG + j * fp4;
        double a = (double)lds_f32(cR[0] + oR);
#pragma unroll
        for (int i = 0; i < SA; ++i) {
          const double b = (double)lds_f32(cR[i + 1] + oR);
          const double v = __dadd_rn(__dmul_rn(mo[i], a), __dmul_rn(mf[i], b));
          a = b;
          const double t = __dsub_rn((double)lds_f32(cL[i] + oL), mean);
          double r = __dsub_rn(__dsub_rn(v, rmean), t);
          // masked columns: r * 0 = +-0 adds nothing to ssr / jr
          if (kMask) r = __dmul_rn(r, mk[i]);
          ssr = __dadd_rn(ssr, __dmul_rn(r, r));
          if (kJr) jr = __dadd_rn(jr, __dmul_rn((double)lds_f32(cL[i] + oG), r));
        }
      }
    };
    // every column in the image (the common case): no mask multiply; a lane
    // only votes for the unmasked pass when its own columns are all inside
    if (__all_sync(__activemask(), inb == kAll)) pass2(std::false_type{});
    else pass2(std::true_type{});
    ev.msq = __ddiv_rn(ssr, (double)n);
    ev.jr = jr;
    return ev;
  }
  // Validity masks, a runtime patch size, non-contiguous taps or global rows:
  // per-sample predicates on the per-column table.
  int cxi[SA];
  double cfx[SA], comf[SA];
  inb = 0;
#pragma unroll
  for (int i = 0; i < SA; ++i) {
    if (S <= 0 && i >= s) break;
    const double X = __dsub_rn(__dadd_rn(xd0, (double)i), u);  // (cx + offset(i)) - u
    const bool in = X >= 0.0 && X <= wm1;
    const int xi = in ? __double2int_rz(X) : 0;
    cxi[i] = xi;
    cfx[i] = in ? __dsub_rn(X, (double)xi) : 0.0;
    comf[i] = __dsub_rn(1.0, cfx[i]);
    inb |= (unsigned)in << i;
  }
  const int xo = kSmem ? rpad : 0;
  int n = 0;
  double sum = 0.0;
#pragma unroll 1
  for (int j = 0; j < s; ++j) {
    const auto* rr = rw.R + (r0 + j) * rw.rp;
    double b = 0.0;
#pragma unroll
    for (int i = 0; i < SA; ++i) {
      if (S <= 0 && i >= s) break;
      const double a = (double)rr[rw.s8(xo + cxi[i])];
      b = (double)rr[rw.s8(xo + cxi[i] + 1)];
      const double v = __dadd_rn(__dmul_rn(comf[i], a), __dmul_rn(cfx[i], b));
      bool use = (inb >> i) & 1u;
      if (kValid)
        use = use && rw.lq[(r0 + j) * rw.bp + x0 + i] && rw.rq[(r0 + j) * rw.bp + cxi[i]];
      if (use) {
        sum = __dadd_rn(sum, v);
        if (kValid) ++n;
      }
    }
  }
  if (!kValid) n = s * __popc(inb);
  ev.n = n;
  if (n == 0) return ev;
  const double rmean = __ddiv_rn(sum, (double)n);
  double ssr = 0.0, jr = 0.0;
#pragma unroll 1
  for (int j = 0; j < s; ++j) {
    const auto* rr = rw.R + (r0 + j) * rw.rp;
    const float* lr = rw.Lf + (r0 + j) * rw.fp;
    const float* gr = rw.Gf + (r0 + j) * rw.fp;
    double b = 0.0;
#pragma unroll
    for (int i = 0; i < SA; ++i) {
      if (S <= 0 && i >= s) break;
      const double a = (double)rr[rw.s8(xo + cxi[i])];
      b = (double)rr[rw.s8(xo + cxi[i] + 1)];
      bool use = (inb >> i) & 1u;
      if (kValid)
        use = use && rw.lq[(r0 + j) * rw.bp + x0 + i] && rw.rq[(r0 + j) * rw.bp + cxi[i]];
      if (use) {
        const double v = __dadd_rn(__dmul_rn(comf[i], a), __dmul_rn(cfx[i], b));
        const double t = __dsub_rn((double)lr[rw.s4(x0 + i)], mean);
        const double r = __dsub_rn(__dsub_rn(v, rmean), t);
        ssr = __dadd_rn(ssr, __dmul_rn(r, r));
        if (kJr) jr = __dadd_rn(jr, __dmul_rn((double)gr[rw.s4(x0 + i)], r));
      }
    }
  }
  ev.msq = __ddiv_rn(ssr, (double)n);
  ev.jr = jr;
  return ev;
}

}  // namespace


template <int S, bool kSmem, bool kValid>
__global__ void __launch_bounds__(256, S == -16 ? 2 : 0) k_patches(Level L, Level P, PatchParams pp, BandPlan bp) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Grid& g = L.g;
  const int s = S > 0 ? S : g.size;
  const int w = L.w, h = L.h;
  const long long pair = blockIdx.y;
  const int ky0 = blockIdx.x * bp.rb;
  const int ky1 = min(ky0 + bp.rb, g.ny);
  const int npb = (ky1 - ky0) * g.nx;
  const int nwin = pp.nwin;
  const int tid = threadIdx.x, nt = blockDim.x;
  auto row_start = [&](int ky) { return ky == g.ny - 1 ? g.lasty0 : ky * g.stride; };
  auto col_start = [&](int kx) { return kx == g.nx - 1 ? g.lastx0 : kx * g.stride; };
  // band-local patch index -> (column, row) by a multiply: p / nx as
  // umulhi(p, ceil(2^32 / nx)), exact for p * nx < 2^32 (checked by the planner)
  auto row_of = [&](int p) { return (int)__umulhi((unsigned)p, bp.nx_magic); };
  const int ylo = row_start(ky0);
  const int nrows = row_start(ky1 - 1) + s - ylo;

  // ---- shared-memory carve-up (mirrors band_layout on the host)
  const BandLayout lay = band_layout(bp.use_smem ? bp.smem_rows : 0, bp.rpitch, bp.fpitch,
                                     bp.bpitch, bp.npb, nwin, kValid, bp.threads);
  float* sR = (float*)(smem + lay.oR);
  const int rpad = kSmem ? bp.rpad : 0;
  float* sL = (float*)(smem + lay.oL);
  float* sG = (float*)(smem + lay.oG);
  uint8_t* sLQ = smem + lay.oLQ;
  uint8_t* sRQ = smem + lay.oRQ;
  double* st_mean = (double*)(smem + lay.oMean);
  double* st_hess = (double*)(smem + lay.oHess);
  double* st_tmsq = (double*)(smem + lay.oTmsq);
  double* st_u = (double*)(smem + lay.oU);
  double* st_wres = (double*)(smem + lay.oWres);
  int* st_cnt = (int*)(smem + lay.oCnt);
  int* pool = (int*)(smem + lay.oPool);
  int* wlist = (int*)(smem + lay.oWlist);
  int* counters = (int*)(smem + lay.oCounters);
  double* sl_u = (double*)(smem + lay.oSlotU);
  double* sl_prev = (double*)(smem + lay.oSlotPrev);
  double* sl_lastd = (double*)(smem + lay.oSlotLastd);
  int* sl_p = (int*)(smem + lay.oSlotP);
  int* sl_it = (int*)(smem + lay.oSlotIt);
  uint8_t* st_stage = smem + lay.oStage;
  uint8_t* st_wok = smem + lay.oWok;

  const long long pbase = pair * L.plane;
  // Levels after the first are launched programmatically behind the previous
  // level: their band staging reads only the pyramid (complete before that
  // level passed its own wait), so it overlaps the previous level's tail; the
  // records of the coarser level are read only after griddep_wait below.
  if (!pp.have_prev) griddep_wait();
  Rows<kSmem> rw;
  int rofs;  // row index of image row y in rw is y - rofs
  if constexpr (kSmem) {
    // ---- stage the band (coalesced global reads, padded shared writes)
    const int gpitch = rpad_pitch(w);
    const float* gR = L.rpad + pair * (long long)gpitch * h + (long long)ylo * gpitch;
    // right rows with rpad zero slots either side (x in [-rpad, w + rpad])
    const int rw2 = w + 1 + 2 * rpad;
    // asynchronous copies (cp.async): every thread queues all of its
    // elements before waiting once, instead of a few loads in flight
    // (row, column) of the flat index q advance incrementally: no division
    {
      int r = tid / rw2, xs = tid - r * rw2;  // xs = x + rpad
      const int dr = nt / rw2, dx = nt - dr * rw2;
#pragma unroll 4
      for (int q = tid; q < nrows * rw2; q += nt) {
        const int x = xs - rpad;
        float* dst = sR + r * bp.rpitch + Rows<true>::s8(xs);
        if (x >= 0 && x <= w) cp_async4(dst, gR + r * gpitch + x);
        else *dst = 0.0f;
        xs += dx;
        r += dr;
        if (xs >= rw2) xs -= rw2, ++r;
      }
    }
    const float* gl0 = L.left + pbase + (long long)ylo * w;
    const float* gg0 = L.grad + pbase + (long long)ylo * w;
    {
      int r = tid / w, x = tid - r * w;
      const int dr = nt / w, dx = nt - dr * w;
#pragma unroll 4
      for (int q = tid; q < nrows * w; q += nt) {
        cp_async4(sL + r * bp.fpitch + Rows<true>::s4(x), gl0 + q);
        cp_async4(sG + r * bp.fpitch + Rows<true>::s4(x), gg0 + q);
        x += dx;
        r += dr;
        if (x >= w) x -= w, ++r;
      }
    }
    cp_async_wait_all();
    for (int r = 0; r < nrows; ++r) {
      if (kValid) {
        const uint8_t* lq = L.lq + pbase + (long long)(ylo + r) * w;
        const uint8_t* rq = L.rq + pbase + (long long)(ylo + r) * w;
        for (int x = tid; x < w; x += nt) {
          sLQ[r * bp.bpitch + x] = lq[x];
          sRQ[r * bp.bpitch + x] = rq[x];
        }
      }
    }
    rw.R = sR;
    rw.Lf = sL;
    rw.Gf = sG;
    rw.lq = sLQ;
    rw.rq = sRQ;
    rw.rp = bp.rpitch;
    rw.fp = bp.fpitch;
    rw.bp = bp.bpitch;
    rofs = ylo;
  } else {
    rw.R = L.rpad + pair * (long long)rpad_pitch(w) * h;
    rw.Lf = L.left + pbase;
    rw.Gf = L.grad + pbase;
    rw.lq = L.lq + pbase;
    rw.rq = L.rq + pbase;
    rw.rp = rpad_pitch(w);
    rw.fp = w;
    rw.bp = w;
    rofs = 0;
  }
  if (pp.have_prev) griddep_wait();
  griddep_launch();  // our predecessors are complete: the next level may start staging
  if (tid < 32) counters[tid] = 0;
  __syncthreads();

  // ---- phase 1: extract_patch + precompute_patch_system + u0 (:250-262)
  for (int p = tid; p < npb; p += nt) {
    const int prow = row_of(p);
    const int kx = p - prow * g.nx, ky = ky0 + prow;
    const int x0 = col_start(kx);
    const int r0 = row_start(ky) - rofs;
    uint8_t stage = kSkipped;
    double sum = 0.0;
    int count = 0;
    // fully valid inputs in shared memory: the template columns as byte
    // offsets, rows through the uniform datapath (as in eval_patch)
    constexpr bool kFastRows = kSmem && !kValid && S > 0;
    constexpr int SP = kFastRows ? S : 1;
    unsigned pc[SP];
    unsigned pbL = 0, pbG = 0, pf4 = 0;
    if constexpr (kFastRows) {
#pragma unroll
      for (int i = 0; i < SP; ++i) pc[i] = byte_ofs(r0 * rw.fp + rw.s4(x0 + i));
      pbL = (unsigned)__cvta_generic_to_shared(rw.Lf);
      pbG = (unsigned)__cvta_generic_to_shared(rw.Gf);
      pf4 = rw.fp * 4;
#pragma unroll 2
      for (int j = 0; j < SP; ++j) {
        const unsigned o = pbL + j * pf4;
#pragma unroll
        for (int i = 0; i < SP; ++i) sum = __dadd_rn(sum, (double)lds_f32(pc[i] + o));
      }
      count = SP * SP;
    } else {
      for (int j = 0; j < s; ++j) {
        const float* lr = rw.Lf + (r0 + j) * rw.fp;
        for (int i = 0; i < s; ++i) {
          if (kValid && !rw.lq[(r0 + j) * rw.bp + x0 + i]) continue;
          sum = __dadd_rn(sum, (double)lr[rw.s4(x0 + i)]);
          ++count;
        }
      }
    }
    double mean = 0.0, hess = 0.0, tsq = 0.0;
    bool ok = count > 0;
    if (ok) {
      mean = __ddiv_rn(sum, (double)count);
      ok = !(__ddiv_rn((double)count, (double)(s * s)) < pp.vpr);  // :251
    }
    if (ok) {
      if constexpr (kFastRows) {
#pragma unroll 2
        for (int j = 0; j < SP; ++j) {
          const unsigned oL = pbL + j * pf4, oG = pbG + j * pf4;
#pragma unroll
          for (int i = 0; i < SP; ++i) {
            const double gv = (double)lds_f32(pc[i] + oG);
            hess = __dadd_rn(hess, __dmul_rn(gv, gv));
            const double t = __dsub_rn((double)lds_f32(pc[i] + oL), mean);
            tsq = __dadd_rn(tsq, __dmul_rn(t, t));
          }
        }
      } else {
        for (int j = 0; j < s; ++j) {
          const float* lr = rw.Lf + (r0 + j) * rw.fp;
          const float* gr = rw.Gf + (r0 + j) * rw.fp;
          for (int i = 0; i < s; ++i) {
            if (kValid && !rw.lq[(r0 + j) * rw.bp + x0 + i]) continue;
            const double gv = (double)gr[rw.s4(x0 + i)];
            hess = __dadd_rn(hess, __dmul_rn(gv, gv));
            const double t = __dsub_rn((double)lr[rw.s4(x0 + i)], mean);
            tsq = __dadd_rn(tsq, __dmul_rn(t, t));
          }
        }
      }
      ok = (hess >= 1e-8) && isfinite(hess);  // degenerate (:254, lk_solver.cpp:33)
    }
    if (ok) {
      stage = kSolved;
      const double cx = kx == g.nx - 1 ? g.cmax_x : __dadd_rn(g.c0, (double)kx * g.stride);
      const double cy = ky == g.ny - 1 ? g.cmax_y : __dadd_rn(g.c0, (double)ky * g.stride);
      double u = 0.0;
      bool weak = false;  // no confident prior: the long LK solves (measured)
      if (pp.have_prev) {
        const int ix = clampi(lround_i(cx), 0, w - 1);
        const int iy = clampi(lround_i(cy), 0, h - 1);
        const Fused f = gather<false, false>(P, pair, min(ix / 2, P.w - 1), min(iy / 2, P.h - 1),
                                            pp.prev_mask);
        if (!(f.sw <= 0.0)) u = __dmul_rn(2.0, __ddiv_rn(f.swu, f.sw));
        weak = !(f.sw >= 1.0);
      }
      st_mean[p] = mean;
      st_hess[p] = hess;
      st_tmsq[p] = __ddiv_rn(tsq, (double)count);
      st_u[p] = u;
      st_cnt[p] = count;
      const double xc = __dsub_rn(cx, u);  // in_bounds(cx - u0, cy), lk_solver.cpp:89
      // pool order: patches without a confident coarse prior first -- they
      // take ~11 LK iterations against ~2-3 for the rest, so starting them in
      // the first round shortens the CTA's critical path (order never changes
      // a result); the rest are parked in wlist (unused until phase 2)
      if (xc >= 0.0 && xc <= (double)(w - 1)) {
        if (weak) pool[atomicAdd(&counters[0], 1)] = p;  // cNPool
        else wlist[atomicAdd(&counters[1], 1)] = p;
      }
    }
    st_stage[p] = stage;
  }
  __syncthreads();
  {
    const int nw = counters[0], ns = counters[1];
    for (int q = tid; q < ns; q += nt) pool[nw + q] = wlist[q];
    __syncthreads();
    if (tid == 0) {
      counters[0] = nw + ns;
      counters[1] = 0;
    }
    __syncthreads();
  }

  // ---- phase 2: rounds of one residual evaluation per busy lane. Slots
  // [0, n_act) hold the running LK solves (src/lk_solver.cpp:83-132), packed to
  // the lowest lanes after every round and refilled from the pool; the next
  // lanes take window samples (src/window_posterior.cpp:10-36) of patches that
  // converged in earlier rounds. Idle warps go straight to the barrier, so a
  // long solve keeps one warp busy, not a quarter of every warp.
  enum { cNPool, cConv, cNAct, cPoolNext = 4, cWNext = 6, cWAvail = 8, cAlive = 10, cFit = 30 };
  {
    const int n_pool = counters[cNPool];
    const int n0 = min(n_pool, nt);
    if (tid < n0) {
      const int p = pool[tid];
      sl_p[tid] = p;
      sl_it[tid] = 0;
      sl_u[tid] = st_u[p];
      sl_prev[tid] = CUDART_INF;
      sl_lastd[tid] = 0.0;
    }
    if (tid == 0) {
      counters[cNAct] = n0;
      counters[cPoolNext] = n0;
      counters[cWNext] = 0;
      counters[cWAvail] = 0;
    }
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
#pragma unroll 1
    for (int par = 0;; par ^= 1) {
      const int na = counters[cNAct + par], pn = counters[cPoolNext + par];
      const int wn = counters[cWNext + par], wa = counters[cWAvail + par] * nwin;
      const int wjobs = min(nt - na, wa - wn);
      if (na == 0 && wjobs == 0) break;
      bool alive = false;
      int p = 0, it = 0, k = -1;
      double u = 0.0, prev = 0.0, lastd = 0.0, ue = 0.0;
      const bool lk = tid < na, busy = tid < na + wjobs;
      if (lk) {
        p = sl_p[tid];
        it = sl_it[tid];
        u = sl_u[tid];
        prev = sl_prev[tid];
        lastd = sl_lastd[tid];
        ue = u;
      } else if (busy) {
        const int j = wn + tid - na;
        p = wlist[j / nwin];
        k = j - (j / nwin) * nwin;
        ue = __dadd_rn(st_u[p], pp.woff[k]);
      }
      // warps holding no LK solve skip the jr chain (warp-uniform choice)
      const bool warp_lk = __any_sync(0xffffffffu, lk);
      if (busy) {
        // one code path per warp for both kinds of job: a warp costs one evaluation
        const int prow = row_of(p);
        const int ex0 = col_start(p - prow * g.nx), er0 = row_start(ky0 + prow) - rofs;
        const Ev ev = warp_lk ? eval_patch<S, kSmem, kValid, true>(rw, w, s, ex0, er0, rpad,
                                                                         st_mean[p], ue)
                              : eval_patch<S, kSmem, kValid, false>(rw, w, s, ex0, er0, rpad,
                                                                          st_mean[p], ue);
        if (!lk) {
          // sample_window: valid iff every template pixel was sampled (:31-36)
          st_wres[p * nwin + k] = ev.msq;
          st_wok[p * nwin + k] = ev.n == st_cnt[p];
        } else {
          // one iteration of solve_patch_disparity (src/lk_solver.cpp:96-127)
          ++it;
          bool done = false, conv = false;
          if (ev.n == 0) {
            done = true;
          } else {
            const double r = ev.msq;
            if (it >= pp.min_it) {
              if (r < pp.stop_good) {
                conv = done = true;
              } else if (r > __dmul_rn(pp.stop_bad, st_tmsq[p])) {
                done = true;
              } else if (isfinite(prev) && __dsub_rn(prev, r) < __dmul_rn(pp.stop_improve, prev)) {
                conv = it > 1 && fabs(lastd) < 1e-2;
                done = true;
              }
            }
            if (!done) {
              const double delta = __ddiv_rn(ev.jr, st_hess[p]);
              u = __dadd_rn(u, delta);
              lastd = delta;
              prev = r;
              if (fabs(delta) < 1e-2) conv = done = true;  // kUpdateEpsilon
              else if (it >= pp.max_it) done = true;
            }
          }
          if (done && conv) {
            st_stage[p] = kConverged;
            st_u[p] = u;
            wlist[atomicAdd(&counters[cConv], 1)] = p;
          }
          alive = !done;
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, alive);
      if (lane == 0) counters[cAlive + warp] = __popc(bal);
      __syncthreads();
      int before = 0, n_alive = 0;
      for (int q = 0; q < (nt >> 5); ++q) {
        const int c = counters[cAlive + q];
        before += q < warp ? c : 0;
        n_alive += c;
      }
      if (alive) {
        const int d = before + __popc(bal & ((1u << lane) - 1u));
        sl_p[d] = p;
        sl_it[d] = it;
        sl_u[d] = u;
        sl_prev[d] = prev;
        sl_lastd[d] = lastd;
      }
      const int refill = min(nt - n_alive, n_pool - pn);
      if (tid >= n_alive && tid < n_alive + refill) {
        const int np = pool[pn + tid - n_alive];
        sl_p[tid] = np;
        sl_it[tid] = 0;
        sl_u[tid] = st_u[np];
        sl_prev[tid] = CUDART_INF;
        sl_lastd[tid] = 0.0;
      }
      if (tid == 0) {
        counters[cNAct + (par ^ 1)] = n_alive + refill;
        counters[cPoolNext + (par ^ 1)] = pn + refill;
        counters[cWNext + (par ^ 1)] = wn + wjobs;
        counters[cWAvail + (par ^ 1)] = counters[cConv];
      }
      __syncthreads();
    }
  }

  // ---- phase 3: posterior, propagation, variance and the records (:268-299)
  const long long rec0 = pair * (long long)g.nx * g.ny + (long long)ky0 * g.nx;
  for (int p = tid; p < npb; p += nt) {
    uint8_t stage = st_stage[p];
    double u_out = 0.0, prob_out = 0.0, post_out = 0.0, sig_out = 0.0;
    if (stage == kConverged) {
      const double* res = st_wres + p * nwin;
      const uint8_t* ok = st_wok + p * nwin;
      int invalid = 0;
      for (int q = 0; q < nwin; ++q) invalid += !ok[q];
      bool accept = !(invalid > 1 || !ok[pp.wcenter]);
      double sigma_r = 0.0, posterior = 0.0;
      if (accept) {
        // dynamic_sigma (src/window_posterior.cpp:42-59)
        double ssum = 0.0;
        int cnt = 0;
        for (int q = 0; q < nwin; ++q) {
          if (!ok[q]) continue;
          ssum = __dadd_rn(ssum, res[q]);
          ++cnt;
        }
        const double m = __ddiv_rn(ssum, (double)cnt);
        double ss = 0.0;
        for (int q = 0; q < nwin; ++q) {
          if (!ok[q]) continue;
          const double d = __dsub_rn(res[q], m);
          ss = __dadd_rn(ss, __dmul_rn(d, d));
        }
        const double sd = __dsqrt_rn(__ddiv_rn(ss, (double)cnt));
        sigma_r = (sd < 1e-4) ? 1e-4 : sd;
        // window_priors + patch_posterior (:61-96)
        const double denom = __dmul_rn(
            __dmul_rn(__dmul_rn(__dmul_rn(2.0, sigma_r), sigma_r), (double)s), (double)s);
        double psum = 0.0, pc = 0.0;
        for (int q = 0; q < nwin; ++q) {
          const double pr = ok[q] ? fast_exp(__ddiv_rn(-res[q], denom)) : 0.0;
          psum = __dadd_rn(psum, pr);
          if (q == pp.wcenter) pc = pr;
        }
        accept = !(psum <= 0.0);
        if (accept) {
          posterior = __ddiv_rn(pc, psum);
          const double c = res[pp.wcenter];
          for (int q = 0; q < nwin; ++q) {
            if (q == pp.wcenter || !ok[q]) continue;
            if (!(c < res[q])) {
              accept = false;  // not a strict local minimum (:273)
              break;
            }
          }
        }
        if (accept) {
          const int prow = row_of(p);
          const int kx = p - prow * g.nx, ky = ky0 + prow;
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
          u_out = st_u[p];
          prob_out = pr;
          post_out = posterior;
          if (pp.want_var) {
            // the fit runs below on densely packed lanes: here only ~half the
            // lanes hold an accepted patch (measured 13 of 32 active)
            st_hess[p] = denom;  // the Hessian is dead after phase 2
            pool[atomicAdd(&counters[cFit], 1)] = p;
          }
          stage = kAccepted;
        }
      }
    }
    const long long rec = rec0 + p;
    L.stage[rec] = stage;
    L.u[rec] = u_out;
    L.prob[rec] = prob_out;
    L.post[rec] = post_out;
    L.sigma[rec] = sig_out;
  }
  if (pp.want_var) {
    // estimate_patch_variance (src/depth_variance.cpp:94-170) of the accepted patches
    __syncthreads();
    const int nfit = counters[cFit];
    for (int q = tid; q < nfit; q += nt) {
      const int p = pool[q];
      L.sigma[rec0 + p] = variance_fit(pp.woff, nwin, pp.wcenter, st_wres + p * nwin,
                                       st_wok + p * nwin, st_hess[p]);
    }
  }
}

// ---------------------------------------------------------------------------

static inline int pad4_host(int x) { return x + (x >> 5); }

BandPlan plan_bands(const Level& L, const PatchParams& pp, int max_smem_per_cta) {
  const Grid& g = L.g;
  BandPlan bp{};
  const bool valid = !pp.all_valid;
  auto env = [](const char* k, int d) {
    const char* v = getenv(k);
    return v ? atoi(v) : d;
  };
  bp.rpad = g.size;
  bp.rpitch = pad4_host(L.w + 2 * bp.rpad) + 1;  // x in [-rpad, w + rpad]
  bp.fpitch = pad4_host(L.w - 1) + 1;            // x in [0, w - 1]
  bp.bpitch = valid ? L.w : 0;
  // measured per level width (patch columns): 192-slot CTAs, two per SM, for
  // wide levels; 128-slot CTAs, three per SM, for medium ones; 128-slot CTAs,
  // four per SM, with about 0.8 patches per slot for the narrowest (round 2:
  // three bands per pair at the coarsest config-2 level instead of one
  // whole-level CTA, -1% per step; profiles/r02/k_patches_experiments.md)
  const bool medium = g.nx >= 30 && g.nx < 60;
  // (not at s = 16: +5%; not for launches of more than 256 pairs, whose
  // whole-level CTAs already fill several waves: 320x240 x 1024 +1.5%)
  const bool narrow = g.nx < 30 && g.size <= 12 && pp.n_pairs <= 256;
  int threads = env("PSTEREO_TUNE_THREADS", narrow || medium ? 128 : g.nx < 30 ? 256 : 192);
  int ctas = env("PSTEREO_TUNE_CTAS", narrow ? 4 : medium ? 3 : 2);
  int ppl10 = env("PSTEREO_TUNE_PPL10", narrow ? 8 : 20);
  // tuning runs only: PSTEREO_TUNE_SPEC="e1=192x2,e2=128x3" per level exponent
  if (const char* spec = getenv("PSTEREO_TUNE_SPEC")) {
    char key[16];
    snprintf(key, sizeof key, "e%d=", L.e);
    if (const char* q = strstr(spec, key)) {
      int t = 0, c = 0, pp10 = 0;
      const int got = sscanf(q + strlen(key), "%dx%dx%d", &t, &c, &pp10);
      if (got >= 2 && t >= 32 && t <= 256 && c >= 1) {
        threads = t;
        ctas = c;
        if (got == 3 && pp10 > 0) ppl10 = pp10;
      }
    }
  }
  auto bytes_for = [&](int rb) {
    const int rows = (rb - 1) * g.stride + g.size;
    return band_layout(rows, bp.rpitch, bp.fpitch, bp.bpitch, rb * g.nx, pp.nwin, valid,
                       threads).total;
  };
  // up to ~2 patches per slot of a 192-thread CTA, while two CTAs fit an SM
  // (measured best of a T x ppl x CTAs sweep at the bench workload;
  // PSTEREO_TUNE_THREADS / _PPL10 / _CTAS override, for tuning runs only)
  auto fit = [&](int t, int c) {
    const size_t per_sm = size_t(max_smem_per_cta) / c - 1024;
    int r = std::max(1, std::min(g.ny, (ppl10 * t / 10 + g.nx / 2) / g.nx));
    while (r > 1 && band_layout((r - 1) * g.stride + g.size, bp.rpitch, bp.fpitch, bp.bpitch,
                                r * g.nx, pp.nwin, valid, t).total > per_sm)
      --r;
    return r;
  };
  int rb = fit(threads, ctas);
  // Large patches, wide levels and dense grids make band rows expensive in
  // shared memory: when the default shape's band starves (<= 2 patch rows for
  // s >= 12 or >= 100 patch columns, <= 3 for s >= 16) or the grid is dense
  // and wide (stride <= s/4, >= 60 patch columns), one 256-thread CTA per SM
  // with the whole shared memory and a taller band wins (measured per level,
  // scripts/gpu_shape_sweep.py: s=16 stride 4 finest level 10.2 -> 4.5 ms,
  // 1920x1080 s=8 finest level 2.2 -> 1.3 ms; the bench shape, 640x480 s=8
  // stride 4, is unaffected)
  if (!getenv("PSTEREO_TUNE_SPEC") && !getenv("PSTEREO_TUNE_THREADS") &&
      !getenv("PSTEREO_TUNE_CTAS")) {
    const bool starving =
        (rb <= 2 && (g.size >= 12 || g.nx >= 100)) || (rb <= 3 && g.size >= 16);
    // (s = 12 excepted below 300 patch columns: its instantiation runs the
    // mean pass two rows at a time at 160 registers and measured faster on
    // two 192-thread CTAs there -- 640x480 stride 2 / 3: 7.02 vs 7.18 ms and
    // 3.38 vs 3.54 ms per 128 pairs -- while 1920x1080 stride 2 keeps the
    // one-CTA shape, profiles/r02/k_patches_experiments.md)
    const bool dense = 4 * g.stride <= g.size && g.nx >= 60 && !(g.size == 12 && g.nx < 300);
    if (starving || dense) {
      const int r1 = fit(256, 1);
      if (r1 >= rb + 1) {
        threads = 256;
        ctas = 1;
        rb = r1;
      }
    }
  }
  // small batches: a CTA's rounds are a latency chain, so spread the level
  // over more, smaller bands until every SM has a CTA (single-frame latency)
  const int sms = env("PSTEREO_SMS", pp.fill_sms);
  while (rb > 1 && (long long)((g.ny + rb - 1) / rb) * pp.n_pairs < sms) --rb;
  bp.use_smem = bytes_for(rb) <= size_t(max_smem_per_cta);
  bp.rb = rb;
  bp.n_bands = (g.ny + rb - 1) / rb;
  bp.npb = rb * g.nx;
  bp.nx_magic = (unsigned)((0x100000000ull + (unsigned)g.nx - 1) / (unsigned)g.nx);
  bp.smem_rows = (rb - 1) * g.stride + g.size;
  bp.smem_bytes = bp.use_smem ? bytes_for(rb)
                              : band_layout(0, bp.rpitch, bp.fpitch, bp.bpitch, bp.npb, pp.nwin,
                                            valid, threads).total;
  bp.threads = std::min(threads, std::max(32, ((bp.npb + 31) / 32) * 32));
  return bp;
}

template <int S, bool kSmem, bool kValid>
static cudaError_t launch_t(const Level& L, const Level& P, const PatchParams& pp,
                            const BandPlan& bp, cudaStream_t s) {
  auto kern = k_patches<S, kSmem, kValid>;
  cudaError_t e = ensure_smem_cap((const void*)kern, bp.smem_bytes);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(bp.n_bands, pp.n_pairs);
  cfg.blockDim = dim3(bp.threads);
  cfg.dynamicSmemBytes = bp.smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pp.have_prev ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, L, P, pp, bp);
}

template <bool kSmem, bool kValid>
static cudaError_t launch_s(const Level& L, const Level& P, const PatchParams& pp,
                            const BandPlan& bp, cudaStream_t s) {
  switch (L.g.size) {
    case 8: return launch_t<8, kSmem, kValid>(L, P, pp, bp, s);
    case 10: return launch_t<10, kSmem, kValid>(L, P, pp, bp, s);
    case 12: return launch_t<12, kSmem, kValid>(L, P, pp, bp, s);
    case 16: return launch_t<16, kSmem, kValid>(L, P, pp, bp, s);
    // other sizes: runtime-size instantiations whose column tables hold at
    // most 8 / 16 entries (registers, not local memory), else 32
    default:
      if (L.g.size < 8) return launch_t<-8, kSmem, kValid>(L, P, pp, bp, s);
      if (L.g.size < 16) return launch_t<-16, kSmem, kValid>(L, P, pp, bp, s);
      return launch_t<0, kSmem, kValid>(L, P, pp, bp, s);
  }
}

cudaError_t launch_patches(const Level& L, const Level& P, const PatchParams& pp,
                           const BandPlan& bp, cudaStream_t s) {
  const bool valid = !pp.all_valid;
  if (bp.use_smem) return valid ? launch_s<true, true>(L, P, pp, bp, s)
                                : launch_s<true, false>(L, P, pp, bp, s);
  return valid ? launch_t<0, false, true>(L, P, pp, bp, s)
               : launch_t<0, false, false>(L, P, pp, bp, s);
}

// ---------------------------------------------------------------------------
// Test hook: eval_patch_residual for arbitrary (x0, y0, u) queries on one level,
// through exactly the device function k_patches uses (global-memory mode).
template <bool kValid>
__global__ void k_debug_eval(Level L, int size, int nq, const int* __restrict__ qx,
                             const int* __restrict__ qy, const double* __restrict__ qu,
                             double* __restrict__ msq, double* __restrict__ jr,
                             int* __restrict__ n) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  Rows<false> rw;
  rw.R = L.rpad;
  rw.Lf = L.left;
  rw.Gf = L.grad;
  rw.lq = L.lq;
  rw.rq = L.rq;
  rw.rp = rpad_pitch(L.w);
  rw.fp = L.w;
  rw.bp = L.w;
  const int x0 = qx[q], y0 = qy[q];
  // template mean (extract_patch, src/patch.cpp:15-33)
  double sum = 0.0;
  int cnt = 0;
  for (int j = 0; j < size; ++j)
    for (int i = 0; i < size; ++i) {
      if (kValid && !L.lq[(y0 + j) * L.w + x0 + i]) continue;
      sum = __dadd_rn(sum, (double)L.left[(y0 + j) * L.w + x0 + i]);
      ++cnt;
    }
  const double mean = cnt ? __ddiv_rn(sum, (double)cnt) : 0.0;
  const Ev ev = eval_patch<0, false, kValid>(rw, L.w, size, x0, y0, 0, mean, qu[q]);
  msq[q] = ev.msq;
  jr[q] = ev.jr;
  n[q] = ev.n;
}

cudaError_t launch_debug_eval(const Level& L, int size, int all_valid, int nq, const int* qx,
                              const int* qy, const double* qu, double* msq, double* jr, int* n,
                              cudaStream_t s) {
  const int t = 128;
  if (all_valid) k_debug_eval<false><<<(nq + t - 1) / t, t, 0, s>>>(L, size, nq, qx, qy, qu, msq, jr, n);
  else k_debug_eval<true><<<(nq + t - 1) / t, t, 0, s>>>(L, size, nq, qx, qy, qu, msq, jr, n);
  return cudaGetLastError();
}


}  // namespace bdis
