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
//                           src/depth_variance.cpp:78-86  k_fuse_ccl_local
//   remove_small_components src/depth_variance.cpp:43-76  k_ccl_*
//   upsample_to_full + disparity_to_depth
//                           src/coarse_to_fine.cpp:166-180,328-337,
//                           src/depth_variance.cpp:9-41   k_output
//   MatchStats              src/coarse_to_fine.cpp:302-314 k_stats
// Coarse levels are never fused densely: the next level gathers the fused
// values it needs (init_next_level / inherited probability, :257-283) at its
// patch centres straight from the coarse patch records (bdis::gather).
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>
#include <math.h>
#include <stdint.h>

#include <type_traits>

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
  float* rp = L.rpad + blockIdx.y * (long long)rpad_pitch(w) * h + (long long)y * rpad_pitch(w);
  rp[x] = r[p00];
  if (x == w - 1) rp[w] = r[p00];
}

// Fused pyramid for fully valid inputs: one CTA per (row of the coarsest
// level, pair) builds every level's rows of that band -- to_grayscale on the
// fly from the uint8 raster (or the fp32 plane), then the cascade of
// downsample_half (src/pyramid.cpp:9-28, same ceil dims and edge clamps at
// every level) in shared memory -- and writes, for each stored level, the left
// view, its gradient_x (src/pyramid.cpp:30-42) and the padded right view.
// Replaces k_gray_u8 + k_downsample + k_level_tables: the full-resolution fp32
// planes never touch HBM.
// to_grayscale of one source pixel through shared lookup tables built with
// the reference's own expressions: gray = float(p * (1/255)); RGB: the three
// products 0.299 R, 0.587 G, 0.114 B (doubles), summed left to right.
struct GrayLut {
  const float* g1;   // [256] gray
  const double* c3;  // [3][256] RGB channel products
};

template <bool kU8>
__device__ __forceinline__ float src_px(const PyrArgs& a, const GrayLut& lut, int view,
                                        long long pair, int x, int y) {
  const long long i = pair * (long long)a.W * a.H + (long long)y * a.W + x;
  if (kU8) {
    const uint8_t* p = (view ? a.u8r : a.u8l) + i * a.C;
    if (a.C == 1) return lut.g1[p[0]];
    const double s = __dadd_rn(__dadd_rn(lut.c3[p[0]], lut.c3[256 + p[1]]), lut.c3[512 + p[2]]);
    return __double2float_rn(__dmul_rn(s, 1.0 / 255.0));
  }
  return (view ? a.f0r : a.f0l)[i];
}

__device__ __forceinline__ float down4(float a, float b, float c, float d) {
  return __fmul_rn(0.25f, __fadd_rn(__fadd_rn(__fadd_rn(a, b), c), d));
}

// kRGB: the vectorised RGB level-1 path (its own instantiation, so the gray
// path keeps its register budget)
template <bool kU8, bool kRGB = false>
__global__ void __launch_bounds__(256, kRGB ? 4 : 8) k_pyramid(PyrArgs a) {
  extern __shared__ __align__(16) float sbuf[];
  const long long pair = blockIdx.y;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int ce = a.ce, fe = a.fe;
  // level-1 rows of this band live in buf0 (L then R), level e >= 2 alternate
  // (pointer arithmetic on sbuf, not an indexed pointer array: that went to
  // local memory and turned the cascade's loads into generic LD)
  auto buf_of = [&](int k) { return sbuf + (k ? 2 * a.buf_floats : 0); };
  // grayscale lookup tables after the level buffers (8-byte aligned)
  double* c3 = (double*)(sbuf + ((2 * a.buf_floats + 2 * a.buf1_floats + 1) & ~1));
  float* g1 = (float*)(c3 + 768);
  if (kU8) {
    for (int q = tid; q < 256; q += nt) {
      g1[q] = __double2float_rn(__dmul_rn((double)q, 1.0 / 255.0));  // src/image.cpp:30
      c3[q] = __dmul_rn(0.299, (double)q);                            // src/image.cpp:36
      c3[256 + q] = __dmul_rn(0.587, (double)q);
      c3[512 + q] = __dmul_rn(0.114, (double)q);
    }
    __syncthreads();
  }
  const GrayLut lut{g1, c3};
  auto store = [&](int e, int y0, int rows, const float* Lb, const float* Rb) {
    const int w = a.ws[e];
    const long long pl = pair * (long long)w * a.hs[e];
    const int rpw = rpad_pitch(w);
    const long long pr = pair * (long long)rpw * a.hs[e];
    if ((w & 3) == 0 && w >= 8 && ((Rb - Lb) & 3) == 0 && ((Lb - sbuf) & 3) == 0) {
      // four pixels per thread: 16-byte stores of L and G (rows of 4k floats)
      const int qw = w >> 2;
      for (int q = tid; q < rows * qw; q += nt) {
        const int r = q / qw, x = (q - r * qw) << 2;
        const float* lr = Lb + r * w;
        const float4 l4 = *(const float4*)(lr + x);
        const float lm = x > 0 ? lr[x - 1] : 0.0f, lp = x + 4 < w ? lr[x + 4] : 0.0f;
        const float l[6] = {lm, l4.x, l4.y, l4.z, l4.w, lp};
        float g[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int xx = x + k;
          if (xx == 0) g[k] = __fsub_rn(l[k + 2], l[k + 1]);
          else if (xx == w - 1) g[k] = __fsub_rn(l[k + 1], l[k]);
          else g[k] = __fmul_rn(0.5f, __fsub_rn(l[k + 2], l[k]));
        }
        const long long o = pl + (long long)(y0 + r) * w + x;
        *(float4*)(a.L[e] + o) = l4;
        *(float4*)(a.G[e] + o) = make_float4(g[0], g[1], g[2], g[3]);
        const float4 r4 = *(const float4*)(Rb + r * w + x);
        float* rp = a.Rp[e] + pr + (long long)(y0 + r) * rpw + x;
        *(float4*)rp = r4;  // rows of rpad_pitch(w) floats start 16-byte aligned
        if (x + 4 == w) rp[4] = r4.w;
      }
      return;
    }
    for (int q = tid; q < rows * w; q += nt) {
      const int r = q / w, x = q % w;
      const float* lr = Lb + r * w;
      const float l = lr[x];
      float g = 0.0f;
      if (w >= 2) {
        if (x == 0) g = __fsub_rn(lr[1], lr[0]);
        else if (x == w - 1) g = __fsub_rn(lr[w - 1], lr[w - 2]);
        else g = __fmul_rn(0.5f, __fsub_rn(lr[x + 1], lr[x - 1]));
      }
      const long long o = pl + (long long)(y0 + r) * w + x;
      a.L[e][o] = l;
      a.G[e][o] = g;
      const float rv = Rb[r * w + x];
      float* rp = a.Rp[e] + pr + (long long)(y0 + r) * rpw;
      rp[x] = rv;
      if (x == w - 1) rp[w] = rv;
    }
  };
  // several bands per CTA (grid-stride): amortises the LUT set-up and keeps
  // every thread busy at the narrow coarse levels
  for (int band = blockIdx.x; band < a.hs[a.ce]; band += gridDim.x) {
    if (band != (int)blockIdx.x) __syncthreads();  // level buffers are reused
    // ---- level 0 rows of the band (stored only when finest_exp == 0)
    if (fe == 0) {
      const int r0 = band << ce, r1 = min(r0 + (1 << ce), a.H);
      const int W = a.W;
      const long long pl = pair * (long long)W * a.H, pr = pair * (long long)rpad_pitch(W) * a.H;
      for (int q = tid; q < (r1 - r0) * W; q += nt) {
        const int y = r0 + q / W, x = q % W;
        const float l = src_px<kU8>(a, lut, 0, pair, x, y);
        float g = 0.0f;
        if (W >= 2) {
          if (x == 0) g = __fsub_rn(src_px<kU8>(a, lut, 0, pair, 1, y), l);
          else if (x == W - 1) g = __fsub_rn(l, src_px<kU8>(a, lut, 0, pair, W - 2, y));
          else g = __fmul_rn(0.5f, __fsub_rn(src_px<kU8>(a, lut, 0, pair, x + 1, y),
                                             src_px<kU8>(a, lut, 0, pair, x - 1, y)));
        }
        const long long o = pl + (long long)y * W + x;
        a.L[0][o] = l;
        a.G[0][o] = g;
        const float rv = src_px<kU8>(a, lut, 1, pair, x, y);
        float* rp = a.Rp[0] + pr + (long long)y * rpad_pitch(W);
        rp[x] = rv;
        if (x == W - 1) rp[W] = rv;
      }
    }
    if (ce == 0) continue;
    // ---- level 1 from the source
    {
      const int w = a.ws[1], h = a.hs[1];
      const int y0 = band << (ce - 1), rows = min(1 << (ce - 1), h - y0);
      float* Lb = buf_of(0);
      float* Rb = Lb + a.buf_floats;
      if (kRGB) {
        // RGB rasters, W % 8 == 0, even H: 24 source bytes (8 pixels) of two
        // rows per view, three 8-byte loads each, give 4 level-1 pixels; the
        // luma of every pixel is src_px's (the same table sums, the same order)
        const int qw = w >> 2;
        for (int q = tid; q < rows * qw; q += nt) {
          const int r = q / qw, xq = q - r * qw;
          const long long base =
              3 * (pair * (long long)a.W * a.H + (long long)(2 * (y0 + r)) * a.W + 8 * xq);
  #pragma unroll
          for (int v = 0; v < 2; ++v) {
            const uint8_t* src = (v ? a.u8r : a.u8l) + base;
            unsigned tw[6], bw[6];
  #pragma unroll
            for (int k = 0; k < 3; ++k) {
              const uint2 t = __ldg((const uint2*)src + k);
              const uint2 b = __ldg((const uint2*)(src + 3 * a.W) + k);
              tw[2 * k] = t.x;
              tw[2 * k + 1] = t.y;
              bw[2 * k] = b.x;
              bw[2 * k + 1] = b.y;
            }
            auto byte = [](const unsigned* wd, int n) { return (wd[n >> 2] >> (8 * (n & 3))) & 255u; };
            // the channel products computed, not looked up: 96 random 8-byte
            // table reads per thread made this path shared-memory-bandwidth
            // bound (bank conflicts; issue 33%). (double)q is exact as
            // (2^52 + q) - 2^52, so q * coefficient is the table's value.
            auto prod = [](unsigned q, double coef) {
              return __dmul_rn(coef, __dsub_rn(__hiloint2double(0x43300000, (int)q),
                                               4503599627370496.0));
            };
            auto luma = [&](const unsigned* wd, int px) {
              const double sum = __dadd_rn(__dadd_rn(prod(byte(wd, 3 * px), 0.299),
                                                     prod(byte(wd, 3 * px + 1), 0.587)),
                                           prod(byte(wd, 3 * px + 2), 0.114));
              return __double2float_rn(__dmul_rn(sum, 1.0 / 255.0));
            };
            float o[4];
  #pragma unroll
            for (int k = 0; k < 4; ++k)
              o[k] = down4(luma(tw, 2 * k), luma(tw, 2 * k + 1), luma(bw, 2 * k), luma(bw, 2 * k + 1));
            *(float4*)((v ? Rb : Lb) + r * w + 4 * xq) = make_float4(o[0], o[1], o[2], o[3]);
          }
        }
      } else if (kU8 && a.vec8) {  // C == 1 here: the launcher routes vec8 RGB to kRGB
        // gray rasters, W % 8 == 0, even H: 8 source bytes of two rows per view
        // give 4 level-1 pixels (down4 of the grayscale values, as below)
        const int qw = w >> 2;
        for (int q = tid; q < rows * qw; q += nt) {
          const int r = q / qw, xq = q - r * qw;
          const long long base = pair * (long long)a.W * a.H + (long long)(2 * (y0 + r)) * a.W + 8 * xq;
  #pragma unroll
          for (int v = 0; v < 2; ++v) {
            const uint8_t* src = (v ? a.u8r : a.u8l) + base;
            const uint2 t = __ldg((const uint2*)src);
            const uint2 b = __ldg((const uint2*)(src + a.W));
            const unsigned tw[2] = {t.x, t.y}, bw[2] = {b.x, b.y};
            float o[4];
  #pragma unroll
            for (int k = 0; k < 4; ++k) {
              const unsigned ts = tw[k >> 1] >> (16 * (k & 1)), bs = bw[k >> 1] >> (16 * (k & 1));
              o[k] = down4(g1[ts & 255u], g1[(ts >> 8) & 255u], g1[bs & 255u], g1[(bs >> 8) & 255u]);
            }
            *(float4*)((v ? Rb : Lb) + r * w + 4 * xq) = make_float4(o[0], o[1], o[2], o[3]);
          }
        }
      } else
      for (int q = tid; q < rows * w; q += nt) {
        const int y = y0 + q / w, x = q % w;
        const int sx0 = 2 * x, sx1 = min(2 * x + 1, a.W - 1);
        const int sy0 = 2 * y, sy1 = min(2 * y + 1, a.H - 1);
        Lb[q] = down4(src_px<kU8>(a, lut, 0, pair, sx0, sy0), src_px<kU8>(a, lut, 0, pair, sx1, sy0),
                      src_px<kU8>(a, lut, 0, pair, sx0, sy1), src_px<kU8>(a, lut, 0, pair, sx1, sy1));
        Rb[q] = down4(src_px<kU8>(a, lut, 1, pair, sx0, sy0), src_px<kU8>(a, lut, 1, pair, sx1, sy0),
                      src_px<kU8>(a, lut, 1, pair, sx0, sy1), src_px<kU8>(a, lut, 1, pair, sx1, sy1));
      }
      __syncthreads();
      if (1 >= fe) store(1, y0, rows, Lb, Rb);
    }
    // ---- levels 2..ce from the previous level in shared memory
    for (int e = 2; e <= ce; ++e) {
      const int pw = a.ws[e - 1], ph = a.hs[e - 1];
      const int py0 = band << (ce - e + 1);
      const float* PL = buf_of((e - 2) & 1);
      const float* PR = PL + (((e - 2) & 1) ? a.buf1_floats : a.buf_floats);
      const int w = a.ws[e], h = a.hs[e];
      const int y0 = band << (ce - e), rows = min(1 << (ce - e), h - y0);
      float* Lb = buf_of((e - 1) & 1);
      float* Rb = Lb + (((e - 1) & 1) ? a.buf1_floats : a.buf_floats);
      const unsigned wm = a.wmagic[e];
      for (int q = tid; q < rows * w; q += nt) {
        const int qr = (int)__umulhi((unsigned)q, wm);  // q / w (q * w < 2^32)
        const int y = y0 + qr, x = q - qr * w;
        const int x0 = 2 * x, x1 = min(2 * x + 1, pw - 1);
        const int r0 = 2 * y - py0, r1 = min(2 * y + 1, ph - 1) - py0;
        Lb[q] = down4(PL[r0 * pw + x0], PL[r0 * pw + x1], PL[r1 * pw + x0], PL[r1 * pw + x1]);
        Rb[q] = down4(PR[r0 * pw + x0], PR[r0 * pw + x1], PR[r1 * pw + x0], PR[r1 * pw + x1]);
      }
      __syncthreads();
      if (e >= fe) store(e, y0, rows, Lb, Rb);
    }
  }
}

size_t pyramid_smem_bytes(const PyrArgs& a) {
  const size_t bufs =
      a.ce >= 1 ? size_t((2 * a.buf_floats + 2 * a.buf1_floats + 1) & ~1) * sizeof(float) : 0;
  return bufs + 768 * sizeof(double) + 256 * sizeof(float);  // + grayscale tables
}

cudaError_t ensure_smem_cap(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> cap;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cap[{dev, kernel}];
  if (bytes <= c) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) c = bytes;
  return e;
}

cudaError_t launch_pyramid(const PyrArgs& a, bool u8, cudaStream_t s) {
  const size_t smem = pyramid_smem_bytes(a);
  dim3 grid((a.hs[a.ce] + 1) / 2, a.n_pairs);  // two bands per CTA
  if (u8 && a.vec8 && a.C == 3) {
    ensure_smem_cap((const void*)k_pyramid<true, true>, smem);
    k_pyramid<true, true><<<grid, 256, smem, s>>>(a);
  } else if (u8) {
    ensure_smem_cap((const void*)k_pyramid<true>, smem);
    k_pyramid<true><<<grid, 256, smem, s>>>(a);
  } else {
    ensure_smem_cap((const void*)k_pyramid<false>, smem);
    k_pyramid<false><<<grid, 256, smem, s>>>(a);
  }
  return cudaGetLastError();
}

// --------------------------------------------------------------------------
// finest level: fusion, filter, components, output

// 4-connected components of the thresholded finest mask (the full-resolution
// mask is its block replication, so components and areas carry over with
// per-pixel area weights, src/depth_variance.cpp:43-92). Three passes:
//   k_fuse_ccl_local -- (after the fusion) components inside a 32x32 tile:
//                   horizontal runs from ballots, one smem union per
//                   overlapping run segment, run areas summed at the tile-local
//                   roots; every kept pixel labelled with its tile-local root
//                   (a global index), the roots listed per tile;
//   k_ccl_border -- unions across tile borders in global memory;
//   k_ccl_merge  -- per tile-local root: area added to its global root, link
//                   compressed to point at it (no per-pixel pass, no memset).
// Links always point to the smaller index (atomicMin), so the partition --
// and therefore the kept mask -- does not depend on scheduling.
constexpr int kTileW = 32, kTileH = 64, kTilePx = kTileW * kTileH;
constexpr int kFuseThreads = 256, kFuseWarps = kFuseThreads / 32, kFuseRows = kTileH / kFuseWarps;

template <typename Ptr>
__device__ __forceinline__ int uf_find(Ptr lab, int p) {
  int q = lab[p];
  while (q != p) {
    p = q;
    q = lab[p];
  }
  return p;
}

template <typename Ptr>
__device__ __forceinline__ void uf_union(Ptr lab, int* raw, int a, int b) {
  for (;;) {
    a = uf_find(lab, a);
    b = uf_find(lab, b);
    if (a == b) return;
    if (a < b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(&raw[a], b);
    if (old == a) return;
    a = old;
  }
}

// tile-local index of the first pixel of the run holding `lane` in `bits`
__device__ __forceinline__ int run_start(unsigned bits, int row, int lane) {
  const unsigned starts = bits & ~(bits << 1);
  const unsigned upto = starts & (0xffffffffu >> (31 - lane));
  return row * kTileW + (31 - __clz(upto));
}

// Shared-memory copy of the patch records covering one tile; records that are
// not accepted carry zero weight (prob = u = sigma = 0), which leaves the
// fusion sums bit-identical to skipping them (sums start at +0.0 and never
// become -0.0 under round-to-nearest, so adding +0.0 is the identity).
// One shared array: prob at [0, kTileRec), u at [kTileRec, 2 kTileRec), sigma_k
// after it -- the three loads of a record share one address register and
// differ by immediates.
struct TileRecords {
  const double* base;
  int ky0, kx0, ncol;
};

constexpr int kTileRec = 320;  // records staged per tile; more -> global gather

// Per-thread column list: the (at most K) patch columns covering the thread's
// pixel column, ascending, the clamped last patch after the regular ones;
// unused entries point at the tile's zero column (adds +0.0, the identity).
template <int K>
struct ColList {
  int kxo[K];   // column within the staged records, in bytes
  int moff[K];  // x - footprint start (mask column), in bytes
};

template <int K>
__device__ __forceinline__ bool col_list(const Grid& g, int x, Cover cx, int kx0, int zcol,
                                         ColList<K>* cl) {
  const int nmain = cx.hi - cx.lo + 1;
  const int used = max(nmain, 0) + (cx.last ? 1 : 0);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (k < nmain) {
      cl->kxo[k] = 8 * (cx.lo + k - kx0);
      cl->moff[k] = 8 * (x - (cx.lo + k) * g.stride);
    } else if (cx.last && k == max(nmain, 0)) {
      cl->kxo[k] = 8 * (g.nx - 1 - kx0);
      cl->moff[k] = 8 * (x - g.lastx0);
    } else {
      cl->kxo[k] = 8 * zcol;
      cl->moff[k] = 0;
    }
  }
  return used <= K;
}

template <bool kVar, int K>
__device__ __forceinline__ Fused gather_tile(const Grid& g, const TileRecords& rec, int y,
                                             const ColList<K>& cl, Cover cy,
                                             const double* __restrict__ mask) {
  const int s = g.size, st = g.stride;
  Fused f{0.0, 0.0, 0.0, 0.0};
  auto row = [&](int ky, int y0) {
    const char* mrow = (const char*)(mask + (y - y0) * s);
    const char* qrow = (const char*)(rec.base + (ky - rec.ky0) * rec.ncol);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double* q = (const double*)(qrow + cl.kxo[k]);
      const double pr = q[0];
      const double w = __dmul_rn(pr, *(const double*)(mrow + cl.moff[k]));
      f.sw = __dadd_rn(f.sw, w);
      f.swu = __dadd_rn(f.swu, __dmul_rn(w, q[kTileRec]));
      f.swp = __dadd_rn(f.swp, __dmul_rn(w, pr));
      if (kVar) {
        const double sk = q[2 * kTileRec];
        f.sw2s = __dadd_rn(f.sw2s, __dmul_rn(__dmul_rn(__dmul_rn(w, w), sk), sk));
      }
    }
  };
  // ascending patch index: rows ky ascending, columns kx ascending (:122-135)
  for (int ky = cy.lo; ky <= cy.hi; ++ky) row(ky, ky * st);
  if (cy.last) row(g.ny - 1, g.lasty0);
  return f;
}

// fuse_level at the finest level (src/coarse_to_fine.cpp:101-150) with the
// probability threshold of filter_validity (src/depth_variance.cpp:81-86),
// then the tile-local pass of the component labelling -- one CTA per 32x32
// tile, each warp four rows, each thread one column (its column cover is
// computed once). The records of the covering patches are staged in shared
// memory and each pixel gathers them in ascending patch index.
template <bool kVar, typename T, int K>
__global__ void __launch_bounds__(kFuseThreads, (!kVar && K <= 3) ? 5 : 4) k_fuse_ccl_local(
    Level L, FinestBufs fb, const double* __restrict__ mask, CclBufs cb) {
  __shared__ int sl[kTilePx];
  __shared__ int s_area[kTilePx];
  __shared__ unsigned s_bits[kTileH];
  __shared__ double s_rec[(kVar ? 3 : 2) * kTileRec];
  double* const s_pr = s_rec;
  double* const s_u = s_rec + kTileRec;
  double* const s_sg = s_rec + (kVar ? 2 * kTileRec : 0);  // (unused without variance)
  __shared__ Cover s_cy[kTileH];
  __shared__ double s_mask[kMaxPatch * kMaxPatch];
  __shared__ int s_nroot;
  const Grid& g = L.g;
  const int w = L.w, h = L.h;
  const int tiles_x = (w + kTileW - 1) / kTileW;
  const int tile = blockIdx.x;
  const int tx0 = (tile % tiles_x) * kTileW, ty0 = (tile / tiles_x) * kTileH;
  const long long pair = blockIdx.y;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int x = tx0 + lane;
  const int wl = min(kTileW, w - tx0) - 1, hl = min(kTileH, h - ty0) - 1;
  const Cover cx = cover_of(x, g.nx, g.size, g.stride, g.lastx0);
  // covering_range of the tile's columns from the first / last lane's covers
  const int lo0 = __shfl_sync(0xffffffffu, cx.lo, 0);
  const int hi1 = __shfl_sync(0xffffffffu, cx.hi, wl);
  const bool last1 = __shfl_sync(0xffffffffu, (int)cx.last, wl) != 0;
  const int kx0 = min(g.nx - 1, lo0);
  const int kx1 = max(kx0, last1 ? g.nx - 1 : hi1);
  if (t < kTileH) s_cy[t] = cover_of(ty0 + t, g.ny, g.size, g.stride, g.lasty0);
  for (int q = t; q < g.size * g.size; q += kFuseThreads) s_mask[q] = mask[q];
  if (t == 0) s_nroot = 0;
  __syncthreads();
  const int ky0 = min(g.ny - 1, s_cy[0].lo);
  const int ky1 = max(ky0, s_cy[hl].last ? g.ny - 1 : s_cy[hl].hi);
  // staged records: one row per patch row, the tile's columns plus a zero column
  const int ncol = kx1 - kx0 + 1, pitch = ncol + 1, nrec = pitch * (ky1 - ky0 + 1);
  ColList<K> cl;
  const bool listed = col_list<K>(g, x, cx, kx0, ncol, &cl);
  const bool all_listed = __syncthreads_and(listed || x >= w) != 0;
  const bool staged = nrec <= kTileRec && all_listed;
  if (staged) {
    const long long rbase = pair * (long long)g.nx * g.ny;
    for (int q = t; q < nrec; q += kFuseThreads) {
      const int rr = q / pitch, cc = q - rr * pitch;
      bool acc = false;
      long long r = 0;
      if (cc < ncol) {
        r = rbase + (long long)(ky0 + rr) * g.nx + kx0 + cc;
        acc = L.stage[r] == kAccepted;  // fuse_level skips the rest (:127)
      }
      s_pr[q] = acc ? L.prob[r] : 0.0;
      s_u[q] = acc ? L.u[r] : 0.0;
      if (kVar) s_sg[q] = acc ? L.sigma[r] : 0.0;
    }
  }
  __syncthreads();
  const TileRecords rec{s_rec, ky0, kx0, pitch};
  const long long pbase = pair * L.plane;
#pragma unroll 1
  for (int i = 0; i < kFuseRows; ++i) {
    const int ly = warp + i * kFuseWarps, y = ty0 + ly;
    bool keep = false;
    if (x < w && y < h) {
      const Fused f = staged ? gather_tile<kVar, K>(g, rec, y, cl, s_cy[ly], s_mask)
                             : gather<true, kVar>(L, pair, x, y, mask);
      const long long o = pbase + (long long)y * w + x;
      const bool valid = !(f.sw <= 0.0);  // fuse_level: sw <= 0 stays invalid (:138)
      double d = 0.0, p = 0.0, v = 0.0;
      if (valid) {
        d = __ddiv_rn(f.swu, f.sw);
        p = __ddiv_rn(f.swp, f.sw);
        if (kVar) v = __ddiv_rn(f.sw2s, __dmul_rn(f.sw, f.sw));
      }
      // upsample_to_full values (:166-180): scale 2^fe, 1, 4^fe where valid, else 0
      const double D = valid ? __dmul_rn(fb.scale_d, d) : 0.0;
      const double Pv = valid ? p : 0.0;  // scale 1: p * 1.0 == p exactly
      const double V = valid ? __dmul_rn(fb.scale_v, v) : 0.0;
      const bool deep = D >= 0.1;  // kMinDisparity (inc/depth_variance.hpp:13)
      keep = valid && !(Pv < fb.threshold);  // filter_validity threshold (:84)
      if (fb.disp) ((T*)fb.disp)[o] = (T)D;
      if (fb.prob) ((T*)fb.prob)[o] = (T)Pv;
      if (fb.depth) ((T*)fb.depth)[o] = (T)(deep ? __ddiv_rn(fb.fb, D) : 0.0);
      if (kVar) {
        if (fb.var) ((T*)fb.var)[o] = (T)V;
        if (fb.sigma) {
          double sg = 0.0;
          if (deep && valid) {
            const double vv = (V < 0.0) ? 0.0 : V;  // std::max(var, 0.0)
            sg = __dmul_rn(__ddiv_rn(fb.fb, __dmul_rn(D, D)), __dsqrt_rn(vv));
          }
          ((T*)fb.sigma)[o] = (T)sg;
        }
      }
      fb.flags[o] = (valid ? kFlagMatch : 0) | (keep ? kFlagKeep : 0) | (deep ? kFlagDepth : 0);
    }
    const unsigned bits = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_bits[ly] = bits;
    const int idx = ly * kTileW + lane;
    if (keep && !(lane > 0 && ((bits >> (lane - 1)) & 1u))) {  // run start
      sl[idx] = idx;
      s_area[idx] = 0;
    }
  }
  __syncthreads();
  const long long tid = pair * gridDim.x + tile;
  const int full = 1 << cb.e;
  // ---- dense tiles (every in-image pixel kept): one component rooted at the
  // tile's first pixel -- no unions, no finds
  bool mine_full = true, mine_empty = true;
  const unsigned in_cols = wl >= 31 ? 0xffffffffu : ((2u << wl) - 1u);
  for (int i = 0; i < kFuseRows; ++i) {
    const int ly = warp + i * kFuseWarps;
    mine_full = mine_full && s_bits[ly] == (ty0 + ly < h ? in_cols : 0u);
    mine_empty = mine_empty && s_bits[ly] == 0u;
  }
  if (__syncthreads_and(mine_empty)) {  // nothing kept: no components
    if (t == 0) cb.nroots[tid] = 0;
    return;
  }
  if (__syncthreads_and(mine_full)) {
    const int root_gi = ty0 * w + tx0;
    int a = 0;
    for (int i = 0; i < kFuseRows; ++i) {
      const int ly = warp + i * kFuseWarps, y = ty0 + ly;
      if (y >= h || x >= w) continue;
      cb.label[pbase + (long long)y * w + x] = root_gi;
      a += min(full, cb.full_w - (x << cb.e)) * min(full, cb.full_h - (y << cb.e));
    }
    a = __reduce_add_sync(0xffffffffu, a);
    if (t == 0) s_area[0] = 0;
    __syncthreads();
    if (lane == 0) atomicAdd(&s_area[0], a);
    __syncthreads();
    if (t == 0) {
      cb.larea[pbase + root_gi] = s_area[0];
      cb.roots[tid * kTilePx] = root_gi;
      cb.nroots[tid] = 1;
    }
    if (s_area[0] >= cb.min_px)
      for (int i = 0; i < kFuseRows; ++i) {
        const int y = ty0 + warp + i * kFuseWarps;
        if (y < h && x < w) fb.flags[pbase + (long long)y * w + x] |= kFlagSure;
      }
    return;
  }
  // one union per column segment where a run overlaps the run above it
  volatile int* vl = sl;
  for (int i = 0; i < kFuseRows; ++i) {
    const int ly = warp + i * kFuseWarps;
    if (ly == 0) continue;
    const unsigned b = s_bits[ly], a = s_bits[ly - 1];
    const unsigned both = a & b;
    if (!(((both & ~(both << 1)) >> lane) & 1u)) continue;
    int ra = run_start(b, ly, lane), rb = run_start(a, ly - 1, lane);
    for (;;) {
      while (vl[ra] != ra) {
        const int gg = vl[vl[ra]];
        vl[ra] = gg;
        ra = gg;
      }
      while (vl[rb] != rb) {
        const int gg = vl[vl[rb]];
        vl[rb] = gg;
        rb = gg;
      }
      if (ra == rb) break;
      if (ra < rb) {
        const int tmp = ra;
        ra = rb;
        rb = tmp;
      }
      const int old = atomicMin(&sl[ra], rb);
      if (old == ra) break;
      ra = old;
    }
  }
  __syncthreads();
  // labels and run areas (weights: full-resolution pixels per finest pixel)
  for (int i = 0; i < kFuseRows; ++i) {
    const int ly = warp + i * kFuseWarps, y = ty0 + ly;
    const unsigned bits = s_bits[ly];
    if (!((bits >> lane) & 1u)) continue;
    const int idx = ly * kTileW + lane;
    const int s0 = run_start(bits, ly, lane);
    const int root = uf_find(sl, s0);
    cb.label[pbase + (long long)y * w + x] = (ty0 + root / kTileW) * w + tx0 + root % kTileW;
    if (s0 == idx) {
      const unsigned rest = ~(bits >> lane);
      const int len = rest ? __ffs(rest) - 1 : 32;
      int sx = len << cb.e;
      if (x + len - 1 == w - 1) sx -= full - min(full, cb.full_w - ((w - 1) << cb.e));
      atomicAdd(&s_area[root], sx * min(full, cb.full_h - (y << cb.e)));
    }
  }
  __syncthreads();
  for (int i = 0; i < kFuseRows; ++i) {
    const int ly = warp + i * kFuseWarps;
    const unsigned bits = s_bits[ly];
    if (!((bits >> lane) & 1u)) continue;
    const int root = uf_find(sl, run_start(bits, ly, lane));
    if (s_area[root] >= cb.min_px)
      fb.flags[pbase + (long long)(ty0 + ly) * w + x] |= kFlagSure;
  }
  for (int i = 0; i < kFuseRows; ++i) {
    const int ly = warp + i * kFuseWarps;
    const int idx = ly * kTileW + lane;
    const unsigned bits = s_bits[ly];
    // roots are run starts whose link is themselves (sl holds nothing elsewhere)
    if (!(((bits & ~(bits << 1)) >> lane) & 1u) || sl[idx] != idx) continue;
    const int gi = (ty0 + ly) * w + x;
    cb.larea[pbase + gi] = s_area[idx];
    cb.roots[tid * kTilePx + atomicAdd(&s_nroot, 1)] = gi;
  }
  __syncthreads();
  if (t == 0) cb.nroots[tid] = s_nroot;
}

__global__ void k_ccl_border(int w, int h, long long plane, const uint8_t* __restrict__ mask,
                             int* lab) {
  // threads enumerate tile-border pixels only: vertical borders first
  // (x = k*kTileW, k >= 1, every row), then horizontal ones
  const int tiles_x = (w + kTileW - 1) / kTileW, tiles_y = (h + kTileH - 1) / kTileH;
  const int nv = (tiles_x - 1) * h, nh = (tiles_y - 1) * w;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nv + nh) return;
  int x, y;
  bool left;
  if (q < nv) {
    x = (q / h + 1) * kTileW;
    y = q % h;
    left = true;
  } else {
    x = (q - nv) % w;
    y = ((q - nv) / w + 1) * kTileH;
    left = false;
  }
  const long long base = blockIdx.y * plane;
  const int i = y * w + x;
  if (!(mask[base + i] & kFlagKeep)) return;
  int* l = lab + base;
  volatile int* vl = l;
  const int j = left ? i - 1 : i - w;
  if (!(mask[base + j] & kFlagKeep)) return;
  // both tile-local components already meet the area rule on their own: the
  // union cannot change any keep decision (a smaller component joined to
  // either one still reaches that one's area), so it is skipped
  if ((mask[base + i] & kFlagSure) && (mask[base + j] & kFlagSure)) return;
  // start from the tile-local roots; neighbouring border threads mostly join
  // the same pair of components, so one lane per distinct pair does the union
  const int a = l[i], b = l[j];
  const unsigned long long key = ((unsigned long long)(unsigned)a << 32) | (unsigned)b;
  const unsigned peers = __match_any_sync(__activemask(), key);
  if ((threadIdx.x & 31) == __ffs(peers) - 1) uf_union(vl, l, a, b);
}

// one warp per tile: every tile-local root adds its area to its global root
// (roots never receive from themselves, so the read of a non-root's area does
// not race) and is linked straight to it for k_output's two-load lookup
__global__ void k_ccl_merge(int n_tiles, int n_pairs, long long plane, CclBufs cb) {
  const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= (long long)n_tiles * n_pairs) return;
  const long long pair = wid / n_tiles;
  const int n = cb.nroots[wid];
  const int* rl = cb.roots + wid * kTilePx;
  int* lab = cb.label + pair * plane;
  volatile int* vl = lab;
  for (int k = threadIdx.x & 31; k < n; k += 32) {
    const int r = rl[k];
    const int R = uf_find(vl, r);
    if (R != r) {
      atomicAdd(&cb.larea[pair * plane + R], cb.larea[pair * plane + r]);
      vl[r] = R;
    }
  }
}

// upsample_to_full (src/coarse_to_fine.cpp:166-180, :328-337), the area rule
// of filter_validity (src/depth_variance.cpp:87-90), run_pipeline's mask
// sharing (src/pipeline.cpp:21-22) and disparity_to_depth (:9-41).
template <typename T>
__global__ void k_output(OutputArgs a) {
  // one thread per finest-level pixel: apply the area rule of filter_validity
  // (src/depth_variance.cpp:87-90) and replicate the fused values over the
  // pixel's 2^e x 2^e full-resolution block (nearest upsampling)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.fw * a.fh) return;
  const long long pair = blockIdx.y;
  const int fx = i % a.fw, fy = i / a.fw;
  const long long f = pair * a.fplane + i;
  const uint8_t fl = a.fb.flags[f];
  const bool mv = fl & kFlagMatch;
  bool keep = false;
  if (fl & kFlagSure) {
    keep = true;
  } else if (fl & kFlagKeep) {  // local root -> global root (k_ccl_merge) -> component area
    const int* lab = a.label + pair * a.fplane;
    keep = a.area[pair * a.fplane + lab[lab[i]]] >= a.min_px;
  }
  const bool dv = keep && (fl & kFlagDepth);  // depth valid; sigma valid too (var valid == mv)
  T d = a.fb.disp ? ((const T*)a.fb.disp)[f] : (T)0;
  const T p = a.fb.prob ? ((const T*)a.fb.prob)[f] : (T)0;
  T z = (dv && a.fb.depth) ? ((const T*)a.fb.depth)[f] : (T)0;
  const T v = a.fb.var ? ((const T*)a.fb.var)[f] : (T)0;
  T sg = (dv && a.fb.sigma) ? ((const T*)a.fb.sigma)[f] : (T)0;
  const T md = d;  // MatchResult::disparity keeps its value
  if (a.fill_invalid) {
    const T iv = (T)a.invalid_value;
    if (!keep) d = iv;
    if (!dv) z = iv, sg = iv;
  }
  const int x0 = fx << a.e, x1 = min((fx + 1) << a.e, a.W);
  const int y0 = fy << a.e, y1 = min((fy + 1) << a.e, a.H);
  const long long pbase = pair * (long long)a.W * a.H;
  using T2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  if (a.e == 1 && x1 - x0 == 2 && (a.W & 1) == 0) {
    // 2x2 blocks on an even-width image: vector stores, two rows
    const uchar2 kv{(unsigned char)keep, (unsigned char)keep};
    const uchar2 mv2{(unsigned char)mv, (unsigned char)mv};
    const uchar2 dv2{(unsigned char)dv, (unsigned char)dv};
    for (int y = y0; y < y1; ++y) {
      const long long o = pbase + (long long)(a.flip_rows ? a.H - 1 - y : y) * a.W + x0;
      if (a.out_disp) *(T2*)((T*)a.out_disp + o) = T2{d, d};
      if (a.out_dvalid) *(uchar2*)(a.out_dvalid + o) = kv;
      if (a.out_prob) *(T2*)((T*)a.out_prob + o) = T2{p, p};
      if (a.out_mdisp) *(T2*)((T*)a.out_mdisp + o) = T2{md, md};
      if (a.out_mvalid) *(uchar2*)(a.out_mvalid + o) = mv2;
      if (a.out_depth) *(T2*)((T*)a.out_depth + o) = T2{z, z};
      if (a.out_depth_valid) *(uchar2*)(a.out_depth_valid + o) = dv2;
      if (a.out_var) *(T2*)((T*)a.out_var + o) = T2{v, v};
      if (a.out_sigma) *(T2*)((T*)a.out_sigma + o) = T2{sg, sg};
      if (a.out_sigma_valid) *(uchar2*)(a.out_sigma_valid + o) = dv2;
    }
    return;
  }
  for (int y = y0; y < y1; ++y) {
    for (int x = x0; x < x1; ++x) {
      const long long o = pbase + (long long)(a.flip_rows ? a.H - 1 - y : y) * a.W + x;
      if (a.out_disp) ((T*)a.out_disp)[o] = d;
      if (a.out_dvalid) a.out_dvalid[o] = keep ? 1 : 0;
      if (a.out_prob) ((T*)a.out_prob)[o] = p;
      if (a.out_mdisp) ((T*)a.out_mdisp)[o] = md;
      if (a.out_mvalid) a.out_mvalid[o] = mv ? 1 : 0;
      if (a.out_depth) ((T*)a.out_depth)[o] = z;
      if (a.out_depth_valid) a.out_depth_valid[o] = dv ? 1 : 0;
      if (a.out_var) ((T*)a.out_var)[o] = v;
      if (a.out_sigma) ((T*)a.out_sigma)[o] = sg;
      if (a.out_sigma_valid) a.out_sigma_valid[o] = dv ? 1 : 0;
    }
  }
}

// The same per-pixel rule for the common layout -- 2x2 blocks (finest_exp 1),
// W = 2 fw, H = 2 fh, fw % 4 == 0, 16-byte aligned planes: one thread per
// four finest pixels, vector loads of the finest fields and 16-byte streaming
// stores of the two 8-pixel output rows.
template <typename T>
__device__ __forceinline__ void put_row8(void* base, long long o, T v0, T v1, T v2, T v3) {
  T* p = (T*)base + o;
  if constexpr (sizeof(T) == 4) {
    __stcs((float4*)p, make_float4(v0, v0, v1, v1));
    __stcs((float4*)p + 1, make_float4(v2, v2, v3, v3));
  } else {
    __stcs((double2*)p, make_double2(v0, v0));
    __stcs((double2*)p + 1, make_double2(v1, v1));
    __stcs((double2*)p + 2, make_double2(v2, v2));
    __stcs((double2*)p + 3, make_double2(v3, v3));
  }
}

__device__ __forceinline__ void put_row8_u8(uint8_t* base, long long o, unsigned m4) {
  // m4: one bit per finest pixel -> 8 bytes of 0/1
  const unsigned lo = (m4 & 1u) * 0x0101u | ((m4 >> 1) & 1u) * 0x01010000u;
  const unsigned hi = ((m4 >> 2) & 1u) * 0x0101u | ((m4 >> 3) & 1u) * 0x01010000u;
  __stcs((uint2*)(base + o), make_uint2(lo, hi));
}

template <typename T>
__device__ __forceinline__ void load4(const void* base, long long f, T* v) {
  if constexpr (sizeof(T) == 4) {
    const float4 q = *(const float4*)((const float*)base + f);
    v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
  } else {
    const double2 q0 = *(const double2*)((const double*)base + f);
    const double2 q1 = *((const double2*)((const double*)base + f) + 1);
    v[0] = q0.x, v[1] = q0.y, v[2] = q1.x, v[3] = q1.y;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_output_x4(OutputArgs a) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int qw = a.fw >> 2;
  if (q >= qw * a.fh) return;
  const long long pair = blockIdx.y;
  const int fy = q / qw, fx = (q - fy * qw) << 2;
  const long long f = pair * a.fplane + (long long)fy * a.fw + fx;
  const uchar4 fl = *(const uchar4*)(a.fb.flags + f);
  const uint8_t fls[4] = {fl.x, fl.y, fl.z, fl.w};
  unsigned keep = 0, mv = 0, dv = 0;
  const int* lab = a.label + pair * a.fplane;
  const int* area = a.area + pair * a.fplane;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    mv |= (unsigned)((fls[k] & kFlagMatch) != 0) << k;
    if (fls[k] & kFlagKeep) {  // local root -> global root -> component area
      const bool kp = (fls[k] & kFlagSure) || area[lab[lab[fy * a.fw + fx + k]]] >= a.min_px;
      keep |= (unsigned)kp << k;
      dv |= (unsigned)(kp && (fls[k] & kFlagDepth)) << k;
    }
  }
  T d[4] = {0, 0, 0, 0}, p[4] = {0, 0, 0, 0}, z[4] = {0, 0, 0, 0}, v[4] = {0, 0, 0, 0},
    sg[4] = {0, 0, 0, 0}, md[4];
  if (a.fb.disp) load4<T>(a.fb.disp, f, d);
  if (a.fb.prob) load4<T>(a.fb.prob, f, p);
  if (a.fb.depth) load4<T>(a.fb.depth, f, z);
  if (a.fb.var) load4<T>(a.fb.var, f, v);
  if (a.fb.sigma) load4<T>(a.fb.sigma, f, sg);
  const T iv = (T)a.invalid_value;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    md[k] = d[k];  // MatchResult::disparity keeps its value
    const bool kk = (keep >> k) & 1u, dd = (dv >> k) & 1u;
    if (!dd) z[k] = 0, sg[k] = 0;
    if (a.fill_invalid) {
      if (!kk) d[k] = iv;
      if (!dd) z[k] = iv, sg[k] = iv;
    }
  }
  const long long pbase = pair * (long long)a.W * a.H;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int y = 2 * fy + r;
    const long long o = pbase + (long long)(a.flip_rows ? a.H - 1 - y : y) * a.W + 2 * fx;
    if (a.out_disp) put_row8<T>(a.out_disp, o, d[0], d[1], d[2], d[3]);
    if (a.out_dvalid) put_row8_u8(a.out_dvalid, o, keep);
    if (a.out_prob) put_row8<T>(a.out_prob, o, p[0], p[1], p[2], p[3]);
    if (a.out_mdisp) put_row8<T>(a.out_mdisp, o, md[0], md[1], md[2], md[3]);
    if (a.out_mvalid) put_row8_u8(a.out_mvalid, o, mv);
    if (a.out_depth) put_row8<T>(a.out_depth, o, z[0], z[1], z[2], z[3]);
    if (a.out_depth_valid) put_row8_u8(a.out_depth_valid, o, dv);
    if (a.out_var) put_row8<T>(a.out_var, o, v[0], v[1], v[2], v[3]);
    if (a.out_sigma) put_row8<T>(a.out_sigma, o, sg[0], sg[1], sg[2], sg[3]);
    if (a.out_sigma_valid) put_row8_u8(a.out_sigma_valid, o, dv);
  }
}

// The same for the common request of the filtered disparity alone (plus its
// validity): no other planes in registers, so more CTAs stay resident.
template <typename T>
__global__ void __launch_bounds__(256) k_output_disp_x4(OutputArgs a) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int qw = a.fw >> 2;
  if (q >= qw * a.fh) return;
  const long long pair = blockIdx.y;
  const int fy = q / qw, fx = (q - fy * qw) << 2;
  const long long f = pair * a.fplane + (long long)fy * a.fw + fx;
  const uchar4 fl = *(const uchar4*)(a.fb.flags + f);
  const uint8_t fls[4] = {fl.x, fl.y, fl.z, fl.w};
  T d[4];
  load4<T>(a.fb.disp, f, d);
  unsigned keep = 0;
  const int* lab = a.label + pair * a.fplane;
  const int* area = a.area + pair * a.fplane;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (fls[k] & kFlagKeep)  // local root -> global root -> component area
      keep |= (unsigned)((fls[k] & kFlagSure) ||
                         area[lab[lab[fy * a.fw + fx + k]]] >= a.min_px) << k;
  if (a.fill_invalid) {
    const T iv = (T)a.invalid_value;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (!((keep >> k) & 1u)) d[k] = iv;
  }
  const long long pbase = pair * (long long)a.W * a.H;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int y = 2 * fy + r;
    const long long o = pbase + (long long)(a.flip_rows ? a.H - 1 - y : y) * a.W + 2 * fx;
    put_row8<T>(a.out_disp, o, d[0], d[1], d[2], d[3]);
    if (a.out_dvalid) put_row8_u8(a.out_dvalid, o, keep);
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

void launch_fuse_ccl(const Level& L, const FinestBufs& fb, const double* mask, int want_var,
                     int f64, const CclBufs& cb, int n_pairs, cudaStream_t s) {
  const int w = L.w, h = L.h;
  const long long plane = L.plane;
  const int nt = ccl_tiles(w, h);
  const dim3 grid(nt, n_pairs);
  // covering columns per pixel: at most ceil(size / stride) regular + the last
  const int kcov = (L.g.size + L.g.stride - 1) / L.g.stride + 1;
  auto go = [&](auto kv, auto kk) {
    constexpr bool V = decltype(kv)::value;
    constexpr int K = decltype(kk)::value;
    if (f64) k_fuse_ccl_local<V, double, K><<<grid, kFuseThreads, 0, s>>>(L, fb, mask, cb);
    else k_fuse_ccl_local<V, float, K><<<grid, kFuseThreads, 0, s>>>(L, fb, mask, cb);
  };
  using T3 = std::integral_constant<int, 3>;
  using T4 = std::integral_constant<int, 4>;
  using T6 = std::integral_constant<int, 6>;
  if (want_var) {
    if (kcov <= 3) go(std::true_type{}, T3{});
    else if (kcov <= 4) go(std::true_type{}, T4{});
    else go(std::true_type{}, T6{});
  } else {
    if (kcov <= 3) go(std::false_type{}, T3{});
    else if (kcov <= 4) go(std::false_type{}, T4{});
    else go(std::false_type{}, T6{});
  }
  const int tx = (w + kTileW - 1) / kTileW, ty = (h + kTileH - 1) / kTileH;
  const long long nb = (long long)(tx - 1) * h + (long long)(ty - 1) * w;
  if (nb > 0)
    k_ccl_border<<<dim3(blocks_for(nb, 256), n_pairs), 256, 0, s>>>(w, h, plane, fb.flags, cb.label);
  k_ccl_merge<<<blocks_for((long long)nt * n_pairs * 32, 256), 256, 0, s>>>(nt, n_pairs, plane, cb);
}

int ccl_tiles(int w, int h) { return ((w + kTileW - 1) / kTileW) * ((h + kTileH - 1) / kTileH); }
int ccl_tile_px() { return kTilePx; }

static bool aligned(const void* p, size_t n) { return ((uintptr_t)p % n) == 0; }

void launch_output(const OutputArgs& a, int f64, int n_pairs, cudaStream_t s) {
  const size_t vt = 16;  // float4 / double2
  bool x4 = a.e == 1 && a.W == 2 * a.fw && a.H == 2 * a.fh && a.fw % 4 == 0 &&
            a.fplane % 4 == 0;
  for (const void* p : {(const void*)a.out_disp, (const void*)a.out_prob, (const void*)a.out_mdisp,
                        (const void*)a.out_depth, (const void*)a.out_var, (const void*)a.out_sigma,
                        (const void*)a.fb.disp, (const void*)a.fb.prob, (const void*)a.fb.depth,
                        (const void*)a.fb.var, (const void*)a.fb.sigma})
    x4 = x4 && aligned(p, vt);
  for (const void* p : {(const void*)a.out_dvalid, (const void*)a.out_mvalid,
                        (const void*)a.out_depth_valid, (const void*)a.out_sigma_valid})
    x4 = x4 && aligned(p, 8);
  if (x4) {
    dim3 grid(blocks_for((long long)(a.fw / 4) * a.fh, 256), n_pairs);
    const bool disp_only = a.out_disp && !a.out_prob && !a.out_mdisp && !a.out_mvalid &&
                           !a.out_depth && !a.out_depth_valid && !a.out_var && !a.out_sigma &&
                           !a.out_sigma_valid;
    if (disp_only) {
      if (f64) k_output_disp_x4<double><<<grid, 256, 0, s>>>(a);
      else k_output_disp_x4<float><<<grid, 256, 0, s>>>(a);
      return;
    }
    if (f64) k_output_x4<double><<<grid, 256, 0, s>>>(a);
    else k_output_x4<float><<<grid, 256, 0, s>>>(a);
    return;
  }
  dim3 grid(blocks_for((long long)a.fw * a.fh, 256), n_pairs);
  if (f64) k_output<double><<<grid, 256, 0, s>>>(a);
  else k_output<float><<<grid, 256, 0, s>>>(a);
}

void launch_stats(const StatsArgs& a, int n_pairs, cudaStream_t s) {
  dim3 grid(n_pairs, a.n_levels);
  k_stats<<<grid, 256, 0, s>>>(a);
}

}  // namespace bdis
