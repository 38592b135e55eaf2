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
  float* rp = L.rpad + blockIdx.y * (long long)(w + 1) * h + (long long)y * (w + 1);
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

template <bool kU8>
__global__ void __launch_bounds__(256) k_pyramid(PyrArgs a) {
  extern __shared__ __align__(16) float sbuf[];
  const int band = blockIdx.x;
  const long long pair = blockIdx.y;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int ce = a.ce, fe = a.fe;
  // level-1 rows of this band live in buf0 (L then R), level e >= 2 alternate
  float* buf[2] = {sbuf, sbuf + 2 * a.buf_floats};
  // grayscale lookup tables after the level buffers (8-byte aligned)
  double* c3 = (double*)(sbuf + ((4 * a.buf_floats + 1) & ~1));
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
    const long long pr = pair * (long long)(w + 1) * a.hs[e];
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
      float* rp = a.Rp[e] + pr + (long long)(y0 + r) * (w + 1);
      rp[x] = rv;
      if (x == w - 1) rp[w] = rv;
    }
  };
  // ---- level 0 rows of the band (stored only when finest_exp == 0)
  if (fe == 0) {
    const int r0 = band << ce, r1 = min(r0 + (1 << ce), a.H);
    const int W = a.W;
    const long long pl = pair * (long long)W * a.H, pr = pair * (long long)(W + 1) * a.H;
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
      float* rp = a.Rp[0] + pr + (long long)y * (W + 1);
      rp[x] = rv;
      if (x == W - 1) rp[W] = rv;
    }
  }
  if (ce == 0) return;
  // ---- level 1 from the source
  {
    const int w = a.ws[1], h = a.hs[1];
    const int y0 = band << (ce - 1), rows = min(1 << (ce - 1), h - y0);
    float* Lb = buf[0];
    float* Rb = buf[0] + a.buf_floats;
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
    const float* PL = buf[(e - 2) & 1];
    const float* PR = PL + a.buf_floats;
    const int w = a.ws[e], h = a.hs[e];
    const int y0 = band << (ce - e), rows = min(1 << (ce - e), h - y0);
    float* Lb = buf[(e - 1) & 1];
    float* Rb = Lb + a.buf_floats;
    for (int q = tid; q < rows * w; q += nt) {
      const int y = y0 + q / w, x = q % w;
      const int x0 = 2 * x, x1 = min(2 * x + 1, pw - 1);
      const int r0 = 2 * y - py0, r1 = min(2 * y + 1, ph - 1) - py0;
      Lb[q] = down4(PL[r0 * pw + x0], PL[r0 * pw + x1], PL[r1 * pw + x0], PL[r1 * pw + x1]);
      Rb[q] = down4(PR[r0 * pw + x0], PR[r0 * pw + x1], PR[r1 * pw + x0], PR[r1 * pw + x1]);
    }
    __syncthreads();
    if (e >= fe) store(e, y0, rows, Lb, Rb);
  }
}

size_t pyramid_smem_bytes(const PyrArgs& a) {
  const size_t bufs = a.ce >= 1 ? size_t((4 * a.buf_floats + 1) & ~1) * sizeof(float) : 0;
  return bufs + 768 * sizeof(double) + 256 * sizeof(float);  // + grayscale tables
}

cudaError_t launch_pyramid(const PyrArgs& a, bool u8, cudaStream_t s) {
  const size_t smem = pyramid_smem_bytes(a);
  dim3 grid(a.hs[a.ce], a.n_pairs);
  if (u8) {
    cudaFuncSetAttribute(k_pyramid<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_pyramid<true><<<grid, 256, smem, s>>>(a);
  } else {
    cudaFuncSetAttribute(k_pyramid<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_pyramid<false><<<grid, 256, smem, s>>>(a);
  }
  return cudaGetLastError();
}

// --------------------------------------------------------------------------
// finest level: fusion, filter, components, output

// 4-connected components of the thresholded finest mask (the full-resolution
// mask is its block replication, so components and areas carry over with
// per-pixel area weights, src/depth_variance.cpp:43-92). Three passes:
//   k_fuse_ccl_local -- (after the fusion) union-find inside a 32x16 tile in smem, every
//                   pixel labelled with its tile-local root (a global index);
//   k_ccl_border -- unions across tile borders in global memory;
//   k_ccl_final  -- path compression + warp-aggregated component areas.
// Links always point to the smaller index (atomicMin), so the partition --
// and therefore the kept mask -- does not depend on scheduling.
constexpr int kTileW = 32, kTileH = 16;

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

// Shared-memory copy of the patch records covering one tile.
struct TileRecords {
  const uint8_t* st;
  const double* pr;
  const double* uu;
  const double* sg;
  int ky0, kx0, ncol;
  __device__ __forceinline__ int at(int ky, int kx) const { return (ky - ky0) * ncol + (kx - kx0); }
  __device__ __forceinline__ uint8_t stage(int ky, int kx) const { return st[at(ky, kx)]; }
  __device__ __forceinline__ double prob(int ky, int kx) const { return pr[at(ky, kx)]; }
  __device__ __forceinline__ double u(int ky, int kx) const { return uu[at(ky, kx)]; }
  __device__ __forceinline__ double sigma(int ky, int kx) const { return sg[at(ky, kx)]; }
};

constexpr int kTileRec = 160;  // max covering patches per 32x16 tile (stride >= 2, s <= 32)

// fuse_level at the finest level (src/coarse_to_fine.cpp:101-150) with the
// probability threshold of filter_validity (src/depth_variance.cpp:81-86),
// then the tile-local pass of the component labelling -- one CTA per 32x16
// tile. The records of the covering patches are staged in shared memory and
// each pixel gathers them in ascending patch index (fuse_level's order).
template <bool kVar, typename T>
__global__ void __launch_bounds__(kTileW * kTileH) k_fuse_ccl_local(
    Level L, FinestBufs fb, const double* __restrict__ mask) {
  __shared__ int sl[kTileW * kTileH];
  __shared__ double s_pr[kTileRec], s_u[kTileRec], s_sg[kTileRec];
  __shared__ uint8_t s_st[kTileRec];
  const Grid& g = L.g;
  const int w = L.w, h = L.h;
  const int tiles_x = (w + kTileW - 1) / kTileW;
  const int tx0 = (blockIdx.x % tiles_x) * kTileW, ty0 = (blockIdx.x / tiles_x) * kTileH;
  const long long pair = blockIdx.y;
  const int t = threadIdx.x, lx = t % kTileW, ly = t / kTileW;
  const int x = tx0 + lx, y = ty0 + ly;
  int kx0, kx1, ky0, ky1;
  covering_range(tx0, min(tx0 + kTileW, w) - 1, g.nx, g.size, g.stride, g.lastx0, &kx0, &kx1);
  covering_range(ty0, min(ty0 + kTileH, h) - 1, g.ny, g.size, g.stride, g.lasty0, &ky0, &ky1);
  const int ncol = kx1 - kx0 + 1, nrec = ncol * (ky1 - ky0 + 1);
  const long long rbase = pair * (long long)g.nx * g.ny;
  const bool staged = nrec <= kTileRec;
  // covering ranges per tile column / row (no integer divisions per pixel)
  __shared__ Cover s_cx[kTileW], s_cy[kTileH];
  __shared__ double s_mask[kMaxPatch * kMaxPatch];
  if (t < kTileW) s_cx[t] = cover_of(tx0 + t, g.nx, g.size, g.stride, g.lastx0);
  else if (t < kTileW + kTileH) s_cy[t - kTileW] = cover_of(ty0 + t - kTileW, g.ny, g.size, g.stride, g.lasty0);
  for (int q = t; q < g.size * g.size; q += blockDim.x) s_mask[q] = mask[q];
  if (staged) {
    for (int q = t; q < nrec; q += blockDim.x) {
      const long long r = rbase + (long long)(ky0 + q / ncol) * g.nx + kx0 + q % ncol;
      s_st[q] = L.stage[r];
      s_pr[q] = L.prob[r];
      s_u[q] = L.u[r];
      if (kVar) s_sg[q] = L.sigma[r];
    }
  }
  __syncthreads();
  bool keep = false;
  if (x < w && y < h) {
    Fused f;
    if (staged) {
      const TileRecords rec{s_st, s_pr, s_u, s_sg, ky0, kx0, ncol};
      f = gather_cover<true, kVar>(g, rec, x, y, s_cx[lx], s_cy[ly], s_mask);
    } else {
      f = gather<true, kVar>(L, pair, x, y, mask);
    }
    const long long o = pair * L.plane + (long long)y * w + x;
    const bool valid = !(f.sw <= 0.0);  // fuse_level: sw <= 0 stays invalid (:138)
    double d = 0.0, p = 0.0, v = 0.0;
    if (valid) {
      d = __ddiv_rn(f.swu, f.sw);
      p = __ddiv_rn(f.swp, f.sw);
      if (kVar) v = __ddiv_rn(f.sw2s, __dmul_rn(f.sw, f.sw));
    }
    // upsample_to_full values (:166-180): scale 2^fe, 1, 4^fe where valid, else 0
    const double D = valid ? __dmul_rn(fb.scale_d, d) : 0.0;
    const double Pv = valid ? __dmul_rn(1.0, p) : 0.0;
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
  // ---- tile-local components: run labels (ballot bit tricks) + union-find
  const unsigned bits = __ballot_sync(0xffffffffu, keep);
  const unsigned starts = bits & ~(bits << 1);
  const unsigned upto = starts & (0xffffffffu >> (31 - lx));
  sl[t] = keep ? ly * kTileW + (31 - __clz(upto)) : -1;
  __syncthreads();
  volatile int* vl = sl;
  if (keep && ly > 0 && sl[t - kTileW] >= 0) {
    int a = sl[t], b = sl[t - kTileW];
    for (;;) {
      while (vl[a] != a) {
        const int gg = vl[vl[a]];
        vl[a] = gg;
        a = gg;
      }
      while (vl[b] != b) {
        const int gg = vl[vl[b]];
        vl[b] = gg;
        b = gg;
      }
      if (a == b) break;
      if (a < b) {
        const int tmp = a;
        a = b;
        b = tmp;
      }
      const int old = atomicMin(&sl[a], b);
      if (old == a) break;
      a = old;
    }
  }
  __syncthreads();
  if (keep) {
    const int r = uf_find(vl, t);
    fb.label[pair * L.plane + (long long)y * w + x] = (ty0 + r / kTileW) * w + tx0 + r % kTileW;
  }
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
  if (mask[base + j] & kFlagKeep) uf_union(vl, l, i, j);
}

__global__ void k_ccl_final(int w, int h, long long plane, int full_w, int full_h, int e,
                            const uint8_t* __restrict__ mask, int* lab, int* area) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const long long base = blockIdx.y * plane;
  const bool m = i < w * h && (mask[base + i] & kFlagKeep);
  int root = -1, weight = 0;
  if (m) {
    volatile int* vl = lab + base;
    root = uf_find(vl, i);
    lab[base + i] = root;
    const int x = i % w, y = i / w;
    weight = min(1 << e, full_w - (x << e)) * min(1 << e, full_h - (y << e));
  }
  // one atomic per distinct root in the warp
  unsigned pending = __ballot_sync(0xffffffffu, m);
  while (pending) {
    const int leader = __ffs(pending) - 1;
    const int r = __shfl_sync(0xffffffffu, root, leader);
    const bool mine = m && root == r;
    const int sum = __reduce_add_sync(0xffffffffu, mine ? weight : 0);
    if ((int)(threadIdx.x & 31) == leader) atomicAdd(&area[base + r], sum);
    pending &= ~__ballot_sync(0xffffffffu, mine);
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
  if (fl & kFlagKeep) keep = a.area[pair * a.fplane + a.fb.label[f]] >= a.min_px;
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
      const long long o = pbase + (long long)y * a.W + x0;
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
      const long long o = pbase + (long long)y * a.W + x;
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
                     int f64, int full_w, int full_h, int e, int* area, int n_pairs,
                     cudaStream_t s) {
  const int w = L.w, h = L.h;
  const long long plane = L.plane;
  const int tx = (w + kTileW - 1) / kTileW, ty = (h + kTileH - 1) / kTileH;
  const dim3 grid(tx * ty, n_pairs);
  if (want_var) {
    if (f64) k_fuse_ccl_local<true, double><<<grid, kTileW * kTileH, 0, s>>>(L, fb, mask);
    else k_fuse_ccl_local<true, float><<<grid, kTileW * kTileH, 0, s>>>(L, fb, mask);
  } else {
    if (f64) k_fuse_ccl_local<false, double><<<grid, kTileW * kTileH, 0, s>>>(L, fb, mask);
    else k_fuse_ccl_local<false, float><<<grid, kTileW * kTileH, 0, s>>>(L, fb, mask);
  }
  const long long nb = (long long)(tx - 1) * h + (long long)(ty - 1) * w;
  if (nb > 0)
    k_ccl_border<<<dim3(blocks_for(nb, 256), n_pairs), 256, 0, s>>>(w, h, plane, fb.flags, fb.label);
  k_ccl_final<<<dim3(blocks_for((long long)w * h, 256), n_pairs), 256, 0, s>>>(
      w, h, plane, full_w, full_h, e, fb.flags, fb.label, area);
}

void launch_output(const OutputArgs& a, int f64, int n_pairs, cudaStream_t s) {
  dim3 grid(blocks_for((long long)a.fw * a.fh, 256), n_pairs);
  if (f64) k_output<double><<<grid, 256, 0, s>>>(a);
  else k_output<float><<<grid, 256, 0, s>>>(a);
}

void launch_stats(const StatsArgs& a, int n_pairs, cudaStream_t s) {
  dim3 grid(n_pairs, a.n_levels);
  k_stats<<<grid, 256, 0, s>>>(a);
}

}  // namespace bdis
