// bdis_kernels.h -- launch interface between the host runtime (bdis_capi.cu)
// and the sm_100a kernels (bdis_kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "bdis_device.cuh"

namespace bdis {

constexpr int kMaxLevels = 17;

struct PatchParams {
  int n_pairs;
  int size;
  double vpr;  // valid_patch_ratio
  int min_it, max_it;
  double stop_good, stop_bad, stop_improve;
  int nwin, wcenter;
  double woff[kMaxWin];  // sorted symmetric closure with 0
  int want_var;
  int have_prev;
  const double* prev_mask;  // spatial mask (s*s doubles, device)
  int all_valid;            // every input pixel valid: skip the 4-tap tests
  int fill_sms;             // host planning: spread small launches over >= this many CTAs
};

// Row-band decomposition of one level for k_patches (host-planned).
struct BandPlan {
  int rb;          // patch rows per CTA
  int n_bands;     // ceil(ny / rb)
  int threads;     // CTA size
  int smem_rows;   // (rb - 1) * stride + size
  int rpitch;      // smem slots per right-view row
  int fpitch;      // smem slots per left/gradient row (floats)
  int bpitch;      // bytes per validity row
  int use_smem;    // 0: read the level tables from global memory
  int rpad;        // zero slots either side of a staged right row (= patch size)
  size_t smem_bytes;
  int npb;         // max patches per band = rb * nx
  unsigned nx_magic;  // ceil(2^32 / nx): p / nx == umulhi(p, nx_magic) for p < npb
};

// Shared-memory layout of one k_patches CTA (byte offsets), shared by the
// host planner and the kernel.
struct BandLayout {
  size_t oR, oL, oG, oLQ, oRQ;
  size_t oMean, oHess, oTmsq, oU, oWres;
  size_t oCnt, oPool, oWlist, oCounters;
  size_t oSlotU, oSlotPrev, oSlotLastd, oSlotP, oSlotIt;
  size_t oStage, oWok;
  size_t total;
};

__host__ __device__ inline BandLayout band_layout(int rows, int rpitch, int fpitch, int bpitch,
                                                  int npb, int nwin, bool valid, int nslots) {
  BandLayout l;
  size_t o = 0;
  auto take = [&](size_t bytes, size_t align) {
    o = (o + align - 1) / align * align;
    const size_t r = o;
    o += bytes;
    return r;
  };
  l.oR = take(size_t(rows) * rpitch * 4, 16);
  l.oL = take(size_t(rows) * fpitch * 4, 16);
  l.oG = take(size_t(rows) * fpitch * 4, 16);
  l.oLQ = take(valid ? size_t(rows) * bpitch : 0, 16);
  l.oRQ = take(valid ? size_t(rows) * bpitch : 0, 16);
  l.oMean = take(size_t(npb) * 8, 8);
  l.oHess = take(size_t(npb) * 8, 8);
  l.oTmsq = take(size_t(npb) * 8, 8);
  l.oU = take(size_t(npb) * 8, 8);
  l.oWres = take(size_t(npb) * nwin * 8, 8);
  l.oCnt = take(size_t(npb) * 4, 4);
  l.oPool = take(size_t(npb) * 4, 4);
  l.oWlist = take(size_t(npb) * 4, 4);
  l.oCounters = take(32 * 4, 4);
  l.oSlotU = take(size_t(nslots) * 8, 8);
  l.oSlotPrev = take(size_t(nslots) * 8, 8);
  l.oSlotLastd = take(size_t(nslots) * 8, 8);
  l.oSlotP = take(size_t(nslots) * 4, 4);
  l.oSlotIt = take(size_t(nslots) * 4, 4);
  l.oStage = take(size_t(npb), 1);
  l.oWok = take(size_t(npb) * nwin, 1);
  l.total = (o + 15) / 16 * 16;
  return l;
}

BandPlan plan_bands(const Level& L, const PatchParams& pp, int max_smem_per_cta);

// Fused pyramid (all-valid inputs): levels are indexed by exponent.
struct PyrArgs {
  int n_pairs, W, H, C, ce, fe;
  const uint8_t* u8l;
  const uint8_t* u8r;
  const float* f0l;
  const float* f0r;
  int ws[kMaxLevels], hs[kMaxLevels];
  unsigned wmagic[kMaxLevels];  // ceil(2^32 / ws[e]): q / ws[e] == umulhi(q, wmagic[e]) in a band
  float* L[kMaxLevels];
  float* G[kMaxLevels];
  float* Rp[kMaxLevels];
  int buf_floats;  // floats per view in shared buffer 0 (levels 1, 3): 2^(ce-1) * ws[1]
  int buf1_floats; // floats per view in shared buffer 1 (levels 2, 4), rounded to 4
  int vec8;        // gray or RGB u8, W % 8 == 0, even H, 8-byte aligned rasters
};
size_t pyramid_smem_bytes(const PyrArgs& a);
cudaError_t launch_pyramid(const PyrArgs& a, bool u8, cudaStream_t s);

// Raises a kernel's dynamic shared-memory cap (cudaFuncAttributeMax-
// DynamicSharedMemorySize) on the current device to at least `bytes`. The
// attribute is per function and process-wide, so contexts on other host
// threads launching the same kernel with other sizes would race on a plain
// set; this only ever grows it, under a lock.
cudaError_t ensure_smem_cap(const void* kernel, size_t bytes);

// Finest-level fields written by the fusion kernel, already upsampled values
// in the output element type (disparity scaled by 2^fe, depth and sigma from
// the full-resolution disparity, src/coarse_to_fine.cpp:328-337,
// src/depth_variance.cpp:9-41); null planes are not requested.
struct FinestBufs {
  void* disp;   // scale_d * d           (0 where no patch covers)
  void* prob;   // p
  void* depth;  // D >= 0.1 ? fb / D : 0
  void* var;    // scale_v * v
  void* sigma;  // fb / D^2 * sqrt(max(V, 0)) where D >= 0.1
  uint8_t* flags;
  double scale_d, scale_v, fb, threshold;
};
// kFlagSure: kept, and the pixel's tile-local component alone already meets
// the area rule (its global component is a superset), so k_output needs no
// label lookup for it
enum FinestFlag : uint8_t { kFlagMatch = 1, kFlagKeep = 2, kFlagDepth = 4, kFlagSure = 8 };

// component labelling state at the finest level (per pair: one plane of
// labels and areas, ccl_tiles() root lists of ccl_tile_px() entries)
struct CclBufs {
  int* label;   // kept pixel -> tile-local root; tile-local root -> global root
  int* larea;   // at tile-local roots: tile-local area; at global roots: total
  int* roots;   // [pair][tile][ccl_tile_px()] tile-local roots (global indices)
  int* nroots;  // [pair][tile]
  int full_w, full_h, e;
  long long min_px;  // area rule of filter_validity, in full-resolution pixels
};
int ccl_tiles(int w, int h);
int ccl_tile_px();

struct OutputArgs {
  int W, H, e, fw, fh;
  long long fplane;
  FinestBufs fb;
  const int* label;
  const int* area;  // component area at global roots (CclBufs::larea)
  long long min_px;
  void* out_disp;
  uint8_t* out_dvalid;
  void* out_prob;
  void* out_depth;
  uint8_t* out_depth_valid;
  void* out_sigma;
  uint8_t* out_sigma_valid;
  void* out_mdisp;
  uint8_t* out_mvalid;
  void* out_var;
  int fill_invalid;
  double invalid_value;
  int flip_rows;  // output rows bottom to top (the PFM payload order)
};

struct StatsArgs {
  int n_levels;
  const uint8_t* stage[kMaxLevels];
  int np[kMaxLevels];
  int* out;  // [pair][level][3]: extracted, converged, accepted
};

void launch_gray_u8(const uint8_t* src, int channels, long long n_px, float* out,
                    uint8_t* valid, cudaStream_t s);
void launch_downsample(const float* sl, const uint8_t* slv, const float* sr,
                       const uint8_t* srv, int sw, int sh, float* dl, uint8_t* dlv,
                       float* dr, uint8_t* drv, int dw, int dh, int n_pairs,
                       cudaStream_t s);
void launch_level_tables(const Level& L, int n_pairs, cudaStream_t s);
cudaError_t launch_patches(const Level& L, const Level& P, const PatchParams& pp,
                           const BandPlan& bp, cudaStream_t s);
// fuse_level (finest) + threshold + 4-connected components with area sums
void launch_fuse_ccl(const Level& L, const FinestBufs& fb, const double* mask, int want_var,
                     int f64, const CclBufs& cb, int n_pairs, cudaStream_t s);
cudaError_t launch_debug_eval(const Level& L, int size, int all_valid, int nq, const int* qx,
                              const int* qy, const double* qu, double* msq, double* jr, int* n,
                              cudaStream_t s);
void launch_output(const OutputArgs& a, int f64, int n_pairs, cudaStream_t s);

// compute_metrics (src/metrics.cpp:10-52), one CTA per frame (bdis_metrics.cu)
struct pstereo_frame_metrics_dev {
  long long valid_px, compared;
  int has_errors;
  double mean_err, median_err, coverage_rate;
};
struct MetricsArgs {
  int w, h;
  const double* est;
  const uint8_t* est_valid;
  const double* ref;
  const uint8_t* ref_valid;
  const double* sigma;  // nullable (with sigma_valid)
  const uint8_t* sigma_valid;
  unsigned long long* scratch;  // w*h keys per frame
  pstereo_frame_metrics_dev* out;
};
cudaError_t launch_metrics(const MetricsArgs& a, int n_frames, cudaStream_t s);
void launch_stats(const StatsArgs& a, int n_pairs, cudaStream_t s);

}  // namespace bdis
