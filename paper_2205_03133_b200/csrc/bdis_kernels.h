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
};

struct FinestBufs {
  double* disp;
  double* prob;
  double* var;
  uint8_t* mvalid;
  uint8_t* mask;
  int* label;
};

struct OutputArgs {
  int W, H, e, fw, fh;
  long long fplane;
  const double* disp;
  const double* prob;
  const double* var;
  const uint8_t* mvalid;
  const uint8_t* fmask;
  const int* label;
  const int* area;
  long long min_px;
  double scale_d, scale_v, fb;
  int has_var;
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
void launch_patches(const Level& L, const Level& P, const PatchParams& pp, cudaStream_t s);
void launch_fuse_finest(const Level& L, const FinestBufs& fb, const double* mask,
                        int want_var, double threshold, int n_pairs, cudaStream_t s);
void launch_ccl(int w, int h, long long plane, int full_w, int full_h, int e,
                const uint8_t* mask, int* lab, int* area, int n_pairs, cudaStream_t s);
void launch_output(const OutputArgs& a, int f64, int n_pairs, cudaStream_t s);
void launch_stats(const StatsArgs& a, int n_pairs, cudaStream_t s);

}  // namespace bdis
