// bdis_render.cu -- the reference's analytic scene renderer on the device
// (SURVEY.md §8f row 4): render_scene, src/synth.cpp:209-284, with
// scene_depth_at / scene_intensity_at (:117-207), value_noise (:43-72) and
// gaussian_noise (:33-41).
//
// One thread per pixel of a batch of scenes of one size. A pixel's work is the
// left-view shading, the reference fields, and the right view's inverse warp:
// a 0.25-px scan down from d_max for the first root bracket of
// f(d) = d - disparity(x + d, y), then 50 bisection steps -- ~150 evaluations
// of the scene geometry in FP64, independent per pixel (FP64-pipe bound).
//
// Arithmetic follows the reference operation for operation (no FMA
// contraction: this TU builds with --fmad=false), so the geometry, the
// reference disparity/depth fields and the root search are bit-identical.
// The transcendentals of the shading (log/cos of the Box-Muller noise,
// pow of the specular highlight) are CUDA's, within 1-2 ulp of glibc's; the
// float views they feed are rounded from double, so they agree bit for bit
// except when a double lands within an ulp of a float rounding boundary
// (tests/test_gpu_render.py measures it).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/pstereo_gpu.h"

namespace {

thread_local std::string g_render_error;

__device__ __forceinline__ uint64_t r_splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// hash_unit, src/synth.cpp:24-27
__device__ __forceinline__ double r_hash_unit(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t h = r_splitmix(a ^ r_splitmix(b ^ r_splitmix(c)));
  return (double)(h >> 11) * 0x1.0p-53;
}

// gaussian_noise, src/synth.cpp:33-41
__device__ double r_gaussian(uint64_t seed, uint64_t stream, uint64_t index) {
  const double u1 = 1.0 - r_hash_unit(seed, stream * 2 + 1, index);
  const double u2 = r_hash_unit(seed, stream * 2 + 2, index);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

// value_noise, src/synth.cpp:43-72
__device__ double r_value_noise(double x, double y, uint64_t seed, int octaves, double base) {
  double sum = 0.0, norm = 0.0, amp = 1.0, wavelength = base;
  for (int o = 0; o < octaves; ++o) {
    const double gx = x / wavelength, gy = y / wavelength;
    const double fx = floor(gx), fy = floor(gy);
    const int64_t ix = (int64_t)fx, iy = (int64_t)fy;
    const double sx = gx - fx, sy = gy - fy;
    const double tx = sx * sx * (3.0 - 2.0 * sx);
    const double ty = sy * sy * (3.0 - 2.0 * sy);
    const uint64_t os = r_splitmix(seed + (uint64_t)o);
    const double v00 = r_hash_unit(os, (uint64_t)ix, (uint64_t)iy);
    const double v10 = r_hash_unit(os, (uint64_t)(ix + 1), (uint64_t)iy);
    const double v01 = r_hash_unit(os, (uint64_t)ix, (uint64_t)(iy + 1));
    const double v11 = r_hash_unit(os, (uint64_t)(ix + 1), (uint64_t)(iy + 1));
    const double v =
        (1.0 - ty) * ((1.0 - tx) * v00 + tx * v10) + ty * ((1.0 - tx) * v01 + tx * v11);
    sum += amp * v;
    norm += amp;
    amp *= 0.5;
    wavelength *= 0.5;
  }
  return sum / norm;
}

// sphere_hit, src/synth.cpp:104-113, ray (rx, ry, 1)
__device__ __forceinline__ double r_sphere_hit(const pstereo_scene_spec& s, double rx,
                                               double ry) {
  const double zc = s.sphere_depth + s.sphere_radius;
  const double dd = rx * rx + ry * ry + 1.0 * 1.0;
  const double dc = 1.0 * zc;
  const double disc = dc * dc - dd * (zc * zc - s.sphere_radius * s.sphere_radius);
  if (disc < 0.0) return -1.0;
  const double t = (dc - sqrt(disc)) / dd;
  if (t <= 0.0) return -1.0;
  return t * 1.0;
}

// scene_depth_at, src/synth.cpp:117-129 (pixel_ray :98-101)
__device__ __forceinline__ double r_depth_at(const pstereo_scene_spec& s, double x, double y) {
  const double fb = s.focal_px * s.baseline;
  if (s.surface == PSTEREO_SURFACE_SLANTED) return fb / (s.disparity0 + s.disparity_gradient * x);
  if (s.surface == PSTEREO_SURFACE_SPHERE) {
    const double rx = (x - 0.5 * (s.width - 1)) / s.focal_px;
    const double ry = (y - 0.5 * (s.height - 1)) / s.focal_px;
    const double z = r_sphere_hit(s, rx, ry);
    return z > 0.0 ? z : s.background_depth;
  }
  return fb / s.disparity;
}

// scene_disparity_at, src/synth.cpp:131-133
__device__ __forceinline__ double r_disparity_at(const pstereo_scene_spec& s, double x,
                                                 double y) {
  return s.focal_px * s.baseline / r_depth_at(s, x, y);
}

// reference_depth, src/synth.cpp:84-95
__device__ __forceinline__ double r_reference_depth(const pstereo_scene_spec& s) {
  const double fb = s.focal_px * s.baseline;
  if (s.surface == PSTEREO_SURFACE_SLANTED) return fb / s.disparity0;
  if (s.surface == PSTEREO_SURFACE_SPHERE) return s.background_depth;
  return fb / s.disparity;
}

// texture_at, src/synth.cpp:137-158
__device__ double r_texture_at(const pstereo_scene_spec& s, double wx, double wy) {
  const double wavelength = s.texture_scale * r_reference_depth(s) / s.focal_px;
  if (s.texture == PSTEREO_TEXTURE_PERLIN) {
    const double t = r_value_noise(wx / wavelength * s.texture_scale,
                                   wy / wavelength * s.texture_scale, s.seed, s.texture_octaves,
                                   s.texture_scale);
    return 0.1 + 0.8 * t;
  }
  if (s.texture == PSTEREO_TEXTURE_CHECKER) {
    const int64_t cx = (int64_t)floor(wx / wavelength);
    const int64_t cy = (int64_t)floor(wy / wavelength);
    return ((cx + cy) & 1) ? 0.8 : 0.2;
  }
  return 0.5;
}

// facing_cos, src/synth.cpp:161-188 (std::max(0.0, c) = 0 < c ? c : 0)
__device__ double r_facing_cos(const pstereo_scene_spec& s, double x, double y, double z) {
  if (s.surface == PSTEREO_SURFACE_SLANTED) {
    const double d = s.disparity0 + s.disparity_gradient * x;
    const double fb = s.focal_px * s.baseline;
    const double dzdx = -fb * s.disparity_gradient / (d * d);
    const double xc = x - 0.5 * (s.width - 1);
    const double a = z / s.focal_px + xc / s.focal_px * dzdx;
    const double c = a / sqrt(a * a + dzdx * dzdx);
    return 0.0 < c ? c : 0.0;
  }
  if (s.surface == PSTEREO_SURFACE_SPHERE) {
    const double rx = (x - 0.5 * (s.width - 1)) / s.focal_px;
    const double ry = (y - 0.5 * (s.height - 1)) / s.focal_px;
    const double zhit = r_sphere_hit(s, rx, ry);
    if (zhit <= 0.0) return 1.0;
    const double zc = s.sphere_depth + s.sphere_radius;
    const double nz = (zhit - zc) / s.sphere_radius;
    return 0.0 < -nz ? -nz : 0.0;
  }
  return 1.0;
}

// std::clamp(v, 0, 1)
__device__ __forceinline__ double r_clamp01(double v) {
  return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
}

// scene_intensity_at, src/synth.cpp:192-207
__device__ double r_intensity_at(const pstereo_scene_spec& s, double x, double y) {
  const double z = r_depth_at(s, x, y);
  const double rx = (x - 0.5 * (s.width - 1)) / s.focal_px;
  const double ry = (y - 0.5 * (s.height - 1)) / s.focal_px;
  double v = r_texture_at(s, rx * z, ry * z);
  const double cosa = r_facing_cos(s, x, y, z);
  v *= s.ambient + (1.0 - s.ambient) * cosa;
  if (s.shading == PSTEREO_SHADING_NONLAMBERTIAN) {
    const double h = s.highlight_strength * pow(cosa, s.highlight_falloff);
    v = v * (1.0 - h) + h * 0.95;
  }
  return r_clamp01(v);
}

struct RenderArgs {
  const pstereo_scene_spec* specs;
  int w, h;
  float* left;
  float* right;
  double* ref_disparity;
  double* ref_depth;
};

// render_scene, src/synth.cpp:209-284: one thread per pixel
__global__ void __launch_bounds__(128) k_render(RenderArgs A) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int k = blockIdx.z;
  if (x >= A.w) return;
  const pstereo_scene_spec& s = A.specs[k];
  const double fb = s.focal_px * s.baseline;
  double dmax;
  if (s.surface == PSTEREO_SURFACE_PLANE) {
    dmax = s.disparity + 1.0;
  } else if (s.surface == PSTEREO_SURFACE_SLANTED) {
    const double g = s.disparity_gradient;
    dmax = g > 0.0 ? (s.disparity0 + g * (A.w - 1) + 1.0) / (1.0 - g) : s.disparity0 + 1.0;
  } else {
    dmax = fb / s.sphere_depth + 1.0;
  }
  const size_t idx = (size_t)y * A.w + x;
  const size_t o = (size_t)k * A.w * A.h + idx;
  const double d_ref = r_disparity_at(s, x, y);
  if (A.ref_disparity) A.ref_disparity[o] = d_ref;
  if (A.ref_depth) A.ref_depth[o] = fb / d_ref;
  double v = r_intensity_at(s, x, y);
  if (s.noise_std > 0.0) v += s.noise_std * r_gaussian(s.seed, 0, idx);
  A.left[o] = (float)r_clamp01(v);
  // right(x) = left-view intensity of the surface point that lands here:
  // first root of f(d) = d - disparity(x + d) scanning down from dmax
  double hi = dmax, lo = 0.0;
  const double step = 0.25;
  for (double d = dmax - step; d > 0.0; d -= step) {
    if (d - r_disparity_at(s, x + d, y) <= 0.0) {
      lo = d;
      break;
    }
    hi = d;
  }
  for (int it = 0; it < 50; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid - r_disparity_at(s, x + mid, y) <= 0.0) lo = mid;
    else hi = mid;
  }
  const double d_star = 0.5 * (lo + hi);
  double rv = r_intensity_at(s, x + d_star, y);
  if (s.noise_std > 0.0) rv += s.noise_std * r_gaussian(s.seed, 1, idx);
  A.right[o] = (float)r_clamp01(rv);
}

int fail(int code, const std::string& m) {
  g_render_error = m;
  return code;
}

}  // namespace

extern "C" const char* pstereo_render_last_error(void) { return g_render_error.c_str(); }

extern "C" int pstereo_gpu_render(int device, const pstereo_scene_spec* specs, int n_scenes,
                                  float* left, float* right, double* ref_disparity,
                                  double* ref_depth, void* stream) {
  if (n_scenes < 0 || (n_scenes > 0 && (!specs || !left || !right)))
    return fail(PSTEREO_EINTERNAL, "pstereo_gpu_render: bad arguments");
  if (n_scenes == 0) return PSTEREO_OK;
  char msg[256];
  for (int k = 0; k < n_scenes; ++k) {
    if (pstereo_scene_validate(&specs[k], msg, sizeof msg) != PSTEREO_OK) return fail(PSTEREO_ECONFIG, msg);
    if (specs[k].width != specs[0].width || specs[k].height != specs[0].height)
      return fail(PSTEREO_ECONFIG, "pstereo_gpu_render: scenes of one call share width/height");
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(PSTEREO_EINTERNAL, cudaGetErrorString(e));
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (major != 10) return fail(PSTEREO_EINTERNAL, "pstereo_gpu_render: needs an sm_100 device");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t bytes = sizeof(pstereo_scene_spec) * (size_t)n_scenes;
  void* dspecs = nullptr;
  e = cudaMallocAsync(&dspecs, bytes, st);
  if (e != cudaSuccess) return fail(PSTEREO_EINTERNAL, cudaGetErrorString(e));
  e = cudaMemcpyAsync(dspecs, specs, bytes, cudaMemcpyHostToDevice, st);
  // the specs may live in pageable memory owned by the caller
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) {
    RenderArgs A;
    A.specs = (const pstereo_scene_spec*)dspecs;
    A.w = specs[0].width;
    A.h = specs[0].height;
    A.left = left;
    A.right = right;
    A.ref_disparity = ref_disparity;
    A.ref_depth = ref_depth;
    k_render<<<dim3((A.w + 127) / 128, A.h, n_scenes), 128, 0, st>>>(A);
    e = cudaGetLastError();
  }
  cudaError_t e2 = cudaFreeAsync(dspecs, st);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return fail(PSTEREO_EINTERNAL, cudaGetErrorString(e));
  return PSTEREO_OK;
}

// Host-buffer variant: device scratch, render, copy back (blocking).
extern "C" int pstereo_render_host(int device, const pstereo_scene_spec* specs, int n_scenes,
                                   float* left, float* right, double* ref_disparity,
                                   double* ref_depth) {
  if (n_scenes <= 0) return n_scenes == 0 ? PSTEREO_OK : fail(PSTEREO_EINTERNAL, "bad count");
  if (!specs) return fail(PSTEREO_EINTERNAL, "pstereo_render_host: bad arguments");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(PSTEREO_EINTERNAL, cudaGetErrorString(e));
  const size_t px = (size_t)specs[0].width * specs[0].height * n_scenes;
  char* buf = nullptr;
  e = cudaMalloc(&buf, px * 24);
  if (e != cudaSuccess) return fail(PSTEREO_EINTERNAL, cudaGetErrorString(e));
  float* dl = (float*)buf;
  float* dr = dl + px;
  double* dd = (double*)(buf + px * 8);
  double* dz = dd + px;
  int rc = pstereo_gpu_render(device, specs, n_scenes, dl, dr, ref_disparity ? dd : nullptr,
                              ref_depth ? dz : nullptr, nullptr);
  if (rc == PSTEREO_OK) {
    e = cudaMemcpy(left, dl, px * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(right, dr, px * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && ref_disparity)
      e = cudaMemcpy(ref_disparity, dd, px * 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && ref_depth) e = cudaMemcpy(ref_depth, dz, px * 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = fail(PSTEREO_EINTERNAL, cudaGetErrorString(e));
  }
  cudaFree(buf);
  return rc;
}
