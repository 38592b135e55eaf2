// bdis_synth.cu -- on-device BASELINE.json pair generator.
//
// Produces, for pairs seed0 .. seed0+n-1, the same bytes as the host generator
// pstereo_synth_pair (csrc/synth.c): both evaluate the per-element arithmetic
// of csrc/synth_core.h (integer hashing + IEEE-exact double/float operations,
// no FMA contraction: this TU builds with --fmad=false like the rest), and
// the float blur accumulates its taps in the same order. The generator lets a
// multi-GPU run fill its inputs in HBM instead of generating on the host and
// crossing PCIe.
//
// Per chunk of pairs, four launches:
//   k_syn_hblur   CTA per (row, pair): the row's white noise (edge-clamped,
//                 r extra columns either side) into smem, horizontal taps
//   k_syn_vblur_tile  32 columns x 64 rows per CTA: the column strip staged
//                 in smem, sliding window of 8 outputs per thread (each input
//                 row loaded once), per-pair min/max of the blurred field
//                 (order-free: exact); k_syn_vblur (taps through L1) when the
//                 strip does not fit
//   k_syn_discs   (stress only) CTA per pair: the sequential disc placement
//                 loop with a per-pair coverage map, one disc per iteration
//   k_syn_views   CTA per (row, pair): the row's value-noise lattice into
//                 smem, texture row into smem (left view), then the right view
//                 sampled from it at x + d plus noise
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pstereo_gpu.h"
#include "synth_core.h"

namespace bdis {
// bdis_kernels.cu: grow-only, thread-safe dynamic shared-memory cap
cudaError_t ensure_smem_cap(const void* kernel, size_t bytes);
}  // namespace bdis

namespace {

thread_local std::string g_synth_error;

struct SynthDev {
  int w, h, C;
  int octaves;
  double wavelength, d_min, d_range, noise_sigma;
  int stress;
  int r;                 // blur radius
  uint64_t seed0;        // seed of the chunk's first pair
  const float* weights;  // 2r+1 blur taps
  float* tmp;            // [pair][h][w] horizontal pass
  float* fld;            // [pair][h][w] blurred field
  unsigned* minmax;      // [pair][2]: ~bits(min), bits(max) (non-negative floats)
  uint8_t* cov;          // [pair][h][w] disc coverage (stress)
  double* discs;         // [pair][SYN_MAX_DISCS][4]
  int* n_discs;          // [pair]
  uint8_t* left;         // [pair][h][w][C]
  uint8_t* right;
  float* disparity;      // [pair][h][w] or null
};

// Horizontal pass, four consecutive outputs per thread: the row's line is read
// as float4 (one 16-byte load feeds four taps of four outputs) and the tap
// weights rotate through registers. Output o of a thread takes tap jj - o at
// input jj, in ascending order; out-of-range taps use zero weights, and since
// every weight and every noise value is >= +0, adding +0 * v = +0 to a sum
// that is >= +0 leaves it bit-identical -- the host's sums exactly.
constexpr int kHPad = 4;   // zero weights before tap 0
constexpr int kHTail = 8;  // zero weights after the last tap (the last block overruns by <= 5)

__global__ void k_syn_hblur(SynthDev S) {
  extern __shared__ __align__(16) float sm_h[];
  const int y = blockIdx.x, p = blockIdx.y;
  const int w = S.w, r = S.r, taps = 2 * r + 1;
  const int nline = ((w + 2 * r + 3) & ~3) + 8;           // float4-padded line
  float* line = sm_h;
  float* kw = sm_h + nline;                                // [kHPad zeros][taps][kHTail zeros]
  const uint64_t key = syn_pair_key(S.seed0 + (uint64_t)p);
  for (int i = threadIdx.x; i < taps + kHPad + kHTail; i += blockDim.x) {
    const int t = i - kHPad;
    kw[i] = (t >= 0 && t < taps) ? S.weights[t] : 0.0f;
  }
  for (int i = threadIdx.x; i < nline; i += blockDim.x) {
    int xs = i - r;
    xs = xs < 0 ? 0 : (xs >= w ? w - 1 : xs);
    line[i] = syn_white(key, xs, y);
  }
  __syncthreads();
  float* out = S.tmp + ((size_t)p * S.h + y) * w;
  const float4* line4 = (const float4*)line;
  const int nq = (w + 3) >> 2;
  const int nblk = (taps + 3 + 3) >> 2;  // input steps jj = 0 .. taps + 2
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
    // k1..k3 = weights of taps jj-1, jj-2, jj-3 (zero before tap 0)
    float k1 = 0.0f, k2 = 0.0f, k3 = 0.0f;
    for (int b = 0; b < nblk; ++b) {
      const float4 v4 = line4[q + b];
      const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float k0 = kw[kHPad + 4 * b + u];  // tap jj = 4b + u
        const float v = vv[u];
        a0 = __fadd_rn(a0, __fmul_rn(k0, v));
        a1 = __fadd_rn(a1, __fmul_rn(k1, v));
        a2 = __fadd_rn(a2, __fmul_rn(k2, v));
        a3 = __fadd_rn(a3, __fmul_rn(k3, v));
        k3 = k2;
        k2 = k1;
        k1 = k0;
      }
    }
    const int x = 4 * q;
    out[x] = a0;
    if (x + 1 < w) out[x + 1] = a1;
    if (x + 2 < w) out[x + 2] = a2;
    if (x + 3 < w) out[x + 3] = a3;
  }
}

__global__ void k_syn_vblur(SynthDev S) {
  extern __shared__ float sm_v[];
  const int p = blockIdx.z;
  const int x = blockIdx.x * 32 + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int w = S.w, h = S.h, r = S.r, taps = 2 * r + 1;
  const int tid = threadIdx.y * 32 + threadIdx.x, nt = 32 * blockDim.y;
  for (int i = tid; i < taps; i += nt) sm_v[i] = S.weights[i];
  __syncthreads();
  unsigned mn_inv = 0u, mx = 0u;
  if (x < w && y < h) {
    const float* col = S.tmp + (size_t)p * h * w + x;
    float acc = 0.0f;
    for (int i = 0; i < taps; ++i) {
      int ys = y + i - r;
      ys = ys < 0 ? 0 : (ys >= h ? h - 1 : ys);
      acc = __fadd_rn(acc, __fmul_rn(sm_v[i], __ldg(col + (size_t)ys * w)));
    }
    S.fld[((size_t)p * h + y) * w + x] = acc;
    const unsigned b = __float_as_uint(acc);  // acc >= 0: bit order = value order
    mn_inv = ~b;
    mx = b;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn_inv = max(mn_inv, __shfl_xor_sync(0xffffffffu, mn_inv, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (threadIdx.x == 0) {
    atomicMax(S.minmax + 2 * p, mn_inv);
    atomicMax(S.minmax + 2 * p + 1, mx);
  }
}

// The same vertical pass with the column strip staged in shared memory and
// a sliding window: each thread produces kVR consecutive rows of one column,
// loading each input row once; output o takes its taps in ascending order as
// the input row advances, so every sum is the host's, rounding for rounding.
constexpr int kVR = 8;   // rows per thread
constexpr int kVW = 8;   // warps per CTA -> 64 rows per CTA

__global__ void __launch_bounds__(32 * kVW) k_syn_vblur_tile(SynthDev S) {
  extern __shared__ __align__(16) float sm_t[];
  const int p = blockIdx.z;
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int w = S.w, h = S.h, r = S.r, taps = 2 * r + 1;
  // weights with kVR-1 zeros before tap 0 and kVR+1 after: output o at input jj
  // reads kwp[jj - o + kVR - 1]; the extra terms are +0 * v on sums >= +0
  // (weights and field values are non-negative), i.e. bit-identities
  const int nkw = (taps + 2 * kVR + 3) & ~3;
  float* kwp = sm_t;
  float* tile = sm_t + nkw;  // [(kVR * kVW + 2r) rows][32]
  const int tid = warp * 32 + lane, nt = 32 * kVW;
  const int x0 = blockIdx.x * 32, y_cta = blockIdx.y * (kVR * kVW);
  const int rows = kVR * kVW + 2 * r;
  const float* src = S.tmp + (size_t)p * h * w;
  for (int i = tid; i < nkw; i += nt) {
    const int t = i - (kVR - 1);
    kwp[i] = (t >= 0 && t < taps) ? S.weights[t] : 0.0f;
  }
  for (int q = tid; q < rows * 32; q += nt) {
    const int rr = q >> 5, c = q & 31;
    int ys = y_cta - r + rr;
    ys = ys < 0 ? 0 : (ys >= h ? h - 1 : ys);
    const int xs = min(x0 + c, w - 1);
    tile[q] = src[(size_t)ys * w + xs];
  }
  __syncthreads();
  float acc[kVR], kr[kVR];
#pragma unroll
  for (int o = 0; o < kVR; ++o) {
    acc[o] = 0.0f;
    kr[o] = kwp[kVR - 1 - o];  // weights of input jj = 0
  }
  const float* col = tile + warp * kVR * 32 + lane;
  const int steps = kVR - 1 + taps;
#pragma unroll 8
  for (int jj = 0; jj < steps; ++jj) {
    const float v = col[jj * 32];
#pragma unroll
    for (int o = 0; o < kVR; ++o) acc[o] = __fadd_rn(acc[o], __fmul_rn(kr[o], v));
#pragma unroll
    for (int o = kVR - 1; o > 0; --o) kr[o] = kr[o - 1];
    kr[0] = kwp[jj + kVR];  // weight of tap jj + 1 for output 0
  }
  const int x = x0 + lane;
  unsigned mn_inv = 0u, mx = 0u;
#pragma unroll
  for (int o = 0; o < kVR; ++o) {
    const int y = y_cta + warp * kVR + o;
    if (x < w && y < h) {
      S.fld[((size_t)p * h + y) * w + x] = acc[o];
      const unsigned b = __float_as_uint(acc[o]);  // acc >= 0: bit order = value order
      mn_inv = max(mn_inv, ~b);
      mx = max(mx, b);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn_inv = max(mn_inv, __shfl_xor_sync(0xffffffffu, mn_inv, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    atomicMax(S.minmax + 2 * p, mn_inv);
    atomicMax(S.minmax + 2 * p + 1, mx);
  }
}

// pstereo_synth_discs (csrc/synth.c): discs are placed one after another
// until 30% of the pixels are covered; a disc's newly covered pixels are
// counted in parallel (each pixel belongs to one thread, so the count equals
// the sequential scan's).
__global__ void k_syn_discs(SynthDev S) {
  __shared__ unsigned long long covered;
  __shared__ unsigned added;
  const int p = blockIdx.x;
  const int w = S.w, h = S.h;
  const size_t n = (size_t)w * h;
  const size_t limit = (size_t)(0.30 * (double)n);
  const uint64_t key = syn_pair_key(S.seed0 + (uint64_t)p);
  uint8_t* cov = S.cov + (size_t)p * n;
  double* rec = S.discs + (size_t)p * SYN_MAX_DISCS * 4;
  if (threadIdx.x == 0) covered = 0;
  __syncthreads();
  int nd = 0;
  for (int k = 0; k < SYN_MAX_DISCS; ++k) {
    if (covered >= limit) break;
    double cx, cy, r, val;
    syn_disc(key, k, w, h, &cx, &cy, &r, &val);
    if (threadIdx.x == 0) {
      rec[4 * k + 0] = cx;
      rec[4 * k + 1] = cy;
      rec[4 * k + 2] = r;
      rec[4 * k + 3] = val;
      added = 0;
    }
    ++nd;
    const int x0 = (int)fmax(0.0, cx - r), x1 = (int)fmin(w - 1.0, cx + r);
    const int y0 = (int)fmax(0.0, cy - r), y1 = (int)fmin(h - 1.0, cy + r);
    const int bw = x1 - x0 + 1, bh = y1 - y0 + 1;
    unsigned mine = 0;
    __syncthreads();
    if (bw > 0 && bh > 0) {
      for (int q = threadIdx.x; q < bw * bh; q += blockDim.x) {
        const int x = x0 + q % bw, y = y0 + q / bw;
        const double dx = x - cx, dy = y - cy;
        if (dx * dx + dy * dy <= r * r && !cov[(size_t)y * w + x]) {
          cov[(size_t)y * w + x] = 1;
          ++mine;
        }
      }
    }
    if (mine) atomicAdd(&added, mine);
    __syncthreads();
    if (threadIdx.x == 0) covered += added;
    __syncthreads();
  }
  if (threadIdx.x == 0) S.n_discs[p] = nd;
}

// Value-noise lattice of one image row, octave by octave: the corner values
// syn_unit3(ok, ix, iy) and (ix, iy + 1) for every lattice column the row
// touches, so each pixel reads four cached doubles instead of hashing twelve
// splitmix rounds per octave. Same values, same arithmetic as syn_value_noise.
struct Lattice {
  int oct;                  // octaves
  int off[16];              // first entry of octave o (entries of 2 doubles)
  long long ixlo[16];       // lattice column of entry 0 of octave o
};

__host__ __device__ inline int lattice_entries(int w, int octaves, double base, Lattice* L) {
  int total = 0;
  double wl = base;
  for (int o = 0; o < octaves; ++o) {
    const long long lo = (long long)floor(0.5 / wl);
    const long long hi = (long long)floor(((double)(w - 1) + 0.5) / wl);
    if (L) {
      L->off[o] = total;
      L->ixlo[o] = lo;
    }
    total += (int)(hi - lo + 2);
    wl *= 0.5;
  }
  if (L) L->oct = octaves;
  return total;
}

__device__ __forceinline__ double value_noise_cached(double x, double y, const Lattice& L,
                                                     const double* lat, double wavelength) {
  double sum = 0.0, norm = 0.0, amp = 1.0;
  for (int o = 0; o < L.oct; ++o) {
    const double gx = x / wavelength, gy = y / wavelength;
    const double fx = floor(gx), fy = floor(gy);
    const double tx = syn_smooth(gx - fx), ty = syn_smooth(gy - fy);
    const double* e = lat + 2 * (L.off[o] + (int)((long long)fx - L.ixlo[o]));
    const double v00 = e[0], v01 = e[1], v10 = e[2], v11 = e[3];
    const double v = (1.0 - ty) * ((1.0 - tx) * v00 + tx * v10) +
                     ty * ((1.0 - tx) * v01 + tx * v11);
    sum += amp * v;
    norm += amp;
    amp *= 0.5;
    wavelength *= 0.5;
  }
  return sum / norm;
}

template <bool kCache>
__global__ void k_syn_views(SynthDev S) {
  extern __shared__ double sm_d[];
  const int y = blockIdx.x, p = blockIdx.y;
  const int w = S.w, h = S.h, C = S.C;
  const uint64_t key = syn_pair_key(S.seed0 + (uint64_t)p);
  const int nd = S.stress ? S.n_discs[p] : 0;
  double* tex = sm_d;                              // [w][C]
  double* dsc = tex + (size_t)w * C;               // [4][nd] (cx, cy, r, val planes)
  double* blob = dsc + 4 * SYN_MAX_DISCS;          // [2 views][3][SYN_BLOBS]
  double* lat = blob + 2 * 3 * SYN_BLOBS;          // [C][entries][2] (kCache)
  __shared__ double hp[3];
  Lattice L;
  int n_ent = 0;
  if (kCache) {
    n_ent = lattice_entries(w, S.octaves, S.wavelength, &L);
    const double yc = y + 0.5;
    for (int q = threadIdx.x; q < C * n_ent; q += blockDim.x) {
      const int c = q / n_ent, k = q - c * n_ent;
      int o = 0;
      while (o + 1 < L.oct && k >= L.off[o + 1]) ++o;
      double wl = S.wavelength;
      for (int t = 0; t < o; ++t) wl *= 0.5;
      const long long ix = L.ixlo[o] + (k - L.off[o]);
      const long long iy = (long long)floor(yc / wl);
      const uint64_t ok = syn_mix64(syn_channel_key(key, c) + (uint64_t)o * 0x1000193ull);
      double* e = lat + 2 * ((size_t)c * n_ent + k);
      e[0] = syn_unit3(ok, (uint64_t)ix, (uint64_t)iy);
      e[1] = syn_unit3(ok, (uint64_t)ix, (uint64_t)(iy + 1));
    }
  }
  if (S.stress) {
    const double* rec = S.discs + (size_t)p * SYN_MAX_DISCS * 4;
    for (int i = threadIdx.x; i < 4 * nd; i += blockDim.x)
      dsc[(i & 3) * SYN_MAX_DISCS + (i >> 2)] = rec[i];
    if (threadIdx.x < 2 * SYN_BLOBS) {
      const int v = threadIdx.x / SYN_BLOBS, b = threadIdx.x % SYN_BLOBS;
      double* bb = blob + v * 3 * SYN_BLOBS;
      syn_blob(key, v, b, w, h, &bb[b], &bb[SYN_BLOBS + b], &bb[2 * SYN_BLOBS + b]);
    }
    if (threadIdx.x == 2 * SYN_BLOBS) syn_half_plane(key, w, h, &hp[0], &hp[1], &hp[2]);
  }
  __syncthreads();
  const double* dcx = dsc;
  const double* dcy = dsc + SYN_MAX_DISCS;
  const double* drr = dsc + 2 * SYN_MAX_DISCS;
  const double* dvl = dsc + 3 * SYN_MAX_DISCS;
  // left view = the texture row
  const double gain0 = syn_gain(key, S.stress, 0), gain1 = syn_gain(key, S.stress, 1);
  const size_t row0 = ((size_t)p * h + y) * w;
  for (int x = threadIdx.x; x < w; x += blockDim.x) {
    double spec = 0.0, dark = 1.0;
    if (S.stress) {
      spec = syn_specular(blob, blob + SYN_BLOBS, blob + 2 * SYN_BLOBS, x, y);
      if (hp[0] * x + hp[1] * y > hp[2]) dark = 0.4;
    }
    for (int c = 0; c < C; ++c) {
      double v;
      if (kCache) {
        // syn_texture with the cached lattice
        v = 255.0 * value_noise_cached(x + 0.5, y + 0.5, L, lat + 2 * (size_t)c * n_ent,
                                       S.wavelength);
        for (int k = 0; k < nd; ++k) {
          const double dx = x - dcx[k], dy = y - dcy[k];
          if (dx * dx + dy * dy <= drr[k] * drr[k]) v = dvl[k];
        }
      } else {
        v = syn_texture(x, y, syn_channel_key(key, c), S.octaves, S.wavelength, nd, dcx, dcy,
                        drr, dvl);
      }
      tex[(size_t)x * C + c] = v;
      S.left[(row0 + x) * C + c] = syn_finish(v, gain0, dark, spec);
    }
  }
  __syncthreads();
  // right view: texture at x + d, plus sensor noise
  const float lo = __uint_as_float(~S.minmax[2 * p]);
  const float hi = __uint_as_float(S.minmax[2 * p + 1]);
  const float span = hi > lo ? __fsub_rn(hi, lo) : 1.0f;
  const double* b1 = blob + 3 * SYN_BLOBS;
  for (int x = threadIdx.x; x < w; x += blockDim.x) {
    const size_t i = (size_t)y * w + x;
    const float d = syn_normalise(S.fld[row0 + x], lo, span, S.d_min, S.d_range);
    if (S.disparity) S.disparity[row0 + x] = d;
    double spec = 0.0, dark = 1.0;
    if (S.stress) {
      spec = syn_specular(b1, b1 + SYN_BLOBS, b1 + 2 * SYN_BLOBS, x, y);
      if (hp[0] * x + hp[1] * y > hp[2]) dark = 0.4;
    }
    for (int c = 0; c < C; ++c) {
      double v = syn_right_tex(tex, w, C, c, x, d);
      v += S.noise_sigma * syn_gauss3(key ^ 0xA015Eull, (uint64_t)c, i);
      S.right[(row0 + x) * C + c] = syn_finish(v, gain1, dark, spec);
    }
  }
}

int fail(int code, const std::string& msg) {
  g_synth_error = msg;
  return code;
}

// Stream-ordered scratch from a per-device pool that keeps its memory between
// calls (release threshold: never), so repeated calls do not remap hundreds of
// megabytes of scratch each time.
cudaError_t scratch_alloc(int device, void** p, size_t bytes, cudaStream_t st) {
  static std::mutex mu;
  static std::vector<cudaMemPool_t> pools;
  cudaMemPool_t pool = nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    if ((int)pools.size() <= device) pools.resize(device + 1, nullptr);
    if (!pools[device]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      cudaError_t e = cudaMemPoolCreate(&pools[device], &props);
      if (e != cudaSuccess) return e;
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool = pools[device];
  }
  return cudaMallocFromPoolAsync(p, bytes, pool, st);
}

}  // namespace

extern "C" int pstereo_synth_check(const pstereo_synth_spec* s);

extern "C" const char* pstereo_synth_last_error(void) { return g_synth_error.c_str(); }

extern "C" int pstereo_gpu_synth(int device, const pstereo_synth_spec* s, int n_pairs,
                                 uint64_t seed0, uint8_t* left, uint8_t* right,
                                 float* disparity, void* stream) {
  if (pstereo_synth_check(s)) return fail(PSTEREO_ECONFIG, "pstereo_gpu_synth: bad spec");
  if (n_pairs < 0 || (n_pairs > 0 && (!left || !right)))
    return fail(PSTEREO_EINTERNAL, "pstereo_gpu_synth: bad arguments");
  if (n_pairs == 0) return PSTEREO_OK;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(PSTEREO_EINTERNAL, cudaGetErrorString(e));
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (major != 10) return fail(PSTEREO_EINTERNAL, "pstereo_gpu_synth: needs an sm_100 device");
  cudaStream_t st = (cudaStream_t)stream;
  const int w = s->width, h = s->height, C = s->channels;
  const size_t px = (size_t)w * h;
  const int r = pstereo_synth_blur_weights(s->blur_sigma, nullptr, 0);
  std::vector<float> kw((size_t)(2 * r + 1));
  pstereo_synth_blur_weights(s->blur_sigma, kw.data(), 2 * r + 1);
  const size_t smem_h =
      sizeof(float) * ((size_t)(((w + 2 * r + 3) & ~3) + 8) + (size_t)(2 * r + 1 + kHPad + kHTail));
  const size_t smem_v = sizeof(float) * (size_t)(2 * r + 1);
  const size_t smem_vt =
      sizeof(float) * ((size_t)((2 * r + 1 + 2 * kVR + 3) & ~3) + (size_t)(kVR * kVW + 2 * r) * 32);
  const size_t smem_views =
      sizeof(double) * ((size_t)w * C + 4 * SYN_MAX_DISCS + 2 * 3 * SYN_BLOBS);
  const size_t smem_views_c =
      smem_views + sizeof(double) * 2 * (size_t)C *
                       (size_t)lattice_entries(w, s->octaves, s->base_wavelength, nullptr);
  const bool vcache = s->octaves <= 16 && smem_views_c <= 200 * 1024;
  const size_t smem_cap = 227 * 1024;
  if (smem_h > smem_cap || smem_views > smem_cap)
    return fail(PSTEREO_ECONFIG, "pstereo_gpu_synth: width or blur radius too large");
  bdis::ensure_smem_cap((const void*)k_syn_hblur, smem_h);
  bdis::ensure_smem_cap((const void*)k_syn_vblur, smem_v);
  const bool vtile = smem_vt <= smem_cap;
  if (vtile)
    bdis::ensure_smem_cap((const void*)k_syn_vblur_tile, smem_vt);
  bdis::ensure_smem_cap((const void*)k_syn_views<false>, smem_views);
  if (vcache)
    bdis::ensure_smem_cap((const void*)k_syn_views<true>, smem_views_c);

  // chunked so the scratch stays bounded (~8.1 B per pixel per pair in flight)
  const int chunk = n_pairs < 64 ? n_pairs : 64;
  SynthDev S;
  std::memset(&S, 0, sizeof S);
  S.w = w;
  S.h = h;
  S.C = C;
  S.octaves = s->octaves;
  S.wavelength = s->base_wavelength;
  S.d_min = s->d_min;
  S.d_range = s->d_range;
  S.noise_sigma = s->noise_sigma;
  S.stress = s->stress;
  S.r = r;
  void* base = nullptr;
  const size_t b_w = sizeof(float) * kw.size();
  const size_t b_field = sizeof(float) * px * chunk;
  const size_t b_mm = sizeof(unsigned) * 2 * chunk;
  const size_t b_cov = s->stress ? px * chunk : 0;
  const size_t b_disc = s->stress ? sizeof(double) * SYN_MAX_DISCS * 4 * chunk : 0;
  const size_t b_nd = sizeof(int) * chunk;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t total = al(b_w) + 2 * al(b_field) + al(b_mm) + al(b_cov) + al(b_disc) + al(b_nd);
  e = scratch_alloc(device, &base, total, st);
  if (e != cudaSuccess) return fail(PSTEREO_EINTERNAL, cudaGetErrorString(e));
  char* q = (char*)base;
  S.weights = (const float*)q;
  float* dw = (float*)q;
  q += al(b_w);
  S.tmp = (float*)q;
  q += al(b_field);
  S.fld = (float*)q;
  q += al(b_field);
  S.minmax = (unsigned*)q;
  q += al(b_mm);
  S.cov = (uint8_t*)q;
  q += al(b_cov);
  S.discs = (double*)q;
  q += al(b_disc);
  S.n_discs = (int*)q;
  e = cudaMemcpyAsync(dw, kw.data(), b_w, cudaMemcpyHostToDevice, st);
  // the blur taps live in pageable host memory: wait before `kw` goes away
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  for (int p0 = 0; p0 < n_pairs && e == cudaSuccess; p0 += chunk) {
    const int m = n_pairs - p0 < chunk ? n_pairs - p0 : chunk;
    S.seed0 = seed0 + (uint64_t)p0;
    S.left = left + (size_t)p0 * px * C;
    S.right = right + (size_t)p0 * px * C;
    S.disparity = disparity ? disparity + (size_t)p0 * px : nullptr;
    e = cudaMemsetAsync(S.minmax, 0, sizeof(unsigned) * 2 * m, st);
    if (e == cudaSuccess && s->stress) e = cudaMemsetAsync(S.cov, 0, px * m, st);
    if (e != cudaSuccess) break;
    k_syn_hblur<<<dim3(h, m), 256, smem_h, st>>>(S);
    if (vtile)
      k_syn_vblur_tile<<<dim3((w + 31) / 32, (h + kVR * kVW - 1) / (kVR * kVW), m),
                         dim3(32, kVW), smem_vt, st>>>(S);
    else
      k_syn_vblur<<<dim3((w + 31) / 32, (h + 7) / 8, m), dim3(32, 8), smem_v, st>>>(S);
    if (s->stress) k_syn_discs<<<m, 512, 0, st>>>(S);
    if (vcache) k_syn_views<true><<<dim3(h, m), 128, smem_views_c, st>>>(S);
    else k_syn_views<false><<<dim3(h, m), 128, smem_views, st>>>(S);
    e = cudaGetLastError();
  }
  cudaError_t e2 = cudaFreeAsync(base, st);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return fail(PSTEREO_EINTERNAL, cudaGetErrorString(e));
  return PSTEREO_OK;
}
