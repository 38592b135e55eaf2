// bdis_metrics.cu -- compute_metrics (src/metrics.cpp:10-52) for a batch of
// frames: |estimate - reference| over pixels valid on both sides, mean error,
// median error, 1.96-sigma coverage.
//
// Bit-exact with the reference:
//   * the mean is the reference's sequential sum in pixel-index order
//     (:36-37): producer warps stream 1792-pixel chunks of errors into shared
//     memory (double-buffered) while one consumer thread adds them in order --
//     the DADD chain is the critical path, so frames run as independent CTAs;
//   * the median is an order statistic (nth_element, :40-48), which does not
//     depend on the selection algorithm: radix select over the IEEE bit
//     patterns of the compacted errors (non-negative doubles order like their
//     uint64 bits), 11-bit digits, warp-aggregated shared histograms; for an
//     even count the lower middle value comes from the same select (ties) or
//     one max pass below it;
//   * counts and the coverage ratio are integer / one division (:33, :50).
#include <cuda_runtime.h>
#include <math.h>
#include <math_constants.h>
#include <stdint.h>

#include "bdis_kernels.h"

namespace bdis {

namespace {

constexpr int kMetThreads = 256;
constexpr int kProducers = kMetThreads - 32;  // warps 1..7
constexpr int kPerProducer = 8;
constexpr int kChunk = kProducers * kPerProducer;  // 1792 pixels
constexpr int kDigitBits = 11, kBins = 1 << kDigitBits;

__device__ __forceinline__ unsigned long long dbits(double v) {
  return (unsigned long long)__double_as_longlong(v);
}

__global__ void __launch_bounds__(kMetThreads) k_metrics(MetricsArgs a) {
  __shared__ double s_err[2][kChunk];
  __shared__ unsigned s_hist[kBins];
  __shared__ unsigned long long s_red[kMetThreads / 32][3];
  __shared__ unsigned s_m;
  __shared__ double s_sum;
  const int f = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long n = (long long)a.w * a.h;
  const long long base = (long long)f * n;
  const double* est = a.est + base;
  const double* ref = a.ref + base;
  const uint8_t* ev = a.est_valid + base;
  const uint8_t* rv = a.ref_valid + base;
  const double* sg = a.sigma ? a.sigma + base : nullptr;
  const uint8_t* sv = a.sigma ? a.sigma_valid + base : nullptr;
  unsigned long long* keys = a.scratch + base;
  if (tid == 0) s_m = 0;
  __syncthreads();

  // ---- pass 1: errors in index order (sum), counts, compaction of the keys
  unsigned long long valid_px = 0, compared = 0, covered = 0;
  double sum = 0.0;
  const long long n_chunks = (n + kChunk - 1) / kChunk;
  for (long long c = 0; c <= n_chunks; ++c) {
    if (warp > 0 && c < n_chunks) {
      const int b = int(c & 1);
#pragma unroll
      for (int k = 0; k < kPerProducer; ++k) {
        const int q = (tid - 32) + k * kProducers;  // coalesced per k
        const long long i = c * kChunk + q;
        bool ok = false;
        double e = 0.0;
        if (i < n) {
          const bool evi = ev[i] != 0;
          valid_px += evi;
          ok = evi && rv[i] != 0;
          if (ok) {
            e = fabs(est[i] - ref[i]);
            ++compared;
            if (sg && sv[i] && e <= 1.96 * sg[i]) ++covered;
          }
        }
        s_err[b][q] = e;
        // append the key (order irrelevant for an order statistic)
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        unsigned slot = 0;
        if (lane == 0 && bal) slot = atomicAdd(&s_m, (unsigned)__popc(bal));
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (ok) keys[slot + __popc(bal & ((1u << lane) - 1u))] = dbits(e);
      }
    }
    if (tid == 0 && c > 0) {
      // the reference's sequential sum (:36-37), pixel-index order
      const int b = int((c - 1) & 1);
      const long long rem = n - (c - 1) * kChunk;
      const int len = rem < kChunk ? int(rem) : kChunk;
      // pixels not compared hold +0.0: the sum is never -0.0 (it starts at
      // +0.0, errors are fabs), so adding +0.0 is the identity -- a pure DADD
      // chain with the loads hoisted ahead of it
#pragma unroll 16
      for (int q = 0; q < len; ++q) sum = __dadd_rn(sum, s_err[b][q]);
    }
    __syncthreads();
  }
  // block totals of the counts
  for (int o = 16; o > 0; o >>= 1) {
    valid_px += __shfl_xor_sync(0xffffffffu, valid_px, o);
    compared += __shfl_xor_sync(0xffffffffu, compared, o);
    covered += __shfl_xor_sync(0xffffffffu, covered, o);
  }
  if (lane == 0) {
    s_red[warp][0] = valid_px;
    s_red[warp][1] = compared;
    s_red[warp][2] = covered;
  }
  if (tid == 0) s_sum = sum;
  __syncthreads();
  unsigned long long tv = 0, tc = 0, tcov = 0;
  for (int q = 0; q < kMetThreads / 32; ++q) {
    tv += s_red[q][0];
    tc += s_red[q][1];
    tcov += s_red[q][2];
  }
  const long long m = (long long)s_m;  // == tc

  // ---- median: radix select of rank mid over the compacted keys
  double median = CUDART_NAN;
  if (m > 0) {
    const long long mid = m / 2;
    long long k = mid, less = 0;
    unsigned long long prefix = 0, pmask = 0;
    for (int shift = 64 - kDigitBits; shift > -kDigitBits; shift -= kDigitBits) {
      const int sh = shift < 0 ? 0 : shift;
      const int bits = shift < 0 ? kDigitBits + shift : kDigitBits;
      const unsigned dmask = (1u << bits) - 1u;
      for (int q = tid; q < kBins; q += kMetThreads) s_hist[q] = 0;
      __syncthreads();
      // kKeyIlp keys per thread in flight: the pass is bound by the global
      // load latency, not by the histogram updates
      constexpr int kKeyIlp = 8;
      for (long long i0 = 0; i0 < m; i0 += (long long)kMetThreads * kKeyIlp) {
        unsigned long long kv[kKeyIlp];
#pragma unroll
        for (int u = 0; u < kKeyIlp; ++u) {
          const long long i = i0 + (long long)u * kMetThreads + tid;
          kv[u] = i < m ? __ldcg(keys + i) : ~0ull;
        }
#pragma unroll
        for (int u = 0; u < kKeyIlp; ++u) {
          const long long i = i0 + (long long)u * kMetThreads + tid;
          unsigned d = kBins;  // no bin
          if (i < m && (kv[u] & pmask) == prefix) d = (unsigned)(kv[u] >> sh) & dmask;
          // one atomic per distinct digit in the warp (hot bins are common)
          const unsigned peers = __match_any_sync(0xffffffffu, d);
          if (d != kBins && lane == __ffs(peers) - 1)
            atomicAdd(&s_hist[d], (unsigned)__popc(peers));
        }
      }
      __syncthreads();
      if (tid == 0) {
        long long acc = 0;
        unsigned bsel = 0;
        for (unsigned bq = 0; bq <= dmask; ++bq) {
          const long long c = s_hist[bq];
          if (acc + c > k) {
            bsel = bq;
            break;
          }
          acc += c;
        }
        s_red[0][0] = (unsigned long long)acc;
        s_red[0][1] = bsel;
      }
      __syncthreads();
      const long long acc = (long long)s_red[0][0];
      const unsigned bsel = (unsigned)s_red[0][1];
      k -= acc;
      less += acc;
      prefix |= (unsigned long long)bsel << sh;
      pmask |= (unsigned long long)dmask << sh;
      __syncthreads();
    }
    const double hi = __longlong_as_double((long long)prefix);
    if (m % 2 == 1) {
      median = hi;
    } else {
      double lo = hi;
      if (less > mid - 1) {
        // rank mid-1 is below the value at rank mid: the largest smaller key
        unsigned long long best = 0;
        for (long long i = tid; i < m; i += kMetThreads) {
          const unsigned long long key = __ldcg(keys + i);
          if (key < prefix && key > best) best = key;
        }
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
          best = other > best ? other : best;
        }
        if (lane == 0) s_red[warp][2] = best;
        __syncthreads();
        unsigned long long b2 = 0;
        for (int q = 0; q < kMetThreads / 32; ++q) b2 = s_red[q][2] > b2 ? s_red[q][2] : b2;
        lo = __longlong_as_double((long long)b2);
      }
      median = __dmul_rn(0.5, __dadd_rn(lo, hi));  // 0.5 * (errs[mid-1] + hi), :46
    }
  }
  if (tid == 0) {
    pstereo_frame_metrics_dev& o = a.out[f];
    o.valid_px = (long long)tv;
    o.compared = (long long)tc;
    o.has_errors = tc > 0;
    o.mean_err = tc > 0 ? __ddiv_rn(s_sum, (double)tc) : CUDART_NAN;
    o.median_err = median;
    o.coverage_rate = (a.sigma && tc > 0) ? __ddiv_rn((double)tcov, (double)tc) : CUDART_NAN;
  }
}

}  // namespace

cudaError_t launch_metrics(const MetricsArgs& a, int n_frames, cudaStream_t s) {
  if (n_frames <= 0) return cudaSuccess;
  k_metrics<<<n_frames, kMetThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace bdis
