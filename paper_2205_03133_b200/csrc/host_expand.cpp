// host_expand.cpp -- see host_expand.h. Host side of the drop-in's D2H path:
// upsample_to_full's block replication (src/coarse_to_fine.cpp:166-180)
// applied while the planes land in the caller's buffers.
#include "host_expand.h"

#include <immintrin.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <thread>
#include <vector>

namespace bdis {

void ExpandCounter::add(long n) {
  std::lock_guard<std::mutex> g(m);
  pending += n;
}
void ExpandCounter::done(long n) {
  std::lock_guard<std::mutex> g(m);
  pending -= n;
  if (pending <= 0) cv.notify_all();
}
void ExpandCounter::wait() {
  std::unique_lock<std::mutex> g(m);
  cv.wait(g, [&] { return pending <= 0; });
}

namespace {

template <typename T>
void expand_generic(const ExpandJob& j, const T* src, T* dst) {
  for (int y = 0; y < j.H; ++y) {
    const T* s = src + size_t(std::min(y >> j.e, j.fh - 1)) * j.fw;
    T* o = dst + size_t(j.flip ? j.H - 1 - y : y) * j.W;
    for (int x = 0; x < j.W; ++x) o[x] = s[std::min(x >> j.e, j.fw - 1)];
  }
}

// 2x2 blocks on W = 2 fw: each source row goes to output rows 2y and 2y + 1
// (the second only when it exists: H may be odd). Streaming stores when the
// rows are aligned: the planes are written once and not read back here.
__attribute__((target("avx2"))) void rows2_f32(const float* s, float* o0, float* o1, int fw) {
  const __m256i lo = _mm256_setr_epi32(0, 0, 1, 1, 2, 2, 3, 3);
  const __m256i hi = _mm256_setr_epi32(4, 4, 5, 5, 6, 6, 7, 7);
  int x = 0;
  const bool nt = (((uintptr_t)o0 | (uintptr_t)(o1 ? o1 : o0)) & 31) == 0;
  for (; x + 8 <= fw; x += 8) {
    const __m256 v = _mm256_loadu_ps(s + x);
    const __m256 a = _mm256_permutevar8x32_ps(v, lo), b = _mm256_permutevar8x32_ps(v, hi);
    if (nt) {
      _mm256_stream_ps(o0 + 2 * x, a);
      _mm256_stream_ps(o0 + 2 * x + 8, b);
      if (o1) {
        _mm256_stream_ps(o1 + 2 * x, a);
        _mm256_stream_ps(o1 + 2 * x + 8, b);
      }
    } else {
      _mm256_storeu_ps(o0 + 2 * x, a);
      _mm256_storeu_ps(o0 + 2 * x + 8, b);
      if (o1) {
        _mm256_storeu_ps(o1 + 2 * x, a);
        _mm256_storeu_ps(o1 + 2 * x + 8, b);
      }
    }
  }
  for (; x < fw; ++x) {
    o0[2 * x] = o0[2 * x + 1] = s[x];
    if (o1) o1[2 * x] = o1[2 * x + 1] = s[x];
  }
}

__attribute__((target("avx2"))) void rows2_f64(const double* s, double* o0, double* o1, int fw) {
  int x = 0;
  const bool nt = (((uintptr_t)o0 | (uintptr_t)(o1 ? o1 : o0)) & 31) == 0;
  for (; x + 4 <= fw; x += 4) {
    const __m256d v = _mm256_loadu_pd(s + x);
    const __m256d a = _mm256_permute4x64_pd(v, 0x50), b = _mm256_permute4x64_pd(v, 0xfa);
    if (nt) {
      _mm256_stream_pd(o0 + 2 * x, a);
      _mm256_stream_pd(o0 + 2 * x + 4, b);
      if (o1) {
        _mm256_stream_pd(o1 + 2 * x, a);
        _mm256_stream_pd(o1 + 2 * x + 4, b);
      }
    } else {
      _mm256_storeu_pd(o0 + 2 * x, a);
      _mm256_storeu_pd(o0 + 2 * x + 4, b);
      if (o1) {
        _mm256_storeu_pd(o1 + 2 * x, a);
        _mm256_storeu_pd(o1 + 2 * x + 4, b);
      }
    }
  }
  for (; x < fw; ++x) {
    o0[2 * x] = o0[2 * x + 1] = s[x];
    if (o1) o1[2 * x] = o1[2 * x + 1] = s[x];
  }
}

void rows2_u8(const uint8_t* s, uint8_t* o0, uint8_t* o1, int fw) {  // SSE2: baseline x86-64
  int x = 0;
  const bool nt = (((uintptr_t)o0 | (uintptr_t)(o1 ? o1 : o0)) & 15) == 0;
  for (; x + 16 <= fw; x += 16) {
    const __m128i v = _mm_loadu_si128((const __m128i*)(s + x));
    const __m128i a = _mm_unpacklo_epi8(v, v), b = _mm_unpackhi_epi8(v, v);
    if (nt) {
      _mm_stream_si128((__m128i*)(o0 + 2 * x), a);
      _mm_stream_si128((__m128i*)(o0 + 2 * x + 16), b);
      if (o1) {
        _mm_stream_si128((__m128i*)(o1 + 2 * x), a);
        _mm_stream_si128((__m128i*)(o1 + 2 * x + 16), b);
      }
    } else {
      _mm_storeu_si128((__m128i*)(o0 + 2 * x), a);
      _mm_storeu_si128((__m128i*)(o0 + 2 * x + 16), b);
      if (o1) {
        _mm_storeu_si128((__m128i*)(o1 + 2 * x), a);
        _mm_storeu_si128((__m128i*)(o1 + 2 * x + 16), b);
      }
    }
  }
  for (; x < fw; ++x) {
    o0[2 * x] = o0[2 * x + 1] = s[x];
    if (o1) o1[2 * x] = o1[2 * x + 1] = s[x];
  }
}

template <typename T>
void rows2_plain(const T* s, T* o0, T* o1, int fw) {
  for (int x = 0; x < fw; ++x) {
    o0[2 * x] = o0[2 * x + 1] = s[x];
    if (o1) o1[2 * x] = o1[2 * x + 1] = s[x];
  }
}

const bool g_avx2 = __builtin_cpu_supports("avx2");

template <typename T>
void expand_x2(const ExpandJob& j, const T* src, T* dst) {
  for (int fy = 0; fy < j.fh; ++fy) {
    const int y0 = 2 * fy, y1 = 2 * fy + 1;
    if (y0 >= j.H) break;
    T* o0 = dst + size_t(j.flip ? j.H - 1 - y0 : y0) * j.W;
    T* o1 = y1 < j.H ? dst + size_t(j.flip ? j.H - 1 - y1 : y1) * j.W : nullptr;
    const T* s = src + size_t(fy) * j.fw;
    if constexpr (sizeof(T) == 1) rows2_u8((const uint8_t*)s, (uint8_t*)o0, (uint8_t*)o1, j.fw);
    else if constexpr (sizeof(T) == 4) {
      if (g_avx2) rows2_f32((const float*)s, (float*)o0, (float*)o1, j.fw);
      else rows2_plain(s, o0, o1, j.fw);
    } else {
      if (g_avx2) rows2_f64((const double*)s, (double*)o0, (double*)o1, j.fw);
      else rows2_plain(s, o0, o1, j.fw);
    }
  }
  _mm_sfence();
}

template <typename T>
void expand_typed(const ExpandJob& j, int pair) {
  const T* src = (const T*)j.src + size_t(pair) * j.fw * j.fh;
  T* dst = (T*)j.dst + size_t(pair) * j.W * j.H;
  if (j.e == 1 && j.W == 2 * j.fw) expand_x2<T>(j, src, dst);
  else expand_generic<T>(j, src, dst);
}

struct Unit {
  ExpandJob job;
  int pair;
  ExpandCounter* c;
};

class Pool {
 public:
  static Pool& get() {
    static Pool* p = new Pool;  // never destroyed: workers may outlive static teardown
    return *p;
  }
  int size() const { return int(threads_.size()); }
  void push(const ExpandJob* jobs, int n, ExpandCounter* c) {
    {
      std::lock_guard<std::mutex> g(m_);
      for (int k = 0; k < n; ++k)
        for (int p = 0; p < jobs[k].n_pairs; ++p) q_.push_back(Unit{jobs[k], p, c});
    }
    cv_.notify_all();
  }

 private:
  Pool() {
    // measured on the 16-core bench host: 5-6 workers are the best (4 cannot
    // keep up, 7 and more add memory-controller contention against the H2D
    // DMA reads)
    int n = int(std::thread::hardware_concurrency()) * 3 / 8;
    n = std::max(1, std::min(n, 6));
    if (const char* v = std::getenv("PSTEREO_HOST_THREADS")) n = std::max(1, std::atoi(v));
    for (int t = 0; t < n; ++t) threads_.emplace_back([this] { run(); });
    for (auto& t : threads_) t.detach();
  }
  void run() {
    for (;;) {
      Unit u;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return !q_.empty(); });
        u = q_.front();
        q_.pop_front();
      }
      const auto t0 = std::chrono::steady_clock::now();
      if (!noop_) expand_frame(u.job, u.pair);
      busy_ns_ += std::chrono::duration_cast<std::chrono::nanoseconds>(
                      std::chrono::steady_clock::now() - t0).count();
      ++units_;
      u.c->done(1);
    }
  }
  const bool noop_ = std::getenv("PSTEREO_DEBUG_EXPAND_NOOP") != nullptr;  // timing aid

 public:
  std::atomic<long long> busy_ns_{0}, units_{0};

 private:
  std::mutex m_;
  std::condition_variable cv_;
  std::deque<Unit> q_;
  std::vector<std::thread> threads_;
};

}  // namespace

void expand_frame(const ExpandJob& j, int pair) {
  if (j.esz == 1) expand_typed<uint8_t>(j, pair);
  else if (j.esz == 4) expand_typed<uint32_t>(j, pair);
  else expand_typed<uint64_t>(j, pair);
}

void expand_submit(const ExpandJob* jobs, int n, ExpandCounter* c) { Pool::get().push(jobs, n, c); }

int expand_threads() { return Pool::get().size(); }

void expand_stats(double* busy_ms, long long* frames) {
  *busy_ms = 1e-6 * double(Pool::get().busy_ns_.load());
  *frames = Pool::get().units_.load();
}

}  // namespace bdis
