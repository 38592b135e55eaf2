// host_expand_bench.c -- how fast can the host replicate a quarter-resolution
// fp32 plane 2x2 into a full-resolution buffer (the upsample_to_full
// replication, src/coarse_to_fine.cpp:166-180, done on the host side of the
// D2H copy)?  gcc -O2 -pthread host_expand_bench.c -o host_expand_bench
// usage: host_expand_bench [threads] [pairs] [reps]
#define _GNU_SOURCE
#include <immintrin.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static int W = 320, H = 240, NP = 256, NT = 16, MODE = 0;
static float *src, *dst;
static pthread_barrier_t bar;

__attribute__((target("avx2"))) static void expand_rows_avx2(const float* in, float* out, int w, int rows) {
  const __m256i lo = _mm256_setr_epi32(0, 0, 1, 1, 2, 2, 3, 3);
  const __m256i hi = _mm256_setr_epi32(4, 4, 5, 5, 6, 6, 7, 7);
  for (int y = 0; y < rows; ++y) {
    const float* s = in + (size_t)y * w;
    float* o0 = out + (size_t)(2 * y) * (2 * w);
    float* o1 = o0 + 2 * w;
    for (int x = 0; x < w; x += 8) {
      const __m256 v = _mm256_loadu_ps(s + x);
      const __m256 a = _mm256_permutevar8x32_ps(v, lo);
      const __m256 b = _mm256_permutevar8x32_ps(v, hi);
      _mm256_stream_ps(o0 + 2 * x, a);
      _mm256_stream_ps(o0 + 2 * x + 8, b);
      _mm256_stream_ps(o1 + 2 * x, a);
      _mm256_stream_ps(o1 + 2 * x + 8, b);
    }
  }
  _mm_sfence();
}
static void expand_rows_scalar(const float* in, float* out, int w, int rows) {
  for (int y = 0; y < rows; ++y) {
    const float* s = in + (size_t)y * w;
    float* o0 = out + (size_t)(2 * y) * (2 * w);
    float* o1 = o0 + 2 * w;
    for (int x = 0; x < w; ++x) {
      const float v = s[x];
      o0[2 * x] = v; o0[2 * x + 1] = v; o1[2 * x] = v; o1[2 * x + 1] = v;
    }
  }
}
static int reps = 10;
static void* worker(void* arg) {
  const int t = (int)(intptr_t)arg;
  const size_t rows = (size_t)NP * H;
  const size_t r0 = rows * t / NT, r1 = rows * (t + 1) / NT;
  for (int r = 0; r < reps + 1; ++r) {
    pthread_barrier_wait(&bar);
    if (MODE == 0) expand_rows_avx2(src + r0 * W, dst + r0 * 2 * (size_t)(2 * W), W, (int)(r1 - r0));
    else if (MODE == 1) expand_rows_scalar(src + r0 * W, dst + r0 * 2 * (size_t)(2 * W), W, (int)(r1 - r0));
    else memcpy(dst + r0 * 4 * W, src + (r0 % (rows / 4)) * W, (r1 - r0) * 4 * W * sizeof(float));
    pthread_barrier_wait(&bar);
  }
  return NULL;
}
static double now() { struct timespec ts; clock_gettime(CLOCK_MONOTONIC, &ts); return ts.tv_sec + 1e-9 * ts.tv_nsec; }
int main(int argc, char** argv) {
  if (argc > 1) NT = atoi(argv[1]);
  if (argc > 2) NP = atoi(argv[2]);
  if (argc > 3) reps = atoi(argv[3]);
  const size_t n = (size_t)NP * W * H;
  src = aligned_alloc(64, n * 4);
  dst = aligned_alloc(64, n * 16);
  for (size_t i = 0; i < n; ++i) src[i] = (float)i;
  memset(dst, 0, n * 16);
  for (MODE = 0; MODE < 3; ++MODE) {
    pthread_barrier_init(&bar, NULL, NT + 1);
    pthread_t th[256];
    for (int t = 0; t < NT; ++t) pthread_create(&th[t], NULL, worker, (void*)(intptr_t)t);
    double best = 1e9, tot = 0;
    for (int r = 0; r < reps + 1; ++r) {
      pthread_barrier_wait(&bar);
      const double t0 = now();
      pthread_barrier_wait(&bar);
      const double dt = now() - t0;
      if (r) { tot += dt; if (dt < best) best = dt; }
    }
    for (int t = 0; t < NT; ++t) pthread_join(th[t], NULL);
    pthread_barrier_destroy(&bar);
    printf("{\"mode\": \"%s\", \"threads\": %d, \"pairs\": %d, \"ms_mean\": %.3f, \"ms_best\": %.3f, \"write_GBps_mean\": %.1f}\n",
           MODE == 0 ? "avx2_stream" : MODE == 1 ? "scalar" : "memcpy_same_bytes", NT, NP, 1e3 * tot / reps,
           1e3 * best, n * 16 / (tot / reps) * 1e-9);
  }
  // check
  MODE = 0;
  return 0;
}
