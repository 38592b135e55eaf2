// Dependent-chain latency of FP64 / FP32 / conversion instructions on one
// warp (clock64 per operation): the sequential sums that bit-exactness
// imposes on k_patches and compute_metrics run at this latency.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_bench lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define N 4096

__global__ void k_dadd(double* out, long long* cyc, double a) {
  double x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __dadd_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_dmul(double* out, long long* cyc, double a) {
  double x = threadIdx.x + 1.0;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __dmul_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_fadd(double* out, long long* cyc, double a) {
  float x = threadIdx.x, af = (float)a;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __fadd_rn(x, af);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_f2f(double* out, long long* cyc, double a) {
  float f = threadIdx.x;
  double x = 0;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    x = (double)f;            // F2F.F64.F32
    f = __double2float_rn(x + a);  // keeps the chain dependent
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1024 * sizeof(double));
  cudaMalloc(&c, sizeof(long long));
  long long h;
  const char* names[] = {"DADD", "DMUL", "FADD", "F2F.F64.F32+DADD+F2F.F32.F64"};
  void (*ks[])(double*, long long*, double) = {k_dadd, k_dmul, k_fadd, k_f2f};
  for (int k = 0; k < 4; ++k) {
    for (int rep = 0; rep < 2; ++rep) ks[k]<<<1, 32>>>(d, c, 1.0000001);
    cudaMemcpy(&h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("%-30s %.1f cycles per dependent step\n", names[k], (double)h / N);
  }
  return 0;
}
