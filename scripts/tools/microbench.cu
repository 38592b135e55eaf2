// microbench.cu -- B200 pipe throughputs that decide the k_patches design
// (FP64 add/mul, f32->f64 conversion, double->int truncation, shared-memory
// 8/16-byte loads with the stride-4 patch access pattern).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_dadd(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, b); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, b);
    x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, b); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_dmul(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = __dmul_rn(x0, a); x1 = __dmul_rn(x1, b); x2 = __dmul_rn(x2, a); x3 = __dmul_rn(x3, b);
    x4 = __dmul_rn(x4, a); x5 = __dmul_rn(x5, b); x6 = __dmul_rn(x6, a); x7 = __dmul_rn(x7, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_cvt_f2d(double* out, float a) {
  float f0 = threadIdx.x * a, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3;
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int i = 0; i < ITERS; ++i) {
    // 4 conversions + 4 dadds per iteration
    acc0 = __dadd_rn(acc0, (double)f0); acc1 = __dadd_rn(acc1, (double)f1);
    acc2 = __dadd_rn(acc2, (double)f2); acc3 = __dadd_rn(acc3, (double)f3);
    f0 += 1.0f; f1 += 1.0f; f2 += 1.0f; f3 += 1.0f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

__global__ void k_d2i(int* out, double a) {
  double x0 = threadIdx.x * a, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  int s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < ITERS; ++i) {
    s0 += __double2int_rz(x0); s1 += __double2int_rz(x1);
    s2 += __double2int_rz(x2); s3 += __double2int_rz(x3);
    x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}

__global__ void k_i2d(double* out, int a) {
  int x0 = threadIdx.x * a, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < ITERS; ++i) {
    s0 = __dadd_rn(s0, (double)x0); s1 = __dadd_rn(s1, (double)x1);
    s2 = __dadd_rn(s2, (double)x2); s3 = __dadd_rn(s3, (double)x3);
    x0 += 3; x1 += 3; x2 += 3; x3 += 3;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}

template <typename T>
__global__ void k_lds(double* out, int stride, int pad) {
  extern __shared__ unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const int n = 2048;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    T v;
    memset(&v, 0, sizeof v);
    *reinterpret_cast<float*>(&v) = (float)i;
    sm[i] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int x = lane * stride + (threadIdx.x >> 5);
  double acc = 0;
  for (int i = 0; i < ITERS; ++i) {
    const int slot = x + (pad ? (x >> 4) : 0);
    T v = sm[slot & (n - 1)];
    acc += *reinterpret_cast<float*>(&v);
    x = (x + 1) & 1023;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <typename F>
float time_kernel(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int sms = p.multiProcessorCount;
  const int blocks = sms * 8, threads = 256;
  const double n_thr = double(blocks) * threads;
  double* d;
  int* di;
  cudaMalloc(&d, sizeof(double) * blocks * threads);
  cudaMalloc(&di, sizeof(int) * blocks * threads);
  printf("device %s, %d SMs, max clock %d MHz\n", p.name, sms, clk / 1000);
  auto report = [&](const char* name, float ms, double ops_per_thread) {
    const double ops = n_thr * ops_per_thread;
    const double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
    printf("%-28s %8.3f ms  %8.1f Gop/s  %6.1f ops/clk/SM (at max clock)\n", name, ms,
           ops / (ms * 1e-3) / 1e9, per_clk_sm);
  };
  report("DADD", time_kernel([&] { k_dadd<<<blocks, threads>>>(d, 1e-9, 2e-9); }), 8.0 * ITERS);
  report("DMUL", time_kernel([&] { k_dmul<<<blocks, threads>>>(d, 1.0000001, 0.9999999); }),
         8.0 * ITERS);
  report("F2F.F64.F32 (+DADD)", time_kernel([&] { k_cvt_f2d<<<blocks, threads>>>(d, 0.5f); }),
         4.0 * ITERS);
  report("F2I.F64.TRUNC (+DADD)", time_kernel([&] { k_d2i<<<blocks, threads>>>(di, 0.37); }),
         4.0 * ITERS);
  report("I2F.F64 (+DADD)", time_kernel([&] { k_i2d<<<blocks, threads>>>(d, 3); }), 4.0 * ITERS);
  for (int pad = 0; pad <= 1; ++pad) {
    for (int stride : {1, 4}) {
      char name[64];
      snprintf(name, sizeof name, "LDS.32 stride%d pad%d", stride, pad);
      report(name, time_kernel([&] { k_lds<float><<<blocks, threads, 2048 * 4 + 1024>>>(d, stride, pad); }),
             ITERS);
      snprintf(name, sizeof name, "LDS.64 stride%d pad%d", stride, pad);
      report(name, time_kernel([&] { k_lds<double><<<blocks, threads, 2048 * 8 + 1024>>>(d, stride, pad); }),
             ITERS);
      snprintf(name, sizeof name, "LDS.128 stride%d pad%d", stride, pad);
      report(name, time_kernel([&] { k_lds<double2><<<blocks, threads, 2048 * 16 + 1024>>>(d, stride, pad); }),
             ITERS);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
