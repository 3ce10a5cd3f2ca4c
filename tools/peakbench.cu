// Pipe-rate microbenchmark for the roofline denominators the RSOT evaluator
// is bound by (FP64 DFMA, FP32 FFMA, MUFU.EX2, libdevice exp, table exp2).
// Not part of the product: it measures the machine.  Prints one JSON line.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void ffma_kernel(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  float x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
    x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
    x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void ex2_kernel(float* out, float a) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f;
#pragma unroll 4
  for (int i = 0; i < kIters; ++i) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x2));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x3));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + a;
}

__global__ void dexp_kernel(double* out, double a) {
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  double t = -(threadIdx.x & 31) * 0.37;
#pragma unroll 4
  for (int i = 0; i < kIters / 4; ++i) {
    s0 += exp(t); s1 += exp(t - a); s2 += exp(t - 2 * a); s3 += exp(t - 3 * a);
    t -= 1e-3;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  const int threads = 256, blocks = sms * 8;
  double* dout; float* fout;
  CK(cudaMalloc(&dout, sizeof(double) * threads * blocks));
  CK(cudaMalloc(&fout, sizeof(float) * threads * blocks));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const double n_thr = double(threads) * blocks;
  auto best = [&](auto launch) {
    float b = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (r > 0 && ms < b) b = ms;
    }
    return b;
  };
  float t_dfma = best([&] { dfma_kernel<<<blocks, threads>>>(dout, 0.999, 1e-3); });
  float t_ffma = best([&] { ffma_kernel<<<blocks, threads>>>(fout, 0.999f, 1e-3f); });
  float t_ex2 = best([&] { ex2_kernel<<<blocks, threads>>>(fout, 1.f); });
  float t_dexp = best([&] { dexp_kernel<<<blocks, threads>>>(dout, 0.01); });
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  const double dfma_per_s = n_thr * kIters * 8 / (t_dfma * 1e-3);
  const double ffma_per_s = n_thr * kIters * 8 / (t_ffma * 1e-3);
  const double ex2_per_s = n_thr * kIters * 4 / (t_ex2 * 1e-3);
  const double dexp_per_s = n_thr * kIters / (t_dexp * 1e-3);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"dfma_per_s\": %.4e, \"fp64_tflops\": %.3f, "
         "\"ffma_per_s\": %.4e, \"mufu_ex2_per_s\": %.4e, \"libdevice_exp_per_s\": %.4e}\n",
         sms, clk, dfma_per_s, 2 * dfma_per_s / 1e12, ffma_per_s, ex2_per_s, dexp_per_s);
  return 0;
}
