// Microbenchmark: FP64 mma.sync (DMMA m8n8k4) rate and overlap with DFMA.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kIt = 1024;
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void k(double* out, double a, double b) {
  double c[8][2];
  double x[8];
  for (int i = 0; i < 8; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; x[i] = threadIdx.x + i; }
  double av = 1.0 + threadIdx.x * 1e-9, bv = 0.5;
#pragma unroll 1
  for (int it = 0; it < kIt; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 2) dmma(c[i][0], c[i][1], av, bv);
      if (MODE == 1 || MODE == 2) x[i] = fma(x[i], a, b);
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE> float run(double* out, int blocks) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(e0); k<MODE><<<blocks, 256>>>(out, 0.999, 1e-3); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
  }
  return best;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 8; double* out; cudaMalloc(&out, sizeof(double) * blocks * 256);
  double warps = double(blocks) * 8 * kIt * 8;
  float t0 = run<0>(out, blocks), t1 = run<1>(out, blocks), t2 = run<2>(out, blocks);
  printf("DMMA only: %.3f ms -> %.3e DMMA/s = %.2f TFLOP/s (256 FMA each)\n", t0, warps / (t0 * 1e-3),
         warps * 256 * 2 / (t0 * 1e-3) / 1e12);
  printf("DFMA only: %.3f ms -> %.3e warp-DFMA/s\n", t1, warps / (t1 * 1e-3));
  printf("both     : %.3f ms (sum of separate %.3f)\n", t2, t0 + t1);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
