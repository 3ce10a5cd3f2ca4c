// Microbenchmark: DFMA throughput vs number of distinct register operands
// (register-file bank pressure), sm_100a.  Development aid.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kIt = 2048;
template <int MODE>
__global__ void k(double* out, double a, double b) {
  double x[8], y[8], z[8];
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; y[i] = 1.0 + 1e-9 * i; z[i] = 1e-3 * i; }
#pragma unroll 2
  for (int it = 0; it < kIt; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) x[i] = fma(x[i], a, b);              // 1 reg + 2 const
      if (MODE == 1) x[i] = fma(x[i], y[i], b);           // 2 regs
      if (MODE == 2) x[i] = fma(x[i], y[i], z[i]);        // 3 regs
      if (MODE == 3) x[i] = fma(y[i], z[i], x[i]);        // 3 regs, acc last
      if (MODE == 4) x[i] = x[i] + y[i];                  // DADD 2 regs
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i] + y[i] + z[i];
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
  double ops = double(blocks) * 256 * kIt * 8;
  printf("1reg+2const %.3e/s\n", ops / (run<0>(out, blocks) * 1e-3));
  printf("2reg+const  %.3e/s\n", ops / (run<1>(out, blocks) * 1e-3));
  printf("3reg        %.3e/s\n", ops / (run<2>(out, blocks) * 1e-3));
  printf("3reg acc    %.3e/s\n", ops / (run<3>(out, blocks) * 1e-3));
  printf("dadd 2reg   %.3e/s\n", ops / (run<4>(out, blocks) * 1e-3));
  return 0;
}
