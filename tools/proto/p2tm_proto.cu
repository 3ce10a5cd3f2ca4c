// Prototype (development aid, not part of the product): throughput of a
// target-major phase-2 inner loop -- lane = item, loop over the warp's 64
// atoms (broadcast from shared memory), FP64 exp2 (512-entry table, degree 3)
// masked by a 64-bit per-item atom mask, fixed-point RED per item -- at the
// cfg5 scale (65536 CTAs x 4 warps x ~1000 items).  Compares with the fused
// kernel's phase 2 (~21.6 ms).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kItems = 1000;
__constant__ double kP[4] = {1.0, 0.6931471805599453, 0.2402265069591007, 0.05550410866482158};

__device__ __forceinline__ double ex2acc(double s, double acc, const int2* tbl, bool take) {
  const double kk = __dadd_rn(s, 0x1.8p43);
  int n = __double2loint(kk);
  const double kd = __dadd_rn(kk, -0x1.8p43);
  const double r = __dadd_rn(s, -kd);
  double p = fma(kP[3], r, kP[2]);
  p = fma(p, r, kP[1]);
  p = fma(p, r, kP[0]);
  n = take ? n : -523776;
  const int2 t = tbl[n & 511];
  return fma(p, __hiloint2double(t.y + n * 2048, t.x), acc);
}

__global__ void __launch_bounds__(128, 4) p2tm(const double4* __restrict__ ys, const double* __restrict__ b2s,
                                               const uint4* __restrict__ recs, unsigned long long* gacc, int n) {
  __shared__ double4 atab[4][64];
  __shared__ int2 tbl[512];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 512; i += 128) tbl[i] = make_int2(0, 0x3ff00000 - i * 2048);
  for (int i = lane; i < 64; i += 32)
    atab[warp][i] = make_double4(1e2 * (i % 4 - 1.5), 1e2 * (i / 16 - 1.5), 1e2 * ((i / 4) % 4 - 1.5), -3.0);
  __syncthreads();
  const uint4* r = recs + (static_cast<size_t>(blockIdx.x) * 4 + warp) * kItems;
  for (int c = 0; c < kItems; c += 32) {
    const int i = c + lane;
    const uint4 rec = i < kItems ? r[i] : make_uint4(0, 0, 0, 0);
    const int k = rec.x % n;
    const double4 y = ys[k];
    const double y0 = y.x - 0.5, y1 = y.y - 0.5, y2 = y.z - 0.5;
    const double T = fma(-7213.0, fma(y2, y2, fma(y1, y1, y0 * y0)), b2s[k]) - 1.0;
    const unsigned long long m = (static_cast<unsigned long long>(rec.z) << 32) | rec.y;
    double acc = 0.0;
#pragma unroll 16
    for (int a = 0; a < 64; ++a) {
      const double4 A = atab[warp][a];
      const double s = fma(A.x, y0, fma(A.y, y1, fma(A.z, y2, T + A.w)));
      acc = ex2acc(s, acc, tbl, (m >> a) & 1ull);
    }
    if (i < kItems && acc > 0.0) {
      const unsigned long long v = static_cast<unsigned long long>(acc * 0x1p40);
      atomicAdd(gacc + 3 * static_cast<size_t>(k), v & 0xffffffffull);
      atomicAdd(gacc + 3 * static_cast<size_t>(k) + 1, v >> 32);
    }
  }
}

int main() {
  const int n = 1 << 20, ctas = 65536;
  const size_t nrec = static_cast<size_t>(ctas) * 4 * kItems;
  double4* ys; double* b2; uint4* recs; unsigned long long* g;
  cudaMalloc(&ys, sizeof(double4) * n); cudaMalloc(&b2, sizeof(double) * n);
  cudaMalloc(&recs, sizeof(uint4) * nrec); cudaMalloc(&g, sizeof(unsigned long long) * 3 * n);
  cudaMemset(ys, 0, sizeof(double4) * n); cudaMemset(b2, 0, sizeof(double) * n);
  // records: pseudo-random target index, ~62 % of the mask bits set
  unsigned* h = nullptr;
  cudaMallocHost(&h, sizeof(uint4) * (1 << 20));
  for (size_t i = 0; i < (1u << 20); ++i) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull;
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    uint64_t mk = 0;
    for (int b = 0; b < 64; ++b) { x = x * 6364136223846793005ull + 1442695040888963407ull; if ((x >> 40) % 100 < 62) mk |= 1ull << b; }
    h[4 * i] = static_cast<unsigned>(x >> 11); h[4 * i + 1] = static_cast<unsigned>(mk); h[4 * i + 2] = static_cast<unsigned>(mk >> 32); h[4 * i + 3] = 0;
  }
  for (size_t off = 0; off < nrec; off += (1u << 20))
    cudaMemcpy(recs + off, h, sizeof(uint4) * std::min<size_t>(1u << 20, nrec - off), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(p2tm, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int dyn : {0, 40 * 1024, 60 * 1024}) {  // extra shared memory limits the CTAs per SM
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, p2tm, 128, dyn);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      p2tm<<<ctas, 128, dyn>>>(ys, b2, recs, g, n);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("p2tm: %d CTAs/SM: %.3f ms (%s)\n", nb, ms, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
