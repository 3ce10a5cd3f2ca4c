// block_util.cuh -- fixed-order warp/block reductions and scans.
// Every reduction here has a summation tree that depends only on the block
// size, so results are bitwise reproducible run to run.
#pragma once

#include <cuda_runtime.h>

namespace rsot_cuda {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-order block sum; all threads receive the result.  sh >= 32 doubles.
template <int BLK>
__device__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = (l < BLK / 32) ? sh[l] : 0.0;
    t = warp_sum(t);
    if (l == 0) sh[0] = t;
  }
  __syncthreads();
  return sh[0];
}

template <int BLK>
__device__ double block_max(double v, double* sh) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = (l < BLK / 32) ? sh[l] : -INFINITY;
    t = warp_max(t);
    if (l == 0) sh[0] = t;
  }
  __syncthreads();
  return sh[0];
}

// Bounding box of the block's points (invalid threads pass lo=+inf,
// hi=-inf).  Writes box[0..2] = lo, box[3..5] = hi; an empty block gets a
// zero box.  sh >= 200 doubles.
template <int BLK>
__device__ void block_bbox(const double lo_in[3], const double hi_in[3],
                           double* sh, double box[6]) {
  double v[6] = {lo_in[0], lo_in[1], lo_in[2], -hi_in[0], -hi_in[1], -hi_in[2]};
#pragma unroll
  for (int c = 0; c < 6; ++c) v[c] = warp_min(v[c]);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0)
#pragma unroll
    for (int c = 0; c < 6; ++c) sh[c * 32 + w] = v[c];
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      double t = (l < BLK / 32) ? sh[c * 32 + l] : INFINITY;
      v[c] = warp_min(t);
    }
    if (l == 0) {
      for (int c = 0; c < 3; ++c) {
        const double a = v[c], b = -v[c + 3];
        const bool ok = a <= b;
        sh[192 + c] = ok ? a : 0.0;
        sh[195 + c] = ok ? b : 0.0;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 6; ++c) box[c] = sh[192 + c];
  __syncthreads();
}

// Exclusive block scan of ints; returns this thread's exclusive prefix and
// writes the block total to *total.  sh >= 33 ints.
template <int BLK>
__device__ int block_exclusive_scan(int v, int* sh, int* total) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (l >= o) inc += t;
  }
  __syncthreads();
  if (l == 31) sh[w] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < BLK / 32; ++i) {
      const int t = sh[i];
      sh[i] = run;
      run += t;
    }
    sh[32] = run;
  }
  __syncthreads();
  const int res = sh[w] + inc - v;
  *total = sh[32];
  __syncthreads();
  return res;
}

}  // namespace rsot_cuda
