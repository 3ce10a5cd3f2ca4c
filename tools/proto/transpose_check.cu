#include <cstdio>
__device__ __forceinline__ unsigned warp_transpose32(unsigned x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 16; k >= 1; k >>= 1) {
    const unsigned m = k == 16 ? 0x0000ffffu : k == 8 ? 0x00ff00ffu : k == 4 ? 0x0f0f0f0fu
                     : k == 2 ? 0x33333333u : 0x55555555u;
    const unsigned y = __shfl_xor_sync(0xffffffffu, x, k);
    x = (lane & k) ? (((y >> k) & m) | (x & ~m)) : ((x & m) | ((y & m) << k));
  }
  return x;
}
__global__ void t(unsigned* out) { unsigned x = 0x9E3779B9u * (threadIdx.x + 1) ^ (threadIdx.x << 7); out[threadIdx.x] = x; out[32 + threadIdx.x] = warp_transpose32(x); }
int main() { unsigned* d; cudaMalloc(&d, 256); t<<<1, 32>>>(d); unsigned h[64]; cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost); int bad = 0; for (int b = 0; b < 32; ++b) for (int l = 0; l < 32; ++l) if (((h[32 + b] >> l) & 1) != ((h[l] >> b) & 1)) ++bad; printf("transpose bad bits: %d\n", bad); return 0; }
