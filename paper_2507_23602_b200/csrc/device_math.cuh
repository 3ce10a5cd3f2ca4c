// device_math.cuh -- fp64 building blocks of the RSOT evaluator kernels.
//
// All exponents are carried in base 2:  e2_qj = log2(e) * e_qj, where
// e_qj = (psi_j - 0.5*|x_q - y_j|^2)/eps + ln(nu_j) is the reference's
// per-pair exponent (proj/src/evaluate.cpp:139-140).  With
//   b2_j = log2(e) * (psi_j/eps + ln nu_j),   c2 = log2(e) / (2 eps)
// we have e2_qj = b2_j - c2 * |x_q - y_j|^2.  In local coordinates about an
// origin o (x' = x - o, y' = y - o):
//   e2_qj = (b2_j - c2|y'|^2) - c2|x'|^2 + (2 c2 x') . y'
// so a pair costs three DFMA once the per-target and per-atom constants are
// staged.  The sum of exponentials uses a table-driven exp2 with a degree-5
// near-minimax polynomial (relative error 4.6e-15, vs the reference's libm
// exp at ~1e-16; the parity bar is 1e-10).  The final multiply by 2^k*T[i]
// is fused into the accumulation FMA, so exp2 + accumulate is 9 FP64-pipe
// instructions (3 DADD + 6 DFMA); the integer split runs on the INT pipe.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rsot_cuda {

constexpr double kLog2e = 1.4426950408889634074;   // 0x1.71547652b82fep+0
constexpr double kLn2 = 0.69314718055994530942;    // 0x1.62e42fefa39efp-1

// 1.5 * 2^48: adding it rounds to the 1/16 grid and leaves round(16 s) in
// the low mantissa bits.
constexpr double kExpMagic = 0x1.8p48;

// 2^(i/16), correctly rounded (mpmath, 200 bits).
__device__ __constant__ double kExp2Table[16] = {
    0x1.0000000000000p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0,
    0x1.2387a6e756238p+0, 0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0,
    0x1.4bfdad5362a27p+0, 0x1.5ab07dd485429p+0, 0x1.6a09e667f3bcdp+0,
    0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0, 0x1.9c49182a3f090p+0,
    0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0,
    0x1.ea4afa2a490dap+0};

// Near-minimax degree-5 fit of 2^r on [-1/32, 1/32] (mpmath chebyfit),
// coefficients rounded to double; worst relative error 4.61e-15.
constexpr double kP5 = 0x1.5d897e525c216p-10;
constexpr double kP4 = 0x1.3b2c9b8a6caeap-7;
constexpr double kP3 = 0x1.c6b08d6f2a289p-5;
constexpr double kP2 = 0x1.ebfbdff555824p-3;
constexpr double kP1 = 0x1.62e42fefa39f3p-1;
constexpr double kP0 = 0x1.0000000000014p+0;

// Copies the exp2 table into shared memory (16 doubles = 128 B: a
// half-warp LDS.64 with any index pattern is one conflict-free wavefront).
__device__ __forceinline__ void load_exp2_table(double* smem_tbl) {
  if (threadIdx.x < 16) smem_tbl[threadIdx.x] = kExp2Table[threadIdx.x];
}

// acc + 2^s.  Valid for s in [-1020, 1020]; s below -1020 contributes 0
// (the contribution is < 2^-1020 and is dropped, the reference would add a
// subnormal); s above 1020 yields +inf, which the callers detect and route
// to the exact per-atom path (exponents are taken relative to an upper
// bound, so this only happens for pathological inputs).
__device__ __forceinline__ double exp2_acc(double s, double acc,
                                           const double* __restrict__ tbl) {
  const double kk = __dadd_rn(s, kExpMagic);
  const int n = __double2loint(kk);          // round(16 s)
  const double kd = __dadd_rn(kk, -kExpMagic);
  const double r = __dadd_rn(s, -kd);        // |r| <= 1/32
  double p = fma(kP5, r, kP4);
  p = fma(p, r, kP3);
  p = fma(p, r, kP2);
  p = fma(p, r, kP1);
  p = fma(p, r, kP0);
  const int k = n >> 4;                      // floor division by 16
  const double t = tbl[n & 15];
  int hi = __double2hiint(t) + static_cast<int>(static_cast<unsigned>(k) << 20);
  int lo = __double2loint(t);
  hi = (k < -1020) ? 0 : hi;                 // flush tiny contributions
  lo = (k < -1020) ? 0 : lo;
  hi = (k > 1020) ? 0x7ff00000 : hi;         // overflow -> +inf (the caller
  lo = (k > 1020) ? 0 : lo;                  // flags the atom for the exact path)
  return fma(p, __hiloint2double(hi, lo), acc);
}

// Exact reference predicate (point.hpp:35-40, spatial_index.cpp:54):
// ((dx*dx + dy*dy) + dz*dz) < r2, every operation rounded separately.
__device__ __forceinline__ bool exact_inside(double x0, double x1, double x2,
                                             double y0, double y1, double y2,
                                             double r2) {
  const double dx = __dsub_rn(x0, y0);
  const double dy = __dsub_rn(x1, y1);
  const double dz = __dsub_rn(x2, y2);
  const double d2 =
      __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return d2 < r2;
}

// Reference squared distance (same association, unfused).
__device__ __forceinline__ double exact_sqdist(double x0, double x1, double x2,
                                               double y0, double y1, double y2) {
  const double dx = __dsub_rn(x0, y0);
  const double dy = __dsub_rn(x1, y1);
  const double dz = __dsub_rn(x2, y2);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// The reference per-pair exponent in natural units, operation for operation
// (evaluate.cpp:139-140): (psi - 0.5*d2)/eps + log_nu.
__device__ __forceinline__ double reference_exponent(double psi, double d2,
                                                     double eps, double log_nu) {
  return __dadd_rn(__ddiv_rn(__dsub_rn(psi, __dmul_rn(0.5, d2)), eps), log_nu);
}

// splitmix64 finaliser; the per-atom candidate hash is the wrapping sum of
// this over the candidate set (same definition as oracle/rsot_oracle.c).
__device__ __forceinline__ uint64_t candidate_hash_term(uint64_t j) {
  uint64_t z = j + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

}  // namespace rsot_cuda
