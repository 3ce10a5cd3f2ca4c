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

// 2^(i/16) correctly rounded (mpmath, 200 bits), stored as {lo, hi - (i<<16)}
// so that the scale 2^k * 2^(i/16) for n = 16k + i is the double with words
// {lo, hi' + (n << 16)}: one IMAD instead of split/shift/add.
__device__ __constant__ int2 kExp2Table[16] = {
    {0x00000000, 0x3ff00000}, {0x6cf9890f, 0x3fefb558}, {0x3c7d517b, 0x3fef72b8},
    {0x6e756238, 0x3fef387a}, {0x0a31b715, 0x3fef06fe}, {0x4c123422, 0x3feedea6},
    {(int)0xd5362a27, 0x3feebfda}, {(int)0xdd485429, 0x3feeab07}, {0x667f3bcd, 0x3feea09e},
    {0x73eb0187, 0x3feea114}, {0x422aa0db, 0x3feeace5}, {(int)0x82a3f090, 0x3feec491},
    {(int)0x995ad3ad, 0x3feee89f}, {(int)0xdd85529c, 0x3fef199b}, {(int)0xdcfba487, 0x3fef5818},
    {(int)0xa2a490da, 0x3fefa4af}};

// Near-minimax degree-5 fit of 2^r on [-1/32, 1/32] (mpmath chebyfit),
// coefficients rounded to double; worst relative error 4.61e-15.  Kept in
// constant memory so the DFMAs take them as c[][] operands (no per-loop
// uniform-register materialisation).
__device__ __constant__ double kPoly[6] = {0x1.0000000000014p+0, 0x1.62e42fefa39f3p-1,
                                           0x1.ebfbdff555824p-3, 0x1.c6b08d6f2a289p-5,
                                           0x1.3b2c9b8a6caeap-7, 0x1.5d897e525c216p-10};
#define kP0 (kPoly[0])
#define kP1 (kPoly[1])
#define kP2 (kPoly[2])
#define kP3 (kPoly[3])
#define kP4 (kPoly[4])
#define kP5 (kPoly[5])

// Copies the exp2 table into shared memory (16 x 8 B = 128 B: a half-warp
// LDS.64 with any index pattern is one conflict-free wavefront).
__device__ __forceinline__ void load_exp2_table(int2* smem_tbl) {
  if (threadIdx.x < 16) smem_tbl[threadIdx.x] = kExp2Table[threadIdx.x];
}

// acc + 2^s.  Exact split s = n/16 + r (|r| <= 1/32) by the magic-constant
// addition, 2^r by the polynomial, 2^(n/16) by table + exponent add.  n is
// clamped to [-16320, 16000]: s below -1020 contributes at most 2^-1019
// (the reference would add a subnormal or zero); s above 1000 yields at least
// 2^999, which the callers detect (sum > 2^960) and route to the exact
// per-atom path.  FP64 pipe: 3 DADD + 6 DFMA; INT: 2 IMNMX, LOP3, LEA, IMAD.
template <bool CLAMP = true>
__device__ __forceinline__ double exp2_acc(double s, double acc,
                                           const int2* __restrict__ tbl) {
  const double kk = __dadd_rn(s, kExpMagic);
  int n = __double2loint(kk);  // round(16 s)
  if (CLAMP) n = min(max(n, -16320), 16000);
  const double kd = __dadd_rn(kk, -kExpMagic);
  const double r = __dadd_rn(s, -kd);        // |r| <= 1/32
  double p = fma(kP5, r, kP4);
  p = fma(p, r, kP3);
  p = fma(p, r, kP2);
  p = fma(p, r, kP1);
  p = fma(p, r, kP0);
  const int2 t = tbl[n & 15];
  const double scale = __hiloint2double(t.y + n * 65536, t.x);
  return fma(p, scale, acc);
}

// acc + (take ? 2^s : 0) without a branch.  Lanes that do not take the
// pair get n = -16368 = 16 * (-1023), whose scale word pattern is exactly
// +0.0 (one SEL on the INT pipe).  CLAMP = false is used when the caller has
// proven every taken s lies in [-1020, 1000].
template <bool CLAMP = true>
__device__ __forceinline__ double exp2_acc_masked(double s, double acc,
                                                  const int2* __restrict__ tbl, bool take) {
  const double kk = __dadd_rn(s, kExpMagic);
  int n = __double2loint(kk);
  if (CLAMP) n = min(max(n, -16320), 16000);
  const double kd = __dadd_rn(kk, -kExpMagic);
  const double r = __dadd_rn(s, -kd);
  double p = fma(kP5, r, kP4);
  p = fma(p, r, kP3);
  p = fma(p, r, kP2);
  p = fma(p, r, kP1);
  p = fma(p, r, kP0);
  n = take ? n : -16368;
  const int2 t = tbl[n & 15];
  return fma(p, __hiloint2double(t.y + n * 65536, t.x), acc);
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
