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
// staged.  The sum of exponentials uses a table-driven exp2 (64 entries) with
// a degree-4 near-minimax polynomial (relative error 2.4e-15, vs the reference's libm
// exp at ~1e-16; the parity bar is 1e-10).  The final multiply by 2^k*T[i]
// is fused into the accumulation FMA, so exp2 + accumulate is 8 FP64-pipe
// instructions (3 DADD + 5 DFMA); the integer split runs on the INT pipe.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rsot_cuda {

constexpr double kLog2e = 1.4426950408889634074;   // 0x1.71547652b82fep+0
constexpr double kLn2 = 0.69314718055994530942;    // 0x1.62e42fefa39efp-1

// exp2 split s = n/64 + r: 1.5 * 2^46 added to s rounds it to the 1/64 grid
// and leaves n = round(64 s) in the low mantissa word.
constexpr double kExpMagic = 0x1.8p46;
constexpr int kExpTab = 64;          // table entries 2^(i/64)
constexpr int kExpUnit = 1 << 14;    // n * kExpUnit = (n >> 6) << 20 + (n & 63) << 14
constexpr int kExpNMin = -65280;     // clamp of n: s >= -1020
constexpr int kExpNMax = 64000;      //             s <=  1000
constexpr int kExpZeroN = -65472;    // 64 * (-1023): scale word pattern +0.0

// 2^(i/64) correctly rounded (mpmath, 200 bits; tools/gen_exp2_table.py),
// stored as {lo, hi - (i << 14)} so that the scale 2^k * 2^(i/64) for
// n = 64k + i is the double with words {lo, hi' + n * 2^14}: one IMAD
// instead of split/shift/add.
__device__ __constant__ int2 kExp2Table[kExpTab] = {
    {0x00000000, 0x3ff00000}, {0x3e778061, 0x3fefec9a}, {(int)0xd3158574, 0x3fefd9b0},
    {0x18759bc8, 0x3fefc745}, {0x6cf9890f, 0x3fefb558}, {0x32d3d1a2, 0x3fefa3ec},
    {(int)0xd0125b51, 0x3fef9301}, {(int)0xaea92de0, 0x3fef829a}, {0x3c7d517b, 0x3fef72b8},
    {(int)0xeb6fcb75, 0x3fef635b}, {0x3168b9aa, 0x3fef5487}, {(int)0x88628cd6, 0x3fef463b},
    {0x6e756238, 0x3fef387a}, {0x65e27cdd, 0x3fef2b45}, {(int)0xf51fdee1, 0x3fef1e9d},
    {(int)0xa6e4030b, 0x3fef1285}, {0x0a31b715, 0x3fef06fe}, {(int)0xb26416ff, 0x3feefc08},
    {0x373aa9cb, 0x3feef1a7}, {0x34e59ff7, 0x3feee7db}, {0x4c123422, 0x3feedea6},
    {0x21f72e2a, 0x3feed60a}, {0x6061892d, 0x3feece08}, {(int)0xb5c13cd0, 0x3feec6a2},
    {(int)0xd5362a27, 0x3feebfda}, {0x769d2ca7, 0x3feeb9b2}, {0x569d4f82, 0x3feeb42b},
    {0x36b527da, 0x3feeaf47}, {(int)0xdd485429, 0x3feeab07}, {0x15ad2148, 0x3feea76f},
    {(int)0xb03a5585, 0x3feea47e}, {(int)0x82552225, 0x3feea238}, {0x667f3bcd, 0x3feea09e},
    {0x3c651a2f, 0x3fee9fb2}, {(int)0xe8ec5f74, 0x3fee9f75}, {0x564267c9, 0x3fee9feb},
    {0x73eb0187, 0x3feea114}, {0x36cf4e62, 0x3feea2f3}, {(int)0x994cce13, 0x3feea589},
    {(int)0x9b4492ed, 0x3feea8d9}, {0x422aa0db, 0x3feeace5}, {(int)0x99157736, 0x3feeb1ae},
    {(int)0xb0cdc5e5, 0x3feeb737}, {(int)0x9fde4e50, 0x3feebd82}, {(int)0x82a3f090, 0x3feec491},
    {0x7b5de565, 0x3feecc66}, {(int)0xb23e255d, 0x3feed503}, {0x5579fdbf, 0x3feede6b},
    {(int)0x995ad3ad, 0x3feee89f}, {(int)0xb84f15fb, 0x3feef3a2}, {(int)0xf2fb5e47, 0x3feeff76},
    {(int)0x904bc1d2, 0x3fef0c1e}, {(int)0xdd85529c, 0x3fef199b}, {0x2e57d14b, 0x3fef27f1},
    {(int)0xdcef9069, 0x3fef3720}, {0x4a07897c, 0x3fef472d}, {(int)0xdcfba487, 0x3fef5818},
    {0x03db3285, 0x3fef69e6}, {0x337b9b5f, 0x3fef7c97}, {(int)0xe78b3ff6, 0x3fef902e},
    {(int)0xa2a490da, 0x3fefa4af}, {(int)0xee615a27, 0x3fefba1b}, {0x5b6e4540, 0x3fefd076},
    {(int)0x819e90d8, 0x3fefe7c1}};

// Near-minimax degree-4 fit of 2^r on [-1/128, 1/128] (mpmath chebyfit,
// tools/gen_exp2_table.py), coefficients rounded to double; worst relative
// error 2.44e-15.  In constant memory so the DFMAs take them as c[][]
// operands (no per-loop uniform-register materialisation).
__device__ __constant__ double kPoly[5] = {0x1.0000000000000p+0, 0x1.62e42fefa0352p-1,
                                           0x1.ebfbdff82ac52p-3, 0x1.c6b0c40d8c4e9p-5,
                                           0x1.3b2ad0385b409p-7};
#define kP0 (kPoly[0])
#define kP1 (kPoly[1])
#define kP2 (kPoly[2])
#define kP3 (kPoly[3])
#define kP4 (kPoly[4])

// Copies the exp2 table into shared memory (64 x 8 B = 512 B).
__device__ __forceinline__ void load_exp2_table(int2* smem_tbl) {
  for (int i = threadIdx.x; i < kExpTab; i += blockDim.x) smem_tbl[i] = kExp2Table[i];
}

// acc + 2^s.  Exact split s = n/64 + r (|r| <= 1/128) by the magic-constant
// addition, 2^r by the polynomial, 2^(n/64) by table + exponent add.  n is
// clamped to [64 (-1020), 64 * 1000]: s below -1020 contributes at most 2^-1019
// (the reference would add a subnormal or zero); s above 1000 yields at least
// 2^999, which the callers detect (sum > 2^960) and route to the exact
// per-atom path.  FP64 pipe: 3 DADD + 5 DFMA; INT: 2 IMNMX, LOP3, LEA, IMAD.
template <bool CLAMP = true>
__device__ __forceinline__ double exp2_acc(double s, double acc,
                                           const int2* __restrict__ tbl) {
  const double kk = __dadd_rn(s, kExpMagic);
  int n = __double2loint(kk);  // round(64 s)
  if (CLAMP) n = min(max(n, kExpNMin), kExpNMax);
  const double kd = __dadd_rn(kk, -kExpMagic);
  const double r = __dadd_rn(s, -kd);        // |r| <= 1/128
  double p = fma(kP4, r, kP3);
  p = fma(p, r, kP2);
  p = fma(p, r, kP1);
  p = fma(p, r, kP0);
  const int2 t = tbl[n & (kExpTab - 1)];
  const double scale = __hiloint2double(t.y + n * kExpUnit, t.x);
  return fma(p, scale, acc);
}

// acc + (take ? 2^s : 0) without a branch.  Lanes that do not take the
// pair get n = kExpZeroN = 64 * (-1023), whose scale word pattern is exactly
// +0.0 (one SEL on the INT pipe).  CLAMP = false is used when the caller has
// proven every taken s lies in [-1020, 1000].
template <bool CLAMP = true>
__device__ __forceinline__ double exp2_acc_masked(double s, double acc,
                                                  const int2* __restrict__ tbl, bool take) {
  const double kk = __dadd_rn(s, kExpMagic);
  int n = __double2loint(kk);
  if (CLAMP) n = min(max(n, kExpNMin), kExpNMax);
  const double kd = __dadd_rn(kk, -kExpMagic);
  const double r = __dadd_rn(s, -kd);
  double p = fma(kP4, r, kP3);
  p = fma(p, r, kP2);
  p = fma(p, r, kP1);
  p = fma(p, r, kP0);
  n = take ? n : kExpZeroN;
  const int2 t = tbl[n & (kExpTab - 1)];
  return fma(p, __hiloint2double(t.y + n * kExpUnit, t.x), acc);
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

// 192-bit fixed point (scale 2^150) accumulation of a non-negative double.
__device__ inline void fp_add(unsigned long long* acc, double m) {
  if (!(m > 0.0)) return;
  int e;
  const double fr = frexp(m, &e);                   // m = fr * 2^e, fr in [0.5,1)
  const unsigned long long mant = static_cast<unsigned long long>(ldexp(fr, 53));
  const int sh = e - 53 + 150;                       // value = mant * 2^sh
  unsigned long long l0 = 0, l1 = 0, l2 = 0;
  if (sh < 0) {
    if (sh > -64) l0 = mant >> (-sh);
  } else {
    const int w = sh >> 6, b = sh & 63;
    const unsigned long long lo = mant << b;
    const unsigned long long hi = b ? (mant >> (64 - b)) : 0ull;
    if (w == 0) { l0 = lo; l1 = hi; }
    else if (w == 1) { l1 = lo; l2 = hi; }
    else if (w == 2) { l2 = lo; }
  }
  unsigned long long carry = 0;
  {
    if (l0) {
      const unsigned long long old = atomicAdd(&acc[0], l0);
      carry = (old + l0 < old) ? 1ull : 0ull;
    }
  }
  {
    const unsigned long long add = l1 + carry;
    const unsigned long long c1 = (add < l1) ? 1ull : 0ull;
    carry = c1;
    if (add) {
      const unsigned long long old = atomicAdd(&acc[1], add);
      carry += (old + add < old) ? 1ull : 0ull;
    }
  }
  {
    const unsigned long long add = l2 + carry;
    if (add) atomicAdd(&acc[2], add);
  }
}

__device__ inline double fp_to_double(const unsigned long long* acc) {
  return (static_cast<double>(acc[2]) * 0x1p-22 + static_cast<double>(acc[1]) * 0x1p-86) +
         static_cast<double>(acc[0]) * 0x1p-150;
}

// Gradient accumulator of the truncated kernels: 5 limbs of 32 bits at
// weights 2^(32 i - 150), each limb word a u64 with 2^32 adds of headroom,
// so contributions are added with fire-and-forget reductions (RED, no
// returned value, no carry chain: fp_add's ATOM round trips stalled the
// phase-2 warps on their results).  Integer sums are order independent, so
// the total is deterministic; bits below 2^-150 are dropped as in fp_add.
constexpr int kLimbs = 5;
__device__ __forceinline__ void fp_red(unsigned long long* acc, double m) {
  if (!(m > 0.0)) return;
  int e;
  const double fr = frexp(m, &e);
  unsigned long long mant = static_cast<unsigned long long>(ldexp(fr, 53));
  int sh = e - 53 + 150;  // value = mant * 2^sh (units of 2^-150)
  if (sh < 0) {
    if (sh <= -64) return;
    mant >>= -sh;
    sh = 0;
  }
  const int i0 = sh >> 5;
  const unsigned __int128 w = static_cast<unsigned __int128>(mant) << (sh & 31);  // < 2^85
  const unsigned long long l0 = static_cast<unsigned long long>(w) & 0xffffffffull;
  const unsigned long long l1 = static_cast<unsigned long long>(w >> 32) & 0xffffffffull;
  const unsigned long long l2 = static_cast<unsigned long long>(w >> 64);
  if (l0 && i0 < kLimbs) atomicAdd(acc + i0, l0);
  if (l1 && i0 + 1 < kLimbs) atomicAdd(acc + i0 + 1, l1);
  if (l2 && i0 + 2 < kLimbs) atomicAdd(acc + i0 + 2, l2);
}

__device__ __forceinline__ double fp_limbs_to_double(const unsigned long long* acc) {
  return (((static_cast<double>(acc[4]) * 0x1p-22 + static_cast<double>(acc[3]) * 0x1p-54) +
           static_cast<double>(acc[2]) * 0x1p-86) +
          static_cast<double>(acc[1]) * 0x1p-118) +
         static_cast<double>(acc[0]) * 0x1p-150;
}

// cost.hpp:19-33: dot(p, q) = (p0 q0 + p1 q1) + p2 q2, clamp, acos, square.
__device__ __forceinline__ double geo_cost(double x0, double x1, double x2, double y0, double y1,
                                           double y2) {
  const double d = __dadd_rn(__dadd_rn(__dmul_rn(x0, y0), __dmul_rn(x1, y1)), __dmul_rn(x2, y2));
  const double t = d < -1.0 ? -1.0 : (1.0 < d ? 1.0 : d);
  const double g = acos(t);
  return __dmul_rn(g, g);
}

}  // namespace rsot_cuda
