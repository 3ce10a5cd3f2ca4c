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
// staged.  The sum of exponentials uses a table-driven exp2 (ExpTab64 /
// ExpTab512 below; relative error <= 2.4e-15, vs the reference's libm exp at
// ~1e-16; the parity bar is 1e-10).  The final multiply by 2^k*T[i] is fused
// into the accumulation FMA, so exp2 + accumulate is 8 (7) FP64-pipe
// instructions (3 DADD + 5 (4) DFMA); the integer split runs on the INT pipe.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rsot_cuda {

constexpr double kLog2e = 1.4426950408889634074;   // 0x1.71547652b82fep+0
constexpr double kLn2 = 0.69314718055994530942;    // 0x1.62e42fefa39efp-1

// Two exp2 variants share one scheme, s = n/T + r: adding 1.5 * 2^(52 - b)
// (T = 2^b) rounds s to the 1/T grid and leaves n = round(T s) in the low
// mantissa word; 2^(n/T) comes from a T-entry table of 2^(i/T) (correctly
// rounded, mpmath 200 bits, tools/gen_exp2_table.py b d) stored as
// {lo, hi - (i << (20 - b))}, so the scale 2^k * 2^(i/T) for n = T k + i is
// the double with words {lo, hi' + n * 2^(20 - b)}: one IMAD instead of
// split/shift/add; 2^r by a near-minimax polynomial (mpmath chebyfit,
// coefficients rounded to double, in constant memory so the DFMAs take them
// as c[][] operands).
//   ExpTab64:  64 entries (512 B), degree 4 on |r| <= 1/128, rel. error 2.4e-15
//   ExpTab512: 512 entries (4 KB), degree 3 on |r| <= 1/1024, rel. error 1.1e-15
// The truncated kernels use ExpTab512 (one DFMA less per exponential:
// cfg3/cfg5 -6.5 %); the dense passes keep ExpTab64, whose fewer distinct
// table rows leave fewer shared-memory bank conflicts in the target-major
// gather (pass B +2 % with 512 entries).  A 256-entry degree-3 fit (1.8e-14)
// fails the reference's symmetric-instance check |g| <= 1e-15
// (test_core.cpp:79-80).
__device__ __constant__ int2 kExp2Table64[64] = {
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
__device__ __constant__ int2 kExp2Table512[512] = {
    {0x00000000, 0x3ff00000}, {(int)0x86da1c0a, 0x3feffd8c}, {(int)0xfa5abcbf, 0x3feffb1a},
    {0x5b2cbd11, 0x3feff8ab}, {(int)0xa9fb3335, 0x3feff63d}, {(int)0xe77170b4, 0x3feff3d1},
    {0x143b0281, 0x3feff168}, {0x3103b10e, 0x3fefef00}, {0x3e778061, 0x3fefec9a},
    {0x3d42b027, 0x3fefea36}, {0x2e11bbcc, 0x3fefe7d4}, {0x11915a8a, 0x3fefe574},
    {(int)0xe86e7f85, 0x3fefe315}, {(int)0xb35659d8, 0x3fefe0b9}, {0x72f654b1, 0x3fefde5f},
    {0x27fc1762, 0x3fefdc07}, {(int)0xd3158574, 0x3fefd9b0}, {0x74f0bec2, 0x3fefd75c},
    {0x0e3c1f89, 0x3fefd50a}, {(int)0x9fa6407c, 0x3fefd2b9}, {0x29ddf6de, 0x3fefd06b},
    {(int)0xad925493, 0x3fefce1e}, {0x2b72a836, 0x3fefcbd4}, {(int)0xa42e7d30, 0x3fefc98b},
    {0x18759bc8, 0x3fefc745}, {(int)0x88f8093f, 0x3fefc500}, {(int)0xf66607e0, 0x3fefc2bd},
    {0x61701716, 0x3fefc07d}, {(int)0xcac6f383, 0x3fefbe3e}, {0x331b9715, 0x3fefbc02},
    {(int)0x9b1f3919, 0x3fefb9c7}, {0x03834e52, 0x3fefb78f}, {0x6cf9890f, 0x3fefb558},
    {(int)0xd833d93f, 0x3fefb323}, {0x45e46c85, 0x3fefb0f1}, {(int)0xb6bdae53, 0x3fefaec0},
    {0x2b7247f7, 0x3fefac92}, {(int)0xa4b520ba, 0x3fefaa65}, {0x23395dec, 0x3fefa83b},
    {(int)0xa7b26300, 0x3fefa612}, {0x32d3d1a2, 0x3fefa3ec}, {(int)0xc55189c6, 0x3fefa1c7},
    {0x5fdfa9c5, 0x3fef9fa5}, {0x03328e6d, 0x3fef9d85}, {(int)0xaffed31b, 0x3fef9b66},
    {0x66f951ce, 0x3fef994a}, {0x28d7233e, 0x3fef9730}, {(int)0xf64d9ef1, 0x3fef9517},
    {(int)0xd0125b51, 0x3fef9301}, {(int)0xb6db2dc1, 0x3fef90ed}, {(int)0xab5e2ab6, 0x3fef8edb},
    {(int)0xae51a5c8, 0x3fef8ccb}, {(int)0xc06c31cc, 0x3fef8abd}, {(int)0xe264a0e9, 0x3fef88b1},
    {0x14f204ab, 0x3fef86a8}, {0x58cbae1e, 0x3fef84a0}, {(int)0xaea92de0, 0x3fef829a},
    {0x17425438, 0x3fef8097}, {(int)0x934f312e, 0x3fef7e95}, {0x2388149e, 0x3fef7c96},
    {(int)0xc8a58e51, 0x3fef7a98}, {(int)0x83606e12, 0x3fef789d}, {0x5471c3c2, 0x3fef76a4},
    {0x3c92df73, 0x3fef74ad}, {0x3c7d517b, 0x3fef72b8}, {0x54eaea89, 0x3fef70c5},
    {(int)0x8695bbc0, 0x3fef6ed4}, {(int)0xd23816c9, 0x3fef6ce5}, {0x388c8dea, 0x3fef6af9},
    {(int)0xba4df41f, 0x3fef690e}, {0x58375d2f, 0x3fef6726}, {0x13041dc2, 0x3fef6540},
    {(int)0xeb6fcb75, 0x3fef635b}, {(int)0xe2363cf8, 0x3fef6179}, {(int)0xf8138a1c, 0x3fef5f99},
    {0x2dc40bf0, 0x3fef5dbc}, {(int)0x84045cd4, 0x3fef5be0}, {(int)0xfb91588f, 0x3fef5a06},
    {(int)0x95281c6b, 0x3fef582f}, {0x51860746, 0x3fef565a}, {0x3168b9aa, 0x3fef5487},
    {0x358e15e8, 0x3fef52b6}, {0x5eb44027, 0x3fef50e7}, {(int)0xad999e82, 0x3fef4f1a},
    {0x22fcd91d, 0x3fef4d50}, {(int)0xbf9cda38, 0x3fef4b87}, {(int)0x8438ce4d, 0x3fef49c1},
    {0x7190241e, 0x3fef47fd}, {(int)0x88628cd6, 0x3fef463b}, {(int)0xc96ffc18, 0x3fef447b},
    {0x3578a819, 0x3fef42be}, {(int)0xcd3d09b9, 0x3fef4102}, {(int)0x917ddc96, 0x3fef3f49},
    {(int)0x82fc1f27, 0x3fef3d92}, {(int)0xa27912d1, 0x3fef3bdd}, {(int)0xf0b63bff, 0x3fef3a2a},
    {0x6e756238, 0x3fef387a}, {0x1c78903a, 0x3fef36cc}, {(int)0xfb82140a, 0x3fef351f},
    {0x0c547f15, 0x3fef3376}, {0x4fb2a63f, 0x3fef31ce}, {(int)0xc65fa1ff, 0x3fef3028},
    {0x711ece75, 0x3fef2e85}, {0x50b3cb82, 0x3fef2ce4}, {0x65e27cdd, 0x3fef2b45},
    {(int)0xb16f0a30, 0x3fef29a8}, {0x341ddf29, 0x3fef280e}, {(int)0xeeb3ab98, 0x3fef2675},
    {(int)0xe1f56381, 0x3fef24df}, {0x0ea83f36, 0x3fef234c}, {0x7591bb70, 0x3fef21ba},
    {0x17779965, 0x3fef202b}, {(int)0xf51fdee1, 0x3fef1e9d}, {0x0f50d65c, 0x3fef1d13},
    {0x66d10f13, 0x3fef1b8a}, {(int)0xfc675d1f, 0x3fef1a03}, {(int)0xd0dad990, 0x3fef187f},
    {(int)0xe4f2e280, 0x3fef16fd}, {0x39771b2f, 0x3fef157e}, {(int)0xcf2f6c18, 0x3fef1400},
    {(int)0xa6e4030b, 0x3fef1285}, {(int)0xc15d5346, 0x3fef110c}, {0x1f641589, 0x3fef0f96},
    {(int)0xc1c14833, 0x3fef0e21}, {(int)0xa93e2f56, 0x3fef0caf}, {(int)0xd6a454d2, 0x3fef0b3f},
    {0x4abd886b, 0x3fef09d2}, {0x0653dfe4, 0x3fef0867}, {0x0a31b715, 0x3fef06fe},
    {0x5721b004, 0x3fef0597}, {(int)0xedeeb2fd, 0x3fef0432}, {(int)0xcf63eeac, 0x3fef02d0},
    {(int)0xfc4cd831, 0x3fef0170}, {0x75752b40, 0x3fef0013}, {0x3ba8ea32, 0x3feefeb8},
    {0x4fb45e20, 0x3feefd5f}, {(int)0xb26416ff, 0x3feefc08}, {0x6484ebb4, 0x3feefab4},
    {0x66e3fa2d, 0x3feef962}, {(int)0xba4ea77d, 0x3feef812}, {0x5f929ff1, 0x3feef6c5},
    {0x577dd72b, 0x3feef57a}, {(int)0xa2de883b, 0x3feef431}, {0x428335b4, 0x3feef2eb},
    {0x373aa9cb, 0x3feef1a7}, {(int)0x81d3f669, 0x3feef065}, {0x231e754a, 0x3feeef26},
    {0x1be9c811, 0x3feeede9}, {0x6d05d866, 0x3feeecae}, {0x1742d808, 0x3feeeb76},
    {0x1b7140ef, 0x3feeea40}, {0x7a61d55b, 0x3feee90c}, {0x34e59ff7, 0x3feee7db},
    {0x4bcdf3ea, 0x3feee6ac}, {(int)0xbfec6cf4, 0x3feee57f}, {(int)0x9212ef89, 0x3feee455},
    {(int)0xc313a8e5, 0x3feee32d}, {0x53c10f28, 0x3feee208}, {0x44ede173, 0x3feee0e5},
    {(int)0x976d27fa, 0x3feedfc4}, {0x4c123422, 0x3feedea6}, {0x63b0a09b, 0x3feedd8a},
    {(int)0xdf1c5175, 0x3feedc70}, {(int)0xbf29743f, 0x3feedb59}, {0x04ac801c, 0x3feeda45},
    {(int)0xb07a35df, 0x3feed932}, {(int)0xc367a024, 0x3feed822}, {0x3e4a136a, 0x3feed715},
    {0x21f72e2a, 0x3feed60a}, {0x6f44d8f5, 0x3feed501}, {0x2709468a, 0x3feed3fb},
    {0x4a1af3f1, 0x3feed2f7}, {(int)0xd950a897, 0x3feed1f5}, {(int)0xd5817663, 0x3feed0f6},
    {0x3f84b9d4, 0x3feecffa}, {0x18321a1a, 0x3feecf00}, {0x6061892d, 0x3feece08},
    {0x18eb43ec, 0x3feecd13}, {0x42a7d232, 0x3feecc20}, {(int)0xde7006f4, 0x3feecb2f},
    {(int)0xed1d0057, 0x3feeca41}, {0x6f8827d0, 0x3feec956}, {0x668b3237, 0x3feec86d},
    {(int)0xd3001fe5, 0x3feec786}, {(int)0xb5c13cd0, 0x3feec6a2}, {0x0fa920a1, 0x3feec5c1},
    {(int)0xe192aed2, 0x3feec4e1}, {0x2c5916c4, 0x3feec405}, {(int)0xf0d7d3de, 0x3feec32a},
    {0x2feaada6, 0x3feec253}, {(int)0xea6db7d7, 0x3feec17d}, {0x213d5283, 0x3feec0ab},
    {(int)0xd5362a27, 0x3feebfda}, {0x073537ca, 0x3feebf0d}, {(int)0xb817c114, 0x3feebe41},
    {(int)0xe8bb586b, 0x3feebd78}, {(int)0x99fddd0d, 0x3feebcb2}, {(int)0xccbd7b2a, 0x3feebbee},
    {(int)0x81d8abff, 0x3feebb2d}, {(int)0xba2e35f0, 0x3feeba6e}, {0x769d2ca7, 0x3feeb9b2},
    {(int)0xb804f127, 0x3feeb8f8}, {0x7f4531ee, 0x3feeb841}, {(int)0xcd3deb0d, 0x3feeb78c},
    {(int)0xa2cf6642, 0x3feeb6da}, {0x00da3b14, 0x3feeb62b}, {(int)0xe83f4eef, 0x3feeb57d},
    {0x59dfd53d, 0x3feeb4d3}, {0x569d4f82, 0x3feeb42b}, {(int)0xdf598d78, 0x3feeb385},
    {(int)0xf4f6ad27, 0x3feeb2e2}, {(int)0x98571b06, 0x3feeb242}, {(int)0xca5d920f, 0x3feeb1a4},
    {(int)0x8bed1bdf, 0x3feeb109}, {(int)0xdde910d2, 0x3feeb070}, {(int)0xc1351819, 0x3feeafda},
    {0x36b527da, 0x3feeaf47}, {0x3f4d854c, 0x3feeaeb6}, {(int)0xdbe2c4cf, 0x3feeae27},
    {0x0d59ca07, 0x3feead9c}, {(int)0xd497c7fd, 0x3feead12}, {0x32824135, 0x3feeac8c},
    {0x27ff07cc, 0x3feeac08}, {(int)0xb5f43d92, 0x3feeab86}, {(int)0xdd485429, 0x3feeab07},
    {(int)0x9ee20d1e, 0x3feeaa8b}, {(int)0xfba87a03, 0x3feeaa11}, {(int)0xf482fc8f, 0x3feea99a},
    {(int)0x8a5946b7, 0x3feea926}, {(int)0xbe135acc, 0x3feea8b4}, {(int)0x90998b93, 0x3feea845},
    {0x02d47c65, 0x3feea7d9}, {0x15ad2148, 0x3feea76f}, {(int)0xca0cbf0f, 0x3feea707},
    {0x20dceb71, 0x3feea6a3}, {0x1b078d26, 0x3feea641}, {(int)0xb976dc09, 0x3feea5e1},
    {(int)0xfd15612a, 0x3feea584}, {(int)0xe6cdf6f4, 0x3feea52a}, {0x778bc944, 0x3feea4d3},
    {(int)0xb03a5585, 0x3feea47e}, {(int)0x91c56acd, 0x3feea42c}, {0x1d1929fd, 0x3feea3dd},
    {0x532205d8, 0x3feea390}, {0x34ccc320, 0x3feea346}, {(int)0xc30678b7, 0x3feea2fe},
    {(int)0xfebc8fb7, 0x3feea2b9}, {(int)0xe8dcc390, 0x3feea277}, {(int)0x82552225, 0x3feea238},
    {(int)0xcc140be7, 0x3feea1fb}, {(int)0xc70833f6, 0x3feea1c1}, {0x7420a036, 0x3feea18a},
    {(int)0xd44ca973, 0x3feea155}, {(int)0xe87bfb7a, 0x3feea123}, {(int)0xb19e9538, 0x3feea0f4},
    {0x30a4c8d4, 0x3feea0c8}, {0x667f3bcd, 0x3feea09e}, {0x541ee718, 0x3feea077},
    {(int)0xfa75173e, 0x3feea052}, {0x5a736c75, 0x3feea031}, {0x750bdabf, 0x3feea012},
    {0x4b30aa09, 0x3fee9ff6}, {(int)0xddd47645, 0x3fee9fdc}, {0x2dea2f8a, 0x3fee9fc6},
    {0x3c651a2f, 0x3fee9fb2}, {0x0a38cee8, 0x3fee9fa1}, {(int)0x98593ae5, 0x3fee9f92},
    {(int)0xe7ba9fef, 0x3fee9f86}, {(int)0xf9519484, 0x3fee9f7d}, {(int)0xce1303f6, 0x3fee9f77},
    {0x66f42e87, 0x3fee9f74}, {(int)0xc4eaa988, 0x3fee9f73}, {(int)0xe8ec5f74, 0x3fee9f75},
    {(int)0xd3ef9011, 0x3fee9f7a}, {(int)0x86ead08a, 0x3fee9f82}, {0x02d50b8f, 0x3fee9f8d},
    {0x48a58174, 0x3fee9f9a}, {0x5953c849, 0x3fee9faa}, {0x35d7cbfd, 0x3fee9fbd},
    {(int)0xdf29ce7c, 0x3fee9fd2}, {0x564267c9, 0x3fee9feb}, {(int)0x9c1a861d, 0x3feea006},
    {(int)0xb1ab6e09, 0x3feea024}, {(int)0x97eeba8f, 0x3feea045}, {0x4fde5d3f, 0x3feea069},
    {(int)0xda749e5d, 0x3feea08f}, {0x38ac1cf6, 0x3feea0b9}, {0x6b7fcf03, 0x3feea0e5},
    {0x73eb0187, 0x3feea114}, {0x52e958aa, 0x3feea146}, {0x0976cfdb, 0x3feea17b},
    {(int)0x988fb9ec, 0x3feea1b2}, {0x0130c132, 0x3feea1ed}, {0x4456e7a3, 0x3feea22a},
    {0x62ff86f0, 0x3feea26a}, {0x5e2850ac, 0x3feea2ad}, {0x36cf4e62, 0x3feea2f3},
    {(int)0xedf2e1b9, 0x3feea33b}, {(int)0x8491c491, 0x3feea387}, {(int)0xfbab091f, 0x3feea3d5},
    {0x543e1a12, 0x3feea427}, {(int)0x8f4abaa9, 0x3feea47b}, {(int)0xadd106d9, 0x3feea4d2},
    {(int)0xb0d1736a, 0x3feea52c}, {(int)0x994cce13, 0x3feea589}, {0x68443d9a, 0x3feea5e9},
    {0x1eb941f7, 0x3feea64c}, {(int)0xbdadb46d, 0x3feea6b1}, {0x4623c7ad, 0x3feea71a},
    {(int)0xb91e07f1, 0x3feea785}, {0x179f5b21, 0x3feea7f4}, {0x62ab00ec, 0x3feea865},
    {(int)0x9b4492ed, 0x3feea8d9}, {(int)0xc27004c2, 0x3feea950}, {(int)0xd931a436, 0x3feea9ca},
    {(int)0xe08e1957, 0x3feeaa47}, {(int)0xd98a6699, 0x3feeaac7}, {(int)0xc52be8f7, 0x3feeab4a},
    {(int)0xa478580f, 0x3feeabd0}, {0x7875c644, 0x3feeac59}, {0x422aa0db, 0x3feeace5},
    {0x029db01e, 0x3feead74}, {(int)0xbad61778, 0x3feeae05}, {0x6bdb5598, 0x3feeae9a},
    {0x16b5448c, 0x3feeaf32}, {(int)0xbc6c19e6, 0x3feeafcc}, {0x5e0866d9, 0x3feeb06a},
    {(int)0xfc931857, 0x3feeb10a}, {(int)0x99157736, 0x3feeb1ae}, {0x3499284b, 0x3feeb255},
    {(int)0xd0282c8a, 0x3feeb2fe}, {0x6ccce12c, 0x3feeb3ab}, {0x0b91ffc6, 0x3feeb45b},
    {(int)0xad829e70, 0x3feeb50d}, {0x53aa2fe2, 0x3feeb5c3}, {(int)0xff148396, 0x3feeb67b},
    {(int)0xb0cdc5e5, 0x3feeb737}, {0x69e2802b, 0x3feeb7f6}, {0x2b5f98e5, 0x3feeb8b8},
    {(int)0xf65253d1, 0x3feeb97c}, {(int)0xcbc8520f, 0x3feeba44}, {(int)0xaccf9243, 0x3feebb0f},
    {(int)0x9a7670b3, 0x3feebbdd}, {(int)0x95cba768, 0x3feebcae}, {(int)0x9fde4e50, 0x3feebd82},
    {(int)0xb9bddb5b, 0x3feebe59}, {(int)0xe47a22a2, 0x3feebf33}, {0x21235681, 0x3feec011},
    {0x70ca07ba, 0x3feec0f1}, {(int)0xd47f2598, 0x3feec1d4}, {0x4d53fe0d, 0x3feec2bb},
    {(int)0xdc5a3dd3, 0x3feec3a4}, {(int)0x82a3f090, 0x3feec491}, {0x414380f2, 0x3feec581},
    {0x194bb8d5, 0x3feec674}, {0x0bcfc15e, 0x3feec76a}, {0x19e32323, 0x3feec863},
    {0x4499c647, 0x3feec95f}, {(int)0x8d07f29e, 0x3feeca5e}, {(int)0xf4424fcb, 0x3feecb60},
    {0x7b5de565, 0x3feecc66}, {0x23701b15, 0x3feecd6f}, {(int)0xed8eb8bb, 0x3feece7a},
    {(int)0xdacfe68c, 0x3feecf89}, {(int)0xec4a2d33, 0x3feed09b}, {0x231475f7, 0x3feed1b1},
    {(int)0x80460ad8, 0x3feed2c9}, {0x04f696b1, 0x3feed3e5}, {(int)0xb23e255d, 0x3feed503},
    {(int)0x893523d4, 0x3feed625}, {(int)0x8af46052, 0x3feed74a}, {(int)0xb8950a73, 0x3feed872},
    {0x1330b358, 0x3feed99e}, {(int)0x9be14dca, 0x3feedacc}, {0x53c12e59, 0x3feedbfe},
    {0x3beb0b7e, 0x3feedd33}, {0x5579fdbf, 0x3feede6b}, {(int)0xa1897fd2, 0x3feedfa6},
    {0x21356eba, 0x3feee0e5}, {(int)0xd59a09ee, 0x3feee226}, {(int)0xbfd3f37a, 0x3feee36b},
    {(int)0xe100301e, 0x3feee4b3}, {0x3a3c2774, 0x3feee5ff}, {(int)0xcca5a413, 0x3feee74d},
    {(int)0x995ad3ad, 0x3feee89f}, {(int)0xa17a4735, 0x3feee9f4}, {(int)0xe622f2ff, 0x3feeeb4c},
    {0x68742ee4, 0x3feeeca8}, {0x298db666, 0x3feeee07}, {0x2a8fa8cd, 0x3feeef69},
    {0x6c9a8952, 0x3feef0ce}, {(int)0xf0cf3f3a, 0x3feef236}, {(int)0xb84f15fb, 0x3feef3a2},
    {(int)0xc43bbd62, 0x3feef511}, {0x15b749b1, 0x3feef684}, {(int)0xade433c6, 0x3feef7f9},
    {(int)0x8de5593a, 0x3feef972}, {(int)0xb6ddfc87, 0x3feefaee}, {0x29f1c52a, 0x3feefc6e},
    {(int)0xe844bfc6, 0x3feefdf0}, {(int)0xf2fb5e47, 0x3feeff76}, {0x4b3a7804, 0x3fef0100},
    {(int)0xf22749e4, 0x3fef028c}, {(int)0xe8e77680, 0x3fef041c}, {0x30a1064a, 0x3fef05b0},
    {(int)0xca7a67a7, 0x3fef0746}, {(int)0xb79a6f1f, 0x3fef08e0}, {(int)0xf9285775, 0x3fef0a7d},
    {(int)0x904bc1d2, 0x3fef0c1e}, {0x7e2cb5e5, 0x3fef0dc2}, {(int)0xc3f3a207, 0x3fef0f69},
    {0x62c95b60, 0x3fef1114}, {0x5bd71e09, 0x3fef12c2}, {(int)0xb0468d30, 0x3fef1473},
    {0x6141b33d, 0x3fef1628}, {0x6ff301f4, 0x3fef17e0}, {(int)0xdd85529c, 0x3fef199b},
    {(int)0xab23e61e, 0x3fef1b5a}, {(int)0xd9fa652c, 0x3fef1d1c}, {0x6b34e065, 0x3fef1ee2},
    {0x5fffd07a, 0x3fef20ab}, {(int)0xb9881650, 0x3fef2277}, {0x78fafb22, 0x3fef2447},
    {(int)0x9f8630ad, 0x3fef261a}, {0x2e57d14b, 0x3fef27f1}, {0x269e601f, 0x3fef29cb},
    {(int)0x8988c933, 0x3fef2ba8}, {0x584661a1, 0x3fef2d89}, {(int)0x9406e7b5, 0x3fef2f6d},
    {0x3dfa8313, 0x3fef3155}, {0x5751c4db, 0x3fef3340}, {(int)0xe13da7cb, 0x3fef352e},
    {(int)0xdcef9069, 0x3fef3720}, {0x4b994d23, 0x3fef3916}, {0x2e6d1675, 0x3fef3b0f},
    {(int)0x869d8f0f, 0x3fef3d0b}, {0x555dc3fa, 0x3fef3f0b}, {(int)0x9be12cb9, 0x3fef410e},
    {0x5b5bab74, 0x3fef4315}, {(int)0x95018d17, 0x3fef451f}, {0x4a07897c, 0x3fef472d},
    {0x7ba2c38c, 0x3fef493e}, {0x2b08c968, 0x3fef4b53}, {0x596f948c, 0x3fef4d6b},
    {0x080d89f2, 0x3fef4f87}, {0x38197a3c, 0x3fef51a6}, {(int)0xeacaa1d6, 0x3fef53c8},
    {0x2158a91f, 0x3fef55ef}, {(int)0xdcfba487, 0x3fef5818}, {0x1eec14be, 0x3fef5a46},
    {(int)0xe862e6d3, 0x3fef5c76}, {0x3a99745b, 0x3fef5eab}, {0x16c98398, 0x3fef60e3},
    {0x7e2d479d, 0x3fef631e}, {0x71ff6075, 0x3fef655d}, {(int)0xf37adb4a, 0x3fef679f},
    {0x03db3285, 0x3fef69e6}, {(int)0xa45c4dfd, 0x3fef6c2f}, {(int)0xd63a8315, 0x3fef6e7c},
    {(int)0x9ab294e4, 0x3fef70cd}, {(int)0xf301b460, 0x3fef7321}, {(int)0xe065807d, 0x3fef7579},
    {0x641c0658, 0x3fef77d5}, {0x7f63c159, 0x3fef7a34}, {0x337b9b5f, 0x3fef7c97},
    {(int)0x81a2ece1, 0x3fef7efd}, {0x6b197d17, 0x3fef8167}, {(int)0xf11f8220, 0x3fef83d4},
    {0x14f5a129, 0x3fef8646}, {(int)0xd7dcee90, 0x3fef88ba}, {0x3b16ee12, 0x3fef8b33},
    {0x3fe592e8, 0x3fef8daf}, {(int)0xe78b3ff6, 0x3fef902e}, {0x334ac7ee, 0x3fef92b2},
    {0x24676d76, 0x3fef9539}, {(int)0xbc24e350, 0x3fef97c3}, {(int)0xfbc74c83, 0x3fef9a51},
    {(int)0xe4933c7e, 0x3fef9ce3}, {0x77cdb740, 0x3fef9f79}, {(int)0xb6bc3181, 0x3fefa212},
    {(int)0xa2a490da, 0x3fefa4af}, {0x3ccd2be5, 0x3fefa750}, {(int)0x867cca6e, 0x3fefa9f4},
    {(int)0x80faa594, 0x3fefac9c}, {0x2d8e67f1, 0x3fefaf48}, {(int)0x8d802dc2, 0x3fefb1f7},
    {(int)0xa2188510, 0x3fefb4aa}, {0x6ca06dd6, 0x3fefb761}, {(int)0xee615a27, 0x3fefba1b},
    {0x28a52e59, 0x3fefbcda}, {0x1cb6412a, 0x3fefbf9c}, {(int)0xcbdf5be7, 0x3fefc261},
    {0x376bba97, 0x3fefc52b}, {0x60a70c22, 0x3fefc7f8}, {0x48dd7274, 0x3fefcac9},
    {(int)0xf15b82ac, 0x3fefcd9d}, {0x5b6e4540, 0x3fefd076}, {(int)0x88633625, 0x3fefd352},
    {0x798844f8, 0x3fefd632}, {0x302bd526, 0x3fefd916}, {(int)0xad9cbe14, 0x3fefdbfd},
    {(int)0xf32a4b45, 0x3fefdee8}, {0x02243c89, 0x3fefe1d8}, {(int)0xdbdac61d, 0x3fefe4ca},
    {(int)0x819e90d8, 0x3fefe7c1}, {(int)0xf4c0ba54, 0x3fefeabb}, {0x3692d514, 0x3fefedba},
    {0x4866e8ad, 0x3feff0bc}, {0x2b8f71f1, 0x3feff3c2}, {(int)0xe15f6314, 0x3feff6cb},
    {0x6b2a23d9, 0x3feff9d9}, {(int)0xca4391b6, 0x3feffcea}};
__device__ __constant__ double kPoly64[5] = {0x1.0000000000000p+0, 0x1.62e42fefa0352p-1,
                                             0x1.ebfbdff82ac52p-3, 0x1.c6b0c40d8c4e9p-5,
                                             0x1.3b2ad0385b409p-7};
__device__ __constant__ double kPoly512[4] = {0x1.ffffffffffff6p-1, 0x1.62e42fefa39eep-1,
                                              0x1.ebfbe13357103p-3, 0x1.c6b08e1f0e0b5p-5};

struct ExpTab64 {
  static constexpr double kMagic = 0x1.8p46;
  static constexpr int kTab = 64;
  static constexpr int kUnit = 1 << 14;   // n * kUnit = (n >> 6) << 20 + (n & 63) << 14
  static constexpr int kNMin = -65280;    // clamp of n: s >= -1020
  static constexpr int kNMax = 64000;     //             s <=  1000
  static constexpr int kZeroN = -65472;   // 64 * (-1023): scale word pattern +0.0
  __device__ static __forceinline__ const int2* table() { return kExp2Table64; }
  __device__ static __forceinline__ double poly(double r) {
    double p = fma(kPoly64[4], r, kPoly64[3]);
    p = fma(p, r, kPoly64[2]);
    p = fma(p, r, kPoly64[1]);
    return fma(p, r, kPoly64[0]);
  }
};

struct ExpTab512 {
  static constexpr double kMagic = 0x1.8p43;
  static constexpr int kTab = 512;
  static constexpr int kUnit = 1 << 11;   // n * kUnit = (n >> 9) << 20 + (n & 511) << 11
  static constexpr int kNMin = -522240;   // clamp of n: s >= -1020
  static constexpr int kNMax = 512000;    //             s <=  1000
  static constexpr int kZeroN = -523776;  // 512 * (-1023): scale word pattern +0.0
  __device__ static __forceinline__ const int2* table() { return kExp2Table512; }
  __device__ static __forceinline__ double poly(double r) {
    double p = fma(kPoly512[3], r, kPoly512[2]);
    p = fma(p, r, kPoly512[1]);
    return fma(p, r, kPoly512[0]);
  }
};

// Copies the exp2 table into shared memory.
template <class E = ExpTab64>
__device__ __forceinline__ void load_exp2_table(int2* smem_tbl) {
  for (int i = threadIdx.x; i < E::kTab; i += blockDim.x) smem_tbl[i] = E::table()[i];
}

// acc + 2^s.  Exact split s = n/T + r (|r| <= 1/(2T)) by the magic-constant
// addition, 2^r by the polynomial, 2^(n/T) by table + exponent add.  n is
// clamped to [T (-1020), T * 1000]: s below -1020 contributes at most 2^-1019
// (the reference would add a subnormal or zero); s above 1000 yields at least
// 2^999, which the callers detect (sum > 2^960) and route to the exact
// per-atom path.  FP64 pipe: 3 DADD + 5 (ExpTab64) or 4 (ExpTab512) DFMA;
// INT: 2 IMNMX, LOP3, LEA, IMAD.
template <bool CLAMP = true, class E = ExpTab64>
__device__ __forceinline__ double exp2_acc(double s, double acc,
                                           const int2* __restrict__ tbl) {
  const double kk = __dadd_rn(s, E::kMagic);
  int n = __double2loint(kk);  // round(T s)
  if (CLAMP) n = min(max(n, E::kNMin), E::kNMax);
  const double kd = __dadd_rn(kk, -E::kMagic);
  const double r = __dadd_rn(s, -kd);        // |r| <= 1/(2T)
  const double p = E::poly(r);
  const int2 t = tbl[n & (E::kTab - 1)];
  const double scale = __hiloint2double(t.y + n * E::kUnit, t.x);
  return fma(p, scale, acc);
}

// acc + (take ? 2^s : 0) without a branch.  Lanes that do not take the
// pair get n = E::kZeroN = T * (-1023), whose scale word pattern is exactly
// +0.0 (one SEL on the INT pipe).  CLAMP = false is used when the caller has
// proven every taken s lies in [-1020, 1000].
template <bool CLAMP = true, class E = ExpTab64>
__device__ __forceinline__ double exp2_acc_masked(double s, double acc,
                                                  const int2* __restrict__ tbl, bool take) {
  const double kk = __dadd_rn(s, E::kMagic);
  int n = __double2loint(kk);
  if (CLAMP) n = min(max(n, E::kNMin), E::kNMax);
  const double kd = __dadd_rn(kk, -E::kMagic);
  const double r = __dadd_rn(s, -kd);
  const double p = E::poly(r);
  n = take ? n : E::kZeroN;
#ifdef RSOT_EXP_NOTABLE
  const int2 t = make_int2(0, 0x3ff00000 - (n & (E::kTab - 1)) * E::kUnit);
#else
  const int2 t = tbl[n & (E::kTab - 1)];
#endif
  return fma(p, __hiloint2double(t.y + n * E::kUnit, t.x), acc);
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
// Set when a contribution cannot be represented in the accumulator (a single
// term >= 2^41, i.e. masses far from normalised); the C ABI turns it into
// RSOT_CUDA_RUNTIME_ERROR instead of returning a silently wrong gradient.
static __device__ unsigned int g_fp_overflow = 0;

// Limb words past the top limb fold into it (limb 4 is a u64 with 32 bits of
// headroom: a part of value v at limb 4 + k adds v << 32 k).
__device__ __forceinline__ void fp_red_top(unsigned long long* acc, int limb, unsigned long long v) {
  const int k = limb - (kLimbs - 1);
  if (k >= 2 || (k == 1 && (v >> 31))) {
    atomicOr(&g_fp_overflow, 1u);
    return;
  }
  atomicAdd(acc + kLimbs - 1, v << (32 * k));
}

__device__ __forceinline__ void fp_red(unsigned long long* acc, double m) {
  if (!(m > 0.0)) return;
  // m = mant * 2^(e - 53), mant the 53-bit significand (frexp / ldexp done on
  // the bits; subnormals lie far below the last limb)
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(m));
  const int ef = static_cast<int>(bits >> 52);
  if (ef == 0) return;
  unsigned long long mant = (bits & 0x000fffffffffffffull) | 0x0010000000000000ull;
  const int e = ef - 1022;
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
  if (i0 + 2 < kLimbs) {  // (every in-range contribution: m < 2^10)
    if (l0) atomicAdd(acc + i0, l0);
    if (l1) atomicAdd(acc + i0 + 1, l1);
    if (l2) atomicAdd(acc + i0 + 2, l2);
  } else {
    if (l0) (i0 < kLimbs ? atomicAdd(acc + i0, l0) : (fp_red_top(acc, i0, l0), 0ull));
    if (l1) (i0 + 1 < kLimbs ? atomicAdd(acc + i0 + 1, l1) : (fp_red_top(acc, i0 + 1, l1), 0ull));
    if (l2) fp_red_top(acc, i0 + 2, l2);
  }
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
