"""Generates the exp2 table and polynomial of device_math.cuh (development
aid): 2^(i/T) correctly rounded, stored pre-biased as {lo, hi - i*2^(20-b)}
(T = 2^b), and a near-minimax degree-d fit of 2^r on [-1/(2T), 1/(2T)]
(mpmath chebyfit, coefficients rounded to double), with its worst relative
error measured in 200-bit arithmetic."""
import struct
import sys

import mpmath as mp

mp.mp.prec = 200
b = int(sys.argv[1]) if len(sys.argv) > 1 else 6
deg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
T = 1 << b
rows = []
for i in range(T):
    v = float(mp.mpf(2) ** (mp.mpf(i) / T))  # correctly rounded (200-bit -> nearest double)
    bits = struct.unpack("<Q", struct.pack("<d", v))[0]
    lo, hi = bits & 0xFFFFFFFF, bits >> 32
    hi -= i << (20 - b)
    rows.append((lo, hi))
h = mp.mpf(1) / (2 * T)
poly, err = mp.chebyfit(lambda r: mp.mpf(2) ** r, [-h, h], deg + 1, error=True)
coef = [float(c) for c in reversed(poly)]  # c0 .. cdeg
worst = mp.mpf(0)
for k in range(4001):
    r = -h + 2 * h * k / 4000
    p = mp.mpf(0)
    for c in reversed(coef):
        p = p * r + mp.mpf(c)
    worst = max(worst, abs(p / mp.mpf(2) ** r - 1))
print(f"// 2^(i/{T}), {{lo, hi - (i << {20 - b})}}")
line = []
for lo, hi in rows:
    los = f"0x{lo:08x}" if lo < 0x80000000 else f"(int)0x{lo:08x}"
    line.append(f"{{{los}, 0x{hi:08x}}}")
for k in range(0, T, 3):
    print("    " + ", ".join(line[k:k + 3]) + ",")
print("// degree", deg, "coefficients c0..c%d:" % deg, ", ".join(c.hex() for c in coef))
print("// worst relative error", mp.nstr(worst, 4))
