// truncated.cu -- truncated dual objective + gradient over a GPU cell list.
//
// Reference semantics (proj/src/evaluate.cpp:86-174 with a finite cutoff):
//   candidates(q) = {j : ((dx*dx + dy*dy) + dz*dz) < r*r}, r = sqrt(2 C)
//                   (spatial_index.cpp:47-61, cost.hpp:38-42),
//   empty set    -> {nearest target, lowest index on ties} (:129-132),
//   candidate_pairs counts the fallback as 1, empty_candidate_atoms counts it.
//
// Pipeline per evaluation (grid rebuilt only when r leaves its band):
//   gather b2 into sorted target order
//   pass A  (CTA = 128 sorted atoms): scan the x-rows of target cells that
//           can reach the CTA's bounding box, staged through shared memory;
//           per pair an FP32 pre-test on local coordinates decides clear
//           in/out, pairs inside the error band get the exact fp64 reference
//           predicate; accepted pairs accumulate 2^(e2 - B + c2|x'|^2).
//   nearest (warp per empty atom): exact lexicographic (d^2, j) argmin by
//           expanding cell rings; J/D from the single-term LSE; the gradient
//           contribution m_q is added to a 192-bit fixed-point accumulator
//           per target, so the result is order independent (deterministic).
//   pass B  (CTA = 128 sorted targets): same scan over atom cells; gather of
//           2^(e2_qj - log2 S_q + log2 m_q) into the thread's own target.
//   assemble: res[j] = G[j] + empty[j]; fixed-order sums of J, D, counts.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "block_util.cuh"
#include "device_math.cuh"
#include "geodesic.cuh"
#include "truncated.cuh"

namespace rsot_cuda {

namespace {

constexpr int kT = 128;        // threads per CTA = points per chunk
constexpr int kTileT = 256;    // staged points per tile (fp64 kernel)
constexpr int kTileT32 = 384;  // staged points per tile (fp32 kernel)
#ifndef RSOT_FULLIN_RATIO2
#define RSOT_FULLIN_RATIO2 16.0f  // full-in split when r > 4 warp-box half-diagonals
#endif
#ifndef RSOT_P2_TM
#define RSOT_P2_TM 1  // target-major phase 2 over per-warp item records (unsplit non-safe CTAs)
#endif
#ifndef RSOT_P1_LEAN
#define RSOT_P1_LEAN 1
#endif
using ListT = unsigned short;  // per-warp culled-list entry (tile index)
constexpr int kMortonBits = 7; // per dim, position inside a cell
double g_cells_per_radius = 5.0;  // grid cell side ~ r / 5 (env RSOT_CELLS_PER_RADIUS; swept 2-8: r/5-r/6 best
                                  // for cfg3/cfg5 in both precisions since the phase-2 mask replay)

struct GridDev {
  double lo[3];
  double h, inv_h;
  int dims[3];
};

GridDev to_dev(const GridDesc& g) {
  GridDev d;
  for (int i = 0; i < 3; ++i) {
    d.lo[i] = g.lo[i];
    d.dims[i] = g.dims[i];
  }
  d.h = g.h;
  d.inv_h = 1.0 / g.h;
  return d;
}

__device__ __forceinline__ int cell_of(const GridDev& g, int d, double v) {
  const double t = floor((v - g.lo[d]) * g.inv_h);
  if (!(t >= 0.0)) return 0;
  if (t >= static_cast<double>(g.dims[d] - 1)) return g.dims[d] - 1;
  return static_cast<int>(t);
}

// Distance from the interval [a, b] to the slab of cell c in dim d; edge
// cells extend to infinity (points outside the grid are clamped into them).
__device__ __forceinline__ double slab_dist(const GridDev& g, int d, int c,
                                            double a, double b) {
  const double pad = 1e-7 * g.h;
  const double s0 = (c == 0) ? -INFINITY : g.lo[d] + c * g.h - pad;
  const double s1 = (c == g.dims[d] - 1) ? INFINITY : g.lo[d] + (c + 1) * g.h + pad;
  return fmax(0.0, fmax(s0 - b, a - s1));
}

__device__ __forceinline__ uint32_t spread3(uint32_t v) {
  // 7 bits -> every third bit
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < kMortonBits; ++i) r |= ((v >> i) & 1u) << (3 * i);
  return r;
}

__global__ void cell_keys_kernel(const double4* __restrict__ pts, int n,
                                 GridDev g, uint64_t* __restrict__ keys,
                                 int* __restrict__ idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = pts[i];
  const double v[3] = {p.x, p.y, p.z};
  int c[3];
  uint32_t m[3];
  for (int d = 0; d < 3; ++d) {
    c[d] = cell_of(g, d, v[d]);
    double f = (v[d] - g.lo[d]) * g.inv_h - c[d];
    f = fmin(fmax(f, 0.0), 0.999999);
    m[d] = static_cast<uint32_t>(f * (1 << kMortonBits));
  }
  const uint64_t cell = (static_cast<uint64_t>(c[2]) * g.dims[1] + c[1]) * g.dims[0] + c[0];
  const uint32_t mort = spread3(m[0]) | (spread3(m[1]) << 1) | (spread3(m[2]) << 2);
  keys[i] = (cell << (3 * kMortonBits)) | mort;
  idx[i] = i;
}

// Hilbert index (Skilling's transpose algorithm, 3 dims x kHilBits bits) of
// each point quantised over the set's bounding box.
constexpr int kHilBits = 16;

__global__ void hilbert_keys_kernel(const double4* __restrict__ pts, int n, double lo0,
                                    double lo1, double lo2, double s0, double s1, double s2,
                                    uint64_t* __restrict__ keys, int* __restrict__ idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = pts[i];
  const double v[3] = {(p.x - lo0) * s0, (p.y - lo1) * s1, (p.z - lo2) * s2};
  uint32_t X[3];
  const double top = static_cast<double>((1u << kHilBits) - 1);
#pragma unroll
  for (int d = 0; d < 3; ++d) X[d] = static_cast<uint32_t>(fmin(fmax(v[d], 0.0), top));
  const uint32_t M = 1u << (kHilBits - 1);
  for (uint32_t Q = M; Q > 1; Q >>= 1) {
    const uint32_t P = Q - 1;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (X[d] & Q) {
        X[0] ^= P;
      } else {
        const uint32_t t = (X[0] ^ X[d]) & P;
        X[0] ^= t;
        X[d] ^= t;
      }
    }
  }
  X[1] ^= X[0];
  X[2] ^= X[1];
  uint32_t t = 0;
  for (uint32_t Q = M; Q > 1; Q >>= 1)
    if (X[2] & Q) t ^= Q - 1;
  X[0] ^= t;
  X[1] ^= t;
  X[2] ^= t;
  uint64_t key = 0;
  for (int b = kHilBits - 1; b >= 0; --b)
    key = (key << 3) | (((X[0] >> b) & 1u) << 2) | (((X[1] >> b) & 1u) << 1) | ((X[2] >> b) & 1u);
  keys[i] = key;
  idx[i] = i;
}

__global__ void gather_d_kernel(const double* __restrict__ src, const int* __restrict__ idx,
                                int n, double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void gather4_kernel(const double4* __restrict__ src,
                               const int* __restrict__ perm, int n,
                               double4* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

__global__ void cell_start_kernel(const uint64_t* __restrict__ keys, int n,
                                  long long ncells, int* __restrict__ start) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > n) return;
  const long long prev = (k == 0) ? -1 : static_cast<long long>(keys[k - 1] >> (3 * kMortonBits));
  const long long cur = (k == n) ? ncells : static_cast<long long>(keys[k] >> (3 * kMortonBits));
  for (long long c = prev + 1; c <= cur; ++c) start[c] = k;
}


// Scan-region setup shared by both passes: chunk bbox, origin, FP32 band.
struct Region {
  double box[6];
  double o[3];
  float lo_thr, hi_thr;
  int c_lo[3], c_hi[3];
  bool wide;
  float xy_max;  // >= |2 c2 x'.y'| of any taken pair (|x'| <= hd, |y'| <= hd + r)
  float wy_max;  // >= c2 |y'|^2 of any taken pair's target
};

__device__ void setup_region(const GridDev& g, const double lo[3], const double hi[3],
                             double r2, double r_scan, double c2, double* sh, Region& R) {
  block_bbox<kT>(lo, hi, sh, R.box);
  double hd2 = 0.0;
  for (int d = 0; d < 3; ++d) {
    R.o[d] = 0.5 * (R.box[d] + R.box[d + 3]);
    const double e = 0.5 * (R.box[d + 3] - R.box[d]);
    hd2 += e * e;
  }
  // Bound on |x'|, |y'| for pairs near the decision boundary, and the FP32
  // error band (9x the worst-case rounding of the FP32 distance).
  R.wide = c2 * hd2 > 400.0;
  const double r = sqrt(r2);
  {
    const double hd = sqrt(hd2), yb = hd + r;
    R.xy_max = __double2float_ru(2.0 * c2 * hd * yb * (1.0 + 1e-6));
    R.wy_max = __double2float_ru(c2 * yb * yb * (1.0 + 1e-6));
  }
  const double Rb = sqrt(hd2) + r_scan + 1.75 * g.h;
  const double band = 0x1p-21 * (8.0 * r * Rb + 4.0 * r2);
  R.lo_thr = __double2float_rd(r2 - band);
  R.hi_thr = __double2float_ru(r2 + band);
  if (!(r2 - band > 1e-30)) R.lo_thr = -1.0f;  // tiny radius: always exact
  for (int d = 0; d < 3; ++d) {
    R.c_lo[d] = cell_of(g, d, R.box[d] - r_scan);
    R.c_hi[d] = cell_of(g, d, R.box[d + 3] + r_scan);
  }
}

// Computes one candidate row (index ri over the (cy, cz) rectangle) and
// returns its [start, start+len) range in the sorted order of `cell_start`.
__device__ __forceinline__ void row_range(const GridDev& g, const Region& R,
                                          double r_scan, const int* __restrict__ cell_start,
                                          int ri, int& start, int& len) {
  start = 0;
  len = 0;
  const int ny = R.c_hi[1] - R.c_lo[1] + 1;
  const int cy = R.c_lo[1] + ri % ny;
  const int cz = R.c_lo[2] + ri / ny;
  const double dy = slab_dist(g, 1, cy, R.box[1], R.box[4]);
  const double dz = slab_dist(g, 2, cz, R.box[2], R.box[5]);
  const double rem = r_scan * r_scan - dy * dy - dz * dz;
  if (rem < 0.0) return;
  const double rx = sqrt(rem);
  const int x0 = cell_of(g, 0, R.box[0] - rx);
  const int x1 = cell_of(g, 0, R.box[3] + rx);
  const long long row = (static_cast<long long>(cz) * g.dims[1] + cy) * g.dims[0];
  start = cell_start[row + x0];
  len = cell_start[row + x1 + 1] - start;
}

__device__ __forceinline__ int find_row(const int* pref, int s) {
  // largest r in [0, kT) with pref[r] <= s
  int lo = 0, hi = kT;  // pref[kT] = total > s
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pref[mid] <= s) lo = mid; else hi = mid;
  }
  return lo;
}

// Row of batch position s when 8 consecutive threads hold 8 consecutive
// positions (a kGroup of the tile map, or a run of a contiguous tile): the
// group's first thread runs the binary search, the others step forward from
// its row (one search per 8 entries; ncu: the per-entry searches were 3 % of
// the fused kernel's warp samples).  All 32 lanes must call it.
__device__ __forceinline__ int find_row_group(const int* pref, int s, bool valid) {
  const int lane = threadIdx.x & 31;
  int r = 0;
  if ((lane & 7) == 0 && valid) r = find_row(pref, s);
  r = __shfl_sync(0xffffffffu, r, lane & ~7);
  if (valid)
    while (pref[r + 1] <= s) ++r;
  return r;
}

// Interleaved tiles (load balance between the CTA's warps): a row batch's
// `total` positions form ng = ceil(total / kGroup) groups of kGroup
// consecutive (cell-ordered, hence close) targets, and tile k holds groups
// k, k + ntile, k + 2 ntile, ...  Every tile then samples the whole scanned
// region, so each warp's culled share of a tile tracks its share of the
// batch; contiguous tiles (a few cell rows each) loaded the warps whose box
// is nearest those rows and left the others waiting at the tile barrier
// (ncu: 15 % of the cfg5 warp samples at the two per-tile barriers).
// Groups keep the staging loads coalesced (8 x 32 B of target records).
// Measured: fp64 cfg5 -2 %, cfg3 unchanged; the fp32 kernel keeps contiguous
// tiles (interleaving is neutral there: +-0.3 %).
constexpr int kGroup = 8;
struct TileMap {
  int total, tile, ng, ntile;
  bool inter;  // interleaved groups (fp64 kernel) or contiguous tiles (fp32 kernel)
};
__device__ __forceinline__ TileMap tile_map(int total, int tile, bool inter) {
  TileMap m;
  m.total = total;
  m.tile = tile;
  m.inter = inter;
  m.ng = (total + kGroup - 1) / kGroup;
  const int gpt = tile / kGroup;
  m.ntile = inter ? (m.ng + gpt - 1) / gpt : (total + tile - 1) / tile;
  return m;
}
// Positions in tile k (< ntile); at most `tile`.
__device__ __forceinline__ int tile_count(const TileMap& m, int k) {
  if (!m.inter) return min(m.tile, m.total - k * m.tile);
  const int nu = (m.ng - k + m.ntile - 1) / m.ntile;
  const int last = k + (nu - 1) * m.ntile;
  return (nu - 1) * kGroup + min(kGroup, m.total - last * kGroup);
}
// Batch position of entry t of tile k.
__device__ __forceinline__ int tile_pos(const TileMap& m, int k, int t) {
  if (!m.inter) return k * m.tile + t;
  return (k + (t / kGroup) * m.ntile) * kGroup + (t % kGroup);
}

// Warp bounding box (local fp32 coordinates) of the warp's own points.
struct WarpBox {
  float lo0, lo1, lo2, hi0, hi1, hi2;
};

__device__ __forceinline__ WarpBox warp_box(bool valid, float a, float b, float c) {
  WarpBox w;
  w.lo0 = valid ? a : INFINITY; w.hi0 = valid ? a : -INFINITY;
  w.lo1 = valid ? b : INFINITY; w.hi1 = valid ? b : -INFINITY;
  w.lo2 = valid ? c : INFINITY; w.hi2 = valid ? c : -INFINITY;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    w.lo0 = fminf(w.lo0, __shfl_xor_sync(0xffffffffu, w.lo0, o));
    w.lo1 = fminf(w.lo1, __shfl_xor_sync(0xffffffffu, w.lo1, o));
    w.lo2 = fminf(w.lo2, __shfl_xor_sync(0xffffffffu, w.lo2, o));
    w.hi0 = fmaxf(w.hi0, __shfl_xor_sync(0xffffffffu, w.hi0, o));
    w.hi1 = fmaxf(w.hi1, __shfl_xor_sync(0xffffffffu, w.hi1, o));
    w.hi2 = fmaxf(w.hi2, __shfl_xor_sync(0xffffffffu, w.hi2, o));
  }
  return w;
}


// Warp-cooperative exact nearest target (lexicographic (d^2, j) argmin) by
// expanding Chebyshev rings of cells.  A ring is a set of cell rows; the
// cells of a row are contiguous in the cell-sorted targets, so each row (or
// the two end cells of an inner row) is one target range.  Lanes fetch the
// ranges of 32 rows at once and drop rows whose box lies farther than the
// best distance so far; the surviving ranges are then scanned by the whole
// warp, lanes over targets.  The search stops once the scanned box provably
// contains the minimum.
__device__ __forceinline__ double range_lb2(const GridDev& g, const double* v, int cy, int cz,
                                            int a0, int a1) {
  const double dx = slab_dist(g, 0, a0, v[0], v[0]);
  const double dx1 = slab_dist(g, 0, a1, v[0], v[0]);
  const double ddx = (a0 <= cell_of(g, 0, v[0]) && cell_of(g, 0, v[0]) <= a1) ? 0.0 : fmin(dx, dx1);
  const double dy = slab_dist(g, 1, cy, v[1], v[1]);
  const double dz = slab_dist(g, 2, cz, v[2], v[2]);
  return fma(ddx, ddx, fma(dy, dy, dz * dz));
}

__device__ __forceinline__ void scan_range(int b, int e, double x0, double x1, double x2,
                                           const double4* __restrict__ ys,
                                           const int* __restrict__ tperm, double& bd, int& bj,
                                           int& bk) {
  const int lane = threadIdx.x & 31;
  unsigned m = __ballot_sync(0xffffffffu, e > b);
  while (m) {
    const int l = __ffs(m) - 1;
    m &= m - 1;
    const int rb = __shfl_sync(0xffffffffu, b, l), re = __shfl_sync(0xffffffffu, e, l);
    for (int t = rb + lane; t < re; t += 32) {
      const double4 y = ys[t];
      const double d2 = exact_sqdist(x0, x1, x2, y.x, y.y, y.z);
      const int j = tperm[t];
      if (d2 < bd || (d2 == bd && j < bj)) { bd = d2; bj = j; bk = t; }
    }
  }
}

__device__ void warp_nearest(const GridDev& g, const double4* __restrict__ ys,
                             const int* __restrict__ tperm,
                             const int* __restrict__ cell_start, double x0,
                             double x1, double x2, double& best_d2, int& best_j,
                             int& best_k) {
  const int lane = threadIdx.x & 31;
  const double v[3] = {x0, x1, x2};
  int cc[3];
  for (int d = 0; d < 3; ++d) cc[d] = cell_of(g, d, v[d]);
  double bd = INFINITY;
  int bj = 0x7fffffff, bk = -1;
  const int maxk = g.dims[0] + g.dims[1] + g.dims[2];
  for (int k = 0; k <= maxk; ++k) {
    const int zlo = max(0, cc[2] - k), zhi = min(g.dims[2] - 1, cc[2] + k);
    const int ylo = max(0, cc[1] - k), yhi = min(g.dims[1] - 1, cc[1] + k);
    const int xlo = max(0, cc[0] - k), xhi = min(g.dims[0] - 1, cc[0] + k);
    const int ny = yhi - ylo + 1;
    const int nrows = ny * (zhi - zlo + 1);
    // rows whose box is beyond the warp's best so far cannot improve it
    const double prune = bd * (1.0 + 1e-9);
    for (int r0 = 0; r0 < nrows; r0 += 32) {
      const int ri = r0 + lane;
      int b0 = 0, e0 = 0, b1 = 0, e1 = 0;
      if (ri < nrows) {
        const int cy = ylo + ri % ny, cz = zlo + ri / ny;
        const bool full = (abs(cz - cc[2]) == k) || (abs(cy - cc[1]) == k);
        const long long row = (static_cast<long long>(cz) * g.dims[1] + cy) * g.dims[0];
        if (full) {
          if (!(range_lb2(g, v, cy, cz, xlo, xhi) > prune)) {
            b0 = cell_start[row + xlo];
            e0 = cell_start[row + xhi + 1];
          }
        } else {
          const int a = cc[0] - k, c = cc[0] + k;
          if (a >= 0 && !(range_lb2(g, v, cy, cz, a, a) > prune)) {
            b0 = cell_start[row + a];
            e0 = cell_start[row + a + 1];
          }
          if (c <= g.dims[0] - 1 && !(range_lb2(g, v, cy, cz, c, c) > prune)) {
            b1 = cell_start[row + c];
            e1 = cell_start[row + c + 1];
          }
        }
      }
      scan_range(b0, e0, x0, x1, x2, ys, tperm, bd, bj, bk);
      scan_range(b1, e1, x0, x1, x2, ys, tperm, bd, bj, bk);
    }
    // warp lexicographic min
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
      if (od < bd || (od == bd && oj < bj)) { bd = od; bj = oj; bk = ok; }
    }
    double margin = INFINITY;
    bool left = false;
    for (int d = 0; d < 3; ++d) {
      if (cc[d] - k > 0) {
        margin = fmin(margin, v[d] - (g.lo[d] + (cc[d] - k) * g.h));
        left = true;
      }
      if (cc[d] + k < g.dims[d] - 1) {
        margin = fmin(margin, (g.lo[d] + (cc[d] + k + 1) * g.h) - v[d]);
        left = true;
      }
    }
    if (!left) break;
    margin = margin * (1.0 - 1e-9) - 1e-7 * g.h;
    if (bk >= 0 && margin > 0.0 && margin * margin > bd * (1.0 + 1e-9)) break;
  }
  best_d2 = bd;
  best_j = bj;
  best_k = bk;
}

// Nearest target given a candidate (cell-order position seed_k, e.g. a
// neighbouring query's answer): every target that beats it, (d2, j)
// lexicographically, lies in the ball through the seed, so one sweep of the
// cell rows meeting that ball (row_range, as the candidate scan) finds the
// minimum -- O(K^2) row visits instead of the rings' O(K^3).  Balls wider than
// kSeedRows rows fall back to the ring search.
constexpr int kSeedRows = 512;

__device__ void warp_nearest_seeded(const GridDev& g, const double4* __restrict__ ys,
                                    const int* __restrict__ tperm, const int* __restrict__ cell_start,
                                    double x0, double x1, double x2, int seed_k, double& best_d2,
                                    int& best_j, int& best_k) {
  const double4 ys0 = ys[seed_k];
  double bd = exact_sqdist(x0, x1, x2, ys0.x, ys0.y, ys0.z);
  int bj = tperm[seed_k], bk = seed_k;
  const double rad = sqrt(bd) * (1.0 + 1e-9) + 1e-300;
  Region R;
  R.box[0] = R.box[3] = x0;
  R.box[1] = R.box[4] = x1;
  R.box[2] = R.box[5] = x2;
  for (int d = 0; d < 3; ++d) {
    R.c_lo[d] = cell_of(g, d, R.box[d] - rad);
    R.c_hi[d] = cell_of(g, d, R.box[d + 3] + rad);
  }
  const int nrows = (R.c_hi[1] - R.c_lo[1] + 1) * (R.c_hi[2] - R.c_lo[2] + 1);
  if (nrows > kSeedRows) {
    warp_nearest(g, ys, tperm, cell_start, x0, x1, x2, best_d2, best_j, best_k);
    return;
  }
  const int lane = threadIdx.x & 31;
  for (int r0 = 0; r0 < nrows; r0 += 32) {
    int st = 0, ln = 0;
    if (r0 + lane < nrows) row_range(g, R, rad, cell_start, r0 + lane, st, ln);
    scan_range(st, st + ln, x0, x1, x2, ys, tperm, bd, bj, bk);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
    const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
    const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
    if (od < bd || (od == bd && oj < bj)) { bd = od; bj = oj; bk = ok; }
  }
  best_d2 = bd;
  best_j = bj;
  best_k = bk;
}

template <bool DEBUG>
__global__ void trunc_nearest_empty(const double4* __restrict__ xs, int nq,
                                    const uint32_t* __restrict__ cnt,
                                    const double4* __restrict__ ys,
                                    const int* __restrict__ tperm,
                                    const int* __restrict__ cell_start, GridDev g,
                                    const double* __restrict__ psi, double eps,
                                    double* __restrict__ atomL,
                                    double* __restrict__ atomJ,
                                    double* __restrict__ atomD,
                                    unsigned long long* __restrict__ empty_fp,
                                    uint64_t* __restrict__ hash_out, const int* __restrict__ range) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int lo = range ? range[0] : 0, hi = range ? range[1] : nq;  // this rank's atoms
  for (int base = (lo & ~31) + warp * 32; base < hi; base += nwarps * 32) {
    const int q = base + lane;
    const bool empty = q >= lo && q < hi && cnt[q] == 0;
    unsigned mask = __ballot_sync(0xffffffffu, empty);
    int seed = -1;  // empty atoms of a Hilbert group are neighbours: seed each with the last answer
    while (mask) {
      const int l = __ffs(mask) - 1;
      mask &= mask - 1;
      const int qq = base + l;
      const double4 a = xs[qq];
      double bd;
      int bj, bk;
      if (seed >= 0)
        warp_nearest_seeded(g, ys, tperm, cell_start, a.x, a.y, a.z, seed, bd, bj, bk);
      else
        warp_nearest(g, ys, tperm, cell_start, a.x, a.y, a.z, bd, bj, bk);
      seed = bk;
      if (lane == 0) {
        const double L = reference_exponent(psi[bj], bd, eps, ys[bk].w);
        atomL[qq] = L;
        atomJ[qq] = eps * L * a.w;
        atomD[qq] = a.w * exp(-L);
        fp_red(empty_fp + kLimbs * static_cast<size_t>(bk), a.w);
        if (DEBUG) hash_out[qq] = candidate_hash_term(static_cast<uint64_t>(bj));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Fused truncated evaluation: one atom-major kernel does both passes.
//
// CTA = 256 Hilbert-consecutive atoms, 2 per thread (a = lane, b = lane+32
// of the warp's 64-atom slice).  Phase 1 scans the target cell rows within
// reach (staged tiles, per-warp culling, packed FP32x2 pre-test for both
// atoms, exact fp64 band test) and accumulates S~_q.  Between the phases the
// CTA finalises its atoms (J_q, D_q, counters), resolves empty candidate
// sets (warp-cooperative exact nearest) and recomputes atoms whose shifted
// sum left [2^-960, 2^960] with the reference's per-atom max shift.  Phase 2
// rescans the same tiles, recomputes the same exponentials with the
// polynomial coefficients pre-scaled by w_q = m_q / S~_q (no extra FP64
// work), sums each target's column over the warp's 64 atoms with a
// transposed shuffle butterfly (16 targets per batch), over the 4 warps in
// fixed order, and adds the CTA's partial into a 192-bit fixed-point
// accumulator per target (order independent => deterministic).

constexpr int kFA = 2 * kT;  // atoms per CTA
// Mask slots: a resident CTA holds one (at most 4 x 148 are resident), kMaskWords
// words per thread (+1 scratch word); CTAs that need more recompute the masks
// in phase 2; slot kMaskSlots is the shared scratch of CTAs without a slot.
constexpr int kMaskSlots = 1024;
constexpr int kMaskWords = 2048;
constexpr int kSlotsPerSm = 4;
constexpr int kRecCap = 131072;  // item indices per warp stream (cfg3's heaviest unsplit chunks: ~64 K)
constexpr int kRecSlots = 160 * kSlotsPerSm;  // streams exist for the slots of SM ids < 160 (1.3 GB)
// Word-major pool: word w of every slot (and of every thread of a slot) is
// contiguous, so the words in use -- a few dozen per thread at cfg5 -- form
// one compact region at the start of the pool that the L2 can hold (see
// mask_l2_window) instead of 1024 scattered 1 MB slots.
constexpr size_t kMaskWordStride = static_cast<size_t>(kMaskSlots + 1) * kT;

struct FusedSmem {
  // 16-byte strided arrays: the culled lists hold byte offsets t << 4, so
  // the step's shared loads need no address arithmetic
  double2 tDa[kTileT];                 // {y0', y1'}
  double2 tDb[kTileT];                 // {y2', w_j}
  float4 tN0[kTileT];                  // {-y0', -y0', -y1', -y1'}  (FP32x2 pairs)
  float4 tN1[kTileT];                  // {-y2', -y2', 0, 0}
  int tK[kTileT];                      // cell-order target position
  int tJ[kTileT];                      // original target index
  int rowStart[kT];
  int rowPref[kT + 1];
  ListT wlist[kT / 32][kTileT];
  alignas(32) double colW[kT / 32][kTileT];  // (also the atom table of phase2_tm: double4)
  double4 rawY[kTileT];                // cp.async landing zone of the next tile
  double rawB2[kTileT];
  int rawJ[kTileT];
  int rawK[kTileT];
  Region R;                            // CTA-uniform scan region (kept out of registers)
  int mslot;                           // this CTA's mask slot (-1: none)
  int mok;                             // 1: phase 1 stored every step's pair mask
  int nrec[kT / 32];                   // mixed / full-in item indices written by each warp
  int nfulrec[kT / 32];                //   (target-major phase 2)
  int rok;                             // 1: every warp's records fit its stream
  int2 tbl[ExpTab512::kTab];
  double sh[200];
  int shi[40];
};

struct FusedAtoms {
  double Xa[3], Xb[3];       // 2 c2 x'
  double xsqa, xsqb;         // c2 |x'|^2
  float2 F0, F1, F2;         // local FP32 coordinates of (a, b)
  float lo_thr, hi_thr;      // FP32 decision thresholds
  int qa, qb;                // Hilbert positions of the two atoms
  double Sa, Sb;             // phase 1 sums
  uint32_t ca, cb;           // accepted pairs per atom
  uint64_t ha, hb;           // candidate hashes (debug)
  double wa, wb;             // phase 2: m_q / S~_q (0 for empty / exact-path atoms)
  int Fa, Fb;                // floor(512 c2 |x'|^2) (exponent-side predicate; huge for invalid atoms)
};

struct FusedArgs {
  const double4* xs; int nq;             // atoms, Hilbert order
  const double4* ys; const double* b2s;  // targets, cell order
  const int* tperm; const int* cell_start;
  GridDev g;
  const double* scal; const double* psi;
  double c2, r2, r_scan, eps;
  double* atomJ; double* atomD; double* cntd; double* emptyd;
  unsigned long long* gacc;              // [kLimbs N] fixed point (fp_red), cell-order index
  uint32_t* dbg_cnt; uint64_t* dbg_hash; double* dbg_logs;  // Hilbert order
  uint32_t* cnt_out;                     // 0 = empty candidate set (Hilbert order)
  const int* chunk_order;                // CTA -> atom chunk (heaviest first) or null
  const unsigned char* role;             // per chunk: kRoleOther / kRoleMine / kRoleSplit, or null
  const int* heavy_count;                // split chunks: chunk_order[0, heavy_count)
  int* queue;                            // trunc_fused_split work counter
  uint32_t* mbuf;                        // phase-1 pair masks for phase 2 (kMaskSlots slots), or null
  int* mbusy;                            // per slot: held by a resident CTA
  unsigned* mticket;                     // slot search start
  int mslots;                            // 0: no slots (phase 2 recomputes the masks)
  int mwords;                            // words per thread a slot may hold (<= kMaskWords)
  int* rbuf;                             // cell-order indices of the warps' culled items: one stream of
  int rcap;                              //   rcap entries per (slot, warp), or null / 0
};

// chunk roles (chunk_role)
constexpr unsigned char kRoleOther = 0, kRoleMine = 1, kRoleSplit = 2;
// Chunk work model, in units of one scanned target (cfg3 per-rank times fit
// 7.4e-8 ms per scanned target + 3.8e-9 ms per accepted pair; the chunk's
// pairs are ~256 x the targets within reach of its centre, so a centre-ball
// target weighs 256 x 0.051 = 13; fixed cost per chunk ~0.25 us per slot; an
// empty-set atom's nearest search ~32 units: cfg3 0.9 ms for 3.8e5 of them
// against 58 ms for 7.8e8 units)
constexpr unsigned long long kChunkBase = 128;
constexpr unsigned long long kPairWeight = 13;
constexpr unsigned long long kEmptyAtomCost = 32;

// Another rank's chunk: nothing to do (the sums and trunc_nearest_empty
// only read this rank's atom range); the debug outputs are zeroed.
template <bool DEBUG>
__device__ __forceinline__ void fused_skip_chunk(const FusedArgs& A, int chunk) {
  if constexpr (DEBUG) {
    for (int t = threadIdx.x; t < kFA; t += kT) {
      const int q = chunk * kFA + t;
      if (q >= A.nq) break;
      A.dbg_cnt[q] = 0u;
      A.dbg_hash[q] = 0u;
      A.dbg_logs[q] = 0.0;
    }
  }
}

__device__ __forceinline__ double chain3(const double (&X)[3], const double4& y) {
  return fma(X[0], y.x, fma(X[1], y.y, fma(X[2], y.z, y.w)));
}

// w_a 2^sa [ta] + w_b 2^sb [tb] (the weights multiply the table scales:
// one DMUL each, fewer live registers than per-atom scaled polynomials).
template <bool CLAMP>
__device__ __forceinline__ double exp2_pair_weighted(double sa, double sb, double wa, double wb,
                                                     const int2* __restrict__ tbl, bool ta,
                                                     bool tb) {
  const double kka = __dadd_rn(sa, ExpTab512::kMagic);
  const double kkb = __dadd_rn(sb, ExpTab512::kMagic);
  int na = __double2loint(kka);
  int nb = __double2loint(kkb);
  if (CLAMP) {
    na = min(max(na, ExpTab512::kNMin), ExpTab512::kNMax);
    nb = min(max(nb, ExpTab512::kNMin), ExpTab512::kNMax);
  }
  const double ra = __dadd_rn(sa, -__dadd_rn(kka, -ExpTab512::kMagic));
  const double rb = __dadd_rn(sb, -__dadd_rn(kkb, -ExpTab512::kMagic));
  const double qa = ExpTab512::poly(ra);
  const double qb = ExpTab512::poly(rb);
  na = ta ? na : ExpTab512::kZeroN;  // scale word pattern 0 -> +0.0
  nb = tb ? nb : ExpTab512::kZeroN;
#ifdef RSOT_EXP_NOTABLE
  const int2 Ta = make_int2(0, 0x3ff00000 - (na & 511) * ExpTab512::kUnit);
  const int2 Tb = make_int2(0, 0x3ff00000 - (nb & 511) * ExpTab512::kUnit);
#else
  const int2 Ta = tbl[na & (ExpTab512::kTab - 1)];
  const int2 Tb = tbl[nb & (ExpTab512::kTab - 1)];
#endif
  const double sca = __hiloint2double(Ta.y + na * ExpTab512::kUnit, Ta.x) * wa;
  const double scb = __hiloint2double(Tb.y + nb * ExpTab512::kUnit, Tb.x) * wb;
  return fma(qa, sca, qb * scb);
}

// Transposed butterfly: v[i] (this lane's contribution to item i of the
// batch of 16) -> lane l returns the warp total of item (l >> 1).
__device__ __forceinline__ double butterfly16(double (&v)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = 8, o = 16; h >= 1; h >>= 1, o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? v[i] : v[i + h];
      const double keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Stages tile [base, base + cnt) of the current row batch.
// Asynchronous copies global -> shared (LDGSTS): the next tile's raw target
// data lands while the CTA computes the current one.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Issues the copies of tile [base, base + cnt) of the current row batch
// (each thread its entries tid + u kT; the same thread converts them).
__device__ __forceinline__ void fused_prefetch(FusedSmem& sm, const FusedArgs& A, const TileMap& m,
                                               int tk, int cnt) {
  for (int u = 0; u < (kTileT + kT - 1) / kT; ++u) {  // (uniform trip count: the row search shuffles)
    const int t = threadIdx.x + u * kT;
    const bool valid = t < cnt;
    const int s = valid ? tile_pos(m, tk, t) : 0;
    const int r = find_row_group(sm.rowPref, s, valid);
    if (!valid) continue;
    const int k = sm.rowStart[r] + (s - sm.rowPref[r]);
    sm.rawK[t] = k;  // tK of the tile being computed is still in use
    cp_async16(&sm.rawY[t], &A.ys[k]);
    cp_async16(reinterpret_cast<char*>(&sm.rawY[t]) + 16, reinterpret_cast<const char*>(&A.ys[k]) + 16);
    cp_async8(&sm.rawB2[t], &A.b2s[k]);
    cp_async4(&sm.rawJ[t], &A.tperm[k]);
  }
  cp_async_commit();
}

// Converts the landed tile into the staged layout (local coordinates,
// per-target exponent term, FP32 pre-test coordinates).
__device__ __forceinline__ void fused_convert(FusedSmem& sm, const FusedArgs& A, double B, int cnt) {
  cp_async_wait_all();
  const double o0 = sm.R.o[0], o1 = sm.R.o[1], o2 = sm.R.o[2];
  for (int t = threadIdx.x; t < cnt; t += kT) {
    const double4 y = sm.rawY[t];
    const double y0 = y.x - o0, y1 = y.y - o1, y2 = y.z - o2;
    const double yy = fma(y2, y2, fma(y1, y1, y0 * y0));
    const double w = fmax(fma(-A.c2, yy, sm.rawB2[t]) - B, -1.0e5);
    sm.tDa[t] = make_double2(y0, y1);
    sm.tDb[t] = make_double2(y2, w);
    const float f0 = -static_cast<float>(y0), f1 = -static_cast<float>(y1),
                f2 = -static_cast<float>(y2);
    sm.tN0[t] = make_float4(f0, f0, f1, f1);
    // floor(512 (b2_j - B - c2 r^2)): the target side of the exponent-side
    // pair predicate (step64i), clamped far from int overflow
    const double th = fmin(fmax(512.0 * ((sm.rawB2[t] - B) - A.c2 * A.r2), -1.0e8), 1.0e8);
    sm.tN1[t] = make_float4(f2, f2, __int_as_float(__double2int_rd(th)), __int_as_float(sm.rawK[t]));
    sm.tJ[t] = sm.rawJ[t];
    sm.tK[t] = sm.rawK[t];
  }
}

// Phase 2: the CTA's column sums of the last computed tile (its `cnt`
// entries), added once per target into the fixed-point accumulator.  Called
// after a barrier, with the thread -> entry map of fused_convert, so the
// same thread reads an entry's tJ before converting the next tile over it.
__device__ __forceinline__ void fused_flush_cols(const FusedSmem& sm, const FusedArgs& A, int cnt) {
  for (int s = threadIdx.x; s < cnt; s += kT) {
    const double c = ((sm.colW[0][s] + sm.colW[1][s]) + sm.colW[2][s]) + sm.colW[3][s];
    if (c > 0.0) fp_red(A.gacc + kLimbs * static_cast<size_t>(sm.tK[s]), c);
  }
}

// Culling with full-in split: staged targets whose FARTHEST point of the
// warp box is still inside lo (conservatively: far^2 < full_thr) are in for
// every atom of the warp, with no per-pair test; they go to the back of the
// list (list[cap - 1 - i], i < *nfull), the others to the front.
template <class SM, int SHIFT = 4>
__device__ __forceinline__ int fused_cull2(const SM& sm, int cnt, const WarpBox& w, float thr,
                                           float full_thr, ListT* __restrict__ list, int cap,
                                           int* nfull) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int nsel = 0, nf = 0;
  for (int g = 0; g < cnt; g += 32) {
    const int t = g + lane;
    bool keep = false, full = false;
    if (t < cnt) {
      const float4 a = sm.tN0[t];
      const float bz = sm.tN1[t].x;
      const float dx = fmaxf(fmaxf(w.lo0 + a.x, -a.x - w.hi0), 0.f);
      const float dy = fmaxf(fmaxf(w.lo1 + a.z, -a.z - w.hi1), 0.f);
      const float dz = fmaxf(fmaxf(w.lo2 + bz, -bz - w.hi2), 0.f);
      keep = fmaf(dz, dz, fmaf(dy, dy, dx * dx)) <= thr;
      const float fx = fmaxf(-a.x - w.lo0, w.hi0 + a.x);
      const float fy = fmaxf(-a.z - w.lo1, w.hi1 + a.z);
      const float fz = fmaxf(-bz - w.lo2, w.hi2 + bz);
      full = keep && fmaf(fz, fz, fmaf(fy, fy, fx * fx)) < full_thr;
      keep = keep && !full;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    const unsigned mf = __ballot_sync(0xffffffffu, full);
    if (keep) list[nsel + __popc(m & lt)] = static_cast<ListT>(t << SHIFT);
    if (full) list[cap - 1 - (nf + __popc(mf & lt))] = static_cast<ListT>(t << SHIFT);
    nsel += __popc(m);
    nf += __popc(mf);
  }
  __syncwarp();
  *nfull = nf;
  return nsel;
}

// SHIFT > 0: list entries are t << SHIFT (byte offsets into 16-byte arrays,
// so the step's shared loads need no address arithmetic).
template <class SM, int SHIFT = 0>
__device__ __forceinline__ int fused_cull(const SM& sm, int cnt, const WarpBox& w,
                                          float thr, ListT* __restrict__ list) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int nsel = 0;
  for (int g = 0; g < cnt; g += 32) {
    const int t = g + lane;
    bool keep = false;
    if (t < cnt) {
      const float4 a = sm.tN0[t];
      const float bz = sm.tN1[t].x;
      const float dx = fmaxf(fmaxf(w.lo0 + a.x, -a.x - w.hi0), 0.f);
      const float dy = fmaxf(fmaxf(w.lo1 + a.z, -a.z - w.hi1), 0.f);
      const float dz = fmaxf(fmaxf(w.lo2 + bz, -bz - w.hi2), 0.f);
      keep = fmaf(dz, dz, fmaf(dy, dy, dx * dx)) <= thr;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) list[nsel + __popc(m & lt)] = static_cast<ListT>(t << SHIFT);
    nsel += __popc(m);
  }
  __syncwarp();
  return nsel;
}

// Element at byte offset o of a 16-byte strided staged array.
template <class T>
__device__ __forceinline__ const T& at16(const T* arr, int o) {
  return *reinterpret_cast<const T*>(reinterpret_cast<const char*>(arr) + o);
}

// Packed FP32x2 squared distances of the item at byte offset o (t << 4) to
// the thread's atoms (a, b).
template <class SM, class AT>
__device__ __forceinline__ float2 fused_d2(const SM& sm, const AT& at, int o) {
  const float4 n01 = at16(sm.tN0, o);
  const float4 n2 = at16(sm.tN1, o);
  const float2 dx = __fadd2_rn(at.F0, make_float2(n01.x, n01.y));
  const float2 dy = __fadd2_rn(at.F1, make_float2(n01.z, n01.w));
  const float2 dz = __fadd2_rn(at.F2, make_float2(n2.x, n2.y));
  float2 d2 = __fmul2_rn(dx, dx);
  d2 = __ffma2_rn(dy, dy, d2);
  return __ffma2_rn(dz, dz, d2);
}


// 4-bit pair masks for items (t0, t1) x atoms (a, b): bit 2i = atom a,
// bit 2i+1 = atom b.  in: d2 < lo (sign of d2 - lo is exact); border:
// lo <= d2 < hi (decided by the exact fp64 predicate).
__device__ __forceinline__ void fused_masks(float2 d0, float2 d1, float2 nlo, float2 nhi, bool v1,
                                            unsigned& in, unsigned& border) {
  const float lo = -nlo.x, hi = -nhi.x;
  const bool i0 = d0.x < lo, i1 = d0.y < lo;
  const bool i2 = v1 && d1.x < lo, i3 = v1 && d1.y < lo;
  const bool b0 = !i0 && d0.x < hi, b1 = !i1 && d0.y < hi;
  const bool b2 = v1 && !i2 && d1.x < hi, b3 = v1 && !i3 && d1.y < hi;
  in = static_cast<unsigned>(i0) | (static_cast<unsigned>(i1) << 1) |
       (static_cast<unsigned>(i2) << 2) | (static_cast<unsigned>(i3) << 3);
  border = static_cast<unsigned>(b0) | (static_cast<unsigned>(b1) << 1) |
           (static_cast<unsigned>(b2) << 2) | (static_cast<unsigned>(b3) << 3);
}

// Per-scan constants of the FP32 step.
struct Step32 {
  float lo;        // pairs with d2 < lo are in (FP32 decision)
  float nmid, hw;  // band [lo, hi] <=> |d2 - mid| <= hw (inflated: no misses)
  float nbig, lobig;  // indicator sat(lo*BIG - d2*BIG) = [d2 < lo] exactly
  float2 nlo, nhi;
  float2 nc2;
  float2 nmid2;    // (-mid, -mid) for the packed band test
};

__device__ __forceinline__ float sat_fma(float a, float b, float c) {
  float r;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ Step32 make_step(float lo_thr, float hi_thr) {
  Step32 K;
  K.lo = lo_thr;
  K.nlo = make_float2(-lo_thr, -lo_thr);
  K.nhi = make_float2(-hi_thr, -hi_thr);
  {
    // [lo, hi] inside [mid - hw, mid + hw] after every FP32 rounding: the
    // rounding of mid and of d2 - mid is covered by 4 ulp(hi) of slack
    const double lo = lo_thr, hi = hi_thr;
    const float mid = static_cast<float>(0.5 * (lo + hi));
    K.nmid = -mid;
    K.nmid2 = make_float2(-mid, -mid);
    K.hw = static_cast<float>(fmax(hi - mid, mid - lo) * (1.0 + 0x1p-20) +
                              4.0 * fabs(hi) * 0x1p-23) + 1e-30f;
  }
  // power of two: lo * BIG and d2 * BIG are exact, so the FMA rounds
  // BIG (lo - d2) once: >= 2^77 when d2 < lo, <= 0 otherwise
  const float big = lo_thr > 0.f ? ldexpf(1.f, 100 - ilogbf(lo_thr)) : 0.f;
  K.nbig = -big;
  K.lobig = lo_thr * big;
  K.nc2 = make_float2(0.f, 0.f);
  return K;
}

// Band test of a step: some pair with |d2 - mid| <= hw, i.e. possibly in
// [lo, hi] where the exact fp64 predicate decides (false positives harmless).
template <bool PAIR>
__device__ __forceinline__ bool step_in_band(const Step32& K, float2 d0, float2 d1) {
  const float2 a = __fadd2_rn(d0, K.nmid2);  // (same roundings as scalar adds)
  float bm = fminf(fabsf(a.x), fabsf(a.y));
  if (PAIR) {
    const float2 b = __fadd2_rn(d1, K.nmid2);
    bm = fminf(bm, fminf(fabsf(b.x), fabsf(b.y)));
  }
  return bm <= K.hw;
}

// Exact reference predicate for the pairs inside the FP32 error band (rare).
template <class SM>
__device__ __forceinline__ unsigned fused_exact(const SM& sm, const FusedArgs& A, int qa, int qb,
                                                int t0, int t1, unsigned border, unsigned in) {
  for (int bit = 0; bit < 4; ++bit) {
    if (!((border >> bit) & 1u)) continue;
    const double4 yg = A.ys[sm.tK[bit < 2 ? t0 : t1]];
    const double4 x = A.xs[(bit & 1) ? qb : qa];
    if (exact_inside(x.x, x.y, x.z, yg.x, yg.y, yg.z, A.r2)) in |= 1u << bit;
  }
  return in;
}

// Pair bitmask of a step that has a pair in the FP32 error band (bit 2i:
// atom a, 2i+1: atom b of item i): FP32 decision outside the band, exact fp64
// predicate inside.  Out of line to keep the unrolled fast paths compact.
template <class SM>
__device__ __noinline__ unsigned slow_mask(const SM& sm, const FusedArgs& A, int qa, int qb,
                                           const Step32& K, int t0, int t1, float2 d0, float2 d1,
                                           bool pair) {
  unsigned in, bd;
  fused_masks(d0, d1, K.nlo, K.nhi, pair, in, bd);
  if (bd) in = fused_exact(sm, A, qa, qb, t0, t1, bd, in);
  return in;
}

// Step of 2 targets (t0, t1; PAIR = false: t0 only) x atoms (a, b) of the
// fp64 kernel.  The FP32 pre-test decides clear pairs with 4 FSETP; a step
// with a pair in the error band (warp-uniform, rare) takes the bitmask path
// with the exact fp64 predicate (also used in DEBUG builds for the hashes).
// PHASE 1 accumulates S~ of both atoms and the accepted pair counts (floats,
// exact per tile); PHASE 2 returns the weighted column values of t0, t1.
// SAFE: CTA whose exponents may leave [-1020, 1000] (spread chunk or huge
// psi range): per-atom shift carried in every exponent when wide, and the
// exponent split clamped.
// The exponential part of a step for given pair predicates (kxy: item x,
// atom y).
// COUNT = false: the pair counts come from the stored mask words instead.
template <int PHASE, bool PAIR, bool SAFE, bool COUNT = true>
__device__ __forceinline__ double2 exp_part64(const FusedSmem& sm, FusedAtoms& at, bool wide,
                                              int t0, int t1, bool k0a, bool k0b, bool k1a,
                                              bool k1b, float2& cnt) {
  double2 out = make_double2(0.0, 0.0);
  {
    const double2 y0a = at16(sm.tDa, t0), y0b = at16(sm.tDb, t0);
    const double4 y0 = make_double4(y0a.x, y0a.y, y0b.x, y0b.y);
    double sa0 = chain3(at.Xa, y0), sb0 = chain3(at.Xb, y0);
    if (wide) {
      sa0 -= at.xsqa;
      sb0 -= at.xsqb;
    }
    if (PHASE == 1) {
      if (COUNT) cnt = __fadd2_rn(cnt, make_float2(k0a ? 1.f : 0.f, k0b ? 1.f : 0.f));
      at.Sa = exp2_acc_masked<SAFE, ExpTab512>(sa0, at.Sa, sm.tbl, k0a);
      at.Sb = exp2_acc_masked<SAFE, ExpTab512>(sb0, at.Sb, sm.tbl, k0b);
    } else {
      out.x = exp2_pair_weighted<SAFE>(sa0, sb0, at.wa, at.wb, sm.tbl, k0a, k0b);
    }
    if (PAIR) {
      const double2 y1a = at16(sm.tDa, t1), y1b = at16(sm.tDb, t1);
      const double4 y1 = make_double4(y1a.x, y1a.y, y1b.x, y1b.y);
      double sa1 = chain3(at.Xa, y1), sb1 = chain3(at.Xb, y1);
      if (wide) {
        sa1 -= at.xsqa;
        sb1 -= at.xsqb;
      }
      if (PHASE == 1) {
        if (COUNT) cnt = __fadd2_rn(cnt, make_float2(k1a ? 1.f : 0.f, k1b ? 1.f : 0.f));
        at.Sa = exp2_acc_masked<SAFE, ExpTab512>(sa1, at.Sa, sm.tbl, k1a);
        at.Sb = exp2_acc_masked<SAFE, ExpTab512>(sb1, at.Sb, sm.tbl, k1b);
      } else {
        out.y = exp2_pair_weighted<SAFE>(sa1, sb1, at.wa, at.wb, sm.tbl, k1a, k1b);
      }
    }
  }
  return out;
}

// Pair masks of phase 1, replayed in phase 2 (same tiles, same culled lists,
// same step order): phase 2 skips the FP32 pre-test, the band vote and the
// exact band path.  4 bits per step (bit 2i: atom a, 2i+1: atom b of item
// i), 8 steps per word, each tile's stream padded to a word; thread t's words
// are p[0], p[kT], ... of its CTA's region (coalesced).  CTAs whose region
// does not fit recompute the masks in phase 2 (identical results).
struct MaskIO {
  uint32_t* base;  // thread's first word (words base[i * kT])
  int* ok;         // &sm.mok (cleared on overflow)
  int cap;         // words this thread may store
  uint32_t ca, cb; // accepted pairs of atoms a, b in the stored words
  int widx;        // next word
  int n;           // steps in w (the first in the top bits)
  uint32_t w;
};
__device__ __forceinline__ void mask_store(MaskIO& m) {
  m.base[static_cast<size_t>(min(m.widx, m.cap)) * kMaskWordStride] = m.w;  // (overflow: scratch word)
  m.ca += __popc(m.w & 0x55555555u);  // (bits 4s, 4s + 2: atom a; 4s + 1, 4s + 3: atom b)
  m.cb += __popc(m.w & 0xAAAAAAAAu);
  if (m.widx >= m.cap) *m.ok = 0;
  ++m.widx;
  m.w = 0u;
  m.n = 0;
}
__device__ __forceinline__ void mask_put(MaskIO& m, bool k0a, bool k0b, bool k1a, bool k1b) {
  const uint32_t b = (k0a ? 1u : 0u) | (k0b ? 2u : 0u) | (k1a ? 4u : 0u) | (k1b ? 8u : 0u);
  m.w = (m.w << 4) | b;
  if (++m.n == 8) mask_store(m);
}
__device__ __forceinline__ void mask_flush(MaskIO& m) {
  if (m.n) {
    m.w <<= 4 * (8 - m.n);
    mask_store(m);
  }
}
// Bits of step p (0..7) of a word.
__device__ __forceinline__ uint32_t mask_bits(uint32_t w, int p) { return w >> (28 - 4 * p); }

template <int PHASE, bool PAIR, bool SAFE, bool DEBUG, bool CHECK = true, bool MASK = false>
__device__ __forceinline__ double2 step64d(const FusedSmem& sm, const FusedArgs& A, FusedAtoms& at,
                                           const Step32& K, bool wide, int t0, int t1, float2 d0,
                                           float2 d1, float2& cnt, bool& hit,
                                           MaskIO* mio = nullptr) {
  // culled steps always hold accepted pairs (no all-out steps in practice):
  // no vote on the work, masked pairs contribute +0
  if (DEBUG || (CHECK && __any_sync(0xffffffffu, step_in_band<PAIR>(K, d0, d1)))) {
    hit = true;
    const unsigned in = slow_mask(sm, A, at.qa, at.qb, K, t0 >> 4, t1 >> 4, d0, d1, PAIR);
    if (DEBUG && PHASE == 1) {
      if (in & 1u) at.ha += candidate_hash_term(static_cast<uint64_t>(sm.tJ[t0 >> 4]));
      if (in & 4u) at.ha += candidate_hash_term(static_cast<uint64_t>(sm.tJ[t1 >> 4]));
      if (in & 2u) at.hb += candidate_hash_term(static_cast<uint64_t>(sm.tJ[t0 >> 4]));
      if (in & 8u) at.hb += candidate_hash_term(static_cast<uint64_t>(sm.tJ[t1 >> 4]));
    }
    // the exact decisions, re-expressed as distances on either side of lo:
    // both paths meet in the FP32 registers and the predicates below come
    // straight from FSETP (merging bool masks materialised them as bytes)
    d0.x = (in & 1u) ? -INFINITY : INFINITY;
    d0.y = (in & 2u) ? -INFINITY : INFINITY;
    d1.x = (in & 4u) ? -INFINITY : INFINITY;
    d1.y = (in & 8u) ? -INFINITY : INFINITY;
  }
  const bool k0a = d0.x < K.lo, k0b = d0.y < K.lo;
  const bool k1a = PAIR && d1.x < K.lo, k1b = PAIR && d1.y < K.lo;
  if (PHASE == 1 && MASK) mask_put(*mio, k0a, k0b, k1a, k1b);
  return exp_part64<PHASE, PAIR, SAFE, !(PHASE == 1 && MASK)>(sm, at, wide, t0, t1, k0a, k0b, k1a, k1b,
                                                               cnt);
}

template <int PHASE, bool PAIR, bool SAFE, bool DEBUG, bool CHECK = true, bool MASK = false>
__device__ __forceinline__ double2 step64(const FusedSmem& sm, const FusedArgs& A, FusedAtoms& at,
                                          const Step32& K, bool wide, int t0, int t1,
                                          float2& cnt, bool& hit, MaskIO* mio = nullptr) {
  const float2 d0 = fused_d2(sm, at, t0);
  const float2 d1 = PAIR ? fused_d2(sm, at, t1) : d0;
  return step64d<PHASE, PAIR, SAFE, DEBUG, CHECK, MASK>(sm, A, at, K, wide, t0, t1, d0, d1, cnt, hit,
                                                        mio);
}

// acc + (take ? 2^s : 0) from a precomputed magic sum kk = s + M (its low
// word n = round(512 s) already served the pair predicate).
__device__ __forceinline__ double exp2_acc_kk(double s, double kk, int n, double acc,
                                              const int2* __restrict__ tbl, bool take) {
  const double kd = __dadd_rn(kk, -ExpTab512::kMagic);
  const double r = __dadd_rn(s, -kd);
  const double p = ExpTab512::poly(r);
  n = take ? n : ExpTab512::kZeroN;
  const int2 t = tbl[n & (ExpTab512::kTab - 1)];
  return fma(p, __hiloint2double(t.y + n * ExpTab512::kUnit, t.x), acc);
}

// Phase-1 step (2 targets x atoms a, b; non-wide CTAs) whose pair predicates
// come from the exponent itself instead of an FP32 distance pre-test.  With
// s = T_j + X.y' (the chain, in log2 units about the CTA origin),
//   c2 d^2 = c2 |x'|^2 + (b2_j - B) - s, so d^2 < r^2  <=>  s > phi_q + theta_j,
// phi_q = c2 |x'|^2, theta_j = b2_j - B - c2 r^2.  The exp2 split already has
// n = round(512 s); with F_q = floor(512 phi_q) and T_j = floor(512 theta_j)
// (staged), n - F_q - T_j >= 3 proves the pair in and <= -1 proves it out
// (512 (phi + theta) lies in [F + T, F + T + 2), 512 s within 1/2 of n, and
// every rounding of s, phi, theta and the reference's own d^2 is orders of
// magnitude below one unit); pairs with n - F - T in {0, 1, 2} -- a band of
// 3 / (512 c2) in d^2 -- take the exact reference predicate (fused_exact,
// warp-uniform branch, ~5 % of the steps at cfg3 / cfg5).  Replaces the
// packed FP32 distances, their band test and the predicate merge.
__device__ __forceinline__ void step64i(const FusedSmem& sm, const FusedArgs& A, FusedAtoms& at, int t0,
                                        int t1, MaskIO& mio) {
  const double2 y0a = at16(sm.tDa, t0), y0b = at16(sm.tDb, t0);
  const double2 y1a = at16(sm.tDa, t1), y1b = at16(sm.tDb, t1);
  const int T0 = __float_as_int(at16(sm.tN1, t0).z), T1 = __float_as_int(at16(sm.tN1, t1).z);
  const double4 y0 = make_double4(y0a.x, y0a.y, y0b.x, y0b.y);
  const double4 y1 = make_double4(y1a.x, y1a.y, y1b.x, y1b.y);
  const double sa0 = chain3(at.Xa, y0), sb0 = chain3(at.Xb, y0);
  const double sa1 = chain3(at.Xa, y1), sb1 = chain3(at.Xb, y1);
  const double ka0 = __dadd_rn(sa0, ExpTab512::kMagic), kb0 = __dadd_rn(sb0, ExpTab512::kMagic);
  const double ka1 = __dadd_rn(sa1, ExpTab512::kMagic), kb1 = __dadd_rn(sb1, ExpTab512::kMagic);
  const int na0 = __double2loint(ka0), nb0 = __double2loint(kb0);
  const int na1 = __double2loint(ka1), nb1 = __double2loint(kb1);
  const int da0 = na0 - at.Fa - T0, db0 = nb0 - at.Fb - T0;
  const int da1 = na1 - at.Fa - T1, db1 = nb1 - at.Fb - T1;
  bool k0a = da0 >= 3, k0b = db0 >= 3, k1a = da1 >= 3, k1b = db1 >= 3;
  const unsigned border = (static_cast<unsigned>(da0) < 3u ? 1u : 0u) | (static_cast<unsigned>(db0) < 3u ? 2u : 0u) |
                          (static_cast<unsigned>(da1) < 3u ? 4u : 0u) | (static_cast<unsigned>(db1) < 3u ? 8u : 0u);
  if (__any_sync(0xffffffffu, border != 0u)) {
    unsigned in = (k0a ? 1u : 0u) | (k0b ? 2u : 0u) | (k1a ? 4u : 0u) | (k1b ? 8u : 0u);
    if (border) in = fused_exact(sm, A, at.qa, at.qb, t0 >> 4, t1 >> 4, border, in);
    k0a = in & 1u;
    k0b = in & 2u;
    k1a = in & 4u;
    k1b = in & 8u;
  }
  mask_put(mio, k0a, k0b, k1a, k1b);
  at.Sa = exp2_acc_kk(sa0, ka0, na0, at.Sa, sm.tbl, k0a);
  at.Sb = exp2_acc_kk(sb0, kb0, nb0, at.Sb, sm.tbl, k0b);
  at.Sa = exp2_acc_kk(sa1, ka1, na1, at.Sa, sm.tbl, k1a);
  at.Sb = exp2_acc_kk(sb1, kb1, nb1, at.Sb, sm.tbl, k1b);
}

// Shared-memory loads at a register address plus a compile-time offset (the
// staged arrays of FusedSmem lie at fixed distances from tDa): one LDS each,
// no per-load address arithmetic.
template <int OFF>
__device__ __forceinline__ double2 lds_d2(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(v.x), "=d"(v.y) : "r"(addr), "n"(OFF));
  return v;
}
template <int OFF>
__device__ __forceinline__ int lds_i(unsigned addr) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(OFF));
  return v;
}
__device__ __forceinline__ int2 lds_i2(unsigned addr) {
  int2 v;
  asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
// Shared address of table entry n & 511 (AND, then one shift-add).
__device__ __forceinline__ unsigned tbl_addr(unsigned tbl, int n) {
  unsigned a;
  asm("{\n\t.reg .b32 t;\n\tand.b32 t, %1, 511;\n\tshl.b32 t, t, 3;\n\tadd.u32 %0, t, %2;\n\t}"
      : "=r"(a) : "r"(n), "r"(tbl));
  return a;
}
// acc + (take ? 2^s : 0) from the magic sum kk = s + M (n = its low word).
__device__ __forceinline__ double exp2_acc_x(double s, double kk, int n, double acc, unsigned tbl, bool take) {
  const double kd = __dadd_rn(kk, -ExpTab512::kMagic);
  const double r = __dadd_rn(s, -kd);
  const double p = ExpTab512::poly(r);
  n = take ? n : ExpTab512::kZeroN;
  const int2 t = lds_i2(tbl_addr(tbl, n));
  return fma(p, __hiloint2double(t.y + n * ExpTab512::kUnit, t.x), acc);
}
__device__ __forceinline__ int exact_x(const FusedSmem& sm, const FusedArgs& A, int q, int t) {
  const double4 yg = A.ys[sm.tK[t]];
  const double4 x = A.xs[q];
  return exact_inside(x.x, x.y, x.z, yg.x, yg.y, yg.z, A.r2) ? -1 : 3;
}

// step64i with the decisions kept as integers: x = F_q + 2 + T_j - n is
// negative for a pair proven in, >= 3 for one proven out, and 0..2 inside the
// band that takes the exact predicate (which then rewrites x to -1 or 3).
// The step's mask bits are the sign bits of the four x, shifted into the
// mask word by funnel shifts, and the accumulation is predicated on x < 0:
// no boolean merges, selects or byte permutes in the step.
// sb: shared address of sm.tDa[0]; o0, o1: byte offsets (t << 4).
__device__ __forceinline__ void step64x(const FusedSmem& sm, const FusedArgs& A, FusedAtoms& at,
                                        unsigned sb, unsigned tbl, int o0, int o1, MaskIO& mio) {
  constexpr int kDb = offsetof(FusedSmem, tDb) - offsetof(FusedSmem, tDa);
  constexpr int kN1 = offsetof(FusedSmem, tN1) - offsetof(FusedSmem, tDa) + 8;  // tN1[t].z
  const unsigned a0 = sb + o0, a1 = sb + o1;
  const double2 y0a = lds_d2<0>(a0), y0b = lds_d2<kDb>(a0);
  const double2 y1a = lds_d2<0>(a1), y1b = lds_d2<kDb>(a1);
  const int T0 = lds_i<kN1>(a0), T1 = lds_i<kN1>(a1);
  const double4 y0 = make_double4(y0a.x, y0a.y, y0b.x, y0b.y);
  const double4 y1 = make_double4(y1a.x, y1a.y, y1b.x, y1b.y);
  const double sa0 = chain3(at.Xa, y0), sb0 = chain3(at.Xb, y0);
  const double sa1 = chain3(at.Xa, y1), sb1 = chain3(at.Xb, y1);
  const double ka0 = __dadd_rn(sa0, ExpTab512::kMagic), kb0 = __dadd_rn(sb0, ExpTab512::kMagic);
  const double ka1 = __dadd_rn(sa1, ExpTab512::kMagic), kb1 = __dadd_rn(sb1, ExpTab512::kMagic);
  const int na0 = __double2loint(ka0), nb0 = __double2loint(kb0);
  const int na1 = __double2loint(ka1), nb1 = __double2loint(kb1);
  // (at.Fa, at.Fb hold F + 2 here)
  int xa0 = at.Fa + T0 - na0, xb0 = at.Fb + T0 - nb0;
  int xa1 = at.Fa + T1 - na1, xb1 = at.Fb + T1 - nb1;
  const unsigned lowest = min(__vimin3_u32(static_cast<unsigned>(xa0), static_cast<unsigned>(xb0),
                                           static_cast<unsigned>(xa1)), static_cast<unsigned>(xb1));
  if (__any_sync(0xffffffffu, lowest < 3u)) {
    // (inline: the same fix-up as an out-of-line call measured +2.6 % at cfg5)
    if (static_cast<unsigned>(xa0) < 3u) xa0 = exact_x(sm, A, at.qa, o0 >> 4);
    if (static_cast<unsigned>(xb0) < 3u) xb0 = exact_x(sm, A, at.qb, o0 >> 4);
    if (static_cast<unsigned>(xa1) < 3u) xa1 = exact_x(sm, A, at.qa, o1 >> 4);
    if (static_cast<unsigned>(xb1) < 3u) xb1 = exact_x(sm, A, at.qb, o1 >> 4);
  }
  // nibble layout of mask_put: bit 0 = (t0, a), 1 = (t0, b), 2 = (t1, a), 3 = (t1, b)
  uint32_t w = mio.w;
  w = __funnelshift_l(static_cast<unsigned>(xb1), w, 1);
  w = __funnelshift_l(static_cast<unsigned>(xa1), w, 1);
  w = __funnelshift_l(static_cast<unsigned>(xb0), w, 1);
  w = __funnelshift_l(static_cast<unsigned>(xa0), w, 1);
  // (the four predicates from the nibble just shifted in: one R2P)
  at.Sa = exp2_acc_x(sa0, ka0, na0, at.Sa, tbl, w & 1u);
  at.Sb = exp2_acc_x(sb0, kb0, nb0, at.Sb, tbl, w & 2u);
  at.Sa = exp2_acc_x(sa1, ka1, na1, at.Sa, tbl, w & 4u);
  at.Sb = exp2_acc_x(sb1, kb1, nb1, at.Sb, tbl, w & 8u);
  mio.w = w;
  if (++mio.n == 8) mask_store(mio);
}

// acc + (take ? 2^s : 0), non-clamped (phase2_tm).
__device__ __forceinline__ double exp2_acc_t(double s, double acc, unsigned tbl, bool take) {
  const double kk = __dadd_rn(s, ExpTab512::kMagic);
  return exp2_acc_x(s, kk, __double2loint(kk), acc, tbl, take);
}

// Target-major phase 2 of an unsplit non-safe CTA.  Phase 1 left, per warp,
// the cell-order indices of its culled items in list order (mixed items from
// the front of the warp's index stream, each tile padded to 16; full-in items
// from the back) next to the pair-mask words (16 mixed items a word).  Each
// warp walks its items, lane = item: the item's 64-atom mask is transposed out
// of the lanes' mask words by ballots (2 per item, against ~1200 instructions
// of pair work per item), and the item's column is summed over the warp's 64
// atoms, broadcast from shared memory as {2 c2 x', log2(m_q / S_q)}.  No
// tiles, staging, culling, barriers or cross-lane reduction; the per-target
// factor 2^(w_j) multiplies the finished column (the exponents X.y' + log2 w
// and w_j are bounded by the caller).  The item's local coordinates and w_j
// are recomputed from the target record exactly as fused_convert staged them.
// Bit-matrix transpose across the warp: returns in lane b the word whose bit
// l is bit b of lane l's x (5 butterfly rounds).
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

// Local coordinates and exponent term of target k about the CTA origin (as
// fused_convert stages them).
struct TmItem {
  double y0, y1, y2, w;
};
__device__ __forceinline__ TmItem tm_load(const FusedSmem& sm, const FusedArgs& A, double B, int k) {
  const double4 y = A.ys[k];
  TmItem t;
  t.y0 = y.x - sm.R.o[0];
  t.y1 = y.y - sm.R.o[1];
  t.y2 = y.z - sm.R.o[2];
  const double yy = fma(t.y2, t.y2, fma(t.y1, t.y1, t.y0 * t.y0));
  t.w = fmax(fma(-A.c2, yy, A.b2s[k]) - B, -1.0e5);
  return t;
}
__device__ __forceinline__ void tm_flush(const FusedSmem& sm, const FusedArgs& A, int k, double w, double acc) {
  if (acc > 0.0) fp_red(A.gacc + kLimbs * static_cast<size_t>(k), acc * exp2_acc<true, ExpTab512>(w, 0.0, sm.tbl));
}
// Two items per lane against the warp's 64 atoms (mask bit a: atom a of the
// table): each broadcast atom entry serves both items; 16 atoms per unrolled
// block, the masks shifted down between blocks (immediate bit tests).
__device__ __forceinline__ void tm_items2(const FusedSmem& sm, const FusedArgs& A, const double4* atab,
                                          unsigned tb, double B, int k0, unsigned long long m0, int k1,
                                          unsigned long long m1) {
  const TmItem i0 = tm_load(sm, A, B, k0), i1 = tm_load(sm, A, B, k1);
  double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 1
  for (int h = 0; h < 4; ++h) {
    const unsigned b0 = static_cast<unsigned>(m0), b1 = static_cast<unsigned>(m1);
    m0 >>= 16;
    m1 >>= 16;
    if (!__any_sync(0xffffffffu, ((b0 | b1) & 0xffffu) != 0u)) continue;  // no item of the pass takes these atoms
#pragma unroll
    for (int a = 0; a < 16; ++a) {
      const double4 X = atab[16 * h + a];
      acc0 = exp2_acc_t(fma(X.x, i0.y0, fma(X.y, i0.y1, fma(X.z, i0.y2, X.w))), acc0, tb, (b0 >> a) & 1u);
      acc1 = exp2_acc_t(fma(X.x, i1.y0, fma(X.y, i1.y1, fma(X.z, i1.y2, X.w))), acc1, tb, (b1 >> a) & 1u);
    }
  }
  tm_flush(sm, A, k0, i0.w, acc0);
  tm_flush(sm, A, k1, i1.w, acc1);
}

// The lane's item of a 32-item block (mask words wA: items 0..15, wB: items
// 16..31 of the block starting at entry e0): index and 64-atom mask.
// 32 x 32 bit transposes of the two words across the warp: lane b then holds
// bit b of every lane's word, i.e. the 32-atom mask of one (item, atom slot).
// Bits b, b + 1 (b even) of a word belong to the item of step (28 - b) / 4
// (b % 4 == 0: slot 0) or (30 - b) / 4 (slot 1): even lanes take that item
// of word A, odd lanes (b = lane - 1) of word B.
__device__ __forceinline__ void tm_gather(uint32_t wA, uint32_t wB, int e0, int nmix, const int* ks,
                                          unsigned EA, unsigned EB, int& k, unsigned long long& m) {
  const int lane = threadIdx.x & 31;
  const unsigned tA = warp_transpose32(wA), tB = warp_transpose32(wB);
  const unsigned pA = __shfl_xor_sync(0xffffffffu, tA, 1), pB = __shfl_xor_sync(0xffffffffu, tB, 1);
  const bool odd = lane & 1;
  const unsigned mA = (odd ? pB : tA) & EA, mB = (odd ? tB : pA) & EB;
  const int bpos = lane & ~1;
  const int slot = (bpos >> 1) & 1, step = ((slot ? 30 : 28) - bpos) >> 2;
  const int e = e0 + (odd ? 16 : 0) + 2 * step + slot;
  k = e < nmix ? ks[e] : 0;
  m = (static_cast<unsigned long long>(mB) << 32) | mA;
}

__device__ __forceinline__ void phase2_tm(FusedSmem& sm, const FusedArgs& A, const FusedAtoms& at, double B,
                                          double la, double lb, bool ea, bool eb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double4* const atab = reinterpret_cast<double4*>(&sm.colW[0][0]) + warp * 64;
  atab[lane] = make_double4(at.Xa[0], at.Xa[1], at.Xa[2], la);
  atab[32 + lane] = make_double4(at.Xb[0], at.Xb[1], at.Xb[2], lb);
  const unsigned EA = __ballot_sync(0xffffffffu, ea), EB = __ballot_sync(0xffffffffu, eb);
  __syncwarp();
  const unsigned tb = static_cast<unsigned>(__cvta_generic_to_shared(&sm.tbl[0]));
  const int* const ks = A.rbuf + (static_cast<size_t>(sm.mslot) * (kT / 32) + warp) * static_cast<size_t>(A.rcap);
  const uint32_t* const mw = A.mbuf + static_cast<size_t>(sm.mslot) * kT + threadIdx.x;
  const int nmix = sm.nrec[warp], nful = sm.nfulrec[warp];
  const int nw = (nmix + 15) >> 4;                 // mask words of the warp's stream
  const int pm = (nmix + 63) >> 6, pf = (nful + 63) >> 6;
  const unsigned long long EF = (static_cast<unsigned long long>(EB) << 32) | EA;
#pragma unroll 1
  for (int pass = 0; pass < pm + pf; ++pass) {  // 64 items a pass, two per lane
    int k0, k1;
    unsigned long long m0, m1;
    if (pass < pm) {
      const int e0 = pass << 6, w0 = pass << 2;
      uint32_t w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = w0 + u < nw ? mw[static_cast<size_t>(w0 + u) * kMaskWordStride] : 0u;
      tm_gather(w[0], w[1], e0, nmix, ks, EA, EB, k0, m0);
      tm_gather(w[2], w[3], e0 + 32, nmix, ks, EA, EB, k1, m1);
    } else {  // full-in items: every enabled atom
      const int e = ((pass - pm) << 6) + lane;
      k0 = e < nful ? ks[A.rcap - 1 - e] : 0;
      k1 = e + 32 < nful ? ks[A.rcap - 1 - (e + 32)] : 0;
      m0 = e < nful ? EF : 0ull;
      m1 = e + 32 < nful ? EF : 0ull;
    }
    tm_items2(sm, A, atab, tb, B, k0, m0, k1, m1);
  }
}

// Phase-2 batch replaying the stored masks (word = the batch's 8 steps).
// No guards on the steps (one basic block of 8 steps): items past nsel read
// stale but finite staged entries (fused_body zeroes the list and staging
// arrays once) and carry zero mask bits (phase 1 pads each tile's last word
// with zeros), so they add +0; only the column writes are guarded.
template <bool SAFE>
__device__ __forceinline__ void batch64_masked(const FusedSmem& sm, FusedAtoms& at, bool wide,
                                               const ListT* list, int b0, int nsel, uint32_t mw,
                                               double* col) {
  const int lane = threadIdx.x & 31;
  double v[16];
  float2 dummy = make_float2(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int i = b0 + 2 * p;
    const uint32_t b = mask_bits(mw, p);
    const double2 val = exp_part64<2, true, SAFE>(sm, at, wide, list[i], list[i + 1], b & 1u, b & 2u,
                                                  b & 4u, b & 8u, dummy);
    v[2 * p] = val.x;
    v[2 * p + 1] = val.y;
  }
  const double tot = butterfly16(v);
  const int item = b0 + (lane >> 1);
  if (!(lane & 1) && item < nsel) col[list[item] >> 4] = tot;
}

template <bool SAFE, bool DEBUG, bool CHECK>
__device__ __forceinline__ void batch64(const FusedSmem& sm, const FusedArgs& A, FusedAtoms& at,
                                        const Step32& K, bool wide, const ListT* list,
                                        int b0, int nsel, double* col) {
  const int lane = threadIdx.x & 31;
  double v[16];
  float2 dummy = make_float2(0.f, 0.f);
  bool hit = false;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int i = b0 + 2 * p;
    double2 val = make_double2(0.0, 0.0);
    if (i < nsel) {
      // a lone last item pairs with itself; its second column is dropped
      const int t0 = list[i];
      const int t1 = i + 1 < nsel ? list[i + 1] : t0;
      val = step64<2, true, SAFE, DEBUG, CHECK>(sm, A, at, K, wide, t0, t1, dummy, hit);
    }
    v[2 * p] = val.x;
    v[2 * p + 1] = i + 1 < nsel ? val.y : 0.0;
  }
  const double tot = butterfly16(v);
  const int item = b0 + (lane >> 1);
  if (!(lane & 1) && item < nsel) col[list[item] >> 4] = tot;
}

// Phase-2 batch over full-in items (every pair of valid atoms taken).
template <bool SAFE>
__device__ __forceinline__ void batch64_full(const FusedSmem& sm, FusedAtoms& at, bool wide,
                                             const ListT* full, int b0, int nfull, bool va, bool vb,
                                             double* col) {
  const int lane = threadIdx.x & 31;
  double v[16];
  float2 dummy = make_float2(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int i = b0 + 2 * p;  // (unguarded: items past nfull are stale entries taken by no atom)
    const bool in0 = i < nfull, in1 = i + 1 < nfull;
    const double2 val = exp_part64<2, true, SAFE>(sm, at, wide, full[-i], full[-(i + 1)], in0 && va,
                                                  in0 && vb, in1 && va, in1 && vb, dummy);
    v[2 * p] = val.x;
    v[2 * p + 1] = val.y;
  }
  const double tot = butterfly16(v);
  const int item = b0 + (lane >> 1);
  if (!(lane & 1) && item < nfull) col[full[-item] >> 4] = tot;
}

// KS > 1: this CTA is split `split` of KS sharing one chunk (heavy chunks,
// trunc_fused_split): every split walks all row batches and takes the tiles
// split, split + KS, ... of each batch's concatenated targets (tile size
// shrunk for small batches so every split gets several), which balances the
// splits to within a tile (every-KS-th-row interleaving left the cluster
// waiting on its longest rows: 14 % of the samples at the cluster barrier).
template <int PHASE, bool SAFE, bool DEBUG, int KS = 1>
__device__ void fused_scan(FusedSmem& sm, const FusedArgs& A, const WarpBox& wb, float cull_thr,
                           double B, FusedAtoms& at, int split = 0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ListT* const list = sm.wlist[warp];
  const bool wide = SAFE && sm.R.wide;
  const Step32 K = make_step(at.lo_thr, at.hi_thr);
  // Full-in split only when the ball is large against the warp box (r > 4
  // half-diagonals; cfg3: ~half the culled targets are full-in, cfg5 (4.9
  // half-diagonals): ~1/8).  With the tiled phase 2 the threshold was 7: the
  // split list handling cost more than it saved at cfg5 (+5 %); with the
  // target-major phase 2, where a full-in item costs what a mixed one does,
  // it pays there too (cfg5 39.65 -> 38.61 ms).
  float full_thr = -1.0f;
  if (!DEBUG && at.lo_thr > 0.f) {
    const float hx = wb.hi0 - wb.lo0, hy = wb.hi1 - wb.lo1, hz = wb.hi2 - wb.lo2;
    const float hd2 = 0.25f * fmaf(hz, hz, fmaf(hy, hy, hx * hx));
    if (at.lo_thr > RSOT_FULLIN_RATIO2 * hd2) full_thr = at.lo_thr * (1.0f - 1e-5f);
  }
  const ListT* const full = list + (kTileT - 1);  // full-in items: full[-i]
  const bool va = at.qa < A.nq, vb = at.qb < A.nq;
  const int ny = sm.R.c_hi[1] - sm.R.c_lo[1] + 1;
  const int nrows = ny * (sm.R.c_hi[2] - sm.R.c_lo[2] + 1);
  int pend = 0;  // phase 2: entries of the previous tile with pending column sums
  // stored pair masks (fused_body holds a slot for this CTA; phase 2 replays
  // them when phase 1 stored every step's)
  // (phase 1 always stores when the kernel has a mask buffer: CTAs without a
  // slot write a shared scratch slot, so the step loop has no branch on it)
  constexpr bool kStore = !DEBUG && KS == 1;
#ifdef RSOT_EXP_NOINTPRED
  constexpr bool kIntPred = false;
#else
  constexpr bool kIntPred = kStore && !SAFE && PHASE == 1;  // (step64i stores the masks it decides)
#endif
  // kRec: the non-safe phase 1 of an unsplit CTA also writes, per tile, the
  // cell-order indices of the warp's culled items for the target-major
  // phase 2 (phase2_tm): mixed items in list order from the front of the
  // warp's stream (two per step: an odd tail item is followed by a pad), full-in
  // items from the back.  The mask stream then runs on across the tiles (no
  // per-tile padding to a word: item e belongs to word e / 16), so the tiled
  // phase 2 cannot replay it: a kRec CTA that falls back recomputes.
  constexpr bool kRec = kIntPred && RSOT_P1_LEAN && RSOT_P2_TM;
  int* const kstream = kRec && A.rbuf != nullptr && sm.mslot >= 0 && sm.mslot < kRecSlots
                           ? A.rbuf + (static_cast<size_t>(sm.mslot) * (kT / 32) + warp) * static_cast<size_t>(A.rcap)
                           : nullptr;
  int rmix = 0, rful = 0;  // entries written so far
  bool rroom = kstream != nullptr;
  const bool mon = kStore && A.mbuf && (PHASE == 1 || (sm.mslot >= 0 && sm.mok));
  MaskIO mio;
  mio.base = A.mbuf + static_cast<size_t>(sm.mslot < 0 ? kMaskSlots : sm.mslot) * kT + threadIdx.x;
  mio.ok = &sm.mok;
  mio.cap = A.mwords;
  mio.ca = mio.cb = 0u;
  mio.widx = 0;
  mio.n = 0;
  mio.w = 0u;
  for (int rb = 0; rb < nrows; rb += kT) {
    int st = 0, ln = 0;
    if (rb + threadIdx.x < nrows)
      row_range(A.g, sm.R, A.r_scan, A.cell_start, rb + threadIdx.x, st, ln);
    int total = 0;
    const int pre = block_exclusive_scan<kT>(ln, sm.shi, &total);
    sm.rowStart[threadIdx.x] = st;
    sm.rowPref[threadIdx.x] = pre;
    if (threadIdx.x == 0) sm.rowPref[kT] = total;
    __syncthreads();  // row ranges visible; previous batch fully consumed
    int tile = kTileT;
    if (KS > 1) tile = min(kTileT, max(32, (total + 4 * KS - 1) / (4 * KS))) & ~(kGroup - 1);
    const TileMap tm = tile_map(total, tile, true);
    if (split < tm.ntile) fused_prefetch(sm, A, tm, split, tile_count(tm, split));
    for (int tk = split; tk < tm.ntile; tk += KS) {
      const int cnt = tile_count(tm, tk);
      __syncthreads();  // every warp is done with the previous tile
      if (PHASE == 2) {  // its column sums, before its entries are overwritten
        fused_flush_cols(sm, A, pend);
        pend = 0;
      }
      fused_convert(sm, A, B, cnt);
      __syncthreads();  // staged tile visible, landing zone free
      if (tk + KS < tm.ntile) fused_prefetch(sm, A, tm, tk + KS, tile_count(tm, tk + KS));
      int nfull = 0;
      const int nsel = fused_cull2(sm, cnt, wb, cull_thr, full_thr, list, kTileT, &nfull);
      if (PHASE == 1) {
        // software-pipelined: the next step's list entries and distances are
        // loaded before this step's exponentials (hides LDS latency)
        float2 cn = make_float2(0.f, 0.f);
        bool hit = false;
        int i = 0;
        if (kRec) {
          // (a tile whose items do not fit the stream any more: no further
          // entries from this warp, phase 2 of the CTA recomputes)
          const int pad = (nsel + 1) & ~1;  // (an odd tail item is a step of its own)
          if (rroom && rmix + pad + rful + nfull > A.rcap) {
            if (lane == 0) sm.rok = 0;
            rroom = false;
          }
          if (rroom) {
            for (int e = lane; e < pad; e += 32)
              kstream[rmix + e] = e < nsel ? __float_as_int(at16(sm.tN1, list[e]).w) : 0;
            for (int f = lane; f < nfull; f += 32)
              kstream[A.rcap - 1 - (rful + f)] = __float_as_int(at16(sm.tN1, full[-f]).w);
          }
          rmix += pad;
          rful += nfull;
        }
        if (kIntPred && nsel >= 2) {
          int t0 = list[0], t1 = list[1];
#if RSOT_P1_LEAN
          const unsigned sb = static_cast<unsigned>(__cvta_generic_to_shared(&sm.tDa[0]));
          const unsigned tb = static_cast<unsigned>(__cvta_generic_to_shared(&sm.tbl[0]));
          at.Fa += 2;  // (step64x: x = F + 2 + T - n)
          at.Fb += 2;
#endif
          for (; i + 1 < nsel; i += 2) {
#ifdef RSOT_P1_NOPIPE
            const int c0 = list[i], c1 = list[i + 1];
#else
            const int c0 = t0, c1 = t1;
#ifdef RSOT_P1_NOGUARD
            {  // (reads up to two entries past the list end: other list entries, unused)
#else
            if (i + 3 < nsel) {
#endif
              t0 = list[i + 2];
              t1 = list[i + 3];
            }
#endif
#if RSOT_P1_LEAN
            step64x(sm, A, at, sb, tb, c0, c1, mio);
#else
            step64i(sm, A, at, c0, c1, mio);
#endif
          }
#if RSOT_P1_LEAN
          at.Fa -= 2;
          at.Fb -= 2;
#endif
        } else if (nsel >= 2) {
          int t0 = list[0], t1 = list[1];
          float2 d0 = fused_d2(sm, at, t0), d1 = fused_d2(sm, at, t1);
          for (; i + 1 < nsel; i += 2) {
            const int c0 = t0, c1 = t1;
            const float2 e0 = d0, e1 = d1;
            if (i + 3 < nsel) {
              t0 = list[i + 2];
              t1 = list[i + 3];
              d0 = fused_d2(sm, at, t0);
              d1 = fused_d2(sm, at, t1);
            }
            step64d<1, true, SAFE, DEBUG, true, kStore>(sm, A, at, K, wide, c0, c1, e0, e1, cn, hit, &mio);
          }
        }
        if (i < nsel)
          step64<1, false, SAFE, DEBUG, true, kStore>(sm, A, at, K, wide, list[i], list[i], cn, hit, &mio);
        if (kStore && !kRec) mask_flush(mio);  // each tile's stream starts on a word
        // full-in items, 4 per iteration without guards (items past nfull:
        // stale entries taken by no atom; f <= 252, so f + 3 stays in the list)
        for (int f = 0; f < nfull; f += 4) {
          const bool i1 = f + 1 < nfull, i2 = f + 2 < nfull, i3 = f + 3 < nfull;
          exp_part64<1, true, SAFE, false>(sm, at, wide, full[-f], full[-(f + 1)], va, vb, i1 && va, i1 && vb,
                                           cn);
          exp_part64<1, true, SAFE, false>(sm, at, wide, full[-(f + 2)], full[-(f + 3)], i2 && va, i2 && vb,
                                           i3 && va, i3 && vb, cn);
        }
        // (every valid atom of the warp takes every full-in item: counted here, not per pair)
        at.ca += va ? static_cast<uint32_t>(nfull) : 0u;
        at.cb += vb ? static_cast<uint32_t>(nfull) : 0u;
        at.ca += static_cast<uint32_t>(cn.x);
        at.cb += static_cast<uint32_t>(cn.y);
      } else {
        double* const col = sm.colW[warp];
        for (int s = lane; s < cnt; s += 32) col[s] = 0.0;
        __syncwarp();
        // (a band-free second instantiation, as in fused_scan32, costs more in
        // instruction-cache misses than it saves here: measured +6 %)
        if (mon) {  // one word per batch of 8 steps (the next one prefetched)
          uint32_t nw = mio.base[static_cast<size_t>(mio.widx) * kMaskWordStride];
          for (int b0 = 0; b0 < nsel; b0 += 16) {
            const uint32_t mw = nw;
            ++mio.widx;
            nw = mio.base[static_cast<size_t>(mio.widx) * kMaskWordStride];
            batch64_masked<SAFE>(sm, at, wide, list, b0, nsel, mw, col);
          }
        } else {
          for (int b0 = 0; b0 < nsel; b0 += 16)
            batch64<SAFE, DEBUG, true>(sm, A, at, K, wide, list, b0, nsel, col);
        }
        for (int b0 = 0; b0 < nfull; b0 += 16) batch64_full<SAFE>(sm, at, wide, full, b0, nfull, va, vb, col);
        pend = cnt;  // summed after the next tile barrier (one barrier less per tile)
      }
    }
    __syncthreads();
    if (PHASE == 2) {
      fused_flush_cols(sm, A, pend);
      pend = 0;
    }
  }
  if (kRec) mask_flush(mio);  // (the stream's last word, before its pairs are counted)
  if (PHASE == 1 && kStore) {  // the mixed-list pairs were counted in the mask words
    at.ca += mio.ca;
    at.cb += mio.cb;
  }
  if (kRec) {
    if (lane == 0) {
      sm.nrec[warp] = rmix;
      sm.nfulrec[warp] = rful;
    }
  }
}

// Exact LSE (reference per-atom max shift) of one atom by the whole warp,
// and, for the gradient, its exact contributions p_qj m_q into gacc.
__device__ __noinline__ void warp_exact_atom(const FusedArgs& A, double x0, double x1, double x2,
                                             double m, double* L_out) {
  const int lane = threadIdx.x & 31;
  const double x[3] = {x0, x1, x2};
  int c_lo[3], c_hi[3];
  for (int d = 0; d < 3; ++d) {
    c_lo[d] = cell_of(A.g, d, x[d] - A.r_scan);
    c_hi[d] = cell_of(A.g, d, x[d] + A.r_scan);
  }
  double mx = -INFINITY, sum = 0.0;
  for (int pass = 0; pass < 3; ++pass) {
    double acc = pass == 0 ? -INFINITY : 0.0;
    for (int cz = c_lo[2]; cz <= c_hi[2]; ++cz)
      for (int cy = c_lo[1]; cy <= c_hi[1]; ++cy) {
        const long long row = (static_cast<long long>(cz) * A.g.dims[1] + cy) * A.g.dims[0];
        const int b = A.cell_start[row + c_lo[0]], e = A.cell_start[row + c_hi[0] + 1];
        for (int k = b + lane; k < e; k += 32) {
          const double4 y = A.ys[k];
          const double d2 = exact_sqdist(x0, x1, x2, y.x, y.y, y.z);
          if (!(d2 < A.r2)) continue;
          const int j = A.tperm[k];
          const double ex = reference_exponent(A.psi[j], d2, A.eps, y.w);
          if (pass == 0) acc = fmax(acc, ex);
          else if (pass == 1) acc += exp(ex - mx);
          else fp_red(A.gacc + kLimbs * static_cast<size_t>(k), exp(ex - mx) * (m / sum));
        }
      }
    if (pass == 0) mx = warp_max(acc);
    else if (pass == 1) sum = warp_sum(acc);
  }
  *L_out = mx + log(sum);
}

// Per-atom finalisation between the phases (all lanes of the warp call it:
// empty and flagged atoms are resolved warp-cooperatively).  Of the CTAs
// sharing a split chunk only the primary writes the per-atom results and
// runs the exact path; the others just take its phase-2 weights.
template <bool DEBUG>
__device__ __forceinline__ void fused_finalize(const FusedArgs& A, double B, bool wide, bool valid,
                                               bool nonempty, double cnt_contrib, uint32_t dbg_count,
                                               double S, double xsq, int q, uint64_t hash,
                                               double& W, double smin = 0x1p-960,
                                               bool primary = true) {
  const int lane = threadIdx.x & 31;
  const double4 p = valid ? A.xs[q] : make_double4(0, 0, 0, 0);
  const double shift = wide ? 0.0 : xsq;
  const double m = p.w;
  const bool empty = valid && !nonempty;
  const bool flag = valid && nonempty && (!(S >= smin) || !(S <= 0x1p960));
  double L = (B - shift + log2(S)) * kLn2;
  double w = valid && nonempty ? m / S : 0.0;
  // Empty candidate sets: resolved after this kernel by trunc_nearest_empty
  // (warp per empty atom over the whole GPU, no CTA barrier in the way);
  // their phase-2 weight is 0 and their J/D/L are written there.
  if (valid && primary) A.cnt_out[q] = empty ? 0u : 1u;
  if (!primary) {
    W = flag ? 0.0 : w;
    return;
  }
  unsigned mf = __ballot_sync(0xffffffffu, flag);
  while (mf) {
    const int l = __ffs(mf) - 1;
    mf &= mf - 1;
    double Lx;
    warp_exact_atom(A, __shfl_sync(0xffffffffu, p.x, l), __shfl_sync(0xffffffffu, p.y, l),
                    __shfl_sync(0xffffffffu, p.z, l), __shfl_sync(0xffffffffu, m, l), &Lx);
    if (lane == l) {
      L = Lx;
      w = 0.0;  // its gradient contributions are already in gacc
    }
  }
  W = w;
  if (valid) {
    A.atomJ[q] = A.eps * L * m;
    A.atomD[q] = m * exp(-L);
    A.cntd[q] = empty ? 1.0 + cnt_contrib : cnt_contrib;
    A.emptyd[q] = empty ? 1.0 : 0.0;
    if (DEBUG) {
      A.dbg_cnt[q] = empty ? 1u : dbg_count;
      A.dbg_hash[q] = hash;
      A.dbg_logs[q] = L;
    }
  }
}

// Phase-1 partials of one split CTA, read by its cluster peers through
// distributed shared memory (aliases colW, which phase 1 does not use).
struct SplitXchg {
  double S[2][kT];
  uint64_t H[2][kT];
  uint32_t C[2][kT];
};
static_assert(sizeof(SplitXchg) <= sizeof(double) * (kT / 32) * kTileT, "exchange fits colW");

// One chunk of kFA Hilbert-consecutive atoms; KS > 1: split `split` of a
// cluster of KS CTAs sharing the chunk (each scans every KS-th target row;
// the phase-1 sums, counts and hashes are combined in rank order, so every
// CTA of the cluster holds the same S_q and the result is deterministic).
template <bool DEBUG, int KS>
__device__ __forceinline__ void fused_body(FusedSmem& sm, const FusedArgs& A, int chunk, int split) {
  load_exp2_table<ExpTab512>(sm.tbl);
  // finite, in-range stale entries for the unguarded replay batches
  for (int t = threadIdx.x; t < kTileT; t += kT) {
    sm.tDa[t] = make_double2(0.0, 0.0);
    sm.tDb[t] = make_double2(0.0, 0.0);
  }
  for (int t = threadIdx.x; t < (kT / 32) * kTileT; t += kT) (&sm.wlist[0][0])[t] = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  FusedAtoms at;
  at.qa = chunk * kFA + warp * 64 + lane;
  at.qb = at.qa + 32;
  const bool va = at.qa < A.nq, vb = at.qb < A.nq;
  double4 pa = va ? A.xs[at.qa] : make_double4(0, 0, 0, 0);
  double4 pb = vb ? A.xs[at.qb] : make_double4(0, 0, 0, 0);
  {
    double lo[3], hi[3];
    lo[0] = fmin(va ? pa.x : INFINITY, vb ? pb.x : INFINITY);
    lo[1] = fmin(va ? pa.y : INFINITY, vb ? pb.y : INFINITY);
    lo[2] = fmin(va ? pa.z : INFINITY, vb ? pb.z : INFINITY);
    hi[0] = fmax(va ? pa.x : -INFINITY, vb ? pb.x : -INFINITY);
    hi[1] = fmax(va ? pa.y : -INFINITY, vb ? pb.y : -INFINITY);
    hi[2] = fmax(va ? pa.z : -INFINITY, vb ? pb.z : -INFINITY);
    Region R;
    setup_region(A.g, lo, hi, A.r2, A.r_scan, A.c2, sm.sh, R);
    if (threadIdx.x == 0) {
      sm.R = R;
      // a mask slot for phase 2: slots kSlotsPerSm * smid + j belong to this
      // SM, whose resident CTAs (at most RSOT_FUSED_MIN_BLOCKS by registers
      // and shared memory) hold at most that many, so a few CAS always find
      // one.  (Linear probing of the whole table from a ticket, as before,
      // failed for some CTAs at cfg3: the probe of a late CTA chases the
      // moving band of just-taken slots, 1024 CAS in ~350 us without a hit.)
      // Fallback for SM ids beyond the table: the global probe.
      int slot = -1;
      if (!DEBUG && KS == 1 && A.mbuf && A.mslots) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        if (smid < static_cast<unsigned>(kMaskSlots / kSlotsPerSm)) {
          for (int j = 0; j < kSlotsPerSm; ++j) {
            const int c = static_cast<int>(smid) * kSlotsPerSm + j;
            if (atomicCAS(A.mbusy + c, 0, 1) == 0) {
              slot = c;
              break;
            }
          }
        } else {
          const unsigned t0 = atomicAdd(A.mticket, 1u);
          for (unsigned k = 0; k < static_cast<unsigned>(kMaskSlots); ++k) {
            const int c = static_cast<int>((t0 + k) & (kMaskSlots - 1));
            if (atomicCAS(A.mbusy + c, 0, 1) == 0) {
              slot = c;
              break;
            }
          }
        }
      }
      sm.mslot = slot;
      sm.mok = slot >= 0 ? 1 : 0;
      sm.rok = slot >= 0 ? 1 : 0;
    }
    __syncthreads();
  }
  const double o0 = sm.R.o[0], o1 = sm.R.o[1], o2 = sm.R.o[2];
  const double ax = pa.x - o0, ay = pa.y - o1, az = pa.z - o2;
  const double bx = pb.x - o0, by = pb.y - o1, bz = pb.z - o2;
  const double c2x2 = 2.0 * A.c2;
  at.Xa[0] = c2x2 * ax; at.Xa[1] = c2x2 * ay; at.Xa[2] = c2x2 * az;
  at.Xb[0] = c2x2 * bx; at.Xb[1] = c2x2 * by; at.Xb[2] = c2x2 * bz;
  at.xsqa = A.c2 * fma(az, az, fma(ay, ay, ax * ax));
  at.xsqb = A.c2 * fma(bz, bz, fma(by, by, bx * bx));
  // (step64i; invalid atoms get a threshold no exponent reaches)
  at.Fa = va ? __double2int_rd(512.0 * at.xsqa) : (1 << 30);
  at.Fb = vb ? __double2int_rd(512.0 * at.xsqb) : (1 << 30);
  const float big = 1e30f;
  at.F0 = make_float2(va ? static_cast<float>(ax) : big, vb ? static_cast<float>(bx) : big);
  at.F1 = make_float2(va ? static_cast<float>(ay) : big, vb ? static_cast<float>(by) : big);
  at.F2 = make_float2(va ? static_cast<float>(az) : big, vb ? static_cast<float>(bz) : big);
  at.lo_thr = sm.R.lo_thr;
  at.hi_thr = sm.R.hi_thr;
  at.Sa = at.Sb = 0.0;
  at.ca = at.cb = 0;
  at.ha = at.hb = 0;
  WarpBox wb;
  {
    const WarpBox w1 = warp_box(va, at.F0.x, at.F1.x, at.F2.x);
    const WarpBox w2 = warp_box(vb, at.F0.y, at.F1.y, at.F2.y);
    wb.lo0 = fminf(w1.lo0, w2.lo0); wb.lo1 = fminf(w1.lo1, w2.lo1); wb.lo2 = fminf(w1.lo2, w2.lo2);
    wb.hi0 = fmaxf(w1.hi0, w2.hi0); wb.hi1 = fmaxf(w1.hi1, w2.hi1); wb.hi2 = fmaxf(w1.hi2, w2.hi2);
  }
  const float cull_thr = sm.R.hi_thr * 1.0001f;
  const double B = A.scal[kSlotB];
  // Exponents of taken pairs lie in [bmin - B - c2 r^2, c2 |x'|^2] (shifted)
  // or [bmin - B - c2 r^2, 0] (wide); outside [-1000, 400] use the safe path.
  const bool wide = sm.R.wide;
  const bool safe = wide || (A.scal[kSlotBmin] - B) - A.c2 * A.r2 < -1000.0;

  if (safe)
    fused_scan<1, true, DEBUG, KS>(sm, A, wb, cull_thr, B, at, split);
  else
    fused_scan<1, false, DEBUG, KS>(sm, A, wb, cull_thr, B, at, split);

  if constexpr (KS > 1) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    SplitXchg* x = reinterpret_cast<SplitXchg*>(&sm.colW[0][0]);
    const int t = threadIdx.x;
    x->S[0][t] = at.Sa; x->S[1][t] = at.Sb;
    x->C[0][t] = at.ca; x->C[1][t] = at.cb;
    if (DEBUG) { x->H[0][t] = at.ha; x->H[1][t] = at.hb; }
    cl.sync();  // partials of every split visible cluster-wide
    double sa = 0.0, sb = 0.0;
    uint32_t ca = 0, cb = 0;
    uint64_t ha = 0, hb = 0;
#pragma unroll
    for (int r = 0; r < KS; ++r) {  // rank order: identical in every CTA
      const SplitXchg* xr = cl.map_shared_rank(x, r);
      sa += xr->S[0][t]; sb += xr->S[1][t];
      ca += xr->C[0][t]; cb += xr->C[1][t];
      if (DEBUG) { ha += xr->H[0][t]; hb += xr->H[1][t]; }
    }
    cl.sync();  // no CTA reuses colW (phase 2) while a peer still reads it
    at.Sa = sa; at.Sb = sb; at.ca = ca; at.cb = cb; at.ha = ha; at.hb = hb;
  }

  // pair counter: the lane's accepted pairs are booked on atom a
  const bool primary = split == 0;
  fused_finalize<DEBUG>(A, B, wide, va, at.ca != 0u, static_cast<double>(at.ca + at.cb), at.ca,
                        at.Sa, at.xsqa, at.qa, at.ha, at.wa, 0x1p-960, primary);
  fused_finalize<DEBUG>(A, B, wide, vb, at.cb != 0u, 0.0, at.cb, at.Sb, at.xsqb, at.qb, at.hb,
                        at.wb, 0x1p-960, primary);

#ifndef RSOT_EXP_NOPHASE2
  if constexpr (!DEBUG && KS == 1 && RSOT_P1_LEAN && RSOT_P2_TM) {
    // Unsplit CTAs: target-major phase 2 over the item records when phase 1
    // wrote them all and every exponent involved stays in range -- the pairs'
    // 2^(X.y' + log2 w_q) and the targets' 2^(w_j), bounded from the region.
    // Any other CTA (safe, no slot, stream overflow, out of range) runs the
    // tiled phase 2 in its safe instantiation, which handles every case.
    const bool ea = at.wa > 0.0, eb = at.wb > 0.0;
    const double la = ea ? log2(at.wa) : 0.0, lb = eb ? log2(at.wb) : 0.0;
    const double xy = sm.R.xy_max;
    const bool fits = fmax(la, lb) + xy <= 1000.0 && fmin(la, lb) - xy >= -1000.0;
    const bool all_fit = __syncthreads_and(fits);  // (also: nrec / rok of phase 1 visible)
    const bool tm = !safe && A.rbuf != nullptr && A.mbuf != nullptr && sm.mslot >= 0 && sm.mslot < kRecSlots &&
                    sm.rok && sm.mok && all_fit &&
                    (A.scal[kSlotBmin] - B) - static_cast<double>(sm.R.wy_max) >= -1000.0;
#ifdef RSOT_LAM_TRACE
    if (!tm && threadIdx.x == 0)
      printf("tmfallback chunk %d safe %d mslot %d rok %d mok %d fit %d nrec %d %d %d %d ful %d\n", chunk, (int)safe,
             sm.mslot, sm.rok, sm.mok, (int)all_fit, sm.nrec[0], sm.nrec[1], sm.nrec[2], sm.nrec[3], sm.nfulrec[0]);
#endif
    if (tm) {
      phase2_tm(sm, A, at, B, la, lb, ea, eb);
    } else {
      if (!safe) {  // (a non-safe CTA's mask stream is not tile-aligned: recompute)
        __syncthreads();
        if (threadIdx.x == 0) sm.mok = 0;
        __syncthreads();
      }
      fused_scan<2, true, DEBUG, KS>(sm, A, wb, cull_thr, B, at, split);
    }
  } else {
    if (safe)
      fused_scan<2, true, DEBUG, KS>(sm, A, wb, cull_thr, B, at, split);
    else
      fused_scan<2, false, DEBUG, KS>(sm, A, wb, cull_thr, B, at, split);
  }
#endif
  if (!DEBUG && KS == 1 && A.mbuf) {
    __syncthreads();  // every thread is done with the slot
    if (threadIdx.x == 0 && sm.mslot >= 0) {
      __threadfence();
      atomicExch(A.mbusy + sm.mslot, 0);
    }
  }
}

#ifndef RSOT_FUSED_MIN_BLOCKS
#define RSOT_FUSED_MIN_BLOCKS 4
#endif
template <bool DEBUG>
__global__ void __launch_bounds__(kT, RSOT_FUSED_MIN_BLOCKS)
trunc_fused(FusedArgs A) {
  __shared__ FusedSmem sm;
  int chunk = static_cast<int>(blockIdx.x);
  if (A.chunk_order) {  // the split chunks lead the order (trunc_fused_split)
    const int pos = *A.heavy_count + chunk;
    if (pos >= (A.nq + kFA - 1) / kFA) return;
    chunk = A.chunk_order[pos];
  }
  if (A.role) {
    const unsigned char r = A.role[chunk];
    if (r == kRoleOther) return fused_skip_chunk<DEBUG>(A, chunk);
    if (r == kRoleSplit) return;  // run by trunc_fused_split
  }
  fused_body<DEBUG, 1>(sm, A, chunk, 0);
}

// Heavy chunks (chunk_role_kernel): a cluster of kSplit CTAs per chunk, so
// the longest chunks no longer bound the kernel (cfg3: one chunk held ~the
// whole GPU's per-slot share of pairs).  Persistent: one resident wave of
// clusters pulls the split chunks heaviest first from a queue (any count,
// no host round trip).
constexpr int kSplit = 8;  // (16, non-portable: +40 % at cfg3 8-way)

template <bool DEBUG>
__global__ void __cluster_dims__(kSplit, 1, 1) __launch_bounds__(kT, 4)
trunc_fused_split(FusedArgs A) {
  __shared__ FusedSmem sm;
  __shared__ int next;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int split = static_cast<int>(cl.block_rank());
  const int count = *A.heavy_count;
  for (;;) {
    // dynamic queue over the heaviest-first split list: the cluster's rank 0
    // takes the next chunk; its peers read it through distributed shared
    // memory (rank 0 writes again only after fused_body's cluster barriers)
    if (split == 0 && threadIdx.x == 0) next = atomicAdd(A.queue, 1);
    cl.sync();
    const int h = *cl.map_shared_rank(&next, 0);
    if (h >= count) {  // uniform across the cluster
      cl.sync();       // rank 0's shared memory stays alive until every peer has read it
      break;
    }
    fused_body<DEBUG, kSplit>(sm, A, A.chunk_order[h], split);
    __syncthreads();  // shared memory free for the next chunk
  }
}

// ---------------------------------------------------------------------------
// Mixed-precision (fp32) truncated evaluation (BASELINE cfg5 "fp32"): the
// same scan, culling and exact candidate sets as trunc_fused; the exponent
// s = (b2_j - B) - c2 d^2 is formed in FP32 from the FP32 pre-test distance
// and 2^s runs on the MUFU (ex2.approx.ftz); tile sums in FP32 are added into
// fp64 per-atom sums.  The shift B is per CTA: the running max of the staged
// b2 (phase 1 rescales its sums when a tile raises it), so any psi range
// keeps the sums in range.  Atoms whose sum falls below 2^-80 take the exact
// fp64 path; empty sets use the same exact nearest kernel.  Observed
// deviation from the fp64 result (tools/fp32_error.py, cfg3/cfg5): J 3e-9 -
// 1.5e-8 relative, gradient 7e-8 of the marginal scale; the tests assert 2e-5.

struct Fused32Smem {
  float4 tN0[kTileT32];                  // {-y0', -y0', -y1', -y1'}
  float4 tN1[kTileT32];                  // {-y2', -y2', b2_j - B, b2_j - B}
  int tK[kTileT32];                      // cell-order target position
  int tJ[kTileT32];                      // original target index
  double4 rawY[kTileT32];                // cp.async landing zone of the next tile
  double rawB2[kTileT32];
  int rawJ[kTileT32];
  int rawK[kTileT32];
  int rowStart[kT];
  int rowPref[kT + 1];
  ListT wlist[kT / 32][kTileT32];
  alignas(16) float colW[kT / 32][kTileT32];  // (also the split exchange: 8-byte fields)
  float wmax[kT / 32];
  Region R;
  double sh[200];
  int shi[40];
};

struct Atoms32 {
  float2 F0, F1, F2;         // local FP32 coordinates of (a, b)
  float lo_thr, hi_thr;
  int qa, qb;
  double Sa, Sb;             // phase 1 sums relative to the CTA shift
  uint32_t ca, cb;           // accepted pairs per atom
  uint64_t ha, hb;           // candidate hashes (debug)
  float wa, wb;              // phase 2 weights m_q / S_q
};

__device__ __forceinline__ float fast_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float butterfly16f(float (&v)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = 8, o = 16; h >= 1; h >>= 1, o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const float send = up ? v[i] : v[i + h];
      const float keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Next tile's raw target data (each thread its entries tid + u kT).
__device__ __forceinline__ void fused_prefetch32(Fused32Smem& sm, const FusedArgs& A,
                                                 const TileMap& m, int tk, int cnt) {
  for (int u = 0; u < (kTileT32 + kT - 1) / kT; ++u) {  // (uniform trip count: the row search shuffles)
    const int t = threadIdx.x + u * kT;
    const bool valid = t < cnt;
    const int s = valid ? tile_pos(m, tk, t) : 0;
    const int r = find_row_group(sm.rowPref, s, valid);
    if (!valid) continue;
    const int k = sm.rowStart[r] + (s - sm.rowPref[r]);
    sm.rawK[t] = k;
    cp_async16(&sm.rawY[t], &A.ys[k]);
    cp_async16(reinterpret_cast<char*>(&sm.rawY[t]) + 16, reinterpret_cast<const char*>(&A.ys[k]) + 16);
    cp_async8(&sm.rawB2[t], &A.b2s[k]);
    cp_async4(&sm.rawJ[t], &A.tperm[k]);
  }
  cp_async_commit();
}

// Stages the landed tile: its b2 maximum is reduced first (phase 1 raises
// the CTA shift and rescales the sums), then the staged exponent offsets are
// written relative to the updated shift.  Two barriers per tile.
// Phase 2 column sums of the last computed tile (see fused_flush_cols).
__device__ __forceinline__ void fused_flush_cols32(const Fused32Smem& sm, const FusedArgs& A, int cnt) {
  for (int s = threadIdx.x; s < cnt; s += kT) {
    const double c = ((static_cast<double>(sm.colW[0][s]) + sm.colW[1][s]) + sm.colW[2][s]) +
                     sm.colW[3][s];
    if (c > 0.0) fp_red(A.gacc + kLimbs * static_cast<size_t>(sm.tK[s]), c);
  }
}

template <int PHASE>
__device__ __forceinline__ void fused_stage32(Fused32Smem& sm, const FusedArgs& A, int cnt,
                                              double& Bc, Atoms32& at, int& pend) {
  cp_async_wait_all();
  if (PHASE == 1) {
    float mx = -INFINITY;
    for (int t = threadIdx.x; t < cnt; t += kT) mx = fmaxf(mx, __double2float_ru(sm.rawB2[t]));
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) sm.wmax[threadIdx.x >> 5] = mx;
  }
  __syncthreads();  // previous tile fully consumed; wmax visible
  if (PHASE == 2) {  // its column sums, before its entries are overwritten
    fused_flush_cols32(sm, A, pend);
    pend = 0;
  }
  if (PHASE == 1) {
    // CTA-uniform running shift (same value in every thread)
    const float tm = fmaxf(fmaxf(sm.wmax[0], sm.wmax[1]), fmaxf(sm.wmax[2], sm.wmax[3]));
    const double Bn = fmax(Bc, static_cast<double>(tm));
    if (Bn > Bc) {
      const double f = exp2(Bc - Bn);
      at.Sa *= f;
      at.Sb *= f;
      Bc = Bn;
    }
  }
  const double o0 = sm.R.o[0], o1 = sm.R.o[1], o2 = sm.R.o[2];
  for (int t = threadIdx.x; t < cnt; t += kT) {
    const double4 y = sm.rawY[t];
    const float f0 = -static_cast<float>(y.x - o0), f1 = -static_cast<float>(y.y - o1),
                f2 = -static_cast<float>(y.z - o2);
    const float w = static_cast<float>(sm.rawB2[t] - Bc);
    sm.tN0[t] = make_float4(f0, f0, f1, f1);
    sm.tN1[t] = make_float4(f2, f2, w, w);
    sm.tK[t] = sm.rawK[t];
    sm.tJ[t] = sm.rawJ[t];
  }
  __syncthreads();  // staged tile visible, landing zone free
}

// FP32x2 squared distances of item t to atoms (a, b) and the item's offset.
// o: byte offset of the item (t << 4) into the 16-byte staged arrays.
template <class SM>
__device__ __forceinline__ float2 fused_d2w(const SM& sm, const Atoms32& at, int o, float& w) {
  const float4 n01 = *reinterpret_cast<const float4*>(reinterpret_cast<const char*>(sm.tN0) + o);
  const float4 n2 = *reinterpret_cast<const float4*>(reinterpret_cast<const char*>(sm.tN1) + o);
  const float2 dx = __fadd2_rn(at.F0, make_float2(n01.x, n01.y));
  const float2 dy = __fadd2_rn(at.F1, make_float2(n01.z, n01.w));
  const float2 dz = __fadd2_rn(at.F2, make_float2(n2.x, n2.y));
  w = n2.z;
  float2 d2 = __fmul2_rn(dx, dx);
  d2 = __ffma2_rn(dy, dy, d2);
  return __ffma2_rn(dz, dz, d2);
}

// Step of 2 targets (t0, t1; PAIR = false: t0 only) x atoms (a, b).
// PHASE 1 accumulates the masked exponentials into acc and the accepted
// pair counts into cnt (floats, exact per tile); PHASE 2 returns the
// weighted column values of t0 and t1.  Pairs in the FP32 error band take
// the exact fp64 predicate (warp-uniform slow path, also used in DEBUG
// builds for the candidate hashes).
template <int PHASE, bool PAIR, bool DEBUG, bool CHECK, class SM>
__device__ __forceinline__ float2 step32(const SM& sm, const FusedArgs& A, Atoms32& at,
                                         const Step32& K, int o0, int o1, float2& acc,
                                         float2& cnt, bool& hit) {
  // o0, o1: byte offsets (t << 4) of the two items
  float w0, w1 = 0.f;
  const float2 d0 = fused_d2w(sm, at, o0, w0);
  const float2 d1 = PAIR ? fused_d2w(sm, at, o1, w1) : d0;
  const int t0 = o0 >> 4, t1 = o1 >> 4;
  float2 i0, i1 = make_float2(0.f, 0.f);
  if (DEBUG || (CHECK && __any_sync(0xffffffffu, step_in_band<PAIR>(K, d0, d1)))) {
    hit = true;
    const unsigned in = slow_mask(sm, A, at.qa, at.qb, K, t0, t1, d0, d1, PAIR);
    i0 = make_float2((in & 1u) ? 1.f : 0.f, (in & 2u) ? 1.f : 0.f);
    if (PAIR) i1 = make_float2((in & 4u) ? 1.f : 0.f, (in & 8u) ? 1.f : 0.f);
    if (DEBUG && PHASE == 1) {
      if (in & 1u) at.ha += candidate_hash_term(static_cast<uint64_t>(sm.tJ[t0]));
      if (in & 4u) at.ha += candidate_hash_term(static_cast<uint64_t>(sm.tJ[t1]));
      if (in & 2u) at.hb += candidate_hash_term(static_cast<uint64_t>(sm.tJ[t0]));
      if (in & 8u) at.hb += candidate_hash_term(static_cast<uint64_t>(sm.tJ[t1]));
    }
  } else {
    i0 = make_float2(sat_fma(d0.x, K.nbig, K.lobig), sat_fma(d0.y, K.nbig, K.lobig));
    if (PAIR) i1 = make_float2(sat_fma(d1.x, K.nbig, K.lobig), sat_fma(d1.y, K.nbig, K.lobig));
  }
  float2 out = make_float2(0.f, 0.f);
  {
    const float2 s0 = __ffma2_rn(K.nc2, d0, make_float2(w0, w0));
    const float2 e0 = __fmul2_rn(make_float2(fast_ex2(s0.x), fast_ex2(s0.y)), i0);
    float2 e1 = make_float2(0.f, 0.f);
    if (PAIR) {
      const float2 s1 = __ffma2_rn(K.nc2, d1, make_float2(w1, w1));
      e1 = __fmul2_rn(make_float2(fast_ex2(s1.x), fast_ex2(s1.y)), i1);
    }
    if (PHASE == 1) {
      acc = __fadd2_rn(acc, e0);
      cnt = __fadd2_rn(cnt, i0);
      if (PAIR) {
        acc = __fadd2_rn(acc, e1);
        cnt = __fadd2_rn(cnt, i1);
      }
    } else {
      out.x = fmaf(at.wb, e0.y, at.wa * e0.x);
      if (PAIR) out.y = fmaf(at.wb, e1.y, at.wa * e1.x);
    }
  }
  return out;
}

template <bool FULL, bool DEBUG, bool CHECK, class SM>
__device__ __forceinline__ void batch32(const SM& sm, const FusedArgs& A, Atoms32& at,
                                        const Step32& K, const ListT* list, int b0, int nsel,
                                        float* col) {
  const int lane = threadIdx.x & 31;
  float v[16];
  float2 dummy = make_float2(0.f, 0.f), dummy2 = dummy;
  bool hit = false;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int i = b0 + 2 * p;
    float2 val = make_float2(0.f, 0.f);
    if (FULL || i + 1 < nsel)
      val = step32<2, true, DEBUG, CHECK>(sm, A, at, K, list[i], list[i + 1], dummy, dummy2, hit);
    else if (i < nsel)
      val = step32<2, false, DEBUG, CHECK>(sm, A, at, K, list[i], list[i], dummy, dummy2, hit);
    v[2 * p] = val.x;
    v[2 * p + 1] = val.y;
  }
  const float tot = butterfly16f(v);
  const int item = b0 + (lane >> 1);
  if (!(lane & 1) && item < nsel) col[list[item] >> 4] = tot;
}

template <int PHASE, bool DEBUG, int KS = 1>
__device__ void fused_scan32(Fused32Smem& sm, const FusedArgs& A, const WarpBox& wb,
                             float cull_thr, double& Bc, Atoms32& at, unsigned& bandmask,
                             int split = 0) {
  // bandmask bit i: phase 1 met a pair in the FP32 error band in this warp's
  // tile i; phase 2 re-tests only those tiles (same tiles, same lists)
  int tix = 0;
  int pend = 0;  // phase 2: entries of the previous tile with pending column sums
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ListT* const list = sm.wlist[warp];
  Step32 K = make_step(at.lo_thr, at.hi_thr);
  const float nc2f = static_cast<float>(-A.c2);
  K.nc2 = make_float2(nc2f, nc2f);
  const int ny = sm.R.c_hi[1] - sm.R.c_lo[1] + 1;
  const int nrows = ny * (sm.R.c_hi[2] - sm.R.c_lo[2] + 1);
  for (int rb = 0; rb < nrows; rb += kT) {
    int st = 0, ln = 0;
    if (rb + threadIdx.x < nrows)
      row_range(A.g, sm.R, A.r_scan, A.cell_start, rb + threadIdx.x, st, ln);
    int total = 0;
    const int pre = block_exclusive_scan<kT>(ln, sm.shi, &total);
    sm.rowStart[threadIdx.x] = st;
    sm.rowPref[threadIdx.x] = pre;
    if (threadIdx.x == 0) sm.rowPref[kT] = total;
    __syncthreads();  // the prefetch reads every thread's row range
    int tile = kTileT32;  // (split: as fused_scan)
    if (KS > 1) tile = min(kTileT32, max(32, (total + 4 * KS - 1) / (4 * KS))) & ~(kGroup - 1);
    const TileMap tm = tile_map(total, tile, false);
    if (split < tm.ntile) fused_prefetch32(sm, A, tm, split, tile_count(tm, split));
    for (int tk = split; tk < tm.ntile; tk += KS) {
      const int cnt = tile_count(tm, tk);
      fused_stage32<PHASE>(sm, A, cnt, Bc, at, pend);
      if (tk + KS < tm.ntile) fused_prefetch32(sm, A, tm, tk + KS, tile_count(tm, tk + KS));
      const int nsel = fused_cull<Fused32Smem, 4>(sm, cnt, wb, cull_thr, list);
      if (PHASE == 1) {
        float2 acc = make_float2(0.f, 0.f), cn = make_float2(0.f, 0.f);
        bool hit = false;
        int i = 0;
        for (; i + 1 < nsel; i += 2)
          step32<1, true, DEBUG, true>(sm, A, at, K, list[i], list[i + 1], acc, cn, hit);
        if (i < nsel) step32<1, false, DEBUG, true>(sm, A, at, K, list[i], list[i], acc, cn, hit);
        if (hit && tix < 32) bandmask |= 1u << tix;
        at.Sa += static_cast<double>(acc.x);
        at.Sb += static_cast<double>(acc.y);
        at.ca += static_cast<uint32_t>(cn.x);
        at.cb += static_cast<uint32_t>(cn.y);
      } else {
        float* const col = sm.colW[warp];
        for (int s = lane; s < cnt; s += 32) col[s] = 0.f;
        __syncwarp();
        int b0 = 0;
        if (tix >= 32 || ((bandmask >> tix) & 1u)) {
          for (; b0 + 16 <= nsel; b0 += 16) batch32<true, DEBUG, true>(sm, A, at, K, list, b0, nsel, col);
          if (b0 < nsel) batch32<false, DEBUG, true>(sm, A, at, K, list, b0, nsel, col);
        } else {
          for (; b0 + 16 <= nsel; b0 += 16) batch32<true, DEBUG, false>(sm, A, at, K, list, b0, nsel, col);
          if (b0 < nsel) batch32<false, DEBUG, false>(sm, A, at, K, list, b0, nsel, col);
        }
        pend = cnt;  // summed after the next tile barrier
      }
      ++tix;
    }
    __syncthreads();
    if (PHASE == 2) {
      fused_flush_cols32(sm, A, pend);
      pend = 0;
    }
  }
}

// Phase-1 partials of one fp32 split CTA (aliases colW; see SplitXchg).
struct SplitXchg32 {
  double S[2][kT];
  uint64_t H[2][kT];
  uint32_t C[2][kT];
  double B;  // the CTA's running shift
};
static_assert(sizeof(SplitXchg32) <= sizeof(float) * (kT / 32) * kTileT32, "exchange fits colW");

// fp32 chunk body (fused_body's counterpart).  KS > 1: the splits' shifts
// combine to B = max_r B_r and S = sum_r S_r 2^(B_r - B) in rank order, the
// shift an unsplit CTA would have reached; phase 2 runs at B.
template <bool DEBUG, int KS>
__device__ __forceinline__ void fused32_body(Fused32Smem& sm, const FusedArgs& A, int chunk, int split) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Atoms32 at;
  at.qa = chunk * kFA + warp * 64 + lane;
  at.qb = at.qa + 32;
  const bool va = at.qa < A.nq, vb = at.qb < A.nq;
  const double4 pa = va ? A.xs[at.qa] : make_double4(0, 0, 0, 0);
  const double4 pb = vb ? A.xs[at.qb] : make_double4(0, 0, 0, 0);
  {
    double lo[3], hi[3];
    lo[0] = fmin(va ? pa.x : INFINITY, vb ? pb.x : INFINITY);
    lo[1] = fmin(va ? pa.y : INFINITY, vb ? pb.y : INFINITY);
    lo[2] = fmin(va ? pa.z : INFINITY, vb ? pb.z : INFINITY);
    hi[0] = fmax(va ? pa.x : -INFINITY, vb ? pb.x : -INFINITY);
    hi[1] = fmax(va ? pa.y : -INFINITY, vb ? pb.y : -INFINITY);
    hi[2] = fmax(va ? pa.z : -INFINITY, vb ? pb.z : -INFINITY);
    Region R;
    setup_region(A.g, lo, hi, A.r2, A.r_scan, A.c2, sm.sh, R);
    if (threadIdx.x == 0) sm.R = R;
    __syncthreads();
  }
  const double o0 = sm.R.o[0], o1 = sm.R.o[1], o2 = sm.R.o[2];
  const float big = 1e30f;
  at.F0 = make_float2(va ? static_cast<float>(pa.x - o0) : big, vb ? static_cast<float>(pb.x - o0) : big);
  at.F1 = make_float2(va ? static_cast<float>(pa.y - o1) : big, vb ? static_cast<float>(pb.y - o1) : big);
  at.F2 = make_float2(va ? static_cast<float>(pa.z - o2) : big, vb ? static_cast<float>(pb.z - o2) : big);
  at.lo_thr = sm.R.lo_thr;
  at.hi_thr = sm.R.hi_thr;
  at.Sa = at.Sb = 0.0;
  at.ca = at.cb = 0;
  at.ha = at.hb = 0;
  WarpBox wb;
  {
    const WarpBox w1 = warp_box(va, at.F0.x, at.F1.x, at.F2.x);
    const WarpBox w2 = warp_box(vb, at.F0.y, at.F1.y, at.F2.y);
    wb.lo0 = fminf(w1.lo0, w2.lo0); wb.lo1 = fminf(w1.lo1, w2.lo1); wb.lo2 = fminf(w1.lo2, w2.lo2);
    wb.hi0 = fmaxf(w1.hi0, w2.hi0); wb.hi1 = fmaxf(w1.hi1, w2.hi1); wb.hi2 = fmaxf(w1.hi2, w2.hi2);
  }
  const float cull_thr = sm.R.hi_thr * 1.0001f;
  double Bc = -0x1p1000;  // running CTA shift (log2 units)

  unsigned bandmask = 0;
  fused_scan32<1, DEBUG, KS>(sm, A, wb, cull_thr, Bc, at, bandmask, split);

  if constexpr (KS > 1) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    SplitXchg32* x = reinterpret_cast<SplitXchg32*>(&sm.colW[0][0]);
    const int t = threadIdx.x;
    x->S[0][t] = at.Sa; x->S[1][t] = at.Sb;
    x->C[0][t] = at.ca; x->C[1][t] = at.cb;
    if (DEBUG) { x->H[0][t] = at.ha; x->H[1][t] = at.hb; }
    if (t == 0) x->B = Bc;
    cl.sync();  // partials of every split visible cluster-wide
    double Bm = -0x1p1000;
#pragma unroll
    for (int r = 0; r < KS; ++r) Bm = fmax(Bm, cl.map_shared_rank(x, r)->B);
    double sa = 0.0, sb = 0.0;
    uint32_t ca = 0, cb = 0;
    uint64_t ha = 0, hb = 0;
#pragma unroll
    for (int r = 0; r < KS; ++r) {  // rank order: identical in every CTA
      const SplitXchg32* xr = cl.map_shared_rank(x, r);
      const double f = exp2(xr->B - Bm);
      sa += xr->S[0][t] * f; sb += xr->S[1][t] * f;
      ca += xr->C[0][t]; cb += xr->C[1][t];
      if (DEBUG) { ha += xr->H[0][t]; hb += xr->H[1][t]; }
    }
    cl.sync();  // no CTA reuses colW (phase 2) while a peer still reads it
    at.Sa = sa; at.Sb = sb; at.ca = ca; at.cb = cb; at.ha = ha; at.hb = hb;
    Bc = Bm;
  }

  const bool primary = split == 0;
  double wa, wb2;
  fused_finalize<DEBUG>(A, Bc, true, va, at.ca != 0u, static_cast<double>(at.ca + at.cb), at.ca,
                        at.Sa, 0.0, at.qa, at.ha, wa, 0x1p-80, primary);
  fused_finalize<DEBUG>(A, Bc, true, vb, at.cb != 0u, 0.0, at.cb, at.Sb, 0.0, at.qb, at.hb, wb2,
                        0x1p-80, primary);
  at.wa = static_cast<float>(wa);
  at.wb = static_cast<float>(wb2);

  fused_scan32<2, DEBUG, KS>(sm, A, wb, cull_thr, Bc, at, bandmask, split);
}

template <bool DEBUG>
__global__ void __launch_bounds__(kT, 4)
trunc_fused32(FusedArgs A) {
  __shared__ Fused32Smem sm;
  int chunk = static_cast<int>(blockIdx.x);
  if (A.chunk_order) {  // the split chunks lead the order (trunc_fused32_split)
    const int pos = *A.heavy_count + chunk;
    if (pos >= (A.nq + kFA - 1) / kFA) return;
    chunk = A.chunk_order[pos];
  }
  if (A.role) {
    const unsigned char r = A.role[chunk];
    if (r == kRoleOther) return fused_skip_chunk<DEBUG>(A, chunk);
    if (r == kRoleSplit) return;  // run by trunc_fused32_split
  }
  fused32_body<DEBUG, 1>(sm, A, chunk, 0);
}

template <bool DEBUG>
__global__ void __cluster_dims__(kSplit, 1, 1) __launch_bounds__(kT, 4)
trunc_fused32_split(FusedArgs A) {
  __shared__ Fused32Smem sm;
  __shared__ int next;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int split = static_cast<int>(cl.block_rank());
  const int count = *A.heavy_count;
  for (;;) {  // as trunc_fused_split
    if (split == 0 && threadIdx.x == 0) next = atomicAdd(A.queue, 1);
    cl.sync();
    const int h = *cl.map_shared_rank(&next, 0);
    if (h >= count) {
      cl.sync();
      break;
    }
    fused32_body<DEBUG, kSplit>(sm, A, A.chunk_order[h], split);
    __syncthreads();
  }
}

// Chunk cost = the chunk's candidate pairs of the last evaluation; key =
// (~cost << 32 | chunk) so an ascending sort puts the heaviest first.
// Bounding box of every Hilbert chunk (warp per chunk; cached with the order).
__global__ void chunk_box_kernel(const double4* __restrict__ xs, int nq, int nblk, double* __restrict__ box) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= nblk) return;
  double v[6] = {INFINITY, INFINITY, INFINITY, INFINITY, INFINITY, INFINITY};  // lo, -hi
  for (int k = lane; k < kFA; k += 32) {
    const int q = c * kFA + k;
    if (q >= nq) break;
    const double4 p = xs[q];
    v[0] = fmin(v[0], p.x); v[1] = fmin(v[1], p.y); v[2] = fmin(v[2], p.z);
    v[3] = fmin(v[3], -p.x); v[4] = fmin(v[4], -p.y); v[5] = fmin(v[5], -p.z);
  }
#pragma unroll
  for (int d = 0; d < 6; ++d) v[d] = warp_min(v[d]);
  if (lane == 0) {
    double* o = box + 6 * static_cast<size_t>(c);
    o[0] = v[0]; o[1] = v[1]; o[2] = v[2];
    o[3] = -v[3]; o[4] = -v[4]; o[5] = -v[5];
  }
}

// Targets within reach of a box (its cell rows, as fused_scan forms them).
__device__ __forceinline__ unsigned warp_rows_count(const GridDev& g, const double* bx, double r,
                                                    const int* __restrict__ cell_start, int lane) {
  Region R;
  for (int d = 0; d < 6; ++d) R.box[d] = bx[d];
  for (int d = 0; d < 3; ++d) {
    R.c_lo[d] = cell_of(g, d, R.box[d] - r);
    R.c_hi[d] = cell_of(g, d, R.box[d + 3] + r);
  }
  const int nrows = (R.c_hi[1] - R.c_lo[1] + 1) * (R.c_hi[2] - R.c_lo[2] + 1);
  unsigned acc = 0;
  for (int ri = lane; ri < nrows; ri += 32) {
    int st, ln;
    row_range(g, R, r, cell_start, ri, st, ln);
    acc += static_cast<unsigned>(ln);
  }
  return __reduce_add_sync(0xffffffffu, acc);
}

// Work estimate per chunk (warp per chunk): the targets its CTA scans (rows
// within reach of the chunk box: pre-tests, staging) plus kPairWeight x the
// targets within reach of the chunk centre (~ accepted pairs / 256), plus a
// fixed cost and, when nothing is within reach of the centre, the nearest
// searches of its atoms.  Depends only on the atoms, targets and cutoff, so the roles
// below (and with them the summation order of the result) are deterministic.
__global__ void chunk_scan_cost(const double* __restrict__ box, int nblk, GridDev g, double r_scan,
                                const int* __restrict__ cell_start, unsigned long long* __restrict__ cost,
                                unsigned long long* __restrict__ w) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= nblk) return;
  double bx[6], ctr[6];
  for (int d = 0; d < 6; ++d) bx[d] = box[6 * static_cast<size_t>(c) + d];
  for (int d = 0; d < 3; ++d) ctr[d] = ctr[d + 3] = 0.5 * (bx[d] + bx[d + 3]);
  const unsigned scan = warp_rows_count(g, bx, r_scan, cell_start, lane);
  const unsigned ball = warp_rows_count(g, ctr, r_scan, cell_start, lane);
  if (lane == 0) {
    // (an empty centre ball: most atoms of the chunk take the nearest path)
    const unsigned long long wc = scan + kPairWeight * ball + kChunkBase + (ball == 0 ? kFA * kEmptyAtomCost : 0);
    cost[c] = wc;
    w[c] = wc;
  }
}

// Per-chunk role for this rank.  Multi-rank partitioned atoms: the Hilbert
// chunk sequence is cut into `world` contiguous ranges of equal weight
// (scan cost + kChunkBase; a chunk goes to the rank holding the midpoint of
// its interval in the exclusive prefix `pre`), the same on every rank since
// the costs are.  This rank's chunks whose scan exceeds max(alpha x its
// per-slot share, floor) run split.  range = {first atom, end atom, atom
// count, split count, split queue} of this rank.
__global__ void chunk_role_kernel(const unsigned long long* __restrict__ cost,
                                  const unsigned long long* __restrict__ w,
                                  const unsigned long long* __restrict__ pre, int nblk, int nq, int rank,
                                  int world, double slots, double alpha, double floor_t,
                                  unsigned char* __restrict__ role, int* __restrict__ range) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nblk) return;
  const double tot = static_cast<double>(pre[nblk - 1] + w[nblk - 1]);
  const double wc = static_cast<double>(w[c]);
  const bool mine = world == 1 ||
                    min(world - 1, static_cast<int>((static_cast<double>(pre[c]) + 0.5 * wc) / tot * world)) == rank;
  const double thr = fmax(alpha * tot / (static_cast<double>(world) * slots), floor_t);
  const bool heavy = mine && alpha >= 0.0 && static_cast<double>(cost[c]) > thr;
  role[c] = !mine ? kRoleOther : heavy ? kRoleSplit : kRoleMine;
  if (heavy) atomicAdd(range + 3, 1);
  if (mine) {
    const int q1 = min(nq, (c + 1) * kFA);
    atomicMin(range, c * kFA);
    atomicMax(range + 1, q1);
    atomicAdd(range + 2, q1 - c * kFA);
  }
}

__global__ void chunk_range_init(int* __restrict__ range, int nq) {
  range[0] = nq;
  range[1] = 0;
  range[2] = 0;
  range[3] = 0;
  range[4] = 0;
}

__global__ void chunk_range_final(int* __restrict__ range, double* __restrict__ visited) {
  if (range[2] == 0) range[0] = range[1] = 0;  // (no atoms: empty range)
  if (visited) *visited = static_cast<double>(range[2]);
}

// The schedule (chunk_order): this rank's split chunks, then its other
// chunks, each heaviest first by scan cost (inverted log2 bucket in key bits
// 32-47, the class in bits 48-49; stable, so ties keep chunk order), then
// the other ranks' chunks.  Scheduling only; results do not depend on it.
__global__ void chunk_order_keys(const unsigned long long* __restrict__ cost,
                                 const unsigned char* __restrict__ role, int nblk,
                                 uint64_t* __restrict__ keys, int* __restrict__ idx) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nblk) return;
  const unsigned char r = role[c];
  const uint32_t cls = r == kRoleSplit ? 0u : r == kRoleMine ? 1u : 2u;
  // quarter-octave cost buckets, Hilbert order inside a bucket: the heavy
  // chunks still lead, while chunks of similar cost (all of them on a
  // uniform instance) keep their spatial order, so concurrently resident
  // CTAs share staged target rows in L2 (a fine-grained cost sort scattered
  // them: cfg5 DRAM traffic 1.4 -> 5.5 GB per evaluation)
  const uint32_t bucket =
      0xFFFFu - min(0xFFFFu, static_cast<uint32_t>(log2(static_cast<double>(cost[c]) + 1.0) * 4.0));
  keys[c] = (static_cast<uint64_t>((cls << 16) | bucket) << 32) | static_cast<uint32_t>(c);
  idx[c] = c;
}

// The accumulator is indexed by cell-order position k (a CTA's reductions
// land in the few contiguous runs of its scanned rows: L2-friendly), the
// result by original target index tperm[k].
__global__ void trunc_assemble_fp(const unsigned long long* __restrict__ gacc,
                                  const int* __restrict__ tperm, int n, double* __restrict__ res) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) res[tperm[k]] = fp_limbs_to_double(gacc + kLimbs * static_cast<size_t>(k));
}

__global__ void set_visited(double* __restrict__ res, int n, double nq) {
  res[n + kResVisited] = nq;
}

template <typename T>
__global__ void scatter_debug(const T* __restrict__ src, const int* __restrict__ perm,
                              int nq, T* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq) dst[perm[i]] = src[i];
}

__global__ void dense_debug_kernel(const double* __restrict__ atomL, int nq, int n,
                                   uint32_t* __restrict__ count,
                                   uint64_t* __restrict__ hash,
                                   double* __restrict__ log_s) {
  __shared__ unsigned long long hsum;
  if (threadIdx.x == 0) hsum = 0;
  __syncthreads();
  unsigned long long h = 0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) h += candidate_hash_term(j);
  atomicAdd(&hsum, h);
  __syncthreads();
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    count[q] = static_cast<uint32_t>(n);
    hash[q] = hsum;
    log_s[q] = atomL[q];
  }
}

__global__ void nearest_points_kernel(const double* __restrict__ pts, int m,
                                      const double4* __restrict__ ys,
                                      const int* __restrict__ tperm,
                                      const int* __restrict__ cell_start, GridDev g,
                                      unsigned long long* __restrict__ out,
                                      double* __restrict__ d2_out) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < m; i += nwarps) {
    double bd;
    int bj, bk;
    warp_nearest(g, ys, tperm, cell_start, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], bd, bj, bk);
    if (lane == 0) {
      out[i] = static_cast<unsigned long long>(bj);
      if (d2_out) d2_out[i] = bd;
    }
  }
}

__global__ void atoms_to_pts(const double4* __restrict__ x, int nq, double* __restrict__ pts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq) {
    pts[3 * i] = x[i].x;
    pts[3 * i + 1] = x[i].y;
    pts[3 * i + 2] = x[i].z;
  }
}

__global__ void max_cost_kernel(const double* __restrict__ d2, int m, double* __restrict__ out) {
  __shared__ double sh[256];
  double mx = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) mx = fmax(mx, 0.5 * d2[i]);
  mx = block_max<256>(mx, sh);
  if (threadIdx.x == 0) *out = mx;
}


double cells_per_radius() {
  static const double v = [] {
    const char* e = std::getenv("RSOT_CELLS_PER_RADIUS");
    const double x = e ? std::atof(e) : 0.0;
    return x >= 1.0 && x <= 16.0 ? x : g_cells_per_radius;
  }();
  return v;
}

template <typename T>
cudaError_t grow(T*& p, size_t& cap, size_t n) {
  if (n <= cap && p) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc(&p, sizeof(T) * (n ? n : 1));
  if (e == cudaSuccess) cap = n;
  return e;
}

template <typename T>
cudaError_t realloc_exact(T*& p, size_t n) {
  if (p) cudaFree(p);
  p = nullptr;
  return cudaMalloc(&p, sizeof(T) * (n ? n : 1));
}

uint64_t g_next_grid_id = 1;

#define TCK(call)                                                       \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) {                                            \
      err = std::string(#call) + ": " + cudaGetErrorString(e_);         \
      return 1;                                                         \
    }                                                                   \
  } while (0)

int ensure_key_buffers(TruncWorkspace& ws, int n, std::string& err) {
  if (static_cast<size_t>(n) <= ws.keys_cap && ws.keys) return 0;
  const size_t c = std::max(n, 1);
  TCK(realloc_exact(ws.keys, c));
  TCK(realloc_exact(ws.keys2, c));
  TCK(realloc_exact(ws.idx, c));
  TCK(realloc_exact(ws.idx2, c));
  ws.keys_cap = ws.idx_cap = c;
  return 0;
}

// Stable radix sort of ws.keys/ws.idx (n entries, end_bit key bits); the
// sorted permutation lands in ws.idx2 and the sorted keys in ws.keys2.
int radix_sort(TruncWorkspace& ws, int n, int end_bit, cudaStream_t s, std::string& err,
               int begin_bit = 0) {
  size_t bytes = 0;
  TCK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, ws.keys, ws.keys2, ws.idx, ws.idx2, n, begin_bit,
                                      end_bit, s));
  if (bytes > ws.cub_bytes) {
    if (ws.cub_tmp) cudaFree(ws.cub_tmp);
    ws.cub_tmp = nullptr;
    TCK(cudaMalloc(&ws.cub_tmp, bytes));
    ws.cub_bytes = bytes;
  }
  bytes = ws.cub_bytes;
  TCK(cub::DeviceRadixSort::SortPairs(ws.cub_tmp, bytes, ws.keys, ws.keys2, ws.idx, ws.idx2, n,
                                      begin_bit, end_bit, s));
  return 0;
}

// Hilbert order of a point set (radius independent; built once).
int build_hilbert(TruncWorkspace& ws, const double4* pts, int n, PointOrders& po,
                  cudaStream_t s, std::string& err) {
  if (po.hil_valid && po.n == n) return 0;
  if (ensure_key_buffers(ws, n, err)) return 1;
  TCK(realloc_exact(po.ph, n));
  TCK(realloc_exact(po.perm_h, n));
  if (n > 0) {
    // isotropic scale (the largest extent spans the curve): chunks of a flat
    // point set (e.g. one rank's slab) stay compact in space instead of
    // being squashed along the thin axis
    double ext = 0.0;
    for (int d = 0; d < 3; ++d) ext = std::max(ext, po.bbox_hi[d] - po.bbox_lo[d]);
    double sc[3];
    for (int d = 0; d < 3; ++d)
      sc[d] = (ext > 0.0 && po.bbox_hi[d] > po.bbox_lo[d]) ? static_cast<double>(1u << kHilBits) / ext
                                                           : 0.0;
    (note_launch(), hilbert_keys_kernel<<<(n + 255) / 256, 256, 0, s>>>(pts, n, po.bbox_lo[0], po.bbox_lo[1],
                                                        po.bbox_lo[2], sc[0], sc[1], sc[2],
                                                        ws.keys, ws.idx));
    if (radix_sort(ws, n, 3 * kHilBits, s, err)) return 1;
    (note_launch(), gather4_kernel<<<(n + 255) / 256, 256, 0, s>>>(pts, ws.idx2, n, po.ph));
    TCK(cudaMemcpyAsync(po.perm_h, ws.idx2, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
  }
  TCK(cudaGetLastError());
  po.n = n;
  po.hil_valid = true;
  return 0;
}

// Cell order for grid g.
int build_cells(TruncWorkspace& ws, const double4* pts, int n, const GridDesc& g,
                PointOrders& po, cudaStream_t s, std::string& err) {
  if (po.cell_valid && po.grid_id == g.id && po.ncell_pts == n) return 0;
  if (ensure_key_buffers(ws, n, err)) return 1;
  TCK(realloc_exact(po.pc, n));
  TCK(realloc_exact(po.perm_c, n));
  TCK(realloc_exact(po.cell_start, g.ncells + 1));
  const GridDev gd = to_dev(g);
  if (n > 0) {
    (note_launch(), cell_keys_kernel<<<(n + 255) / 256, 256, 0, s>>>(pts, n, gd, ws.keys, ws.idx));
    int end_bit = 3 * kMortonBits;
    while ((1ll << (end_bit - 3 * kMortonBits)) < g.ncells) ++end_bit;
    if (radix_sort(ws, n, end_bit, s, err)) return 1;
    (note_launch(), gather4_kernel<<<(n + 255) / 256, 256, 0, s>>>(pts, ws.idx2, n, po.pc));
    TCK(cudaMemcpyAsync(po.perm_c, ws.idx2, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
  }
  (note_launch(), cell_start_kernel<<<(n + 1 + 255) / 256, 256, 0, s>>>(ws.keys2, n, g.ncells, po.cell_start));
  TCK(cudaGetLastError());
  po.grid_id = g.id;
  po.ncell_pts = n;
  po.cell_valid = true;
  return 0;
}

// Grid over the target bounding box with cell side ~max(r/2, spacing).
GridDesc plan_grid(const double blo[3], const double bhi[3], int n, double r) {
  GridDesc g;
  int active = 0;
  double vol = 1.0;
  for (int d = 0; d < 3; ++d)
    if (bhi[d] > blo[d]) {
      ++active;
      vol *= bhi[d] - blo[d];
    }
  double hmin = 1.0;
  if (active > 0) hmin = std::pow(vol / std::max(1.0, n / 2.0), 1.0 / active);
  // cell side ~ r / cells_per_radius on a quarter-octave ladder: the grid is
  // a function of (bounding box, n, r) alone, so every rank of a multi-GPU
  // run cuts the same chunk costs (chunk_scan_cost) whatever it evaluated
  // before, and the cached grid is reused while r stays on its rung
  double want = r / cells_per_radius();
  if (want > 0.0 && std::isfinite(want)) want = std::exp2(std::round(4.0 * std::log2(want)) * 0.25);
  double h = std::max(want, hmin);
  if (!(h > 0.0) || !std::isfinite(h)) h = 1.0;
  for (;;) {
    long long nc = 1;
    for (int d = 0; d < 3; ++d) {
      const double ext = bhi[d] - blo[d];
      g.dims[d] = ext > 0.0 ? static_cast<int>(std::min(std::floor(ext / h) + 1.0, 8192.0)) : 1;
      nc *= g.dims[d];
    }
    if (nc <= (1ll << 26)) {
      g.ncells = nc;
      break;
    }
    h *= 1.25;
  }
  for (int d = 0; d < 3; ++d) g.lo[d] = blo[d];
  g.h = h;
  return g;
}

// ---------------------------------------------------------------------------
// PlanView (proj/src/plan.cpp) on the GPU: explicit candidate lists (the
// ctor's ball query + nearest fallback, ascending per atom) and the
// plan-density reductions over them (target marginals, first moments,
// barycentric and modal maps).

// Warp per atom: candidate indices into idx[off[q], off[q+1]) (unordered;
// sorted afterwards), the nearest target when the ball is empty.
__global__ void plan_fill_kernel(const double4* __restrict__ xs, int nq,
                                 const double4* __restrict__ ys, const int* __restrict__ tperm,
                                 const int* __restrict__ cell_start, GridDev g, double r2,
                                 double r_scan, int scan, const unsigned long long* __restrict__ off,
                                 unsigned long long* __restrict__ idx, int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int q = warp; q < nq; q += nwarps) {
    const double4 x = xs[q];
    const unsigned long long base = off[q];
    unsigned long long pos = 0;
    if (scan) {
      const double v[3] = {x.x, x.y, x.z};
      int c_lo[3], c_hi[3];
      for (int d = 0; d < 3; ++d) {
        c_lo[d] = cell_of(g, d, v[d] - r_scan);
        c_hi[d] = cell_of(g, d, v[d] + r_scan);
      }
      for (int cz = c_lo[2]; cz <= c_hi[2]; ++cz)
        for (int cy = c_lo[1]; cy <= c_hi[1]; ++cy) {
          const long long row = (static_cast<long long>(cz) * g.dims[1] + cy) * g.dims[0];
          const int b = cell_start[row + c_lo[0]], e = cell_start[row + c_hi[0] + 1];
          for (int k0 = b; k0 < e; k0 += 32) {
            const int k = k0 + lane;
            bool in = false;
            if (k < e) {
              const double4 y = ys[k];
              in = exact_inside(x.x, x.y, x.z, y.x, y.y, y.z, r2);
            }
            const unsigned m = __ballot_sync(0xffffffffu, in);
            if (in) idx[base + pos + __popc(m & lt)] = static_cast<unsigned long long>(tperm[k]);
            pos += __popc(m);
          }
        }
    }
    if (pos == 0) {
      double bd;
      int bj, bk;
      warp_nearest(g, ys, tperm, cell_start, x.x, x.y, x.z, bd, bj, bk);  // index.nearest
      if (lane == 0) idx[base] = static_cast<unsigned long long>(bj);
      pos = 1;
    }
    if (lane == 0 && pos != off[q + 1] - base) atomicExch(bad, 1);
  }
}

// Geodesic cost: full scan {j : c < cutoff} in index order (evaluate.cpp /
// plan.cpp full-scan branch) decided as clamped dot >= tmin
// (geo_dot_threshold: the reference's acos on the host), Euclidean nearest
// when empty.
__global__ void plan_fill_geo_kernel(const double4* __restrict__ xs, int nq,
                                     const double4* __restrict__ yo, int n, double tmin,
                                     const double4* __restrict__ ys, const int* __restrict__ tperm,
                                     const int* __restrict__ cell_start, GridDev g,
                                     const unsigned long long* __restrict__ off,
                                     unsigned long long* __restrict__ idx, int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int q = warp; q < nq; q += nwarps) {
    const double4 x = xs[q];
    const unsigned long long base = off[q];
    unsigned long long pos = 0;
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int k = k0 + lane;
      bool in = false;
      if (k < n) {
        const double4 y = yo[k];
        const double d = __dadd_rn(__dadd_rn(__dmul_rn(x.x, y.x), __dmul_rn(x.y, y.y)), __dmul_rn(x.z, y.z));
        in = (d < -1.0 ? -1.0 : (1.0 < d ? 1.0 : d)) >= tmin;
      }
      const unsigned m = __ballot_sync(0xffffffffu, in);
      if (in) idx[base + pos + __popc(m & lt)] = static_cast<unsigned long long>(k);
      pos += __popc(m);
    }
    if (pos == 0) {
      double bd;
      int bj, bk;
      warp_nearest(g, ys, tperm, cell_start, x.x, x.y, x.z, bd, bj, bk);
      if (lane == 0) idx[base] = static_cast<unsigned long long>(bj);
      pos = 1;
    }
    if (lane == 0 && pos != off[q + 1] - base) atomicExch(bad, 1);
  }
}

// Warp per atom over its candidates (all targets when off == nullptr):
// p = exp(e - log_S_q) exactly as plan_density (plan.cpp:70-83); target
// mass and first moments into 192-bit fixed point (moments of x - lo, so
// every term is non-negative; order independent), barycentric image and
// modal argmax (lowest index on ties) per atom.
template <bool GEO>
__global__ void plan_moments_kernel(const double4* __restrict__ xs, int nq,
                                    const double4* __restrict__ ys, int n,
                                    const double* __restrict__ psi, double eps,
                                    const double* __restrict__ log_s,
                                    const unsigned long long* __restrict__ off,
                                    const unsigned long long* __restrict__ idx, double lo0,
                                    double lo1, double lo2, unsigned long long* __restrict__ acc,
                                    double* __restrict__ map, unsigned long long* __restrict__ modal) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int q = warp; q < nq; q += nwarps) {
    const double4 x = xs[q];
    const double L = log_s[q];
    const unsigned long long b = off ? off[q] : 0ull;
    const unsigned long long e = off ? off[q + 1] : static_cast<unsigned long long>(n);
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    double best = -INFINITY;
    unsigned long long bj = ~0ull;
    for (unsigned long long k = b + lane; k < e; k += 32) {
      const unsigned long long j = off ? idx[k] : k;
      const double4 y = ys[j];
      const double c = GEO ? geo_cost(x.x, x.y, x.z, y.x, y.y, y.z)
                           : __dmul_rn(0.5, exact_sqdist(x.x, x.y, x.z, y.x, y.y, y.z));
      const double ex = __dadd_rn(__ddiv_rn(__dsub_rn(psi[j], c), eps), y.w);
      const double p = exp(__dsub_rn(ex, L));
      if (acc) {
        const double w = __dmul_rn(p, x.w);
        unsigned long long* a = acc + 12 * j;
        fp_add(a, w);
        fp_add(a + 3, __dmul_rn(w, x.x - lo0));
        fp_add(a + 6, __dmul_rn(w, x.y - lo1));
        fp_add(a + 9, __dmul_rn(w, x.z - lo2));
      }
      t0 = __dadd_rn(t0, __dmul_rn(p, y.x));
      t1 = __dadd_rn(t1, __dmul_rn(p, y.y));
      t2 = __dadd_rn(t2, __dmul_rn(p, y.z));
      const double score = __dadd_rn(__dsub_rn(psi[j], c), __dmul_rn(eps, y.w));
      if (score > best || (score == best && j < bj)) {
        best = score;
        bj = j;
      }
    }
    t0 = warp_sum(t0);
    t1 = warp_sum(t1);
    t2 = warp_sum(t2);
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const unsigned long long oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ob > best || (ob == best && oj < bj)) {
        best = ob;
        bj = oj;
      }
    }
    if (lane == 0) {
      if (map) {
        map[3 * q] = t0;
        map[3 * q + 1] = t1;
        map[3 * q + 2] = t2;
      }
      if (modal) modal[q] = bj;
    }
  }
}

__global__ void plan_assemble_kernel(const unsigned long long* __restrict__ acc, int n, double lo0,
                                     double lo1, double lo2, double* __restrict__ marginal,
                                     double* __restrict__ moment) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const unsigned long long* a = acc + 12 * static_cast<size_t>(j);
  const double t = fp_to_double(a);
  if (marginal) marginal[j] = t;
  if (moment) {
    moment[3 * j] = fp_to_double(a + 3) + lo0 * t;
    moment[3 * j + 1] = fp_to_double(a + 6) + lo1 * t;
    moment[3 * j + 2] = fp_to_double(a + 9) + lo2 * t;
  }
}

}  // namespace

void AtomCells::release() {
  if (chunk_box) cudaFree(chunk_box);
  chunk_box = nullptr;
  box_chunks = 0;
  PointOrders::release();
}

void PointOrders::release() {
  void* ptrs[] = {ph, perm_h, pc, perm_c, cell_start};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  ph = pc = nullptr;
  perm_h = perm_c = cell_start = nullptr;
  hil_valid = cell_valid = false;
}

void TruncWorkspace::release() {
  void* ptrs[] = {cub_tmp, keys, keys2, idx, idx2, b2s, S, atomL, atomJ, atomD, cntd, emptyd, cnt,
                  hash, empty_fp, pts, near_out, red, chunk_cost, heavy_flag,
                  chunk_w, chunk_pre, part_range, mbuf, mbusy, mticket, rbuf};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (fork_ev) cudaEventDestroy(fork_ev);
  if (join_ev) cudaEventDestroy(join_ev);
  if (side) cudaStreamDestroy(side);
  *this = TruncWorkspace();
}

static double env_double(const char* name, double dflt) {
  const char* e = std::getenv(name);
  if (!e || !*e) return dflt;
  char* end = nullptr;
  const double v = std::strtod(e, &end);
  return end != e ? v : dflt;
}

cudaError_t trunc_read_overflow(unsigned* h_flag, cudaStream_t s) {
  return cudaMemcpyFromSymbolAsync(h_flag, g_fp_overflow, sizeof(unsigned), 0, cudaMemcpyDeviceToHost, s);
}

cudaError_t trunc_clear_overflow() {
  const unsigned zero = 0;
  return cudaMemcpyToSymbol(g_fp_overflow, &zero, sizeof(unsigned));
}

// Keeps the mask pool's leading words resident in L2 (access-policy window,
// persisting): phase 1 writes them and phase 2 of the same CTA reads them
// back milliseconds later, while the streamed atoms and targets would
// otherwise evict them to DRAM (round-1 ncu: ~2.6 GB of the 4.3 GB per cfg5
// evaluation).  RSOT_CUDA_L2_PERSIST=0 disables it.  Best effort: errors
// only leave the pool uncached-preferred.
static void mask_l2_window(TruncWorkspace& ws, cudaStream_t s) {
  if (env_double("RSOT_CUDA_L2_PERSIST", 1.0) == 0.0) return;
  int dev = 0, max_persist = 0, max_win = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  const size_t want = static_cast<size_t>(64) << 20;  // ~120 words of every slot
  const size_t win = std::min<size_t>({want, static_cast<size_t>(max_persist), static_cast<size_t>(max_win)});
  if (win == 0) return;
  size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
  if (cur < win) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, win);
  cudaStreamAttrValue v = {};
  v.accessPolicyWindow.base_ptr = ws.mbuf;
  v.accessPolicyWindow.num_bytes = win;
  v.accessPolicyWindow.hitRatio = 1.0f;
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
  if (ws.side) cudaStreamSetAttribute(ws.side, cudaStreamAttributeAccessPolicyWindow, &v);
  cudaGetLastError();  // (best effort)
}

static int ensure_target_cells(TruncWorkspace& ws, const DeviceTargets& t, TargetCells& tc,
                               double r, cudaStream_t s, std::string& err) {
  if (!tc.bbox_set) {
    err = "target bounding box not set";
    return 1;
  }
  GridDesc g = plan_grid(tc.bbox_lo, tc.bbox_hi, t.n, r);
  if (tc.cell_valid && tc.g.h == g.h && tc.g.dims[0] == g.dims[0] && tc.g.dims[1] == g.dims[1] &&
      tc.g.dims[2] == g.dims[2])
    return 0;
  g.id = g_next_grid_id++;
  tc.cell_valid = false;
  if (build_cells(ws, t.y, t.n, g, tc, s, err)) return 1;
  tc.g = g;
  tc.built_r = r;
  return 0;
}

static int ensure_atom_order(TruncWorkspace& ws, const DeviceAtoms& a, AtomCells& ac,
                             cudaStream_t s, std::string& err) {
  if (!ac.bbox_set) {
    err = "atom bounding box not set";
    return 1;
  }
  if (build_hilbert(ws, a.x, a.nq, ac, s, err)) return 1;
  const int nblk = (a.nq + kFA - 1) / kFA;
  if (ac.box_chunks != nblk && nblk > 0) {
    TCK(realloc_exact(ac.chunk_box, 6 * static_cast<size_t>(nblk)));
    (note_launch(), chunk_box_kernel<<<(nblk + 7) / 8, 256, 0, s>>>(ac.ph, a.nq, nblk, ac.chunk_box));
    ac.box_chunks = nblk;
  }
  return 0;
}

static int ensure_trunc_ws(TruncWorkspace& ws, int nq, int n, std::string& err) {
  if (static_cast<size_t>(nq) > ws.atom_cap || !ws.S) {
    const size_t c = std::max<size_t>(nq, 1);
    TCK(realloc_exact(ws.S, c));
    TCK(realloc_exact(ws.atomL, c));
    TCK(realloc_exact(ws.atomJ, c));
    TCK(realloc_exact(ws.atomD, c));
    TCK(realloc_exact(ws.cntd, c));
    TCK(realloc_exact(ws.emptyd, c));
    TCK(realloc_exact(ws.cnt, c));
    TCK(realloc_exact(ws.hash, c));
    ws.atom_cap = c;
  }
  if (static_cast<size_t>(n) > ws.tgt_cap || !ws.b2s) {
    const size_t c = std::max<size_t>(n, 1);
    TCK(realloc_exact(ws.b2s, c));
    TCK(realloc_exact(ws.empty_fp, kLimbs * c));
    ws.tgt_cap = c;
  }
  if (!ws.red) TCK(cudaMalloc(&ws.red, sizeof(double) * 4096));
  const size_t nblk = (static_cast<size_t>(nq) + kFA - 1) / kFA;
  if (nblk > ws.chunk_cap || !ws.chunk_cost) {
    const size_t c = std::max<size_t>(nblk, 1);
    TCK(realloc_exact(ws.chunk_cost, c));
    TCK(realloc_exact(ws.chunk_w, c));
    TCK(realloc_exact(ws.chunk_pre, c));
    TCK(realloc_exact(ws.heavy_flag, c));
    if (!ws.part_range) TCK(cudaMalloc(&ws.part_range, 5 * sizeof(int)));
    ws.chunk_cap = c;
  }
  if (ws.split_clusters == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kSplit);
    cfg.blockDim = dim3(kT);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kSplit;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0, ncl32 = 0;
    TCK(cudaOccupancyMaxActiveClusters(&ncl, trunc_fused_split<false>, &cfg));
    TCK(cudaOccupancyMaxActiveClusters(&ncl32, trunc_fused32_split<false>, &cfg));
    ws.split_clusters = std::max(1, ncl);
    ws.split_clusters32 = std::max(1, ncl32);
  }
  if (!ws.side) {
    int least = 0, greatest = 0;
    TCK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    TCK(cudaStreamCreateWithPriority(&ws.side, cudaStreamNonBlocking, greatest));
    TCK(cudaEventCreateWithFlags(&ws.fork_ev, cudaEventDisableTiming));
    TCK(cudaEventCreateWithFlags(&ws.join_ev, cudaEventDisableTiming));
  }
  return 0;
}

int run_truncated(TruncWorkspace& ws, const DeviceAtoms& a, AtomCells& ac,
                  const DeviceTargets& t, TargetCells& tc, EvalBuffers& b,
                  double eps, double cutoff, int num_sms, DebugOut* dbg,
                  cudaStream_t s, std::string& err, bool fp32, int part_rank, int part_world) {
  // cost.hpp:38-42 and spatial_index.cpp:50,54, evaluated on the host exactly
  // as the reference does.
  const double radius = cutoff < 0.0 ? 0.0 : std::sqrt(2.0 * cutoff);
  const double r2 = radius * radius;
  const bool scan = radius > 0.0;
  const double r_use = scan ? radius : 0.0;
  const double r_scan = r_use * (1.0 + 1e-9) + 1e-300;
  const int n = t.n, nq = a.nq;
  if (ensure_target_cells(ws, t, tc, r_use, s, err)) return 1;
  if (ensure_atom_order(ws, a, ac, s, err)) return 1;
  if (ensure_trunc_ws(ws, nq, n, err)) return 1;
  const GridDev g = to_dev(tc.g);
  const double c2 = kLog2e / (2.0 * eps);

  TCK(cudaMemsetAsync(b.scal + kSlotFlagCount, 0, sizeof(double), s));
  TCK(cudaMemsetAsync(ws.empty_fp, 0, sizeof(unsigned long long) * kLimbs * static_cast<size_t>(n), s));
  (note_launch(), gather_d_kernel<<<(n + 255) / 256, 256, 0, s>>>(b.b2, tc.perm_c, n, ws.b2s));
  if (nq > 0) {
    FusedArgs A;
    A.xs = ac.ph; A.nq = nq; A.ys = tc.pc; A.b2s = ws.b2s; A.tperm = tc.perm_c;
    A.cell_start = tc.cell_start; A.g = g; A.scal = b.scal; A.psi = b.psi;
    A.c2 = c2; A.r2 = r2; A.r_scan = r_scan; A.eps = eps;
    A.atomJ = ws.atomJ; A.atomD = ws.atomD; A.cntd = ws.cntd; A.emptyd = ws.emptyd;
    A.gacc = ws.empty_fp;
    A.dbg_cnt = reinterpret_cast<uint32_t*>(ws.S); A.dbg_hash = ws.hash; A.dbg_logs = ws.atomL;
    A.cnt_out = ws.cnt;
    const int nblk = (nq + kFA - 1) / kFA;
    A.chunk_order = nullptr;
    A.role = nullptr;
    A.heavy_count = ws.part_range + 3;
    A.queue = ws.part_range + 4;
    // phase-1 pair masks replayed by phase 2 (fp64 kernel; RSOT_CUDA_PAIR_MASKS=0: off)
    A.mbuf = nullptr; A.mbusy = nullptr; A.mticket = nullptr; A.mslots = 0; A.mwords = 0;
    A.rbuf = nullptr; A.rcap = 0;
    if (!fp32 && !dbg) {
      if (!ws.mbuf) {
        TCK(cudaMalloc(&ws.mbuf, sizeof(uint32_t) * (static_cast<size_t>(kMaskSlots) + 1) * (kMaskWords + 1) * kT));
        mask_l2_window(ws, s);
        TCK(cudaMalloc(&ws.mbusy, sizeof(int) * kMaskSlots));
        TCK(cudaMalloc(&ws.mticket, sizeof(unsigned)));
        TCK(cudaMemsetAsync(ws.mbusy, 0, sizeof(int) * kMaskSlots, s));
        TCK(cudaMemsetAsync(ws.mticket, 0, sizeof(unsigned), s));
      }
      if (!ws.rbuf && RSOT_P2_TM)
        TCK(cudaMalloc(&ws.rbuf, sizeof(int) * static_cast<size_t>(kRecSlots) * (kT / 32) * kRecCap));
      A.mbuf = ws.mbuf; A.mbusy = ws.mbusy; A.mticket = ws.mticket;
      A.mslots = env_double("RSOT_CUDA_PAIR_MASKS", 1.0) != 0.0 ? 1 : 0;  // 0: phase 2 recomputes
      // (tests: a small cap forces the overflow fallback in most CTAs)
      A.mwords = static_cast<int>(std::min<double>(kMaskWords, std::max(0.0, env_double("RSOT_CUDA_MASK_WORDS",
                                                                                        kMaskWords))));
      // item records of the target-major phase 2 (the same switches: no slots
      // -> no streams; a small word cap also caps the streams, 8 records a word)
      A.rbuf = ws.rbuf;
      A.rcap = A.mwords < kMaskWords ? 16 * A.mwords : kRecCap;
    }
    // Scan costs of the chunks -> roles (partitioned atoms: this rank's
    // work-balanced range; heavy chunks run split across a CTA cluster) and a
    // heaviest-first schedule.  RSOT_CUDA_SPLIT_ALPHA / RSOT_CUDA_SPLIT_FLOOR
    // override the split threshold (alpha < 0: off).
    // (one GPU: the heaviest-first order already hides chunks below a slot's
    // share, and split CTAs cost ~10 % more per target)
    const bool part = part_world > 1;
    const double alpha = env_double("RSOT_CUDA_SPLIT_ALPHA", part ? 0.5 : 1.0);
    const double floor_t = env_double("RSOT_CUDA_SPLIT_FLOOR", 131072.0);
    const bool split = alpha >= 0.0;
    const int* range = nullptr;
    if (nblk > 1 || part) {
      if (ensure_key_buffers(ws, nblk, err)) return 1;
      (note_launch(), chunk_scan_cost<<<(nblk + 7) / 8, 256, 0, s>>>(ac.chunk_box, nblk, g, r_scan, tc.cell_start,
                                                                    ws.chunk_cost, ws.chunk_w));
      size_t scan_bytes = 0, sort_bytes = 0;  // (sized together: no reallocation between the uses)
      TCK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, ws.chunk_w, ws.chunk_pre, nblk, s));
      TCK(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, ws.keys, ws.keys2, ws.idx, ws.idx2, nblk, 32, 50,
                                          s));
      if (std::max(scan_bytes, sort_bytes) > ws.cub_bytes) {
        if (ws.cub_tmp) cudaFree(ws.cub_tmp);
        ws.cub_tmp = nullptr;
        ws.cub_bytes = std::max(scan_bytes, sort_bytes);
        TCK(cudaMalloc(&ws.cub_tmp, ws.cub_bytes));
      }
      scan_bytes = ws.cub_bytes;
      TCK(cub::DeviceScan::ExclusiveSum(ws.cub_tmp, scan_bytes, ws.chunk_w, ws.chunk_pre, nblk, s));
      (note_launch(), chunk_range_init<<<1, 1, 0, s>>>(ws.part_range, nq));
      (note_launch(), chunk_role_kernel<<<(nblk + 255) / 256, 256, 0, s>>>(
          ws.chunk_cost, ws.chunk_w, ws.chunk_pre, nblk, nq, part_rank, part_world, 4.0 * num_sms, alpha,
          floor_t, ws.heavy_flag, ws.part_range));
      (note_launch(), chunk_range_final<<<1, 1, 0, s>>>(ws.part_range, part ? b.res + n + kResVisited : nullptr));
      (note_launch(), chunk_order_keys<<<(nblk + 255) / 256, 256, 0, s>>>(ws.chunk_cost, ws.heavy_flag, nblk,
                                                                         ws.keys, ws.idx));
      if (radix_sort(ws, nblk, 50, s, err, 32)) return 1;  // (class + bucket fields only)
      A.role = ws.heavy_flag;
      A.chunk_order = ws.idx2;
      if (part) range = ws.part_range;
    } else {
      (note_launch(), chunk_range_init<<<1, 1, 0, s>>>(ws.part_range, nq));  // (split count 0)
    }
    if (b.timing) cudaEventRecord(b.timing[1], s);
    if (fp32) {
      if (split && A.role) {
        TCK(cudaEventRecord(ws.fork_ev, s));
        TCK(cudaStreamWaitEvent(ws.side, ws.fork_ev, 0));
        const int grid = ws.split_clusters32 * kSplit;
        if (dbg)
          (note_launch(), trunc_fused32_split<true><<<grid, kT, 0, ws.side>>>(A));
        else
          (note_launch(), trunc_fused32_split<false><<<grid, kT, 0, ws.side>>>(A));
        TCK(cudaEventRecord(ws.join_ev, ws.side));
      }
      if (dbg)
        (note_launch(), trunc_fused32<true><<<nblk, kT, 0, s>>>(A));
      else
        (note_launch(), trunc_fused32<false><<<nblk, kT, 0, s>>>(A));
      if (split && A.role) TCK(cudaStreamWaitEvent(s, ws.join_ev, 0));
    } else {
      if (split && A.role) {
        // the split clusters go first on a high-priority stream, the rest
        // fill the GPU around them
        TCK(cudaEventRecord(ws.fork_ev, s));
        TCK(cudaStreamWaitEvent(ws.side, ws.fork_ev, 0));
        const int grid = ws.split_clusters * kSplit;
        if (dbg)
          (note_launch(), trunc_fused_split<true><<<grid, kT, 0, ws.side>>>(A));
        else
          (note_launch(), trunc_fused_split<false><<<grid, kT, 0, ws.side>>>(A));
        TCK(cudaEventRecord(ws.join_ev, ws.side));
      }
      if (dbg)
        (note_launch(), trunc_fused<true><<<nblk, kT, 0, s>>>(A));
      else
        (note_launch(), trunc_fused<false><<<nblk, kT, 0, s>>>(A));
      if (split && A.role) TCK(cudaStreamWaitEvent(s, ws.join_ev, 0));
    }
    if (b.timing) cudaEventRecord(b.timing[2], s);
    const int nb_near = std::min(4 * num_sms, (nq + 255) / 256 * 8 + 1);
    if (dbg)
      (note_launch(), trunc_nearest_empty<true><<<nb_near, 256, 0, s>>>(ac.ph, nq, ws.cnt, tc.pc, tc.perm_c,
                                                        tc.cell_start, g, b.psi, eps, ws.atomL,
                                                        ws.atomJ, ws.atomD, ws.empty_fp, ws.hash, range));
    else
      (note_launch(), trunc_nearest_empty<false><<<nb_near, 256, 0, s>>>(ac.ph, nq, ws.cnt, tc.pc, tc.perm_c,
                                                         tc.cell_start, g, b.psi, eps, ws.atomL,
                                                         ws.atomJ, ws.atomD, ws.empty_fp, ws.hash, range));
    if (b.timing) {
      cudaEventRecord(b.timing[3], s);
      cudaEventRecord(b.timing[4], s);
    }
    (note_launch(), trunc_assemble_fp<<<(n + 255) / 256, 256, 0, s>>>(ws.empty_fp, tc.perm_c, n, b.res));
    // J, D, pairs, empty in res[n + 0..3] (fixed-order sums of this rank's atoms)
    launch_det_sum4(ws.atomJ, ws.atomD, ws.cntd, ws.emptyd, nq, range, ws.red, b.res + n + kResJ, s);
    if (dbg) {
      (note_launch(), scatter_debug<uint32_t><<<(nq + 255) / 256, 256, 0, s>>>(
          reinterpret_cast<uint32_t*>(ws.S), ac.perm_h, nq, dbg->count));
      (note_launch(), scatter_debug<unsigned long long><<<(nq + 255) / 256, 256, 0, s>>>(
          reinterpret_cast<unsigned long long*>(ws.hash), ac.perm_h, nq,
          reinterpret_cast<unsigned long long*>(dbg->hash)));
      (note_launch(), scatter_debug<double><<<(nq + 255) / 256, 256, 0, s>>>(ws.atomL, ac.perm_h, nq,
                                                                          dbg->log_s));
    }
  } else {
    TCK(cudaMemsetAsync(b.res, 0, sizeof(double) * (n + kResTail), s));
  }
  if (!(part_world > 1 && nq > 0))  // (partitioned: chunk_role counted this rank's atoms)
    (note_launch(), set_visited<<<1, 1, 0, s>>>(b.res, n, static_cast<double>(nq)));
  TCK(cudaGetLastError());
  return 0;
}

void launch_dense_debug(const DeviceAtoms& a, const DeviceTargets& t, const EvalBuffers& b,
                        const DebugOut& dbg, cudaStream_t s) {
  if (a.nq == 0) return;
  (note_launch(), dense_debug_kernel<<<std::min(1024, (a.nq + 255) / 256), 256, 0, s>>>(
      b.atomL, a.nq, t.n, dbg.count, dbg.hash, dbg.log_s));
}

int run_nearest_points(TruncWorkspace& ws, const DeviceTargets& t, TargetCells& tc,
                       const double* xyz_host, size_t m, uint64_t* out_host, cudaStream_t s,
                       std::string& err) {
  if (ensure_target_cells(ws, t, tc, tc.cell_valid ? tc.built_r : 0.0, s, err)) return 1;
  size_t cap = 0;
  if (3 * m > ws.pts_cap || !ws.pts) {
    TCK(grow(ws.pts, cap, 3 * m));
    cap = 0;
    TCK(grow(ws.near_out, cap, m));
    ws.pts_cap = 3 * m;
  }
  TCK(cudaMemcpyAsync(ws.pts, xyz_host, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, s));
  (note_launch(), nearest_points_kernel<<<static_cast<int>(std::min<size_t>(1024, (m + 7) / 8)), 256, 0, s>>>(
      ws.pts, static_cast<int>(m), tc.pc, tc.perm_c, tc.cell_start, to_dev(tc.g), ws.near_out,
      nullptr));
  TCK(cudaMemcpyAsync(out_host, ws.near_out, sizeof(uint64_t) * m, cudaMemcpyDeviceToHost, s));
  TCK(cudaStreamSynchronize(s));
  return 0;
}

int run_covering_cost(TruncWorkspace& ws, const DeviceAtoms& a, const DeviceTargets& t,
                      TargetCells& tc, double* out, cudaStream_t s, std::string& err) {
  if (a.nq == 0) {
    err = "covering cost: empty input";
    return 1;
  }
  if (ensure_target_cells(ws, t, tc, tc.cell_valid ? tc.built_r : 0.0, s, err)) return 1;
  const size_t m = a.nq;
  double* pts = nullptr;
  double* d2 = nullptr;
  unsigned long long* idx = nullptr;
  double* dres = nullptr;
  TCK(cudaMalloc(&pts, sizeof(double) * 3 * m));
  TCK(cudaMalloc(&d2, sizeof(double) * m));
  TCK(cudaMalloc(&idx, sizeof(unsigned long long) * m));
  TCK(cudaMalloc(&dres, sizeof(double)));
  (note_launch(), atoms_to_pts<<<(a.nq + 255) / 256, 256, 0, s>>>(a.x, a.nq, pts));
  (note_launch(), nearest_points_kernel<<<static_cast<int>(std::min<size_t>(4096, (m + 7) / 8)), 256, 0, s>>>(
      pts, a.nq, tc.pc, tc.perm_c, tc.cell_start, to_dev(tc.g), idx, d2));
  (note_launch(), max_cost_kernel<<<1, 256, 0, s>>>(d2, a.nq, dres));
  TCK(cudaMemcpyAsync(out, dres, sizeof(double), cudaMemcpyDeviceToHost, s));
  TCK(cudaStreamSynchronize(s));
  cudaFree(pts);
  cudaFree(d2);
  cudaFree(idx);
  cudaFree(dres);
  return 0;
}

int run_plan_candidates(TruncWorkspace& ws, const DeviceAtoms& a, const DeviceTargets& t,
                        TargetCells& tc, double cutoff, bool geo, const uint64_t* off_host,
                        uint64_t* idx_host, cudaStream_t s, std::string& err) {
  const int nq = a.nq;
  if (nq == 0) return 0;
  const double radius = geo ? 0.0 : (cutoff < 0.0 ? 0.0 : std::sqrt(2.0 * cutoff));  // cost.hpp:38-42
  const double r2 = radius * radius;
  const bool scan = radius > 0.0;
  const double r_use = scan ? radius : 0.0;
  const double r_scan = r_use * (1.0 + 1e-9) + 1e-300;
  if (ensure_target_cells(ws, t, tc, r_use, s, err)) return 1;
  const size_t total = off_host[nq];
  unsigned long long *off = nullptr, *idx = nullptr, *sorted = nullptr;
  int* bad = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  TCK(cudaMalloc(&off, sizeof(unsigned long long) * (nq + 1)));
  TCK(cudaMalloc(&idx, sizeof(unsigned long long) * std::max<size_t>(total, 1)));
  TCK(cudaMalloc(&sorted, sizeof(unsigned long long) * std::max<size_t>(total, 1)));
  TCK(cudaMalloc(&bad, sizeof(int)));
  TCK(cudaMemcpyAsync(off, off_host, sizeof(unsigned long long) * (nq + 1), cudaMemcpyHostToDevice, s));
  TCK(cudaMemsetAsync(bad, 0, sizeof(int), s));
  if (geo)
    (note_launch(), plan_fill_geo_kernel<<<std::min(8192, (nq + 7) / 8), 256, 0, s>>>(
        a.x, nq, t.y, t.n, std::isfinite(cutoff) ? geo_dot_threshold(cutoff) : -INFINITY, tc.pc, tc.perm_c,
        tc.cell_start, to_dev(tc.g), off, idx, bad));
  else
    (note_launch(), plan_fill_kernel<<<std::min(8192, (nq + 7) / 8), 256, 0, s>>>(
        a.x, nq, tc.pc, tc.perm_c, tc.cell_start, to_dev(tc.g), r2, r_scan, scan ? 1 : 0, off, idx,
        bad));
  TCK(cub::DeviceSegmentedSort::SortKeys(tmp, tmp_bytes, idx, sorted, static_cast<int64_t>(total), nq,
                                         off, off + 1, s));
  TCK(cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 1)));
  TCK(cub::DeviceSegmentedSort::SortKeys(tmp, tmp_bytes, idx, sorted, static_cast<int64_t>(total), nq,
                                         off, off + 1, s));
  int hbad = 0;
  TCK(cudaMemcpyAsync(idx_host, sorted, sizeof(unsigned long long) * total, cudaMemcpyDeviceToHost, s));
  TCK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  TCK(cudaStreamSynchronize(s));
  cudaFree(off);
  cudaFree(idx);
  cudaFree(sorted);
  cudaFree(bad);
  cudaFree(tmp);
  if (hbad) {
    err = "plan candidates: offsets do not match the candidate counts";
    return 1;
  }
  return 0;
}

int run_plan_moments(const DeviceAtoms& a, const DeviceTargets& t, const double* psi_host,
                     double eps, bool geo, const double* log_s_host, const uint64_t* off_host,
                     const uint64_t* idx_host, const double atom_lo[3], double* marginal,
                     double* moment, double* map, uint64_t* modal, cudaStream_t s,
                     std::string& err) {
  const int nq = a.nq, n = t.n;
  const size_t total = off_host ? off_host[nq] : 0;
  double *psi = nullptr, *ls = nullptr, *dmarg = nullptr, *dmom = nullptr, *dmap = nullptr;
  unsigned long long *off = nullptr, *idx = nullptr, *acc = nullptr, *dmodal = nullptr;
  TCK(cudaMalloc(&psi, sizeof(double) * std::max(n, 1)));
  TCK(cudaMalloc(&ls, sizeof(double) * std::max(nq, 1)));
  TCK(cudaMemcpyAsync(psi, psi_host, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  TCK(cudaMemcpyAsync(ls, log_s_host, sizeof(double) * nq, cudaMemcpyHostToDevice, s));
  if (off_host) {
    TCK(cudaMalloc(&off, sizeof(unsigned long long) * (nq + 1)));
    TCK(cudaMalloc(&idx, sizeof(unsigned long long) * std::max<size_t>(total, 1)));
    TCK(cudaMemcpyAsync(off, off_host, sizeof(unsigned long long) * (nq + 1), cudaMemcpyHostToDevice, s));
    TCK(cudaMemcpyAsync(idx, idx_host, sizeof(unsigned long long) * total, cudaMemcpyHostToDevice, s));
  }
  const bool want_acc = marginal || moment;
  if (want_acc) {
    TCK(cudaMalloc(&acc, sizeof(unsigned long long) * 12 * std::max(n, 1)));
    TCK(cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * 12 * std::max(n, 1), s));
    TCK(cudaMalloc(&dmarg, sizeof(double) * std::max(n, 1)));
    TCK(cudaMalloc(&dmom, sizeof(double) * 3 * std::max(n, 1)));
  }
  if (map) TCK(cudaMalloc(&dmap, sizeof(double) * 3 * std::max(nq, 1)));
  if (modal) TCK(cudaMalloc(&dmodal, sizeof(unsigned long long) * std::max(nq, 1)));
  if (nq > 0 && geo)
    (note_launch(), plan_moments_kernel<true><<<std::min(8192, (nq + 7) / 8), 256, 0, s>>>(
        a.x, nq, t.y, n, psi, eps, ls, off, idx, atom_lo[0], atom_lo[1], atom_lo[2], acc, dmap,
        dmodal));
  else if (nq > 0)
    (note_launch(), plan_moments_kernel<false><<<std::min(8192, (nq + 7) / 8), 256, 0, s>>>(
        a.x, nq, t.y, n, psi, eps, ls, off, idx, atom_lo[0], atom_lo[1], atom_lo[2], acc, dmap,
        dmodal));
  if (want_acc && n > 0) {
    (note_launch(), plan_assemble_kernel<<<(n + 255) / 256, 256, 0, s>>>(acc, n, atom_lo[0], atom_lo[1],
                                                                      atom_lo[2], dmarg, dmom));
    if (marginal) TCK(cudaMemcpyAsync(marginal, dmarg, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    if (moment) TCK(cudaMemcpyAsync(moment, dmom, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s));
  }
  if (map && nq) TCK(cudaMemcpyAsync(map, dmap, sizeof(double) * 3 * nq, cudaMemcpyDeviceToHost, s));
  if (modal && nq)
    TCK(cudaMemcpyAsync(modal, dmodal, sizeof(unsigned long long) * nq, cudaMemcpyDeviceToHost, s));
  TCK(cudaStreamSynchronize(s));
  void* ptrs[] = {psi, ls, dmarg, dmom, dmap, off, idx, acc, dmodal};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  TCK(cudaGetLastError());
  return 0;
}

}  // namespace rsot_cuda
