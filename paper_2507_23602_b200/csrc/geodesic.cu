// geodesic.cu -- evaluate_dual for CostKind::SqGeodesicSphere (SURVEY.md
// §8(f) #4; the blue-noise application, proj/src/sphere.cpp:115-168).
//
// Reference semantics (proj/src/evaluate.cpp:86-174 with cost.hpp:19-33):
//   c(x, y) = acos(clamp(x . y, -1, 1))^2 (no Euclidean ball: a finite cutoff
//   selects {j : c(x_q, y_j) < cutoff} by a full scan, evaluate.cpp:124-128),
//   an empty set falls back to the Euclidean nearest target (index.nearest,
//   lowest index on ties), e_qj = (psi_j - c)/eps + ln nu_j.
// Every pair costs an fp64 acos and exp, so this path is compute bound on
// the libdevice transcendental sequences rather than on the tuned exp2 of the
// Euclidean kernels; it shares their packing (res[N + 5]) so the multi-GPU
// reduction and finalisation are the same.  Both sweeps evaluate the cost and
// the candidate predicate with the same unfused operations, so the set used
// for the gradient is exactly the one used for ln S_q.
//   geo_atoms    : thread per atom, targets tiled in shared memory; online
//                  max/rescale LSE, candidate count, Euclidean nearest.
//   geo_targets  : thread per target, atoms tiled; gradient gather in atom
//                  order (deterministic).
//   geo_empty    : empty-set atoms add m_q to their nearest target (fixed
//                  point, order independent).
#include <algorithm>
#include <cmath>

#include "block_util.cuh"
#include "device_math.cuh"
#include "geodesic.cuh"

namespace rsot_cuda {

namespace {

constexpr int kGT = 128;    // threads per block
constexpr int kGTile = 128; // staged points per tile


// cost.hpp:19-33 dot (unfused, (p0 q0 + p1 q1) + p2 q2), clamped to [-1, 1].
__device__ __forceinline__ double geo_clamped_dot(const double4& x, const double4& y) {
  const double d = __dadd_rn(__dadd_rn(__dmul_rn(x.x, y.x), __dmul_rn(x.y, y.y)), __dmul_rn(x.z, y.z));
  return d < -1.0 ? -1.0 : (1.0 < d ? 1.0 : d);
}

template <bool TRUNC>
__global__ void __launch_bounds__(kGT)
geo_atoms(const double4* __restrict__ atoms, int nq, const double4* __restrict__ tgt,
          const double* __restrict__ psi, int n, double eps, double tmin,
          double* __restrict__ L_out, double* __restrict__ J_out, double* __restrict__ D_out,
          double* __restrict__ cnt_out, double* __restrict__ empty_out,
          int* __restrict__ nearest_out, uint64_t* __restrict__ hash_out) {
  __shared__ double4 ty[kGTile];
  __shared__ double tp[kGTile];
  const int q = blockIdx.x * kGT + threadIdx.x;
  const bool valid = q < nq;
  const double4 x = valid ? atoms[q] : make_double4(0, 0, 0, 0);
  double mx = -INFINITY, sum = 0.0, cnt = 0.0;
  uint64_t hash = 0;
  double bd = INFINITY;
  int bj = -1;
  for (int base = 0; base < n; base += kGTile) {
    const int ct = min(kGTile, n - base);
    __syncthreads();
    for (int t = threadIdx.x; t < ct; t += kGT) {
      ty[t] = tgt[base + t];
      tp[t] = psi[base + t];
    }
    __syncthreads();
    if (!valid) continue;
    for (int t = 0; t < ct; ++t) {
      const double4 y = ty[t];
      const double c = geo_cost(x.x, x.y, x.z, y.x, y.y, y.z);
      if (TRUNC) {
        const double d2 = exact_sqdist(x.x, x.y, x.z, y.x, y.y, y.z);
        if (d2 < bd) {  // ascending j: strict < keeps the lowest index
          bd = d2;
          bj = base + t;
        }
        if (!(geo_clamped_dot(x, y) >= tmin)) continue;  // == (c < cutoff) with the host's acos
      }
      const double e = __dadd_rn(__ddiv_rn(__dsub_rn(tp[t], c), eps), y.w);
      if (e > mx) {
        sum = sum * exp(mx - e) + 1.0;
        mx = e;
      } else {
        sum += exp(e - mx);
      }
      cnt += 1.0;
      if (hash_out) hash += candidate_hash_term(static_cast<uint64_t>(base + t));
    }
  }
  if (!valid) return;
  const double m = x.w;
  bool empty = false;
  double L;
  if (cnt == 0.0) {  // evaluate.cpp:129-133: the nearest target alone
    empty = true;
    const double4 y = tgt[bj];
    const double c = geo_cost(x.x, x.y, x.z, y.x, y.y, y.z);
    L = __dadd_rn(__ddiv_rn(__dsub_rn(psi[bj], c), eps), y.w);
    cnt = 1.0;
    hash = candidate_hash_term(static_cast<uint64_t>(bj));
  } else {
    L = mx + log(sum);
  }
  L_out[q] = L;
  J_out[q] = eps * L * m;
  D_out[q] = m * exp(-L);
  cnt_out[q] = cnt;
  empty_out[q] = empty ? 1.0 : 0.0;
  nearest_out[q] = empty ? bj : -1;
  if (hash_out) hash_out[q] = hash;
}

__global__ void geo_debug(const double* __restrict__ L, const double* __restrict__ cnt, int nq,
                          uint32_t* __restrict__ count, double* __restrict__ log_s) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  if (count) count[q] = static_cast<uint32_t>(cnt[q]);
  if (log_s) log_s[q] = L[q];
}

template <bool TRUNC>
__global__ void __launch_bounds__(kGT)
geo_targets(const double4* __restrict__ atoms, int nq, const double* __restrict__ L,
            const int* __restrict__ nearest, const double4* __restrict__ tgt,
            const double* __restrict__ psi, int n, double eps, double tmin,
            double* __restrict__ G) {
  __shared__ double4 ta[kGTile];
  __shared__ double tl[kGTile];
  const int j = blockIdx.x * kGT + threadIdx.x;
  const bool valid = j < n;
  const double4 y = valid ? tgt[j] : make_double4(0, 0, 0, 0);
  const double pj = valid ? psi[j] : 0.0;
  double g = 0.0;
  for (int base = 0; base < nq; base += kGTile) {
    const int ct = min(kGTile, nq - base);
    __syncthreads();
    for (int t = threadIdx.x; t < ct; t += kGT) {
      ta[t] = atoms[base + t];
      // empty-set atoms contribute through geo_empty
      tl[t] = nearest[base + t] >= 0 ? INFINITY : L[base + t];
    }
    __syncthreads();
    if (!valid) continue;
    for (int t = 0; t < ct; ++t) {
      const double lq = tl[t];
      if (lq == INFINITY) continue;
      const double4 x = ta[t];
      if (TRUNC && !(geo_clamped_dot(x, y) >= tmin)) continue;  // == (c < cutoff), see geo_dot_threshold
      const double c = geo_cost(x.x, x.y, x.z, y.x, y.y, y.z);
      const double e = __dadd_rn(__ddiv_rn(__dsub_rn(pj, c), eps), y.w);
      g = fma(exp(e - lq), x.w, g);
    }
  }
  if (valid) G[j] = g;
}

__global__ void geo_empty(const double4* __restrict__ atoms, const int* __restrict__ nearest,
                          int nq, unsigned long long* __restrict__ gacc) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nq && nearest[q] >= 0) fp_add(gacc + 3 * static_cast<size_t>(nearest[q]), atoms[q].w);
}

__global__ void geo_assemble(const double* __restrict__ G, const unsigned long long* __restrict__ gacc,
                             int n, double nq, double* __restrict__ res) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) res[j] = G[j] + fp_to_double(gacc + 3 * static_cast<size_t>(j));
  if (j == 0) res[n + kResVisited] = nq;
}

template <typename T>
cudaError_t grow(T*& p, size_t& cap, size_t n) {
  if (n <= cap && p) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  const cudaError_t e = cudaMalloc(&p, sizeof(T) * (n ? n : 1));
  if (e == cudaSuccess) cap = n;
  return e;
}

}  // namespace

void GeoWorkspace::release() {
  void* ptrs[] = {L, J, D, cnt, empty, nearest, G, gacc, red};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  *this = GeoWorkspace();
}

#define GCK(call)                                                  \
  do {                                                             \
    const cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) {                                       \
      err = std::string(#call) + ": " + cudaGetErrorString(e_);    \
      return 1;                                                    \
    }                                                              \
  } while (0)

// Exact candidate selection without the device's acos: the reference keeps
// a pair iff fl(acos(t))^2 < cutoff with t the clamped dot (cost.hpp:19-33,
// evaluate.cpp:124-128), a non-increasing function of t (libm's acos is
// monotone, squaring on [0, pi] too), so the kept set is {t >= t_min} with
// t_min the smallest double in [-1, 1] that passes -- found here by bisection
// with the host's own acos (the reference's libm call).  The device compares
// the clamped dot with t_min: selection bit for bit as the reference, even
// where libdevice's acos and glibc's differ in the last ulp.  -inf: every
// pair passes; +inf: none.
double geo_dot_threshold(double cutoff) {
  auto pass = [cutoff](double t) {
    const double g = std::acos(t);
    return g * g < cutoff;
  };
  if (!pass(1.0)) return INFINITY;
  if (pass(-1.0)) return -INFINITY;
  double lo = -1.0, hi = 1.0;  // pass(lo) false, pass(hi) true
  for (;;) {
    double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) {  // adjacent doubles
      mid = std::nextafter(lo, hi);
      if (mid >= hi) break;
    }
    if (pass(mid)) hi = mid; else lo = mid;
  }
  return hi;
}

int run_geodesic(GeoWorkspace& w, const DeviceAtoms& a, const DeviceTargets& t, EvalBuffers& b,
                 double eps, double cutoff, cudaStream_t s, std::string& err,
                 uint32_t* dbg_count, uint64_t* dbg_hash, double* dbg_log_s) {
  const int nq = a.nq, n = t.n;
  const bool trunc = std::isfinite(cutoff);
  const double tmin = trunc ? geo_dot_threshold(cutoff) : -INFINITY;
  GCK(grow(w.L, w.atom_cap_L, nq));
  GCK(grow(w.J, w.atom_cap_J, nq));
  GCK(grow(w.D, w.atom_cap_D, nq));
  GCK(grow(w.cnt, w.atom_cap_c, nq));
  GCK(grow(w.empty, w.atom_cap_e, nq));
  GCK(grow(w.nearest, w.atom_cap_n, nq));
  GCK(grow(w.G, w.tgt_cap_G, n));
  GCK(grow(w.gacc, w.tgt_cap_a, 3 * static_cast<size_t>(n)));
  GCK(grow(w.red, w.red_cap, 4096));
  GCK(cudaMemsetAsync(w.gacc, 0, sizeof(unsigned long long) * 3 * static_cast<size_t>(n), s));
  GCK(cudaMemsetAsync(b.res, 0, sizeof(double) * (n + kResTail), s));
  if (nq > 0) {
    const int ga = (nq + kGT - 1) / kGT, gt = (n + kGT - 1) / kGT;
    if (b.timing) cudaEventRecord(b.timing[1], s);
    if (trunc)
      (note_launch(), geo_atoms<true><<<ga, kGT, 0, s>>>(a.x, nq, t.y, b.psi, n, eps, tmin, w.L, w.J,
                                                         w.D, w.cnt, w.empty, w.nearest, dbg_hash));
    else
      (note_launch(), geo_atoms<false><<<ga, kGT, 0, s>>>(a.x, nq, t.y, b.psi, n, eps, tmin, w.L, w.J,
                                                          w.D, w.cnt, w.empty, w.nearest, dbg_hash));
    if (dbg_count || dbg_log_s)
      (note_launch(), geo_debug<<<(nq + 255) / 256, 256, 0, s>>>(w.L, w.cnt, nq, dbg_count, dbg_log_s));
    if (b.timing) {
      cudaEventRecord(b.timing[2], s);
      cudaEventRecord(b.timing[3], s);
    }
    if (trunc)
      (note_launch(), geo_targets<true><<<gt, kGT, 0, s>>>(a.x, nq, w.L, w.nearest, t.y, b.psi, n, eps,
                                                           tmin, w.G));
    else
      (note_launch(), geo_targets<false><<<gt, kGT, 0, s>>>(a.x, nq, w.L, w.nearest, t.y, b.psi, n, eps,
                                                            tmin, w.G));
    if (b.timing) cudaEventRecord(b.timing[4], s);
    (note_launch(), geo_empty<<<(nq + 255) / 256, 256, 0, s>>>(a.x, w.nearest, nq, w.gacc));
    (note_launch(), geo_assemble<<<(n + 255) / 256, 256, 0, s>>>(w.G, w.gacc, n, static_cast<double>(nq),
                                                                b.res));
    launch_det_sum(w.J, nq, w.red, b.res + n + kResJ, s);
    launch_det_sum(w.D, nq, w.red + 1024, b.res + n + kResD, s);
    launch_det_sum(w.cnt, nq, w.red + 2048, b.res + n + kResPairs, s);
    launch_det_sum(w.empty, nq, w.red + 3072, b.res + n + kResEmpty, s);
  }
  GCK(cudaGetLastError());
  return 0;
}

namespace {
// Thread per atom: max over all targets (tiled through shared memory) of the
// clamped unfused dot product; block minimum over the atoms.
__global__ void __launch_bounds__(kGT)
geo_cover_dot(const double4* __restrict__ atoms, int nq, const double4* __restrict__ tgt, int n,
              double* __restrict__ block_min) {
  __shared__ double4 ty[kGTile];
  __shared__ double red[kGT];
  const int q = blockIdx.x * kGT + threadIdx.x;
  const bool valid = q < nq;
  const double4 x = valid ? atoms[q] : make_double4(0, 0, 0, 0);
  double best = -INFINITY;
  for (int base = 0; base < n; base += kGTile) {
    const int ct = min(kGTile, n - base);
    __syncthreads();
    for (int k = threadIdx.x; k < ct; k += kGT) ty[k] = tgt[base + k];
    __syncthreads();
    if (!valid) continue;
    for (int k = 0; k < ct; ++k) {
      const double4 y = ty[k];
      const double d = __dadd_rn(__dadd_rn(__dmul_rn(x.x, y.x), __dmul_rn(x.y, y.y)), __dmul_rn(x.z, y.z));
      best = fmax(best, d);
    }
  }
  // clamp(max) = max(clamp) (cost.hpp:22-23)
  best = best < -1.0 ? -1.0 : (1.0 < best ? 1.0 : best);
  red[threadIdx.x] = valid ? best : INFINITY;
  __syncthreads();
  for (int o = kGT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) block_min[blockIdx.x] = red[0];
}

__global__ void min_final(const double* __restrict__ v, int m, double* __restrict__ out) {
  __shared__ double red[256];
  double b = INFINITY;
  for (int i = threadIdx.x; i < m; i += 256) b = fmin(b, v[i]);
  red[threadIdx.x] = b;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}
}  // namespace

int run_geo_covering_dot(GeoWorkspace& w, const DeviceAtoms& a, const DeviceTargets& t, double* t_star,
                         cudaStream_t s, std::string& err) {
  const int blocks = (a.nq + kGT - 1) / kGT;
  if (blocks == 0 || t.n == 0) {
    err = "covering cost: empty input";
    return 1;
  }
  if (grow(w.red, w.red_cap, std::max<size_t>(4096, static_cast<size_t>(blocks) + 1)) != cudaSuccess) {
    err = "cudaMalloc (covering cost)";
    return 1;
  }
  (note_launch(), geo_cover_dot<<<blocks, kGT, 0, s>>>(a.x, a.nq, t.y, t.n, w.red));
  (note_launch(), min_final<<<1, 256, 0, s>>>(w.red, blocks, w.red + blocks));
  cudaError_t e = cudaMemcpyAsync(t_star, w.red + blocks, sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    err = std::string("covering cost: ") + cudaGetErrorString(e);
    return 1;
  }
  return 0;
}

}  // namespace rsot_cuda
