// refine.cu -- softmax_refine on the GPU.
//
// Reference: rsot::softmax_refine, proj/src/solve.cpp:62-142, the
// prolongation of a coarse-level potential to a finer target level used by
// solve_multilevel (solve.cpp:202-206):
//   phase 1 (:79-118): per atom q, ln S_q = LSE over coarse targets j of
//     (psi_j - c(x_q,y_j))/eps + ln nu_j, candidates {j : c(x_q,y_j) < C}
//     (brute-force cost test, NOT the ball query) or all targets when C is
//     infinite; an empty set falls back to the first minimum of the cost;
//   phase 2 (:120-139): for every fine point y_k,
//     psi_k = -eps * LSE_q( -c(x_q,y_k)/eps - ln S_q + ln m_q ),
//     a dense LSE over all atoms (2.75e11 pairs in BASELINE cfg4).
// Phase 1 reuses the base-2 fixed-shift scheme of the evaluator with the
// reference's exact cost predicate in the FP32 error band; phase 2 is the
// dense target-major gather of dense.cu with b2 = 0 and
// lam_q = log2 m_q - log2 S_q - max_q(...) (all exponents <= 0).
#include <cmath>

#include "block_util.cuh"
#include "device_math.cuh"
#include "kernels.cuh"
#include "refine.cuh"

namespace rsot_cuda {

namespace {

constexpr int kRT = 128;
constexpr int kRTile = 256;

// Phase 1: per atom partial sums over a split of the coarse targets.
template <bool TRUNC>
__global__ void __launch_bounds__(kRT)
refine_phase1(const double4* __restrict__ atoms, int nq, const double4* __restrict__ tgt,
              const double* __restrict__ b2, int n, int per_split,
              const double* __restrict__ scal, double c2, double cutoff,
              double* __restrict__ partS, unsigned* __restrict__ partC,
              double* __restrict__ shiftA) {
  __shared__ double4 tD[kRTile];
  __shared__ float4 tF[kRTile];
  __shared__ int2 tbl[ExpTab64::kTab];
  __shared__ double sh[200];
  load_exp2_table(tbl);
  const int q = blockIdx.x * kRT + threadIdx.x;
  const bool valid = q < nq;
  const double4 a = valid ? atoms[q] : make_double4(0, 0, 0, 0);
  double lo[3] = {valid ? a.x : INFINITY, valid ? a.y : INFINITY, valid ? a.z : INFINITY};
  double hi[3] = {valid ? a.x : -INFINITY, valid ? a.y : -INFINITY, valid ? a.z : -INFINITY};
  double box[6];
  block_bbox<kRT>(lo, hi, sh, box);
  const double o0 = 0.5 * (box[0] + box[3]), o1 = 0.5 * (box[1] + box[4]),
               o2 = 0.5 * (box[2] + box[5]);
  const double hx = 0.5 * (box[3] - box[0]), hy = 0.5 * (box[4] - box[1]),
               hz = 0.5 * (box[5] - box[2]);
  const double hd2 = hx * hx + hy * hy + hz * hz;
  const bool wide = c2 * hd2 > 400.0;
  const double x0 = a.x - o0, x1 = a.y - o1, x2 = a.z - o2;
  const double X0 = 2.0 * c2 * x0, X1 = 2.0 * c2 * x1, X2 = 2.0 * c2 * x2;
  const double xsq = c2 * fma(x2, x2, fma(x1, x1, x0 * x0));
  const float xf0 = valid ? static_cast<float>(x0) : 1e30f;
  const float xf1 = valid ? static_cast<float>(x1) : 1e30f;
  const float xf2 = valid ? static_cast<float>(x2) : 1e30f;
  // cost < C  <=>  d2 < 2C (real numbers); FP32 band as in truncated.cu.
  float lo_thr = -1.0f, hi_thr = INFINITY;
  if (TRUNC) {
    const double r2 = 2.0 * cutoff;
    const double r = sqrt(fmax(r2, 0.0));
    const double band = 0x1p-21 * (8.0 * r * (sqrt(hd2) + 1.01 * r) + 4.0 * r2);
    lo_thr = (r2 - band > 1e-30) ? __double2float_rd(r2 - band) : -1.0f;
    hi_thr = __double2float_ru(r2 + band);
  }
  const double B = scal[kSlotB];
  double S = 0.0;
  unsigned cnt = 0;
  const int j0 = blockIdx.y * per_split;
  const int j1 = min(n, j0 + per_split);
  for (int base = j0; base < j1; base += kRTile) {
    const int ct = min(kRTile, j1 - base);
    __syncthreads();
    for (int t = threadIdx.x; t < ct; t += kRT) {
      const double4 y = tgt[base + t];
      const double y0 = y.x - o0, y1 = y.y - o1, y2 = y.z - o2;
      const double yy = fma(y2, y2, fma(y1, y1, y0 * y0));
      tD[t] = make_double4(y0, y1, y2, fmax(fma(-c2, yy, b2[base + t]) - B, -1.0e5));
      tF[t] = make_float4(static_cast<float>(y0), static_cast<float>(y1), static_cast<float>(y2), 0.f);
    }
    __syncthreads();
    for (int t = 0; t < ct; ++t) {
      bool in = valid;
      if (TRUNC) {
        const float4 yf = tF[t];
        const float dx = xf0 - yf.x, dy = xf1 - yf.y, dz = xf2 - yf.z;
        const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        in = d2 < lo_thr;
        const bool border = !in && d2 <= hi_thr;
        if (__any_sync(0xffffffffu, border) && border) {
          const double4 yg = tgt[base + t];
          in = __dmul_rn(0.5, exact_sqdist(a.x, a.y, a.z, yg.x, yg.y, yg.z)) < cutoff;
        }
      }
      if (__any_sync(0xffffffffu, in)) {
        const double4 y = tD[t];
        double s = fma(X0, y.x, fma(X1, y.y, fma(X2, y.z, y.w)));
        if (wide) s -= xsq;
        S = exp2_acc_masked<true>(s, S, tbl, in);
        cnt += in ? 1u : 0u;
      }
    }
  }
  if (valid) {
    partS[static_cast<size_t>(blockIdx.y) * nq + q] = S;
    partC[static_cast<size_t>(blockIdx.y) * nq + q] = cnt;
    if (blockIdx.y == 0) shiftA[q] = wide ? 0.0 : xsq;
  }
}

// Per atom: log2 S_q, or a flag for the exact paths (empty set / range).
__global__ void refine_finalize1(const double4* __restrict__ atoms, int nq,
                                 const double* __restrict__ partS,
                                 const unsigned* __restrict__ partC, int splits,
                                 const double* __restrict__ shiftA,
                                 const double* __restrict__ scal, double* __restrict__ L2,
                                 int* __restrict__ flag) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  double S = 0.0;
  unsigned c = 0;
  for (int s = 0; s < splits; ++s) {
    S += partS[static_cast<size_t>(s) * nq + q];
    c += partC[static_cast<size_t>(s) * nq + q];
  }
  const bool ok = c > 0 && S >= 0x1p-960 && S <= 0x1p960;
  flag[q] = c == 0 ? 1 : (ok ? 0 : 2);
  L2[q] = ok ? (scal[kSlotB] - shiftA[q]) + log2(S) : 0.0;
}

// Exact per-atom coarse LSE for flagged atoms: empty sets use the first
// minimum of the cost (solve.cpp:86-96); out-of-range sums use the
// reference's max shift (:100-112).  One warp per atom, fixed-order sums.
__global__ void refine_exact1(const double4* __restrict__ atoms, int nq,
                              const double4* __restrict__ tgt, const double* __restrict__ psi,
                              int n, double eps, double cutoff, bool trunc,
                              const int* __restrict__ flag, double* __restrict__ L2) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int base = warp * 32; base < nq; base += nwarps * 32) {
    const int mq = base + lane;
    unsigned todo = __ballot_sync(0xffffffffu, mq < nq && flag[mq] != 0);
    while (todo) {
      const int l = __ffs(todo) - 1;
      todo &= todo - 1;
      const int q = base + l;
      const double4 x = atoms[q];
      const int f = flag[q];
      double L;
      if (f == 1) {
        // first minimum of cost = 0.5 * d2 over all coarse targets
        double bc = INFINITY;
        int bj = 0x7fffffff;
        for (int j = lane; j < n; j += 32) {
          const double4 y = tgt[j];
          const double c = __dmul_rn(0.5, exact_sqdist(x.x, x.y, x.z, y.x, y.y, y.z));
          if (c < bc || (c == bc && j < bj)) { bc = c; bj = j; }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
          const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
          if (oc < bc || (oc == bc && oj < bj)) { bc = oc; bj = oj; }
        }
        const double4 y = tgt[bj];
        L = __dadd_rn(__ddiv_rn(__dsub_rn(psi[bj], bc), eps), y.w);
      } else {
        double mx = -INFINITY;
        for (int j = lane; j < n; j += 32) {
          const double4 y = tgt[j];
          const double c = __dmul_rn(0.5, exact_sqdist(x.x, x.y, x.z, y.x, y.y, y.z));
          if (trunc && !(c < cutoff)) continue;
          mx = fmax(mx, __dadd_rn(__ddiv_rn(__dsub_rn(psi[j], c), eps), y.w));
        }
        mx = warp_max(mx);
        double sum = 0.0;
        for (int j = lane; j < n; j += 32) {
          const double4 y = tgt[j];
          const double c = __dmul_rn(0.5, exact_sqdist(x.x, x.y, x.z, y.x, y.y, y.z));
          if (trunc && !(c < cutoff)) continue;
          sum += exp(__dadd_rn(__ddiv_rn(__dsub_rn(psi[j], c), eps), y.w) - mx);
        }
        sum = warp_sum(sum);
        L = mx + log(sum);
      }
      if (lane == 0) L2[q] = L * kLog2e;
    }
  }
}

// lam_q = log2 m_q - log2 S_q and its block maxima.
__global__ void refine_lam(const double4* __restrict__ atoms, int nq,
                           const double* __restrict__ L2, double* __restrict__ lam,
                           double* __restrict__ part, int chunk) {
  __shared__ double sh[256];
  const int lo = blockIdx.x * chunk, hi = min(nq, lo + chunk);
  double mx = -INFINITY;
  for (int q = lo + threadIdx.x; q < hi; q += blockDim.x) {
    const double v = fmax(log2(atoms[q].w) - L2[q], -1.0e5);
    lam[q] = v;
    mx = fmax(mx, v);
  }
  mx = block_max<256>(mx, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = mx;
}

__global__ void refine_shift_lam(double* __restrict__ lam, int nq, const double* __restrict__ part,
                                 int nblk, double* __restrict__ tmax_out) {
  __shared__ double sh[256];
  double mx = -INFINITY;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) mx = fmax(mx, part[i]);
  mx = block_max<256>(mx, sh);
  if (blockIdx.x == 0 && threadIdx.x == 0) *tmax_out = mx;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x)
    lam[q] -= mx;
}

// psi_k = -eps ln2 (Tmax + log2 G_k); G out of range -> exact fallback flag.
__global__ void refine_psi(const double* __restrict__ G, int n, const double* __restrict__ tmax,
                           double eps, double* __restrict__ psi_out, int* __restrict__ flag,
                           unsigned* __restrict__ nflag) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double g = G[k];
  if (!(g >= 0x1p-960) || !(g <= 0x1p960)) {
    flag[atomicAdd(nflag, 1u)] = k;
    psi_out[k] = 0.0;
    return;
  }
  psi_out[k] = -eps * ((*tmax + log2(g)) * kLn2);
}

// Exact phase 2 (reference max shift, solve.cpp:124-138) for flagged fine
// points; one block per point, fixed-order block reductions.
__global__ void refine_exact2(const double4* __restrict__ atoms, const double* __restrict__ L2,
                              int nq, const double* __restrict__ fine, double eps,
                              const int* __restrict__ flag, const unsigned* __restrict__ nflag,
                              double* __restrict__ psi_out) {
  __shared__ double sh[256];
  const unsigned nf = *nflag;
  for (unsigned f = blockIdx.x; f < nf; f += gridDim.x) {
    const int k = flag[f];
    const double y0 = fine[3 * k], y1 = fine[3 * k + 1], y2 = fine[3 * k + 2];
    double mx = -INFINITY;
    for (int q = threadIdx.x; q < nq; q += blockDim.x) {
      const double4 x = atoms[q];
      const double c = __dmul_rn(0.5, exact_sqdist(x.x, x.y, x.z, y0, y1, y2));
      mx = fmax(mx, -c / eps - L2[q] * kLn2 + log(x.w));
    }
    mx = block_max<256>(mx, sh);
    double sum = 0.0;
    for (int q = threadIdx.x; q < nq; q += blockDim.x) {
      const double4 x = atoms[q];
      const double c = __dmul_rn(0.5, exact_sqdist(x.x, x.y, x.z, y0, y1, y2));
      sum += exp(-c / eps - L2[q] * kLn2 + log(x.w) - mx);
    }
    sum = block_sum<256>(sum, sh);
    if (threadIdx.x == 0) psi_out[k] = -eps * (mx + log(sum));
    __syncthreads();
  }
}

__global__ void fine_to_double4(const double* __restrict__ xyz, int n, double4* __restrict__ out,
                                double* __restrict__ zeros) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) {
    out[k] = make_double4(xyz[3 * k], xyz[3 * k + 1], xyz[3 * k + 2], 0.0);
    zeros[k] = 0.0;
  }
}

}  // namespace

int run_softmax_refine(RefineWorkspace& w, const DeviceAtoms& a, const DeviceTargets& coarse,
                       EvalBuffers& b, const double* fine_xyz_host, int n_fine, double eps,
                       double cutoff, int num_sms, double* psi_host, cudaStream_t s,
                       std::string& err) {
#define RCK(call)                                                     \
  do {                                                                \
    cudaError_t e_ = (call);                                          \
    if (e_ != cudaSuccess) {                                          \
      err = std::string(#call) + ": " + cudaGetErrorString(e_);       \
      return 1;                                                       \
    }                                                                 \
  } while (0)
  const int nq = a.nq, n = coarse.n;
  const bool trunc = std::isfinite(cutoff);
  const double c2 = kLog2e / (2.0 * eps);
  const int splits = std::max(1, std::min((n + 511) / 512, (16 * num_sms * 6 + (nq + kRT - 1) / kRT - 1) /
                                                               std::max(1, (nq + kRT - 1) / kRT)));
  const int per_split = ((n + splits - 1) / splits + kRTile - 1) / kRTile * kRTile;
  const int nsplit = (n + per_split - 1) / per_split;
  const size_t qcap = std::max(1, nq);
  const size_t fcap = std::max(1, n_fine);
  auto grow = [](auto*& p, size_t& cap, size_t want) -> cudaError_t {
    if (p && cap >= want) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, sizeof(*p) * want);
    if (e == cudaSuccess) cap = want;
    return e;
  };
  RCK(grow(w.partS, w.partS_cap, static_cast<size_t>(nsplit) * qcap));
  RCK(grow(w.partC, w.partC_cap, static_cast<size_t>(nsplit) * qcap));
  RCK(grow(w.shiftA, w.shiftA_cap, qcap));
  RCK(grow(w.L2, w.L2_cap, qcap));
  RCK(grow(w.lam, w.lam_cap, qcap));
  RCK(grow(w.flag, w.flag_cap, std::max(qcap, fcap)));
  RCK(grow(w.fine4, w.fine4_cap, fcap));
  RCK(grow(w.zeros, w.zeros_cap, fcap));
  RCK(grow(w.fine, w.fine_cap, 3 * fcap));
  RCK(grow(w.G, w.G_cap, fcap));
  RCK(grow(w.psi, w.psi_cap, fcap));
  RCK(grow(w.partG, w.partG_cap, std::max<size_t>(fcap * 64, 1 << 20)));
  RCK(grow(w.misc, w.misc_cap, 8192));
  RCK(cudaMemcpyAsync(w.fine, fine_xyz_host, sizeof(double) * 3 * n_fine, cudaMemcpyHostToDevice, s));
  (note_launch(), fine_to_double4<<<(n_fine + 255) / 256, 256, 0, s>>>(w.fine, n_fine, w.fine4, w.zeros));
  if (nq > 0) {
    dim3 g1((nq + kRT - 1) / kRT, nsplit);
    if (trunc)
      (note_launch(), refine_phase1<true><<<g1, kRT, 0, s>>>(a.x, nq, coarse.y, b.b2, n, per_split, b.scal,
                                                              c2, cutoff, w.partS, w.partC, w.shiftA));
    else
      (note_launch(), refine_phase1<false><<<g1, kRT, 0, s>>>(a.x, nq, coarse.y, b.b2, n, per_split, b.scal,
                                                               c2, cutoff, w.partS, w.partC, w.shiftA));
    (note_launch(), refine_finalize1<<<(nq + 255) / 256, 256, 0, s>>>(a.x, nq, w.partS, w.partC, nsplit,
                                                                      w.shiftA, b.scal, w.L2, w.flag));
    (note_launch(), refine_exact1<<<4 * num_sms, 256, 0, s>>>(a.x, nq, coarse.y, b.psi, n, eps, cutoff,
                                                              trunc, w.flag, w.L2));
    const int nb = std::min(1024, (nq + 4095) / 4096);
    const int chunk = (nq + nb - 1) / nb;
    double* part = reinterpret_cast<double*>(w.misc);
    double* tmax = part + 4096;
    (note_launch(), refine_lam<<<nb, 256, 0, s>>>(a.x, nq, w.L2, w.lam, part, chunk));
    (note_launch(), refine_shift_lam<<<std::min(1024, (nq + 255) / 256), 256, 0, s>>>(w.lam, nq, part, nb,
                                                                                     tmax));
    launch_dense_gather(a.x, w.lam, nq, w.fine4, w.zeros, n_fine, c2, num_sms, w.partG, w.partG_cap, w.G,
                        s);
    unsigned* nflag = reinterpret_cast<unsigned*>(part + 4100);
    RCK(cudaMemsetAsync(nflag, 0, sizeof(unsigned), s));
    (note_launch(), refine_psi<<<(n_fine + 255) / 256, 256, 0, s>>>(w.G, n_fine, tmax, eps, w.psi, w.flag,
                                                                    nflag));
    (note_launch(), refine_exact2<<<2 * num_sms, 256, 0, s>>>(a.x, w.L2, nq, w.fine, eps, w.flag, nflag,
                                                              w.psi));
  } else {
    RCK(cudaMemsetAsync(w.psi, 0, sizeof(double) * n_fine, s));
  }
  RCK(cudaMemcpyAsync(psi_host, w.psi, sizeof(double) * n_fine, cudaMemcpyDeviceToHost, s));
  RCK(cudaStreamSynchronize(s));
  RCK(cudaGetLastError());
  return 0;
#undef RCK
}

void RefineWorkspace::release() {
  void* ptrs[] = {partS, partC, shiftA, L2, lam, flag, fine4, zeros, fine, G, psi, partG, misc};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  *this = RefineWorkspace();
}

}  // namespace rsot_cuda
