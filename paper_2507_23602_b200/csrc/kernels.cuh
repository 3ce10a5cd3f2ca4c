// kernels.cuh -- launch interface of the RSOT evaluator kernels (internal).
//
// Layout in HBM (all fp64):
//   targets : double4 {y0, y1, y2, ln nu}       32 B / target, original order
//   atoms   : double4 {x0, x1, x2, m}           32 B / atom (this rank's shard)
//   per eval: b2[N]   = log2(e) (psi/eps + ln nu)
//             scal[]  = {B = max b2, sum psi*nu, ...}
//             partS[splitsA][nq], atomL2[nq] (log2 S_q), atomLam[nq]
//             partG[splitsB][N], res[N + 5] packed for the allreduce
#pragma once

#include <cstddef>
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

namespace rsot_cuda {

// Process-wide count of kernels this library has launched
// (rsot_cuda_kernel_launches); every launch site goes through note_launch().
extern std::atomic<unsigned long long> g_kernel_launches;
inline void note_launch() { g_kernel_launches.fetch_add(1, std::memory_order_relaxed); }

// Indices into the per-eval device scalar block.
enum ScalarSlot : int {
  kSlotB = 0,          // max_j b2_j (global exponent shift)
  kSlotPsiNu = 1,      // sum_j psi_j nu_j (fixed-order)
  kSlotNonFinite = 2,  // > 0 when psi had a non-finite entry
  kSlotFlagCount = 3,  // u64 count of atoms needing the exact fallback
  kSlotBmin = 4,       // min_j b2_j (exponent range check)
  kNumSlots = 8
};

// Packed result tail (after the N gradient entries).
enum ResultSlot : int {
  kResJ = 0,
  kResD = 1,
  kResPairs = 2,
  kResEmpty = 3,
  kResVisited = 4,
  kResTail = 5
};

// Element functions of the cross-rank combination, shared by the kernels
// (rank_sum_kernel, finalize_kernel) and their host mirrors in the C ABI.
// Ranks' packed partials summed in rank order (parallel.hpp:24-30 merges the
// workers' partials in worker order): bitwise identical on every rank.
__host__ __device__ inline double rank_sum_element(const double* gathered, int world, size_t len, size_t i) {
  double acc = gathered[i];
  for (int r = 1; r < world; ++r) acc += gathered[static_cast<size_t>(r) * len + i];
  return acc;
}
// evaluate.cpp:157-172: g_j -= nu_j, J -= sum psi nu.
__host__ __device__ inline double finalize_gradient_element(const double* res, const double* nu, size_t j) {
  return res[j] - nu[j];
}
__host__ __device__ inline void finalize_scalars(const double* res, size_t n, double psi_nu, double* out) {
  out[kResJ] = res[n + kResJ] - psi_nu;
  out[kResD] = res[n + kResD];
  out[kResPairs] = res[n + kResPairs];
  out[kResEmpty] = res[n + kResEmpty];
  out[kResVisited] = res[n + kResVisited];
}

struct DeviceTargets {
  const double4* y;   // {y0, y1, y2, ln nu}
  const double* nu;
  int n;
  double3 lo, hi;     // bounding box of the target points
};

struct DeviceAtoms {
  const double4* x;   // {x0, x1, x2, m}
  int nq;
};

// Workspace pointers for one evaluation.
struct EvalBuffers {
  double* psi;        // [N]
  double* b2;         // [N]
  double* scal;       // [kNumSlots]
  double* part;       // reduction partials scratch [>= 2 * 1024]
  double* partS;      // [splitsA * nq]
  double* shiftA;     // [nq]  c2 |x'|^2 about the pass-A origin
  double* atomL;      // [nq]  ln S_q (natural units, reference log_S)
  double* atomLam;    // [nq]  log2 m_q - log2 S_q
  double* atomJ;      // [nq]  eps * ln S_q * m_q
  double* atomD;      // [nq]  m_q exp(-ln S_q)
  int* flagged;       // [nq]  indices of atoms needing the exact path
  double* partG;      // [splitsB * N]
  double* res;        // [N + kResTail]
  double* g_out;      // [N]   final gradient (device)
  double* scalars_out;// [kResTail] final J, D, pairs, empty, visited
  cudaEvent_t* timing = nullptr;  // optional: [0] start [1..2] pass A
                                  // [3..4] pass B [5] end
};

struct DenseLaunch {
  int apt;            // atoms per thread in pass A (1 or 2)
  int splitsA;        // target splits in pass A
  int tpt;            // targets per thread in pass B (1 or 2)
  int splitsB;        // atom splits in pass B
};

DenseLaunch plan_dense(int nq, int n, int num_sms);

// Per-eval prologue: b2, B, sum psi nu, psi finiteness.
void launch_prologue(const DeviceTargets& t, EvalBuffers& b, double eps,
                     cudaStream_t s);

// Dense evaluation of this rank's atoms; leaves the packed partial result
// (before the -nu / -sum psi nu finalisation) in b.res.
void launch_dense(const DeviceAtoms& a, const DeviceTargets& t, EvalBuffers& b,
                  const DenseLaunch& plan, double eps, cudaStream_t s);

// out[i] = sum over r = 0..world-1 (in rank order) of gathered[r * len + i].
void launch_rank_sum(const double* gathered, int world, size_t len, double* out, cudaStream_t s);

// After the (optional) cross-rank sum of b.res: g = res - nu, J -= sum psi nu.
void launch_finalize(const DeviceTargets& t, EvalBuffers& b, cudaStream_t s);

// Deterministic fixed-order sum of x[0..n) into out[0] (two launches).
void launch_det_sum(const double* x, size_t n, double* partials, double* out,
                    cudaStream_t s);
// launch_det_sum of four arrays into out[0..3] (bitwise the same results);
// range = device {lo, hi} or null (entries outside count as zero);
// partials holds 4 x 1024 doubles.
void launch_det_sum4(const double* x0, const double* x1, const double* x2, const double* x3, size_t n,
                     const int* range, double* partials, double* out, cudaStream_t s);

// Dense target-major gather (softmax_refine phase 2), see dense.cu.
void launch_dense_gather(const double4* atoms, const double* lam, int nq, const double4* ty,
                         const double* b2, int n, double c2, int num_sms, double* partG,
                         size_t partG_cap, double* G, cudaStream_t s);

// FP64 DFMA peak probe (roofline denominator), returns DFMA/s.
double measure_dfma_rate(cudaStream_t s);
// FP32 pipe (FFMA lane-ops/s) and MUFU.EX2 (lane-ops/s) probes (the fp32
// path's roofline denominators).
void measure_fp32_rates(cudaStream_t s, double* ffma_per_s, double* ex2_per_s);

}  // namespace rsot_cuda
