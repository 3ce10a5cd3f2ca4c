// refine.cuh -- GPU softmax_refine (proj/src/solve.cpp:62-142), internal.
#pragma once

#include <string>

#include "kernels.cuh"

namespace rsot_cuda {

struct RefineWorkspace {
  double* partS = nullptr; size_t partS_cap = 0;
  unsigned* partC = nullptr; size_t partC_cap = 0;
  double* shiftA = nullptr; size_t shiftA_cap = 0;
  double* L2 = nullptr; size_t L2_cap = 0;
  double* lam = nullptr; size_t lam_cap = 0;
  int* flag = nullptr; size_t flag_cap = 0;
  double4* fine4 = nullptr; size_t fine4_cap = 0;
  double* zeros = nullptr; size_t zeros_cap = 0;
  double* fine = nullptr; size_t fine_cap = 0;
  double* G = nullptr; size_t G_cap = 0;
  double* psi = nullptr; size_t psi_cap = 0;
  double* partG = nullptr; size_t partG_cap = 0;
  double* misc = nullptr; size_t misc_cap = 0;
  void release();
};

// Runs both phases for this rank's atoms (single GPU: the phase-2 LSE runs
// over all atoms, so the atom handle must hold every atom).  b.psi / b.b2 /
// b.scal must hold the coarse prologue (launch_prologue on coarse targets).
int run_softmax_refine(RefineWorkspace& w, const DeviceAtoms& a, const DeviceTargets& coarse,
                       EvalBuffers& b, const double* fine_xyz_host, int n_fine, double eps,
                       double cutoff, int num_sms, double* psi_host, cudaStream_t s,
                       std::string& err);

}  // namespace rsot_cuda
