// geodesic.cuh -- evaluate_dual for CostKind::SqGeodesicSphere (internal).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

#include "kernels.cuh"

namespace rsot_cuda {

struct GeoWorkspace {
  double* L = nullptr; size_t atom_cap_L = 0;
  double* J = nullptr; size_t atom_cap_J = 0;
  double* D = nullptr; size_t atom_cap_D = 0;
  double* cnt = nullptr; size_t atom_cap_c = 0;
  double* empty = nullptr; size_t atom_cap_e = 0;
  int* nearest = nullptr; size_t atom_cap_n = 0;
  double* G = nullptr; size_t tgt_cap_G = 0;
  unsigned long long* gacc = nullptr; size_t tgt_cap_a = 0;
  double* red = nullptr; size_t red_cap = 0;
  void release();
};

// Leaves the packed partial result [g + nu | J + sum psi nu | D | pairs |
// empty | visited] of this rank's atoms in b.res (like launch_dense /
// run_truncated); b.psi must hold psi.  cutoff = +inf: dense.
// Optional per-atom debug outputs (candidate count, hash, ln S_q).
int run_geodesic(GeoWorkspace& w, const DeviceAtoms& a, const DeviceTargets& t, EvalBuffers& b,
                 double eps, double cutoff, cudaStream_t s, std::string& err,
                 uint32_t* dbg_count = nullptr, uint64_t* dbg_hash = nullptr,
                 double* dbg_log_s = nullptr);

// covering_cost for SqGeodesicSphere (spatial_index.cpp:113-119,
// c0 = max_q min_j acos(clamp(x_q . y_j))^2): the cost is a non-increasing
// function of the clamped dot product, so min_j cost = cost(max_j clamp(dot))
// and max_q of that = cost(min_q max_j clamp(dot)).  The device computes
// t* = min_q max_j clamp(x_q . y_j) with the reference's unfused dot
// (cost.hpp:19-33, exact comparisons, order independent); the caller applies
// acos and the square on the host (the same libm call as the reference).
// Smallest clamped dot product t with fl(acos(t))^2 < cutoff under the
// host's libm (the reference's predicate is monotone in t): -inf when every
// t passes, +inf when none does.
double geo_dot_threshold(double cutoff);

int run_geo_covering_dot(GeoWorkspace& w, const DeviceAtoms& a, const DeviceTargets& t, double* t_star,
                         cudaStream_t s, std::string& err);

}  // namespace rsot_cuda
