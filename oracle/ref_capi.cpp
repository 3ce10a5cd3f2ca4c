// ref_capi.cpp -- C entry points into the reference library compiled from
// /root/reference/proj/src (oracle/_ref/librsot_ref.so), so tests and
// bench.py (--impl reference, cpu_baseline) can drive the UNMODIFIED
// reference rsot::evaluate_dual (proj/src/evaluate.cpp:86-174) through
// ctypes.  TEST INFRASTRUCTURE ONLY.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <memory>
#include <string>

#include "rsot/evaluate.hpp"
#include "rsot/measures.hpp"
#include "rsot/plan.hpp"
#include "rsot/solve.hpp"
#include "rsot/spatial_index.hpp"

namespace {

thread_local std::string g_err;

struct RefProblem {
  rsot::SourceAtoms atoms;
  rsot::TargetMeasure target;
  std::unique_ptr<rsot::SpatialIndex> index;
};

rsot::PointList to_points(const double* xyz, size_t n) {
  rsot::PointList p(n);
  if (n) std::memcpy(p.data(), xyz, sizeof(double) * 3 * n);
  return p;
}

}  // namespace

extern "C" {

typedef struct ref_scalars {
  double J;
  double D;
  uint64_t atoms_visited;
  uint64_t candidate_pairs;
  uint64_t empty_candidate_atoms;
} ref_scalars;

const char* ref_last_error(void) { return g_err.c_str(); }

// Builds SourceAtoms (masses used as given), TargetMeasure and the
// per-stage SpatialIndex (solve.cpp:29).  Returns NULL on error.
void* ref_problem_create(int dim, const double* atom_xyz, const double* mass,
                         size_t nq, const double* target_xyz, const double* nu,
                         size_t n) {
  try {
    auto p = std::make_unique<RefProblem>();
    p->atoms.dim = dim;
    p->atoms.points = to_points(atom_xyz, nq);
    p->atoms.masses.assign(mass, mass + nq);
    p->atoms.quad_weights.assign(nq, 1.0);
    p->atoms.densities.assign(nq, 1.0);
    p->target.dim = dim;
    p->target.points = to_points(target_xyz, n);
    p->target.weights.assign(nu, nu + n);
    p->index = std::make_unique<rsot::SpatialIndex>(p->target.points);
    return p.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_problem_destroy(void* p) { delete static_cast<RefProblem*>(p); }

// rsot::evaluate_dual with cfg.epsilon = eps, cfg.workers = workers and
// trunc.cutoff = cutoff (+inf = dense).  Returns 0, -1 on
// std::invalid_argument, -2 on any other exception.
int ref_evaluate_dual(void* prob, const double* psi, size_t n, double eps,
                      double cutoff, int workers, double* g_out,
                      ref_scalars* out) {
  auto* p = static_cast<RefProblem*>(prob);
  try {
    rsot::SolverConfig cfg;
    cfg.epsilon = eps;
    cfg.workers = workers;
    rsot::TruncationState trunc;
    trunc.set_weight_stats(p->target.weights);
    trunc.cutoff = cutoff;
    rsot::DualPotential pot{std::vector<double>(psi, psi + n), rsot::Gauge::Raw};
    const rsot::EvalResult r =
        rsot::evaluate_dual(p->atoms, p->target, pot, cfg, trunc, *p->index);
    std::memcpy(g_out, r.gradient.data(), sizeof(double) * r.gradient.size());
    out->J = r.J;
    out->D = r.D;
    out->atoms_visited = r.atoms_visited;
    out->candidate_pairs = r.candidate_pairs;
    out->empty_candidate_atoms = r.empty_candidate_atoms;
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

// rsot::evaluate_dual with cfg.cost_kind = kind (0 SqEuclidean, 1
// SqGeodesicSphere), single worker.
int ref_evaluate_dual_kind(void* prob, const double* psi, size_t n, double eps, double cutoff,
                           int kind, double* g_out, ref_scalars* out) {
  auto* p = static_cast<RefProblem*>(prob);
  try {
    rsot::SolverConfig cfg;
    cfg.epsilon = eps;
    cfg.workers = 1;
    cfg.cost_kind = kind ? rsot::CostKind::SqGeodesicSphere : rsot::CostKind::SqEuclidean;
    rsot::TruncationState trunc;
    trunc.set_weight_stats(p->target.weights);
    trunc.cutoff = cutoff;
    rsot::DualPotential pot{std::vector<double>(psi, psi + n), rsot::Gauge::Raw};
    const rsot::EvalResult r = rsot::evaluate_dual(p->atoms, p->target, pot, cfg, trunc, *p->index);
    std::memcpy(g_out, r.gradient.data(), sizeof(double) * r.gradient.size());
    out->J = r.J;
    out->D = r.D;
    out->atoms_visited = r.atoms_visited;
    out->candidate_pairs = r.candidate_pairs;
    out->empty_candidate_atoms = r.empty_candidate_atoms;
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

// rsot::covering_cost (spatial_index.cpp:101-121 semantics); kind 0 =
// SqEuclidean, 1 = SqGeodesicSphere (the reference's full scan).
int ref_covering_cost_kind(void* prob, int kind, double* out) {
  auto* p = static_cast<RefProblem*>(prob);
  try {
    *out = rsot::covering_cost(p->atoms, p->target,
                               kind == 1 ? rsot::CostKind::SqGeodesicSphere : rsot::CostKind::SqEuclidean);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_covering_cost(void* prob, double* out) { return ref_covering_cost_kind(prob, 0, out); }

// rsot::softmax_refine (solve.cpp:62-142): prob's targets are the coarse
// level, prob's atoms the atoms; fine points given separately.
int ref_softmax_refine(void* prob, const double* coarse_psi, const double* fine_xyz,
                       size_t n_fine, double eps, double cutoff, int workers,
                       double* psi_out) {
  auto* p = static_cast<RefProblem*>(prob);
  try {
    const std::vector<double> cpsi(coarse_psi, coarse_psi + p->target.size());
    const rsot::PointList fine = to_points(fine_xyz, n_fine);
    const std::vector<double> out =
        rsot::softmax_refine(p->target, cpsi, fine, p->atoms, eps,
                             rsot::CostKind::SqEuclidean, cutoff, workers);
    std::memcpy(psi_out, out.data(), sizeof(double) * n_fine);
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

// rsot::PlanView (plan.cpp) on this problem: candidate counts, target
// marginals, conditional barycentres (starved index or -1), barycentric map
// and modal target indices.  Outputs may be NULL.
int ref_plan_view(void* prob, const double* psi, double eps, double cutoff, uint64_t* count_out,
                  double* marginal_out, double* bary_out, int64_t* starved_out,
                  double* map_out, uint64_t* modal_out) {
  auto* p = static_cast<RefProblem*>(prob);
  try {
    rsot::DualPotential pot{std::vector<double>(psi, psi + p->target.size()), rsot::Gauge::Raw};
    const rsot::PlanView plan(p->atoms, p->target, pot, eps, rsot::CostKind::SqEuclidean, cutoff, 1);
    if (count_out)
      for (size_t q = 0; q < p->atoms.size(); ++q) count_out[q] = plan.candidates(q).size();
    if (marginal_out) {
      const std::vector<double> m = plan.target_marginals();
      std::memcpy(marginal_out, m.data(), sizeof(double) * m.size());
    }
    if (bary_out) {
      *starved_out = -1;
      try {
        const rsot::PointList b = plan.all_conditional_barycenters();
        std::memcpy(bary_out, b.data(), sizeof(double) * 3 * b.size());
      } catch (const std::runtime_error& e) {
        const std::string msg = e.what();
        const auto k = msg.rfind(' ');
        *starved_out = std::stoll(msg.substr(k + 1));
      }
    }
    if (map_out) {
      const rsot::MapSample m = rsot::barycentric_map(plan);
      std::memcpy(map_out, m.mapped.data(), sizeof(double) * 3 * m.mapped.size());
    }
    if (modal_out) {
      const rsot::MapSample m = rsot::modal_map(plan);
      for (size_t q = 0; q < m.target_index.size(); ++q) modal_out[q] = m.target_index[q];
    }
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

// rsot::cutoff_pointwise (evaluate.cpp:22-25) on this problem's weights.
double ref_cutoff_pointwise(double psi_max, double nu_max, double eps,
                            double delta_thr) {
  rsot::TruncationState t;
  t.psi_max = psi_max;
  t.nu_max = nu_max;
  return rsot::cutoff_pointwise(t, eps, delta_thr);
}

}  // extern "C"
