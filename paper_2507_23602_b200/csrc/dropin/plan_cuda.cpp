// plan_cuda.cpp -- drop-in replacement of proj/src/plan.cpp (PlanView and
// the map extractors of proj/include/rsot/plan.hpp, header unchanged).
//
// The O(pairs) work runs on the GPU through the C ABI:
//   ctor                        log_S_q + candidate sets      (plan.cpp:12-59)
//   target_marginals            sum_q p_qj m_q                (plan.cpp:85-91)
//   all_conditional_barycenters first moments / marginals     (plan.cpp:123-140)
//   barycentric_map             sum_j p_qj y_j per atom       (plan.cpp:142-156)
//   modal_map                   argmax_j psi_j - c + eps ln nu_j (plan.cpp:158-182)
// The per-atom / per-target accessors (plan_density, conditional_density,
// conditional_barycenter) and the pointwise helpers (displacement_interpolate,
// transfer_field) are cheap queries over the cached sets and stay host code
// with the reference's semantics.  Both cost kinds run on the GPU (the
// geodesic one by full scans, as the reference).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <iostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "rsot/plan.hpp"
#include "rsot_cuda_context.hpp"

namespace rsot {

namespace {

// e_qj = (psi_j - c(x_q, y_j)) / eps + ln nu_j, as plan_density forms it.
double plan_exponent(const PlanView& plan, std::size_t q, std::size_t j) {
  const double c = cost(plan.cost_kind(), plan.atoms().points[q], plan.target().points[j]);
  return (plan.psi_value(j) - c) / plan.epsilon() + std::log(plan.target().weights[j]);
}

[[noreturn]] void starved(std::size_t j) {
  throw std::runtime_error("target starved: index " + std::to_string(j));
}

}  // namespace

PlanView::PlanView(const SourceAtoms& atoms, const TargetMeasure& target,
                   const DualPotential& psi, double eps, CostKind kind, double cutoff,
                   int workers)
    : atoms_(atoms), target_(target), psi_(psi.values), eps_(eps), kind_(kind) {
  (void)workers;  // host thread count in the reference
  if (psi_.size() != target_.size())
    throw std::invalid_argument("plan view: psi length != target count");
  require_finite(psi_);
  if (target_.points.empty()) throw std::invalid_argument("spatial index: empty point set");
  cuda::plan_build_device(atoms_, target_, psi_, eps_, cutoff, kind_ == CostKind::SqGeodesicSphere,
                          log_S_, candidates_);
}

void PlanView::set_convergence(double grad_l1, double delta_tol) {
  converged_known_ = true;
  converged_ = grad_l1 <= delta_tol;
}

std::vector<std::pair<std::size_t, double>> PlanView::plan_density(std::size_t q) const {
  std::vector<std::pair<std::size_t, double>> out;
  out.reserve(candidates_[q].size());
  for (std::size_t j : candidates_[q]) out.emplace_back(j, std::exp(plan_exponent(*this, q, j) - log_S_[q]));
  return out;
}

std::vector<double> PlanView::target_marginals() const {
  std::vector<double> marg(target_.size(), 0.0);
  cuda::plan_moments_device(atoms_, target_, psi_, eps_, kind_ == CostKind::SqGeodesicSphere, log_S_,
                            candidates_, marg.data(), nullptr, nullptr, nullptr);
  return marg;
}

std::vector<double> PlanView::conditional_density(std::size_t j) const {
  if (converged_known_ && !converged_ && !warned_) {
    std::cerr << "warning: conditional density requested from an unconverged plan\n";
    warned_ = true;
  }
  // the candidate sets are ascending: one binary search per atom finds j
  std::vector<double> mu(atoms_.size(), 0.0);
  double tilde = 0.0;
  for (std::size_t q = 0; q < atoms_.size(); ++q) {
    const auto& c = candidates_[q];
    const auto it = std::lower_bound(c.begin(), c.end(), j);
    if (it == c.end() || *it != j) continue;
    mu[q] = std::exp(plan_exponent(*this, q, j) - log_S_[q]) * atoms_.masses[q];
    tilde += mu[q];
  }
  if (tilde < 1e-30) starved(j);
  for (double& v : mu) v /= tilde;
  return mu;
}

Point PlanView::conditional_barycenter(std::size_t j) const {
  const std::vector<double> mu = conditional_density(j);
  Point t{0.0, 0.0, 0.0};
  for (std::size_t q = 0; q < atoms_.size(); ++q) t = t + mu[q] * atoms_.points[q];
  return t;
}

PointList PlanView::all_conditional_barycenters() const {
  const std::size_t n = target_.size();
  std::vector<double> tilde(n), moment(3 * n);
  cuda::plan_moments_device(atoms_, target_, psi_, eps_, kind_ == CostKind::SqGeodesicSphere, log_S_,
                            candidates_, tilde.data(), moment.data(), nullptr, nullptr);
  PointList out(n);
  for (std::size_t j = 0; j < n; ++j) {
    if (tilde[j] < 1e-30) starved(j);
    const double inv = 1.0 / tilde[j];
    out[j] = Point{inv * moment[3 * j], inv * moment[3 * j + 1], inv * moment[3 * j + 2]};
  }
  return out;
}

// plan.hpp declares MapBuilder a friend of PlanView: the map extractors use
// it to hand the cached log_S_ / candidate sets to the GPU reductions.
struct MapBuilder {
  static void moments(const PlanView& p, double* marginal, double* moment, double* map,
                      std::uint64_t* modal) {
    cuda::plan_moments_device(p.atoms_, p.target_, p.psi_, p.eps_,
                              p.kind_ == CostKind::SqGeodesicSphere, p.log_S_, p.candidates_,
                              marginal, moment, map, modal);
  }
};

MapSample barycentric_map(const PlanView& plan) {
  const auto& atoms = plan.atoms();
  const std::size_t nq = atoms.size();
  std::vector<double> t(3 * nq);
  MapBuilder::moments(plan, nullptr, nullptr, t.data(), nullptr);
  MapSample map;
  map.kind = MapKind::Barycentric;
  map.mapped.resize(nq);
  map.displacement.resize(nq);
  for (std::size_t q = 0; q < nq; ++q) {
    map.mapped[q] = Point{t[3 * q], t[3 * q + 1], t[3 * q + 2]};
    map.displacement[q] = distance(map.mapped[q], atoms.points[q]);
  }
  return map;
}

MapSample modal_map(const PlanView& plan) {
  const auto& atoms = plan.atoms();
  const std::size_t nq = atoms.size();
  std::vector<std::uint64_t> best(nq);
  MapBuilder::moments(plan, nullptr, nullptr, nullptr, best.data());
  MapSample map;
  map.kind = MapKind::Modal;
  map.mapped.resize(nq);
  map.target_index.resize(nq);
  map.displacement.resize(nq);
  for (std::size_t q = 0; q < nq; ++q) {
    map.target_index[q] = best[q];
    map.mapped[q] = plan.target().points[best[q]];
    map.displacement[q] = distance(map.mapped[q], atoms.points[q]);
  }
  return map;
}

// x_alpha = (1 - alpha) x + alpha T(x) (plan.cpp:184-196).
PointList displacement_interpolate(const PlanView& plan, const MapSample& map, double alpha) {
  if (map.kind != MapKind::Barycentric)
    throw std::invalid_argument("interpolation requires a barycentric map");
  if (!(alpha >= 0.0 && alpha <= 1.0)) throw std::invalid_argument("alpha must lie in [0,1]");
  const auto& atoms = plan.atoms();
  PointList out(atoms.size());
  for (std::size_t q = 0; q < atoms.size(); ++q)
    out[q] = (1.0 - alpha) * atoms.points[q] + alpha * map.mapped[q];
  return out;
}

// Pushes a per-atom field through the map; modal maps also resolve
// collisions per target (lowest atom index first, mass-weighted mean)
// (plan.cpp:198-225).
TransferredField transfer_field(const PlanView& plan, const MapSample& map,
                                const std::vector<double>& field) {
  const auto& atoms = plan.atoms();
  if (field.size() != atoms.size()) throw std::invalid_argument("field length != atom count");
  TransferredField out;
  out.points = map.mapped;
  out.values = field;
  if (map.kind != MapKind::Modal) return out;
  const std::size_t n = plan.target().size();
  out.first_value_per_target.assign(n, 0.0);
  out.mean_value_per_target.assign(n, 0.0);
  out.target_hit.assign(n, false);
  std::vector<double> mass(n, 0.0);
  for (std::size_t q = 0; q < atoms.size(); ++q) {
    const std::size_t j = map.target_index[q];
    if (!out.target_hit[j]) {
      out.target_hit[j] = true;
      out.first_value_per_target[j] = field[q];
    }
    out.mean_value_per_target[j] += field[q] * atoms.masses[q];
    mass[j] += atoms.masses[q];
  }
  for (std::size_t j = 0; j < n; ++j)
    if (mass[j] > 0.0) out.mean_value_per_target[j] /= mass[j];
  return out;
}

}  // namespace rsot
