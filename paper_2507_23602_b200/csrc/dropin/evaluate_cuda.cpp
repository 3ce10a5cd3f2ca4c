// evaluate_cuda.cpp -- the B200 drop-in for proj/src/evaluate.cpp.
//
// Implements, against the reference's UNCHANGED header
// proj/include/rsot/evaluate.hpp:
//   - rsot::evaluate_dual (evaluate.hpp:79-82): validates like the reference
//     (evaluate.cpp:90-93, potential.hpp:42-46), then runs the evaluation on
//     the GPU through the C ABI of include/rsot_cuda.h.  No CPU fallback:
//     a missing/unsupported GPU throws std::runtime_error.
//   - the host-side truncation bookkeeping that shares the translation unit
//     in the reference (TruncationState stats, cutoff_* and
//     refresh_truncation, evaluate.cpp:11-72), restated operation for
//     operation because the reference L-BFGS loop (lbfgs.cpp:72,197) uses
//     them on the host.
// cfg.workers (a CPU thread count) is ignored; the GPU count comes from
// rsot_cuda_context.hpp.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <list>
#include <mutex>
#include <stdexcept>
#include <string>

#include "rsot/evaluate.hpp"
#include "rsot/solve.hpp"
#include "rsot_cuda.h"
#include "rsot_cuda_context.hpp"

namespace rsot {

// ---- evaluate.cpp:11-72 (host scalars) -------------------------------------

void TruncationState::set_psi_stats(const std::vector<double>& psi) {
  psi_max = *std::max_element(psi.begin(), psi.end());
  psi_min = *std::min_element(psi.begin(), psi.end());
  psi_range = psi_max - psi_min;
}

void TruncationState::set_weight_stats(const std::vector<double>& nu) {
  nu_max = *std::max_element(nu.begin(), nu.end());
  nu_min = *std::min_element(nu.begin(), nu.end());
}

double cutoff_pointwise(const TruncationState& trunc, double eps, double delta_thr) {
  return trunc.psi_max + eps * std::log(trunc.nu_max / delta_thr);
}

double cutoff_integrated(const TruncationState& trunc, double eps, double tau) {
  const double absJ = std::max(trunc.cached_absJ, 1e-30);
  if (absJ <= 1e-30) throw std::runtime_error("functional estimate degenerate");
  const double c = trunc.psi_max + eps * std::log(eps * trunc.cached_D / (tau * absJ));
  return std::max(c, trunc.covering);
}

double cutoff_geometric(const TruncationState& trunc, double eps, double tau) {
  const double absJ = std::max(trunc.cached_absJ, 1e-30);
  if (absJ <= 1e-30) throw std::runtime_error("functional estimate degenerate");
  const double c = trunc.covering + trunc.psi_range +
                   eps * std::log(eps / (trunc.nu_min * tau * absJ));
  return std::max(c, trunc.covering);
}

double cutoff_bootstrap(const TruncationState& trunc, double eps, double tau) {
  const double c = trunc.covering + trunc.psi_range + eps * std::log(eps / (trunc.nu_min * tau));
  return std::max(c, trunc.covering);
}

void refresh_truncation(TruncationState& trunc, const std::vector<double>& psi,
                        const SolverConfig& cfg) {
  trunc.set_psi_stats(psi);
  switch (cfg.truncation) {
    case TruncationKind::None:
      trunc.cutoff = std::numeric_limits<double>::infinity();
      break;
    case TruncationKind::Pointwise:
      trunc.cutoff = cutoff_pointwise(trunc, cfg.epsilon, cfg.delta_thr);
      break;
    case TruncationKind::Integrated:
      trunc.cutoff = trunc.has_cache ? cutoff_integrated(trunc, cfg.epsilon, cfg.tau)
                                     : cutoff_bootstrap(trunc, cfg.epsilon, cfg.tau);
      break;
    case TruncationKind::Geometric:
      trunc.cutoff = trunc.has_cache ? cutoff_geometric(trunc, cfg.epsilon, cfg.tau)
                                     : cutoff_bootstrap(trunc, cfg.epsilon, cfg.tau);
      break;
  }
}

// ---- device state ------------------------------------------------------------

namespace cuda_detail {

struct Key {
  const void* a = nullptr;
  const void* b = nullptr;
  size_t n = 0;
  uint64_t h = 0;
  bool operator==(const Key& o) const { return a == o.a && b == o.b && n == o.n && h == o.h; }
};

// Sampled FNV-1a over up to 4096 evenly spaced (point, weight) entries.
Key make_key(const PointList& pts, const std::vector<double>& w) {
  Key k;
  k.a = pts.data();
  k.b = w.data();
  k.n = pts.size();
  uint64_t h = 1469598103934665603ull;
  auto mix = [&h](const void* p, size_t bytes) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < bytes; ++i) h = (h ^ c[i]) * 1099511628211ull;
  };
  const size_t n = pts.size();
  const size_t step = n > 4096 ? n / 4096 : 1;
  for (size_t i = 0; i < n; i += step) {
    mix(pts[i].data(), sizeof(double) * 3);
    mix(&w[i], sizeof(double));
  }
  if (n) {
    mix(pts[n - 1].data(), sizeof(double) * 3);
    mix(&w[n - 1], sizeof(double));
  }
  k.h = h;
  return k;
}

[[noreturn]] void raise(int rc, const char* where) {
  const std::string msg = std::string(where) + ": " + rsot_cuda_last_error();
  if (rc == RSOT_CUDA_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct State {
  std::mutex mu;
  int device = -1;
  rsot_cuda_ctx* ctx = nullptr;
  int rank = 0, world = 1;
  std::list<std::pair<Key, rsot_cuda_targets*>> targets;  // MRU first
  std::list<std::pair<Key, rsot_cuda_atoms*>> atoms;
  static constexpr size_t kKeep = 4;

  int default_device() const {
    for (const char* v : {"RSOT_CUDA_DEVICE", "LOCAL_RANK"}) {
      const char* s = std::getenv(v);
      if (s && *s) return std::atoi(s);
    }
    return 0;
  }

  rsot_cuda_ctx* context() {
    if (!ctx) {
      if (device < 0) device = default_device();
      const int rc = rsot_cuda_ctx_create(device, &ctx);
      if (rc) raise(rc, "rsot::evaluate_dual (B200 drop-in)");
    }
    return ctx;
  }

  void clear() {
    for (auto& e : targets) rsot_cuda_targets_destroy(e.second);
    for (auto& e : atoms) rsot_cuda_atoms_destroy(e.second);
    targets.clear();
    atoms.clear();
  }

  rsot_cuda_targets* get_targets(const TargetMeasure& t) {
    const Key k = make_key(t.points, t.weights);
    for (auto it = targets.begin(); it != targets.end(); ++it)
      if (it->first == k) {
        targets.splice(targets.begin(), targets, it);
        return targets.front().second;
      }
    rsot_cuda_targets* h = nullptr;
    const int rc = rsot_cuda_targets_create(context(), t.points.data()->data(), t.weights.data(),
                                            t.points.size(), &h);
    if (rc) raise(rc, "rsot_cuda_targets_create");
    targets.emplace_front(k, h);
    while (targets.size() > kKeep) {
      rsot_cuda_targets_destroy(targets.back().second);
      targets.pop_back();
    }
    return h;
  }

  rsot_cuda_atoms* get_atoms(const SourceAtoms& a, bool full = false) {
    const int world_eff = full ? 1 : world;
    Key k = make_key(a.points, a.masses);
    k.h ^= static_cast<uint64_t>(world_eff) * 0x9E3779B97F4A7C15ull +
           static_cast<uint64_t>(full ? 0 : rank);
    for (auto it = atoms.begin(); it != atoms.end(); ++it)
      if (it->first == k) {
        atoms.splice(atoms.begin(), atoms, it);
        return atoms.front().second;
      }
    // multi-rank: every rank holds all atoms and each evaluation takes its
    // work-balanced share (rsot_cuda_atoms_create_partitioned)
    const size_t nq = a.points.size();
    rsot_cuda_atoms* h = nullptr;
    const double* xyz = nq ? a.points[0].data() : nullptr;
    const double* m = nq ? a.masses.data() : nullptr;
    const int rc = world_eff > 1 ? rsot_cuda_atoms_create_partitioned(context(), xyz, m, nq, &h)
                                 : rsot_cuda_atoms_create(context(), xyz, m, nq, &h);
    if (rc) raise(rc, "rsot_cuda_atoms_create");
    atoms.emplace_front(k, h);
    while (atoms.size() > kKeep) {
      rsot_cuda_atoms_destroy(atoms.back().second);
      atoms.pop_back();
    }
    return h;
  }
};

State& state() {
  static State s;
  return s;
}

}  // namespace cuda_detail

// ---- evaluate.cpp:86-174 on the GPU ---------------------------------------------

EvalResult evaluate_dual(const SourceAtoms& atoms, const TargetMeasure& target,
                         const DualPotential& psi, const SolverConfig& cfg,
                         const TruncationState& trunc, const SpatialIndex& index) {
  (void)index;  // the device cell list lives with the resident targets
  const std::size_t n_targets = target.size();
  if (psi.size() != n_targets)
    throw std::invalid_argument("evaluate_dual: psi length != target count");
  require_finite(psi.values);
  if (atoms.masses.size() != atoms.points.size())
    throw std::invalid_argument("evaluate_dual: atom mass/point size mismatch");

  auto& st = cuda_detail::state();
  std::lock_guard<std::mutex> lock(st.mu);
  rsot_cuda_targets* dt = st.get_targets(target);
  rsot_cuda_atoms* da = st.get_atoms(atoms);
  EvalResult result;
  result.gradient.assign(n_targets, 0.0);
  rsot_cuda_scalars sc{};
  // cost.hpp:17: SqGeodesicSphere runs the full-scan geodesic kernels
  const int kind = cfg.cost_kind == CostKind::SqGeodesicSphere ? RSOT_CUDA_COST_SQGEODESIC
                                                               : RSOT_CUDA_COST_SQEUCLIDEAN;
  const int rc = rsot_cuda_eval_cost(st.context(), da, dt, psi.values.data(), cfg.epsilon,
                                     trunc.cutoff, kind, result.gradient.data(), &sc);
  if (rc) cuda_detail::raise(rc, "rsot_cuda_eval");
  result.J = sc.J;
  result.D = sc.D;
  result.atoms_visited = sc.atoms_visited;
  result.candidate_pairs = sc.candidate_pairs;
  result.empty_candidate_atoms = sc.empty_candidate_atoms;
  return result;
}

// ---- solve.cpp:62-142 on the GPU ----------------------------------------------
// The reference defines softmax_refine in solve.cpp next to solve_multilevel;
// the drop-in build weakens that definition (objcopy --weaken-symbol, see
// csrc/dropin/Makefile) so this one serves both direct callers and the
// reference's own solve_multilevel (its call goes through the PLT).
std::vector<double> softmax_refine(const TargetMeasure& coarse,
                                   const std::vector<double>& coarse_psi,
                                   const PointList& fine_points, const SourceAtoms& atoms,
                                   double eps, CostKind kind, double cutoff, int workers) {
  (void)workers;  // CPU thread count in the reference
  if (coarse_psi.size() != coarse.size())
    throw std::invalid_argument("softmax refine: psi/coarse size mismatch");
  require_finite(coarse_psi);
  if (kind != CostKind::SqEuclidean)
    throw std::invalid_argument(
        "softmax_refine (B200): SqGeodesicSphere is out of scope for the GPU path");
  auto& st = cuda_detail::state();
  std::lock_guard<std::mutex> lock(st.mu);
  rsot_cuda_targets* dt = st.get_targets(coarse);
  rsot_cuda_atoms* da = st.get_atoms(atoms, /*full=*/true);
  std::vector<double> out(fine_points.size());
  const int rc = rsot_cuda_softmax_refine(st.context(), dt, coarse_psi.data(),
                                          fine_points.empty() ? nullptr : fine_points.data()->data(),
                                          fine_points.size(), da, eps, cutoff, out.data());
  if (rc) cuda_detail::raise(rc, "rsot_cuda_softmax_refine");
  return out;
}

namespace cuda {

void set_device(int device) {
  auto& st = cuda_detail::state();
  std::lock_guard<std::mutex> lock(st.mu);
  if (st.ctx) throw std::logic_error("rsot::cuda::set_device after the first evaluation");
  st.device = device;
}

void unique_id(unsigned char id[128]) {
  const int rc = rsot_cuda_comm_unique_id(id);
  if (rc) cuda_detail::raise(rc, "rsot_cuda_comm_unique_id");
}

void set_comm(int rank, int world, const unsigned char id[128]) {
  auto& st = cuda_detail::state();
  std::lock_guard<std::mutex> lock(st.mu);
  st.clear();
  const int rc = rsot_cuda_ctx_set_comm(st.context(), rank, world, id);
  if (rc) cuda_detail::raise(rc, "rsot_cuda_ctx_set_comm");
  st.rank = rank;
  st.world = world;
}

void clear_cache() {
  auto& st = cuda_detail::state();
  std::lock_guard<std::mutex> lock(st.mu);
  st.clear();
}

std::uint64_t kernel_launches() { return rsot_cuda_kernel_launches(); }

// covering_cost on the GPU (spatial_index_cuda.cpp).
double covering_cost_device(const SourceAtoms& atoms, const TargetMeasure& target) {
  auto& st = cuda_detail::state();
  std::lock_guard<std::mutex> lock(st.mu);
  rsot_cuda_targets* dt = st.get_targets(target);
  rsot_cuda_atoms* da = st.get_atoms(atoms);
  double c0 = 0.0;
  const int rc = rsot_cuda_covering_cost(st.context(), da, dt, &c0);
  if (rc) cuda_detail::raise(rc, "rsot_cuda_covering_cost");
  return c0;
}

// ---- PlanView building blocks (plan_cuda.cpp) -------------------------------

void plan_build_device(const SourceAtoms& atoms, const TargetMeasure& target,
                       const std::vector<double>& psi, double eps, double cutoff, bool geodesic,
                       std::vector<double>& log_S,
                       std::vector<std::vector<std::size_t>>& candidates) {
  auto& st = cuda_detail::state();
  std::lock_guard<std::mutex> lock(st.mu);
  rsot_cuda_targets* dt = st.get_targets(target);
  rsot_cuda_atoms* da = st.get_atoms(atoms, /*full=*/true);
  const std::size_t nq = atoms.size(), n = target.size();
  log_S.assign(nq, 0.0);
  std::vector<uint32_t> count(nq);
  std::vector<double> g(n);
  rsot_cuda_scalars sc{};
  const int kind = geodesic ? RSOT_CUDA_COST_SQGEODESIC : RSOT_CUDA_COST_SQEUCLIDEAN;
  int rc = rsot_cuda_eval_debug_cost(st.context(), da, dt, psi.data(), eps, cutoff, kind, g.data(),
                                     &sc, count.data(), nullptr, log_S.data());
  if (rc) cuda_detail::raise(rc, "PlanView (B200 drop-in)");
  std::vector<uint64_t> off(nq + 1, 0);
  for (std::size_t q = 0; q < nq; ++q) off[q + 1] = off[q] + count[q];
  std::vector<uint64_t> idx(std::max<uint64_t>(off[nq], 1));
  rc = rsot_cuda_plan_candidates(st.context(), da, dt, cutoff, kind, off.data(), idx.data());
  if (rc) cuda_detail::raise(rc, "PlanView (B200 drop-in)");
  candidates.assign(nq, {});
  for (std::size_t q = 0; q < nq; ++q)
    candidates[q].assign(idx.begin() + static_cast<std::ptrdiff_t>(off[q]),
                         idx.begin() + static_cast<std::ptrdiff_t>(off[q + 1]));
}

void plan_moments_device(const SourceAtoms& atoms, const TargetMeasure& target,
                         const std::vector<double>& psi, double eps, bool geodesic,
                         const std::vector<double>& log_S,
                         const std::vector<std::vector<std::size_t>>& candidates,
                         double* marginal, double* moment, double* map, std::uint64_t* modal) {
  auto& st = cuda_detail::state();
  std::lock_guard<std::mutex> lock(st.mu);
  rsot_cuda_targets* dt = st.get_targets(target);
  rsot_cuda_atoms* da = st.get_atoms(atoms, /*full=*/true);
  const std::size_t nq = atoms.size(), n = target.size();
  // dense plans (every set = all targets, ascending) need no index upload
  bool dense = true;
  for (std::size_t q = 0; q < nq && dense; ++q) dense = candidates[q].size() == n;
  std::vector<uint64_t> off, idx;
  if (!dense) {
    off.assign(nq + 1, 0);
    for (std::size_t q = 0; q < nq; ++q) off[q + 1] = off[q] + candidates[q].size();
    idx.reserve(std::max<uint64_t>(off[nq], 1));
    for (const auto& c : candidates) idx.insert(idx.end(), c.begin(), c.end());
    if (idx.empty()) idx.push_back(0);
  }
  const int rc = rsot_cuda_plan_moments(st.context(), da, dt, psi.data(), eps,
                                        geodesic ? RSOT_CUDA_COST_SQGEODESIC : RSOT_CUDA_COST_SQEUCLIDEAN,
                                        log_S.data(),
                                        dense ? nullptr : off.data(), dense ? nullptr : idx.data(),
                                        marginal, moment, map, modal);
  if (rc) cuda_detail::raise(rc, "PlanView (B200 drop-in)");
}

}  // namespace cuda
}  // namespace rsot
