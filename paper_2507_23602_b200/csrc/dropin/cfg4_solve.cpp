// cfg4_solve.cpp -- BASELINE config 4: the reference's host optimiser
// driving the B200 evaluator through a full multilevel solve.
//
// The composition follows SURVEY.md §8(d) (solve_multilevel on two levels
// would give the epsilon sequence 1e-1 -> 1e-4 only, solve.cpp:155-160):
//   1. rsot::solve(coarse atoms, coarse targets, eps = 1e-2, 1 scaling step)
//      -> stages eps = 1e-1, 1e-2                      (proj/src/solve.cpp:42-60)
//   2. rsot::softmax_refine(coarse, psi, fine points, fine atoms, eps = 1e-3,
//      last cutoff)                                     (solve.cpp:62-142, GPU)
//   3. rsot::solve(fine atoms, fine targets, eps = 1e-4, 1 scaling step,
//      psi0 = refined) -> stages eps = 1e-3, 1e-4
// Truncation: pointwise, delta_thr = 1e-12; stop at L1 |grad| <= delta_tol.
// All of solve/lbfgs is the reference's code compiled unchanged; only
// evaluate_dual, covering_cost and softmax_refine run on the GPU.
//
// usage: cfg4_solve <dir> [delta_tol] [max_iterations]
//   <dir>/{coarse,fine}_{atoms,masses,targets,nu}.f64  (raw little-endian)
// prints one JSON object.  RSOT_DUMP_STAGE_PSI=<prefix> also writes the
// (raw-gauge) potential entering every stage: <prefix>_{coarse_1e-01,
// coarse_1e-02, fine_1e-03, fine_1e-04}.f64.
//
// usage: cfg4_solve <dir> --stage <level> <eps> <psi_in.f64> [delta_tol] [max_iterations]
//   one stage alone (solve_single through rsot::solve with no scaling
//   steps) from a given potential: per-stage evaluation rates and the
//   behaviour of one stage, e.g. the CPU reference build (cfg4_solve_ref)
//   from the GPU run's potential entering that stage.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "rsot/solve.hpp"
#ifndef RSOT_REFERENCE_BUILD
#include "rsot_cuda_context.hpp"
#endif

namespace {

std::vector<double> read_f64(const std::string& path) {
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  if (!f) throw std::runtime_error("cannot open " + path);
  const std::streamsize bytes = f.tellg();
  f.seekg(0);
  std::vector<double> v(static_cast<size_t>(bytes) / sizeof(double));
  f.read(reinterpret_cast<char*>(v.data()), bytes);
  return v;
}

rsot::PointList to_points(const std::vector<double>& xyz) {
  rsot::PointList p(xyz.size() / 3);
  for (size_t i = 0; i < p.size(); ++i) p[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  return p;
}

rsot::SourceAtoms atoms_of(const std::string& dir, const std::string& lvl) {
  rsot::SourceAtoms a;
  a.dim = 3;
  a.points = to_points(read_f64(dir + "/" + lvl + "_atoms.f64"));
  a.masses = read_f64(dir + "/" + lvl + "_masses.f64");
  a.quad_weights.assign(a.points.size(), 1.0);
  a.densities.assign(a.points.size(), 1.0);
  return a;
}

rsot::TargetMeasure targets_of(const std::string& dir, const std::string& lvl) {
  rsot::TargetMeasure t;
  t.dim = 3;
  t.points = to_points(read_f64(dir + "/" + lvl + "_targets.f64"));
  t.weights = read_f64(dir + "/" + lvl + "_nu.f64");
  return t;
}

void print_stages(const rsot::SolverReport& r, const char* name, bool last) {
  std::printf("  \"%s\": [", name);
  for (size_t i = 0; i < r.stages.size(); ++i) {
    const auto& s = r.stages[i];
    std::printf("%s{\"epsilon\": %.3g, \"iterations\": %d, \"evaluations\": %d, "
                "\"final_grad_l1\": %.6e, \"final_J\": %.17g, \"wall_ms\": %.3f, \"status\": \"%s\", "
                "\"last_cutoff\": %.6e}",
                i ? ", " : "", s.epsilon, s.iterations, s.evaluations, s.final_grad_l1, s.final_J,
                s.wall_ms, rsot::to_string(s.status).c_str(),
                s.cutoff_history.empty() ? NAN : s.cutoff_history.back());
  }
  std::printf("]%s\n", last ? "" : ",");
}

}  // namespace

void dump_psi(const std::string& level, double eps, const std::vector<double>& psi) {
  const char* prefix = std::getenv("RSOT_DUMP_STAGE_PSI");
  if (!prefix) return;
  char tag[64];
  std::snprintf(tag, sizeof(tag), "_%s_%.0e.f64", level.c_str(), eps);
  std::ofstream f(std::string(prefix) + tag, std::ios::binary);
  f.write(reinterpret_cast<const char*>(psi.data()), static_cast<std::streamsize>(sizeof(double) * psi.size()));
}

// rsot::solve one epsilon at a time (the same stages as the scaling loop of
// solve.cpp:42-60), dumping the potential entering each stage.
std::pair<rsot::DualPotential, rsot::SolverReport> solve_staged(const rsot::SourceAtoms& a,
                                                                const rsot::TargetMeasure& t,
                                                                const rsot::SolverConfig& cfg,
                                                                std::vector<double> psi,
                                                                const std::string& level) {
  rsot::SolverReport rep;
  for (double eps : rsot::epsilon_schedule(cfg.epsilon, cfg.scaling_steps)) {
    dump_psi(level, eps, psi);
    rsot::SolverConfig st = cfg;
    st.epsilon = eps;
    st.scaling_steps = 0;
    auto [p, r] = rsot::solve(a, t, st, rsot::DualPotential{psi, rsot::Gauge::Raw});
    psi = p.values;
    for (auto& sr : r.stages) rep.stages.push_back(std::move(sr));
  }
  rep.converged = rep.stages.back().status == rsot::SolveStatus::Converged;
  return {rsot::DualPotential{std::move(psi), rsot::Gauge::Raw}, rep};
}

int run_stage(const std::string& dir, int argc, char** argv) {
  const std::string level = argv[3];
  const double eps = std::atof(argv[4]);
  const std::vector<double> psi0 = read_f64(argv[5]);
  const double tol = argc > 6 ? std::atof(argv[6]) : 1e-8;
  const int max_it = argc > 7 ? std::atoi(argv[7]) : 1000;
  const rsot::SourceAtoms a = atoms_of(dir, level);
  const rsot::TargetMeasure t = targets_of(dir, level);
  rsot::SolverConfig cfg;
  cfg.truncation = rsot::TruncationKind::Pointwise;
  cfg.delta_thr = 1e-12;
  cfg.delta_tol = tol;
  cfg.max_iterations = max_it;
  cfg.scaling_steps = 0;
  cfg.epsilon = eps;
  cfg.workers = std::getenv("RSOT_WORKERS") ? std::atoi(std::getenv("RSOT_WORKERS")) : 1;
  const auto t0 = std::chrono::steady_clock::now();
  auto [psi, rep] = rsot::solve(a, t, cfg, rsot::DualPotential{psi0, rsot::Gauge::Raw});
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  std::printf("{\n  \"workload\": \"cfg4 stage\", \"level\": \"%s\", \"n_atoms\": %zu, \"n_targets\": %zu, "
              "\"workers\": %d, \"max_iterations\": %d, \"wall_ms\": %.3f, \"evals_per_s\": %.4f,\n",
              level.c_str(), a.size(), t.size(), cfg.workers, max_it, ms,
              rep.total_evaluations() / (ms * 1e-3));
  print_stages(rep, "stages", true);
  std::printf("}\n");
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s <dir> [delta_tol] [max_iterations]\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];
  if (argc > 5 && std::string(argv[2]) == "--stage") {
    try {
      return run_stage(dir, argc, argv);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "cfg4_solve: %s\n", e.what());
      return 1;
    }
  }
  const double tol = argc > 2 ? std::atof(argv[2]) : 1e-8;
  const int max_it = argc > 3 ? std::atoi(argv[3]) : 1000;
  try {
    const rsot::SourceAtoms ca = atoms_of(dir, "coarse"), fa = atoms_of(dir, "fine");
    const rsot::TargetMeasure ct = targets_of(dir, "coarse"), ft = targets_of(dir, "fine");
    rsot::SolverConfig cfg;
    cfg.truncation = rsot::TruncationKind::Pointwise;
    cfg.delta_thr = 1e-12;
    cfg.delta_tol = tol;
    cfg.max_iterations = max_it;
    cfg.scaling_steps = 1;

    cfg.workers = std::getenv("RSOT_WORKERS") ? std::atoi(std::getenv("RSOT_WORKERS")) : 1;
    const auto t0 = std::chrono::steady_clock::now();
    cfg.epsilon = 1e-2;
    auto [psi_c, rep_c] = solve_staged(ca, ct, cfg, std::vector<double>(ct.size(), 0.0), "coarse");
    const auto t1 = std::chrono::steady_clock::now();
    const double last_cutoff = rep_c.stages.back().cutoff_history.back();
    const int workers = std::getenv("RSOT_WORKERS") ? std::atoi(std::getenv("RSOT_WORKERS")) : 1;
    cfg.workers = workers;
    std::vector<double> psi_f = rsot::softmax_refine(ct, psi_c.values, ft.points, fa, 1e-3,
                                                     rsot::CostKind::SqEuclidean, last_cutoff, workers);
    const auto t2 = std::chrono::steady_clock::now();
    cfg.epsilon = 1e-4;
    auto [psi, rep_f] = solve_staged(fa, ft, cfg, psi_f, "fine");
    const auto t3 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const int evals = rep_c.total_evaluations() + rep_f.total_evaluations();
    const double total = ms(t0, t3);
    const rsot::DualPotential gf = rsot::gauge_fixed(psi, ft.weights);
    double psi_sum = 0.0, psi_abs = 0.0;
    for (double v : gf.values) {
      psi_sum += v;
      psi_abs += std::fabs(v);
    }
    std::printf("{\n  \"workload\": \"cfg4\", \"n_coarse_atoms\": %zu, \"n_fine_atoms\": %zu, "
                "\"n_coarse_targets\": %zu, \"n_fine_targets\": %zu, \"delta_tol\": %.1e,\n",
                ca.size(), fa.size(), ct.size(), ft.size(), tol);
    std::printf("  \"wall_ms\": {\"coarse_solve\": %.3f, \"softmax_refine\": %.3f, \"fine_solve\": %.3f, "
                "\"total\": %.3f},\n",
                ms(t0, t1), ms(t1, t2), ms(t2, t3), total);
    std::printf("  \"evaluations\": %d, \"evals_per_s\": %.3f, \"converged\": %s, "
                "\"kernel_launches\": %llu,\n",
                evals, evals / (total * 1e-3), (rep_c.converged && rep_f.converged) ? "true" : "false",
#ifdef RSOT_REFERENCE_BUILD
                0ull);
#else
                static_cast<unsigned long long>(rsot::cuda::kernel_launches()));
#endif
    std::printf("  \"psi_gauge_fixed_l1\": %.17g, \"psi_gauge_fixed_sum\": %.6e,\n", psi_abs, psi_sum);
    if (const char* dump = std::getenv("RSOT_DUMP_PSI")) {
      std::ofstream f(dump, std::ios::binary);
      f.write(reinterpret_cast<const char*>(gf.values.data()), sizeof(double) * gf.values.size());
    }
    print_stages(rep_c, "coarse_stages", false);
    print_stages(rep_f, "fine_stages", true);
    std::printf("}\n");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "cfg4_solve: %s\n", e.what());
    return 1;
  }
  return 0;
}
