// plan_check.cpp -- drives the drop-in PlanView (plan_cuda.cpp, reference
// header rsot/plan.hpp unchanged) on raw fp64 inputs for the parity test
// tests/test_gpu_dropin.py::test_dropin_plan_view.
//
// usage: plan_check <dir> <eps> <cutoff>
//   reads  <dir>/{atoms,masses,targets,nu,psi}.f64
//   writes <dir>/{count.u64,marginal.f64,bary.f64,map.f64,modal.u64,starved.txt}
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "rsot/plan.hpp"

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

template <class T>
void write(const std::string& path, const std::vector<T>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(sizeof(T) * v.size()));
}

rsot::PointList to_points(const std::vector<double>& xyz) {
  rsot::PointList p(xyz.size() / 3);
  for (size_t i = 0; i < p.size(); ++i) p[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  return p;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s <dir> <eps> <cutoff>\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];
  const double eps = std::atof(argv[2]);
  const double cutoff = std::strtod(argv[3], nullptr);
  try {
    rsot::SourceAtoms atoms;
    atoms.dim = 3;
    atoms.points = to_points(read_f64(dir + "/atoms.f64"));
    atoms.masses = read_f64(dir + "/masses.f64");
    atoms.quad_weights.assign(atoms.points.size(), 1.0);
    atoms.densities.assign(atoms.points.size(), 1.0);
    rsot::TargetMeasure target;
    target.dim = 3;
    target.points = to_points(read_f64(dir + "/targets.f64"));
    target.weights = read_f64(dir + "/nu.f64");
    const rsot::DualPotential psi{read_f64(dir + "/psi.f64"), rsot::Gauge::Raw};
    const rsot::PlanView plan(atoms, target, psi, eps, rsot::CostKind::SqEuclidean, cutoff);
    std::vector<uint64_t> count(atoms.size()), modal(atoms.size());
    for (size_t q = 0; q < atoms.size(); ++q) count[q] = plan.candidates(q).size();
    write(dir + "/count.u64", count);
    write(dir + "/marginal.f64", plan.target_marginals());
    std::string starved = "-1";
    std::vector<double> bary(3 * target.size(), 0.0);
    try {
      const rsot::PointList b = plan.all_conditional_barycenters();
      for (size_t j = 0; j < b.size(); ++j)
        for (int d = 0; d < 3; ++d) bary[3 * j + d] = b[j][d];
    } catch (const std::runtime_error& e) {
      const std::string msg = e.what();
      starved = msg.substr(msg.rfind(' ') + 1);
    }
    write(dir + "/bary.f64", bary);
    std::ofstream(dir + "/starved.txt") << starved << "\n";
    const rsot::MapSample m = rsot::barycentric_map(plan);
    std::vector<double> mp(3 * atoms.size());
    for (size_t q = 0; q < atoms.size(); ++q)
      for (int d = 0; d < 3; ++d) mp[3 * q + d] = m.mapped[q][d];
    write(dir + "/map.f64", mp);
    const rsot::MapSample md = rsot::modal_map(plan);
    for (size_t q = 0; q < atoms.size(); ++q) modal[q] = md.target_index[q];
    write(dir + "/modal.u64", modal);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "plan_check: %s\n", e.what());
    return 1;
  }
  return 0;
}
