// inplace_check.cpp -- drives the drop-in rsot::evaluate_dual (unchanged
// evaluate.hpp) through the in-place update pattern of the reference's
// barycenter loop (barycenter.cpp:55, `nu.points = points` into the same
// vector) for tests/test_gpu_dropin.py::test_dropin_inplace_edits.
//
// usage: inplace_check <dir> <eps> <cutoff>
//   reads  <dir>/{atoms,masses,targets,targets2,nu,nu2,psi}.f64
//   evaluates (targets, nu), then overwrites the SAME TargetMeasure buffers
//   with targets2 (assignment of an equal-size PointList, as barycenter.cpp:55)
//   and evaluates again, then overwrites the weights in place with nu2 and
//   evaluates a third time, then the atom masses in place (x 2, renormalised
//   by the caller's files: masses2) and a fourth time;
//   writes <dir>/out{1,2,3,4}.f64 = [J, D, pairs, empty, visited, g...]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "rsot/evaluate.hpp"
#include "rsot/spatial_index.hpp"

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

void dump(const std::string& path, const rsot::EvalResult& r) {
  std::vector<double> v = {r.J, r.D, static_cast<double>(r.candidate_pairs),
                           static_cast<double>(r.empty_candidate_atoms), static_cast<double>(r.atoms_visited)};
  v.insert(v.end(), r.gradient.begin(), r.gradient.end());
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(sizeof(double) * v.size()));
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s <dir> <eps> <cutoff>\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];
  try {
    rsot::SourceAtoms atoms;
    atoms.dim = 3;
    atoms.points = to_points(read_f64(dir + "/atoms.f64"));
    atoms.masses = read_f64(dir + "/masses.f64");
    rsot::TargetMeasure nu;
    nu.dim = 3;
    nu.points = to_points(read_f64(dir + "/targets.f64"));
    nu.weights = read_f64(dir + "/nu.f64");
    const rsot::DualPotential psi{read_f64(dir + "/psi.f64"), rsot::Gauge::Raw};
    rsot::SolverConfig cfg;
    cfg.epsilon = std::atof(argv[2]);
    rsot::TruncationState trunc;
    trunc.cutoff = std::atof(argv[3]);
    const double* buf = nu.points.data()->data();
    {
      const rsot::SpatialIndex index(nu.points);
      dump(dir + "/out1.f64", rsot::evaluate_dual(atoms, nu, psi, cfg, trunc, index));
    }
    const rsot::PointList points = to_points(read_f64(dir + "/targets2.f64"));
    nu.points = points;  // barycenter.cpp:55: same size, same buffer
    if (nu.points.data()->data() != buf) throw std::runtime_error("buffer moved");
    {
      const rsot::SpatialIndex index(nu.points);
      dump(dir + "/out2.f64", rsot::evaluate_dual(atoms, nu, psi, cfg, trunc, index));
    }
    const std::vector<double> w2 = read_f64(dir + "/nu2.f64");
    for (size_t j = 0; j < w2.size(); ++j) nu.weights[j] = w2[j];
    {
      const rsot::SpatialIndex index(nu.points);
      dump(dir + "/out3.f64", rsot::evaluate_dual(atoms, nu, psi, cfg, trunc, index));
    }
    const std::vector<double> m2 = read_f64(dir + "/masses2.f64");
    for (size_t q = 0; q < m2.size(); ++q) atoms.masses[q] = m2[q];
    {
      const rsot::SpatialIndex index(nu.points);
      dump(dir + "/out4.f64", rsot::evaluate_dual(atoms, nu, psi, cfg, trunc, index));
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "inplace_check: %s\n", e.what());
    return 1;
  }
  return 0;
}
