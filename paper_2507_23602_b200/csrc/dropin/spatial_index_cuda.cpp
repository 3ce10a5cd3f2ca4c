// spatial_index_cuda.cpp -- the B200 drop-in for proj/src/spatial_index.cpp.
//
// Implements rsot::SpatialIndex (proj/include/rsot/spatial_index.hpp:15-54,
// unchanged) without Boost.Geometry:
//   - evaluate_dual does not use it: its truncation query runs on the GPU
//     cell list that lives with the resident targets (truncated.cu);
//   - covering_cost runs on the GPU for both cost kinds
//     (rsot_cuda_covering_cost_kind: SqEuclidean by the nearest target per
//     atom over expanding cell rings, SqGeodesicSphere by a full scan of
//     clamped dot products; max over atoms and ranks);
//   - the per-point host queries (ball_query / nearest / range_query) serve
//     the reference's out-of-scope host callers (PlanView, plan.cpp:35-49;
//     nearest_atom_density_oracle, hierarchy.cpp:68-74) from worker threads,
//     so they are answered by an immutable exact host grid with the
//     reference semantics: strict squared_distance < radius*radius,
//     ascending output (spatial_index.cpp:47-61), lowest index on exact ties
//     (:70-84).  Safe for concurrent reads.
#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>

#include "rsot/spatial_index.hpp"

namespace rsot {

namespace cuda {
double covering_cost_device(const SourceAtoms& atoms, const TargetMeasure& target, bool geodesic);
}

struct SpatialIndex::Impl {
  PointList pts;
  double lo[3] = {0, 0, 0}, h[3] = {1, 1, 1};
  int dims[3] = {1, 1, 1};
  std::vector<std::size_t> start;  // cells + 1
  std::vector<std::size_t> idx;    // point indices grouped by cell, ascending

  int coord(int d, double v) const {
    const double t = (v - lo[d]) / h[d];
    if (!(t >= 0.0)) return 0;
    if (t >= dims[d]) return dims[d] - 1;
    return static_cast<int>(t);
  }
  std::size_t cell(int x, int y, int z) const {
    return (static_cast<std::size_t>(z) * dims[1] + y) * dims[0] + x;
  }
};

SpatialIndex::SpatialIndex(const PointList& points) {
  if (points.empty()) throw std::invalid_argument("spatial index: empty point set");
  impl_ = std::make_unique<Impl>();
  Impl& g = *impl_;
  g.pts = points;
  double hi[3];
  for (int d = 0; d < 3; ++d) g.lo[d] = hi[d] = points[0][d];
  for (const Point& p : points)
    for (int d = 0; d < 3; ++d) {
      g.lo[d] = std::min(g.lo[d], p[d]);
      hi[d] = std::max(hi[d], p[d]);
    }
  int active = 0;
  double vol = 1.0;
  for (int d = 0; d < 3; ++d)
    if (hi[d] > g.lo[d]) {
      ++active;
      vol *= hi[d] - g.lo[d];
    }
  const double side =
      active ? std::pow(vol / std::max(1.0, points.size() / 2.0), 1.0 / active) : 1.0;
  for (int d = 0; d < 3; ++d) {
    const double ext = hi[d] - g.lo[d];
    if (ext > 0.0) {
      g.dims[d] = static_cast<int>(std::min(std::floor(ext / side) + 1.0, 2048.0));
      g.h[d] = ext / g.dims[d] * (1.0 + 1e-12);
    }
  }
  const std::size_t ncell = static_cast<std::size_t>(g.dims[0]) * g.dims[1] * g.dims[2];
  g.start.assign(ncell + 1, 0);
  std::vector<std::size_t> cell_of(points.size());
  for (std::size_t i = 0; i < points.size(); ++i) {
    cell_of[i] = g.cell(g.coord(0, points[i][0]), g.coord(1, points[i][1]), g.coord(2, points[i][2]));
    ++g.start[cell_of[i] + 1];
  }
  for (std::size_t c = 0; c < ncell; ++c) g.start[c + 1] += g.start[c];
  g.idx.resize(points.size());
  std::vector<std::size_t> fill(g.start.begin(), g.start.end() - 1);
  for (std::size_t i = 0; i < points.size(); ++i) g.idx[fill[cell_of[i]]++] = i;
  count_ = points.size();
}

SpatialIndex::~SpatialIndex() = default;
SpatialIndex::SpatialIndex(SpatialIndex&&) noexcept = default;
SpatialIndex& SpatialIndex::operator=(SpatialIndex&&) noexcept = default;

void SpatialIndex::ball_query(const Point& center, double radius,
                              std::vector<std::size_t>& out) const {
  out.clear();
  if (!(radius > 0.0)) return;
  const Impl& g = *impl_;
  const double r2 = radius * radius;
  int lo[3], hi[3];
  for (int d = 0; d < 3; ++d) {
    lo[d] = std::max(0, g.coord(d, center[d] - radius) - 1);
    hi[d] = std::min(g.dims[d] - 1, g.coord(d, center[d] + radius) + 1);
  }
  for (int z = lo[2]; z <= hi[2]; ++z)
    for (int y = lo[1]; y <= hi[1]; ++y) {
      const std::size_t b = g.start[g.cell(lo[0], y, z)], e = g.start[g.cell(hi[0], y, z) + 1];
      for (std::size_t k = b; k < e; ++k)
        if (squared_distance(center, g.pts[g.idx[k]]) < r2) out.push_back(g.idx[k]);
    }
  std::sort(out.begin(), out.end());
}

std::vector<std::size_t> SpatialIndex::ball_query(const Point& center, double radius) const {
  std::vector<std::size_t> out;
  ball_query(center, radius, out);
  return out;
}

std::size_t SpatialIndex::nearest(const Point& center) const {
  const Impl& g = *impl_;
  int cc[3];
  for (int d = 0; d < 3; ++d) cc[d] = g.coord(d, center[d]);
  double best_d2 = std::numeric_limits<double>::infinity();
  std::size_t best = g.pts.size();
  for (int k = 0;; ++k) {
    for (int z = std::max(0, cc[2] - k); z <= std::min(g.dims[2] - 1, cc[2] + k); ++z)
      for (int y = std::max(0, cc[1] - k); y <= std::min(g.dims[1] - 1, cc[1] + k); ++y)
        for (int x = std::max(0, cc[0] - k); x <= std::min(g.dims[0] - 1, cc[0] + k); ++x) {
          if (std::max({std::abs(x - cc[0]), std::abs(y - cc[1]), std::abs(z - cc[2])}) != k) continue;
          const std::size_t c = g.cell(x, y, z);
          for (std::size_t t = g.start[c]; t < g.start[c + 1]; ++t) {
            const std::size_t j = g.idx[t];
            const double d2 = squared_distance(center, g.pts[j]);
            if (d2 < best_d2 || (d2 == best_d2 && j < best)) {
              best_d2 = d2;
              best = j;
            }
          }
        }
    double margin = std::numeric_limits<double>::infinity();
    bool left = false;
    for (int d = 0; d < 3; ++d) {
      if (cc[d] - k > 0) {
        margin = std::min(margin, center[d] - (g.lo[d] + (cc[d] - k) * g.h[d]));
        left = true;
      }
      if (cc[d] + k < g.dims[d] - 1) {
        margin = std::min(margin, (g.lo[d] + (cc[d] + k + 1) * g.h[d]) - center[d]);
        left = true;
      }
    }
    if (!left) break;
    margin = margin * (1.0 - 1e-9) - 1e-12;
    if (best < g.pts.size() && margin > 0.0 && margin * margin > best_d2 * (1.0 + 1e-9)) break;
  }
  return best;
}

SpatialIndex build_index(const PointList& points) { return SpatialIndex(points); }

std::vector<std::size_t> range_query(const SpatialIndex& index, const Point& center,
                                     double cutoff, CostKind kind) {
  if (cutoff < 0.0) throw std::invalid_argument("range query: negative cutoff");
  const auto radius = ball_radius(kind, cutoff);
  if (!radius)
    throw std::invalid_argument("range query: cost kind has no ball-radius conversion");
  return index.ball_query(center, *radius);
}

double covering_cost(const SourceAtoms& atoms, const TargetMeasure& target, CostKind kind) {
  if (atoms.size() == 0 || target.size() == 0)
    throw std::invalid_argument("covering cost: empty input");
  // both kinds on the GPU (SqGeodesicSphere: the reference's full scan,
  // spatial_index.cpp:113-119, as min_q max_j clamped dot + one host acos)
  return cuda::covering_cost_device(atoms, target, kind == CostKind::SqGeodesicSphere);
}

}  // namespace rsot
