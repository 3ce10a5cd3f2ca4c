/*
 * rsot_oracle.h -- CPU restatement of the reference RSOT dual evaluator.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product (paper_2507_23602_b200/)
 * never links or calls it, and has no CPU fallback.
 *
 * It restates, in plain C with IEEE double and no FP contraction, the
 * reference functions on the hot path (paths relative to
 * /root/reference/proj):
 *   - rsot::evaluate_dual            src/evaluate.cpp:86-174
 *   - rsot::SpatialIndex::ball_query src/spatial_index.cpp:47-61
 *   - rsot::SpatialIndex::nearest    src/spatial_index.cpp:70-84
 *   - rsot::covering_cost            src/spatial_index.cpp:101-121
 *   - cutoff_* / refresh_truncation  src/evaluate.cpp:22-72
 *   - parallel_blocks partition      include/rsot/parallel.hpp:14-31
 * The R*-tree (Boost.Geometry, absent here, version unpinned) is replaced by
 * an exact uniform grid: ball_query output is sorted ascending, so any exact
 * index yields bitwise-identical evaluate_dual results.
 *
 * Parity is pinned by (1) the reference's own frozen values and tests
 * (proj/tests/test_core.cpp, test_geometry.cpp, run against the reference
 * compiled from source in oracle/_ref with this grid behind SpatialIndex),
 * and (2) golden vectors in tests/golden/ produced by that build.
 */
#ifndef RSOT_ORACLE_H_
#define RSOT_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_grid oracle_grid;

typedef struct oracle_scalars {
  double J;
  double D;
  uint64_t atoms_visited;
  uint64_t candidate_pairs;
  uint64_t empty_candidate_atoms;
} oracle_scalars;

/* Error codes (mirror the reference's exception classes). */
enum {
  ORACLE_OK = 0,
  ORACLE_INVALID_ARGUMENT = -1, /* std::invalid_argument */
  ORACLE_RUNTIME_ERROR = -2,    /* std::runtime_error */
  ORACLE_NO_MEMORY = -3
};

const char* oracle_last_error(void);

/* Exact uniform-grid point index over n points (AoS xyz).  Returns NULL and
 * sets ORACLE_INVALID_ARGUMENT on an empty point set
 * (spatial_index.cpp:31-32). */
oracle_grid* oracle_grid_create(const double* xyz, size_t n);
void oracle_grid_destroy(oracle_grid* g);
size_t oracle_grid_size(const oracle_grid* g);

/* {j : squared_distance(center, p_j) < radius*radius}, ascending.  Returns
 * the count; writes up to cap indices to out (out may be NULL to count). */
size_t oracle_grid_ball_query(const oracle_grid* g, const double center[3],
                              double radius, uint64_t* out, size_t cap);

/* Euclidean-nearest point, lowest index on ties. */
uint64_t oracle_grid_nearest(const oracle_grid* g, const double center[3]);

/* Candidate hash used for per-atom selection parity: sum over the candidate
 * set of splitmix64(j), wrapping mod 2^64 (order independent). */
uint64_t oracle_candidate_hash_term(uint64_t j);

/* rsot::evaluate_dual for CostKind::SqEuclidean.
 *   atoms  : nq points (AoS xyz) + masses
 *   target : n points (AoS xyz) + weights nu
 *   cutoff : +inf = dense; finite = ball query with radius sqrt(2*cutoff)
 *   workers: reference SolverConfig::workers (static contiguous partition)
 *   grid   : index over the targets (may be NULL: built internally when
 *            needed)
 * Outputs: g_out[n], scalars; optional per-atom arrays (may be NULL):
 *   cand_count[nq] (candidate set size, 1 for empty-fallback atoms),
 *   cand_hash[nq], log_s[nq] (ln S_q as the reference computes it).
 * Returns ORACLE_OK or ORACLE_INVALID_ARGUMENT (non-finite psi). */
int oracle_evaluate_dual(size_t nq, const double* atom_xyz,
                         const double* atom_mass, size_t n,
                         const double* target_xyz, const double* target_nu,
                         const double* psi, double eps, double cutoff,
                         int workers, const oracle_grid* grid, double* g_out,
                         oracle_scalars* out, uint32_t* cand_count,
                         uint64_t* cand_hash, double* log_s);

/* PlanView (proj/src/plan.cpp), SqEuclidean: per-atom log_S (ctor
 * :47-57) and candidate count; target_marginals (:85-91); unnormalised first
 * moments sum_q p m_q x_q and normalised conditional barycentres (:123-140;
 * *starved_out = first index with marginal < 1e-30, else -1);
 * barycentric_map (:142-156) and modal_map target indices (:158-182).
 * Every output may be NULL (bary needs marginal and moment). */
int oracle_plan_view(size_t nq, const double* atom_xyz, const double* atom_mass,
                     size_t n, const double* target_xyz, const double* target_nu,
                     const double* psi, double eps, double cutoff, double* log_s_out,
                     uint64_t* count_out, double* marginal_out, double* moment_out,
                     double* bary_out, double* map_out, uint64_t* modal_out,
                     int64_t* starved_out);

/* rsot::evaluate_dual for CostKind::SqGeodesicSphere (points on the unit
 * sphere), single worker: full-scan truncation c < cutoff, Euclidean nearest
 * for empty sets (evaluate.cpp:119-133, cost.hpp:19-33).  cand_count and
 * log_s may be NULL. */
int oracle_evaluate_dual_geodesic(size_t nq, const double* atom_xyz, const double* atom_mass,
                                  size_t n, const double* target_xyz, const double* target_nu,
                                  const double* psi, double eps, double cutoff, double* g_out,
                                  oracle_scalars* out, uint32_t* cand_count, double* log_s);

/* rsot::softmax_refine (proj/src/solve.cpp:62-142), SqEuclidean, single
 * worker: psi_out[n_fine] from the coarse potential.  Returns
 * ORACLE_INVALID_ARGUMENT on non-finite input or output (require_finite). */
int oracle_softmax_refine(size_t n_coarse, const double* coarse_xyz,
                          const double* coarse_nu, const double* coarse_psi,
                          size_t n_fine, const double* fine_xyz, size_t nq,
                          const double* atom_xyz, const double* atom_mass,
                          double eps, double cutoff, double* psi_out);

/* rsot::covering_cost, SqEuclidean: max_q min_j 0.5*|x_q - y_j|^2. */
int oracle_covering_cost(size_t nq, const double* atom_xyz, size_t n,
                         const double* target_xyz, double* out);

/* ball_radius (cost.hpp:38-42) for SqEuclidean. */
double oracle_ball_radius(double cutoff);

/* Cutoff formulas (evaluate.cpp:22-49).  The truncation state fields are
 * passed explicitly.  integrated/geometric return ORACLE_RUNTIME_ERROR when
 * the cached |J| is degenerate. */
double oracle_cutoff_pointwise(double psi_max, double nu_max, double eps,
                               double delta_thr);
int oracle_cutoff_integrated(double psi_max, double covering, double cached_D,
                             double cached_absJ, double eps, double tau,
                             double* out);
int oracle_cutoff_geometric(double covering, double psi_range, double nu_min,
                            double cached_absJ, double eps, double tau,
                            double* out);
double oracle_cutoff_bootstrap(double covering, double psi_range,
                               double nu_min, double eps, double tau);

#ifdef __cplusplus
}
#endif

#endif /* RSOT_ORACLE_H_ */
