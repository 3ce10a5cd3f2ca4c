// truncated.cuh -- cell-list truncated evaluation (internal interface).
//
// Replaces the R*-tree ball query of proj/src/spatial_index.cpp:47-61 and
// the nearest-target fallback of :70-84 with a uniform grid over the
// targets.  Targets and atoms are each sorted by (cell key, Morton code of
// the position inside the cell), so
//   - every cell's members are contiguous and every x-row of cells is one
//     contiguous range (the scan unit of both passes), and
//   - 128 consecutive sorted points form a spatially compact CTA chunk.
// The grid is rebuilt only when the truncation radius leaves the band the
// grid was sized for; the selection predicate itself is always the exact
// reference predicate ((dx*dx + dy*dy) + dz*dz) < r*r.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

#include "kernels.cuh"

namespace rsot_cuda {

struct GridDesc {
  double lo[3] = {0, 0, 0};
  double h = 1.0;       // cell side
  int dims[3] = {1, 1, 1};
  long long ncells = 1;
  uint64_t id = 0;      // unique id of this grid build
};

// Point orders:
//   Hilbert order (atoms; radius independent, built once): consecutive runs
//     of kFA points are spatially compact CTA chunks (no long jumps, unlike
//     Morton or row-major orders);
//   cell order (targets; per grid): rows of cells are contiguous scan ranges.
struct PointOrders {
  bool bbox_set = false;     // set once from the host data at creation
  double bbox_lo[3] = {0, 0, 0}, bbox_hi[3] = {0, 0, 0};
  int n = 0;                 // points in the Hilbert order
  bool hil_valid = false;
  double4* ph = nullptr;     // Hilbert-sorted copy
  int* perm_h = nullptr;     // Hilbert position -> original index
  bool cell_valid = false;
  uint64_t grid_id = 0;      // grid the cell order was built for
  int ncell_pts = 0;         // points in the cell order
  double4* pc = nullptr;     // cell-sorted copy
  int* perm_c = nullptr;     // cell position -> original index
  int* cell_start = nullptr; // [ncells + 1]
  void release();
};

struct TargetCells : PointOrders {
  double hmin = 0.0;         // cell side of the radius-free grid
  GridDesc g;
  double built_r = -1.0;
};

struct AtomCells : PointOrders {
  // bounding box of every Hilbert chunk {lo0, lo1, lo2, hi0, hi1, hi2}
  // (radius independent: built with the order; feeds the scan-cost pass)
  double* chunk_box = nullptr;
  int box_chunks = 0;
  void release();  // also frees the boxes
};

struct DebugOut {
  uint32_t* count = nullptr;  // [nq] original atom order
  uint64_t* hash = nullptr;
  double* log_s = nullptr;
};

struct TruncWorkspace {
  // device scratch, grown on demand
  void* cub_tmp = nullptr; size_t cub_bytes = 0;
  uint64_t* keys = nullptr; uint64_t* keys2 = nullptr; size_t keys_cap = 0;
  int* idx = nullptr; int* idx2 = nullptr; size_t idx_cap = 0;
  double* b2s = nullptr; size_t b2s_cap = 0;        // b2 in target cell order
  double* S = nullptr; double* atomL = nullptr;
  double* atomJ = nullptr; double* atomD = nullptr;
  double* cntd = nullptr; double* emptyd = nullptr; uint32_t* cnt = nullptr;
  uint64_t* hash = nullptr; size_t atom_cap = 0;
  unsigned long long* empty_fp = nullptr; size_t tgt_cap = 0;
  double* pts = nullptr; unsigned long long* near_out = nullptr; size_t pts_cap = 0;
  double* red = nullptr;  // reduction partials
  // heavy-chunk split (trunc_fused_split): scanned targets per chunk, flags,
  // the compacted list and its length; the side stream it runs on
  unsigned long long* chunk_cost = nullptr; unsigned char* heavy_flag = nullptr;  // (role per chunk)
  size_t chunk_cap = 0;
  unsigned long long* chunk_w = nullptr; unsigned long long* chunk_pre = nullptr;
  int* part_range = nullptr;                  // [5]: this rank's atoms [lo, hi), atom count, split count, queue
  int split_clusters = 0, split_clusters32 = 0;  // resident clusters of trunc_fused(32)_split
  cudaStream_t side = nullptr; cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  // phase-1 pair masks replayed by phase 2 (trunc_fused): slots held by
  // resident CTAs, busy flags, slot-search ticket
  uint32_t* mbuf = nullptr; int* mbusy = nullptr; unsigned* mticket = nullptr;
  // item indices of the target-major phase 2: one stream per (slot, warp)
  int* rbuf = nullptr;
  void release();
};

// Full truncated evaluation of this rank's atoms (after launch_prologue);
// part_world > 1: `a` holds every atom and this call evaluates the chunks
// chunk_role assigns to rank part_rank (work-balanced over the Hilbert order);
// leaves the packed partial result in b.res like launch_dense.  Returns 0
// or nonzero with err set.
int run_truncated(TruncWorkspace& ws, const DeviceAtoms& a, AtomCells& ac,
                  const DeviceTargets& t, TargetCells& tc, EvalBuffers& b,
                  double eps, double cutoff, int num_sms, DebugOut* dbg,
                  cudaStream_t s, std::string& err, bool fp32 = false,
                  int part_rank = 0, int part_world = 1);

// Dense-path debug outputs (count = N, hash over all targets, ln S_q).
void launch_dense_debug(const DeviceAtoms& a, const DeviceTargets& t,
                        const EvalBuffers& b, const DebugOut& dbg,
                        cudaStream_t s);

// Nearest target (original index, lowest on ties) of m host points.
int run_nearest_points(TruncWorkspace& ws, const DeviceTargets& t,
                       TargetCells& tc, const double* xyz_host, size_t m,
                       uint64_t* out_host, cudaStream_t s, std::string& err);

// covering_cost over this rank's atoms.
// PlanView candidate lists: idx_host[off_host[q] .. off_host[q+1]) receives
// atom q's ascending candidate set (ball query, nearest when empty); the
// offsets must come from the candidate counts of the same cutoff.
int run_plan_candidates(TruncWorkspace& ws, const DeviceAtoms& a, const DeviceTargets& t,
                        TargetCells& tc, double cutoff, bool geo, const uint64_t* off_host,
                        uint64_t* idx_host, cudaStream_t s, std::string& err);

// PlanView reductions over candidate lists (off_host == nullptr: all
// targets): target marginals, first moments (n x 3), barycentric map
// (nq x 3), modal target per atom.  Outputs may be null.
int run_plan_moments(const DeviceAtoms& a, const DeviceTargets& t, const double* psi_host,
                     double eps, bool geo, const double* log_s_host, const uint64_t* off_host,
                     const uint64_t* idx_host, const double atom_lo[3], double* marginal,
                     double* moment, double* map, uint64_t* modal, cudaStream_t s,
                     std::string& err);

int run_covering_cost(TruncWorkspace& ws, const DeviceAtoms& a,
                      const DeviceTargets& t, TargetCells& tc, double* out,
                      cudaStream_t s, std::string& err);

// Gradient accumulator overflow (fp_red: a single contribution >= 2^41):
// enqueues a copy of the device flag into *h_flag (pinned host memory);
// trunc_clear_overflow resets it (synchronous).
cudaError_t trunc_read_overflow(unsigned* h_flag, cudaStream_t s);
cudaError_t trunc_clear_overflow();

}  // namespace rsot_cuda
