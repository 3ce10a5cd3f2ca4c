// rsot_cuda_context.hpp -- the one ADDITIONAL header of the B200 drop-in.
//
// The reference headers (proj/include/rsot/*.hpp) stay byte-identical, so
// the GPU selection and the multi-GPU communicator cannot be SolverConfig
// fields.  They live here instead.  Without any call the
// drop-in uses CUDA device $RSOT_CUDA_DEVICE, else $LOCAL_RANK, else 0, and a
// single GPU.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "rsot/measures.hpp"

namespace rsot::cuda {

// Select the CUDA device for subsequent evaluations (before the first one).
void set_device(int device);

// Attach an NCCL communicator: this process evaluates the atom shard
// [rank's contiguous range) and evaluate_dual returns the global result on
// every rank (one ncclAllGather + rank-ordered sum per evaluation).  `id` is 128 bytes from
// unique_id() on rank 0, shipped to the other ranks out of band.
void unique_id(unsigned char id[128]);
void set_comm(int rank, int world, const unsigned char id[128]);

// Drops all cached device-resident atoms/targets (e.g. between stages when
// memory is tight).  Cached entries are keyed by (data pointer, size, a
// sampled content hash): inputs must not be modified in place while cached
// (SourceAtoms / TargetMeasure are const for a stage in the reference).
void clear_cache();

// Kernel-launch counter of the underlying library (for tests/benchmarks).
std::uint64_t kernel_launches();

// GPU building blocks of the drop-in PlanView (plan_cuda.cpp), single GPU
// (all atoms on this process's device):
//   plan_build_device: log_S_q and the ascending candidate sets of the
//     PlanView ctor (plan.cpp:12-59);
//   plan_moments_device: over those sets, target marginals (n), first
//     moments (3n), barycentric images (3 nq) and modal targets (nq); any
//     output may be null.
void plan_build_device(const SourceAtoms& atoms, const TargetMeasure& target,
                       const std::vector<double>& psi, double eps, double cutoff, bool geodesic,
                       std::vector<double>& log_S,
                       std::vector<std::vector<std::size_t>>& candidates);
void plan_moments_device(const SourceAtoms& atoms, const TargetMeasure& target,
                         const std::vector<double>& psi, double eps, bool geodesic,
                         const std::vector<double>& log_S,
                         const std::vector<std::vector<std::size_t>>& candidates,
                         double* marginal, double* moment, double* map, std::uint64_t* modal);

}  // namespace rsot::cuda
