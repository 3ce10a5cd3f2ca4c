/*
 * rsot_cuda.h -- C ABI of the B200-native RSOT dual evaluator.
 *
 * The drop-in boundary for rsot::evaluate_dual
 * (/root/reference/proj/include/rsot/evaluate.hpp:79-82, implemented at
 * proj/src/evaluate.cpp:86-174) and the target-side state of
 * rsot::SpatialIndex (proj/include/rsot/spatial_index.hpp:15-54).  Plain C:
 * pointers, sizes and status codes; no CUDA or torch types in signatures.
 * Host C++ (paper_2507_23602_b200/csrc/dropin/) re-exposes it under the
 * reference's unchanged C++ headers; Python binds it with ctypes.
 *
 * Layout conventions (identical to the reference's in-memory layout):
 *   points are AoS double[3] per point, contiguous (rsot::Point =
 *   std::array<double,3>, zero-padded for d < 3, point.hpp:10-13), i.e.
 *   std::vector<Point>::data() can be passed as is;
 *   masses / weights / psi / gradient are contiguous double[].
 *
 * Errors: every function returns RSOT_CUDA_OK (0) or a negative status;
 * rsot_cuda_last_error() describes the last failure on the calling thread.
 * RSOT_CUDA_INVALID_ARGUMENT corresponds to the reference's
 * std::invalid_argument (e.g. non-finite psi, potential.hpp:42-46; empty
 * target set, spatial_index.cpp:31-32) and is raised before any device work.
 * There is no CPU fallback: without a usable sm_100 device every entry point
 * that computes returns RSOT_CUDA_NO_DEVICE.
 */
#ifndef RSOT_CUDA_H_
#define RSOT_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSOT_CUDA_ABI_VERSION 1

typedef enum rsot_cuda_status {
  RSOT_CUDA_OK = 0,
  RSOT_CUDA_INVALID_ARGUMENT = -1, /* std::invalid_argument */
  RSOT_CUDA_RUNTIME_ERROR = -2,    /* CUDA / NCCL failure (std::runtime_error) */
  RSOT_CUDA_NO_DEVICE = -3,        /* no usable sm_100 GPU */
  RSOT_CUDA_UNSUPPORTED = -4       /* e.g. CostKind::SqGeodesicSphere */
} rsot_cuda_status;

typedef struct rsot_cuda_ctx rsot_cuda_ctx;         /* device, stream, comm */
typedef struct rsot_cuda_targets rsot_cuda_targets; /* resident targets + cells */
typedef struct rsot_cuda_atoms rsot_cuda_atoms;     /* resident atom shard */

/* EvalResult scalars (evaluate.hpp:15-28).  Counters are global (summed
 * over ranks when a communicator is attached). */
typedef struct rsot_cuda_scalars {
  double J;
  double D;
  uint64_t atoms_visited;
  uint64_t candidate_pairs;
  uint64_t empty_candidate_atoms;
} rsot_cuda_scalars;

int rsot_cuda_abi_version(void);
const char* rsot_cuda_last_error(void);

/* ---- context ------------------------------------------------------------
 * One context per GPU (one process per GPU).  `device` is the CUDA ordinal.
 * Replaces nothing in the reference (which has no device state); GPU count
 * and selection live here, not in SolverConfig. */
int rsot_cuda_ctx_create(int device, rsot_cuda_ctx** out);
int rsot_cuda_ctx_destroy(rsot_cuda_ctx* ctx);
/* Opaque cudaStream_t the context enqueues on (for event timing). */
void* rsot_cuda_ctx_stream(rsot_cuda_ctx* ctx);
int rsot_cuda_ctx_synchronize(rsot_cuda_ctx* ctx);
/* Number of SMs of the context's device. */
int rsot_cuda_ctx_num_sms(rsot_cuda_ctx* ctx);

/* ---- multi-GPU (atoms sharded, targets replicated) ------------------------
 * The gradient and scalars are combined with one collective per evaluation
 * (SURVEY.md §8e): ncclAllGather of the ranks' packed partial buffers and a
 * rank-ordered sum on every rank, so results are bitwise identical across
 * ranks and runs whatever algorithm NCCL picks.  Rank 0 creates the id and ships its 128 bytes
 * to the other ranks out of band (e.g. torch.distributed broadcast). */
int rsot_cuda_comm_unique_id(unsigned char id_out[128]);
int rsot_cuda_ctx_set_comm(rsot_cuda_ctx* ctx, int rank, int world,
                           const unsigned char id[128]);
/* Contiguous shard [lo, hi) of nq atoms for `rank` of `world`
 * (same partition rule as parallel_blocks, parallel.hpp:14-31). */
void rsot_cuda_shard_range(size_t nq, int rank, int world, size_t* lo,
                           size_t* hi);

/* Testing / load-balance diagnostics on one GPU: a context WITHOUT a
 * communicator evaluates partitioned atom handles as rank `rank` of `world`
 * and finalises that rank's partial alone (g_r = partial - nu,
 * J_r = partial - sum psi nu; so g = sum_r g_r + (world-1) nu,
 * J = sum_r J_r + (world-1) sum psi nu, D and the counters add). */
int rsot_cuda_ctx_set_virtual_rank(rsot_cuda_ctx* ctx, int rank, int world);

/* Atoms evaluated whole on this rank: evaluations and covering_cost on this
 * handle never take part in the cross-rank combination, even on a context
 * with a communicator (per-rank work such as PlanView construction, which
 * plan.cpp:35-64 does for the caller's own atoms; no hidden collective). */
int rsot_cuda_atoms_create_local(rsot_cuda_ctx* ctx, const double* xyz,
                                 const double* mass, size_t nq,
                                 rsot_cuda_atoms** out);

/* Testing: one evaluation as `world` virtual ranks of a multi-GPU run on
 * this GPU (partitioned atom handle, context without a communicator).  Every
 * virtual rank's packed partial [g + nu | J + sum psi nu | D | pairs | empty |
 * visited] is computed as that rank computes it and copied to the rank's
 * offset of the gather buffer (in place of ncclAllGather); the rank-ordered
 * sum and finalisation are the launches that follow the collective in a
 * real multi-GPU evaluation (merge order: parallel.hpp:24-30). */
int rsot_cuda_eval_virtual_world(rsot_cuda_ctx* ctx, rsot_cuda_atoms* atoms,
                                 rsot_cuda_targets* targets, const double* psi,
                                 double epsilon, double cutoff, int world,
                                 double* g_out, rsot_cuda_scalars* out);

/* Host mirrors of the cross-rank combination (same element functions as
 * the device kernels; used by the multi-process CPU tests):
 * out[i] = sum over r in rank order of gathered[r * len + i];
 * g_out[j] = res[j] - nu[j], scalars_out = [J - psi_nu, D, pairs, empty,
 * visited] (evaluate.cpp:157-172). */
void rsot_cuda_host_rank_sum(const double* gathered, int world, size_t len,
                             double* out);
void rsot_cuda_host_finalize(const double* res, const double* nu, size_t n,
                             double psi_nu, double* g_out,
                             double* scalars_out);

/* ---- resident data ------------------------------------------------------- */
/* TargetMeasure{points, weights} (measures.hpp:13-19); n >= 1 else
 * RSOT_CUDA_INVALID_ARGUMENT ("spatial index: empty point set"). */
int rsot_cuda_targets_create(rsot_cuda_ctx* ctx, const double* xyz,
                             const double* nu, size_t n,
                             rsot_cuda_targets** out);
int rsot_cuda_targets_destroy(rsot_cuda_targets* t);
size_t rsot_cuda_targets_size(const rsot_cuda_targets* t);

/* SourceAtoms{points, masses} (measures.hpp:24-32) for this rank's shard
 * (quad_weights and densities are not used by the evaluation). */
int rsot_cuda_atoms_create(rsot_cuda_ctx* ctx, const double* xyz,
                           const double* mass, size_t nq,
                           rsot_cuda_atoms** out);
/* The same for ALL atoms on every rank of a multi-rank context: each
 * evaluation then splits the work itself, truncated evaluations by a
 * work-balanced cut of the Hilbert-ordered atom chunks (per-chunk scan cost
 * from the geometry and cutoff, identical on every rank; heavy chunks run
 * split across a CTA cluster), dense and geodesic ones by
 * rsot_cuda_shard_range.  Replaces parallel_blocks' equal atom ranges
 * (parallel.hpp:14-31), which leave clustered truncated problems (BASELINE
 * cfg3) with a 20x spread of work between ranks.  Results are bitwise
 * identical on every rank and run to run.  On a 1-rank context it behaves
 * like rsot_cuda_atoms_create. */
int rsot_cuda_atoms_create_partitioned(rsot_cuda_ctx* ctx, const double* xyz,
                                       const double* mass, size_t nq,
                                       rsot_cuda_atoms** out);
int rsot_cuda_atoms_destroy(rsot_cuda_atoms* a);
size_t rsot_cuda_atoms_size(const rsot_cuda_atoms* a);

/* ---- evaluation ----------------------------------------------------------
 * rsot::evaluate_dual for CostKind::SqEuclidean:
 *   cutoff = +inf            -> dense (evaluate.cpp:119-121)
 *   cutoff finite            -> ball query radius = sqrt(2 cutoff)
 *                               (cost.hpp:38-42), empty sets fall back to the
 *                               nearest target (evaluate.cpp:129-132)
 * psi (length n) and g_out (length n) are HOST pointers; the call copies psi
 * in, evaluates, reduces over ranks and copies g and the scalars back, then
 * synchronises.  Non-finite psi -> RSOT_CUDA_INVALID_ARGUMENT before any
 * device work (evaluate.cpp:91-93). */
int rsot_cuda_eval(rsot_cuda_ctx* ctx, rsot_cuda_atoms* atoms,
                   rsot_cuda_targets* targets, const double* psi, double eps,
                   double cutoff, double* g_out, rsot_cuda_scalars* out);

/* Device-resident variant, asynchronous on the context stream: d_psi and
 * d_g_out are device pointers (length n); scalars land in device memory at
 * d_scalars as 5 doubles {J, D, atoms_visited, candidate_pairs,
 * empty_candidate_atoms}.  Non-finite psi is reported by the next
 * rsot_cuda_ctx_synchronize / rsot_cuda_check_status. */
int rsot_cuda_eval_device(rsot_cuda_ctx* ctx, rsot_cuda_atoms* atoms,
                          rsot_cuda_targets* targets, const double* d_psi,
                          double eps, double cutoff, double* d_g_out,
                          double* d_scalars);
int rsot_cuda_check_status(rsot_cuda_ctx* ctx);

/* rsot_cuda_eval with the reference's CostKind (cost.hpp:17):
 * RSOT_CUDA_COST_SQEUCLIDEAN (c = |x-y|^2/2, the evaluator above) or
 * RSOT_CUDA_COST_SQGEODESIC (c = acos(clamp(x.y, -1, 1))^2 on the unit
 * sphere; a finite cutoff selects {j : c < cutoff} by a full scan and an
 * empty set falls back to the Euclidean nearest target, evaluate.cpp:
 * 119-133; fp64 acos/exp per pair, for the blue-noise application). */
#define RSOT_CUDA_COST_SQEUCLIDEAN 0
#define RSOT_CUDA_COST_SQGEODESIC 1
int rsot_cuda_eval_cost(rsot_cuda_ctx* ctx, rsot_cuda_atoms* atoms,
                        rsot_cuda_targets* targets, const double* psi, double eps,
                        double cutoff, int cost_kind, double* g_out,
                        rsot_cuda_scalars* out);

/* Parity/debug variant of rsot_cuda_eval that also returns, for this rank's
 * atoms, the candidate-set size (1 for empty-fallback atoms), the wrapping
 * sum of splitmix64(j) over the candidate set, and ln S_q.  Any of the three
 * may be NULL. */
int rsot_cuda_eval_debug(rsot_cuda_ctx* ctx, rsot_cuda_atoms* atoms,
                         rsot_cuda_targets* targets, const double* psi,
                         double eps, double cutoff, double* g_out,
                         rsot_cuda_scalars* out, uint32_t* cand_count,
                         uint64_t* cand_hash, double* log_s);
/* rsot_cuda_eval_debug with a cost kind (RSOT_CUDA_COST_*). */
int rsot_cuda_eval_debug_cost(rsot_cuda_ctx* ctx, rsot_cuda_atoms* atoms,
                              rsot_cuda_targets* targets, const double* psi, double eps,
                              double cutoff, int cost_kind, double* g_out,
                              rsot_cuda_scalars* out, uint32_t* cand_count,
                              uint64_t* cand_hash, double* log_s);

/* ---- spatial queries (SpatialIndex / covering_cost) ----------------------
 * nearest target for m host points (lowest index on ties,
 * spatial_index.cpp:70-84). */
int rsot_cuda_nearest(rsot_cuda_ctx* ctx, rsot_cuda_targets* targets,
                      const double* xyz, size_t m, uint64_t* out);
/* covering_cost C0 = max_q min_j 0.5|x_q - y_j|^2 over this rank's atoms,
 * max-reduced over ranks (spatial_index.cpp:101-121). */
int rsot_cuda_covering_cost(rsot_cuda_ctx* ctx, rsot_cuda_atoms* atoms,
                            rsot_cuda_targets* targets, double* out);
/* covering_cost for either cost kind (spatial_index.cpp:101-121).
 * SqGeodesicSphere: the device finds t* = min_q max_j clamp(x_q . y_j) with
 * the reference's unfused dot; acos(t*)^2 is taken on the host (monotone, so
 * equal to the reference's max_q min_j cost). */
int rsot_cuda_covering_cost_kind(rsot_cuda_ctx* ctx, rsot_cuda_atoms* atoms,
                                 rsot_cuda_targets* targets, int cost_kind,
                                 double* out);

/* ---- softmax_refine (multilevel prolongation) -----------------------------
 * rsot::softmax_refine (proj/src/solve.cpp:62-142): psi on the n_fine points
 * fine_xyz (host, AoS double[3]) from the coarse potential coarse_psi (host,
 * length = coarse target count) of `coarse`, using all atoms of `atoms`
 * (single GPU; the atom handle must hold every atom).  cutoff = +inf ->
 * untruncated phase 1; finite -> the reference's brute-force cost test.
 * psi_out (host, n_fine) receives the initial fine potential. */
int rsot_cuda_softmax_refine(rsot_cuda_ctx* ctx, rsot_cuda_targets* coarse,
                             const double* coarse_psi, const double* fine_xyz,
                             size_t n_fine, rsot_cuda_atoms* atoms, double eps,
                             double cutoff, double* psi_out);

/* ---- PlanView (proj/src/plan.cpp) ----------------------------------------
 * The plan induced by a potential, over this handle's atoms.
 * rsot_cuda_plan_candidates: the PlanView ctor's candidate sets (plan.cpp:
 *   37-46): idx_out[offsets[q] .. offsets[q+1]) receives atom q's ascending
 *   candidate list (all targets for cutoff = +inf; the ball query of radius
 *   sqrt(2 cutoff) -- a full scan {j : c < cutoff} for the geodesic cost --
 *   or the nearest target when it is empty).  cost_kind: RSOT_CUDA_COST_*.
 *   offsets[nq+1]
 *   is the prefix sum of the per-atom counts (rsot_cuda_eval_debug's
 *   cand_count for the same cutoff).
 * rsot_cuda_plan_moments: with log_s = the ctor's log_S_q (rsot_cuda_eval_debug
 *   log_s) and the candidate lists (offsets == NULL: every target), the
 *   plan-density reductions of plan.cpp: target_marginals (:85-91,
 *   marginal_out[n]), the unnormalised first moments sum_q p m_q x_q of
 *   all_conditional_barycenters (:123-140, moment_out[3n]), barycentric_map
 *   (:142-156, map_out[3nq]) and modal_map's target index (:158-182,
 *   modal_out[nq], lowest index on ties).  Outputs may be NULL.  Sums are
 *   order independent (fixed point), so results are bitwise reproducible. */
int rsot_cuda_plan_candidates(rsot_cuda_ctx* ctx, rsot_cuda_atoms* atoms,
                              rsot_cuda_targets* targets, double cutoff, int cost_kind,
                              const uint64_t* offsets, uint64_t* idx_out);
int rsot_cuda_plan_moments(rsot_cuda_ctx* ctx, rsot_cuda_atoms* atoms,
                           rsot_cuda_targets* targets, const double* psi, double eps,
                           int cost_kind, const double* log_s, const uint64_t* offsets,
                           const uint64_t* idx, double* marginal_out, double* moment_out,
                           double* map_out, uint64_t* modal_out);

/* ---- precision ------------------------------------------------------------
 * RSOT_CUDA_PRECISION_FP64 (default): every operation in fp64, within 1e-10
 * relative of the reference.  RSOT_CUDA_PRECISION_FP32: truncated
 * evaluations form the exponent in FP32 and exponentiate with the hardware
 * ex2 (sums, J, D and the gradient accumulate in fp64; candidate sets stay
 * exact); observed deviation from fp64 at the BASELINE configs: J 3e-9 - 1.5e-8
 * relative, gradient 7e-8 of the marginal scale; asserted <= 2e-5 in the tests.
 * Dense evaluations (cutoff = +inf) always run in fp64.  BASELINE cfg5 asks
 * for both precisions; the reference has fp64 only. */
#define RSOT_CUDA_PRECISION_FP64 0
#define RSOT_CUDA_PRECISION_FP32 1
int rsot_cuda_ctx_set_precision(rsot_cuda_ctx* ctx, int precision);

/* ---- measurement ----------------------------------------------------------
 * Enables CUDA-event timing of the hot kernels inside each evaluation
 * (events on the launching stream); rsot_cuda_last_kernel_ms returns the
 * durations of the last evaluation's pass A and pass B launches. */
int rsot_cuda_ctx_set_timing(rsot_cuda_ctx* ctx, int enable);
int rsot_cuda_last_kernel_ms(rsot_cuda_ctx* ctx, double* pass_a_ms,
                             double* pass_b_ms, double* total_ms);
/* Number of kernels this library has launched in this process (all
 * contexts); bench.py reports the per-step delta as gpu_launches. */
uint64_t rsot_cuda_kernel_launches(void);
/* Measured FP64 DFMA rate of the device (lane-FMAs per second). */
int rsot_cuda_measure_fp64_peak(rsot_cuda_ctx* ctx, double* dfma_per_s);
/* Measured FP32 FFMA rate and MUFU ex2.approx rate of the device (lane
 * operations per second): the roofline denominators of the fp32 path. */
int rsot_cuda_measure_fp32_peaks(rsot_cuda_ctx* ctx, double* ffma_per_s,
                                 double* ex2_per_s);

#ifdef __cplusplus
}
#endif

#endif /* RSOT_CUDA_H_ */
