// eval_progress.cpp -- measurement aid for the CPU reference build of the
// cfg4 driver (oracle/_ref/cfg4_solve_ref_progress): the link wraps the
// reference's rsot::evaluate_dual (-Wl,--wrap; the reference source is
// unchanged) to print one progress line per evaluation to stderr (count,
// wall seconds of the call, J, L1 gradient norm, candidate pairs, cutoff), so
// a time-capped CPU run still reports how far it got and at what rate.
#include <chrono>
#include <cmath>
#include <cstdio>

#include "rsot/evaluate.hpp"

#define RSOT_EVAL_SYM _ZN4rsot13evaluate_dualERKNS_11SourceAtomsERKNS_13TargetMeasureERKNS_13DualPotentialERKNS_12SolverConfigERKNS_15TruncationStateERKNS_12SpatialIndexE
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)

extern "C" rsot::EvalResult CAT(__real_, RSOT_EVAL_SYM)(const rsot::SourceAtoms&, const rsot::TargetMeasure&,
                                                         const rsot::DualPotential&, const rsot::SolverConfig&,
                                                         const rsot::TruncationState&, const rsot::SpatialIndex&);

extern "C" rsot::EvalResult CAT(__wrap_, RSOT_EVAL_SYM)(const rsot::SourceAtoms& a, const rsot::TargetMeasure& t,
                                                         const rsot::DualPotential& p, const rsot::SolverConfig& c,
                                                         const rsot::TruncationState& tr,
                                                         const rsot::SpatialIndex& idx) {
  static int count = 0;
  const auto t0 = std::chrono::steady_clock::now();
  rsot::EvalResult r = CAT(__real_, RSOT_EVAL_SYM)(a, t, p, c, tr, idx);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  double l1 = 0.0;
  for (double g : r.gradient) l1 += std::fabs(g);
  std::fprintf(stderr, "eval %d eps %.1e  %.3f s  J %.17g  |g|_1 %.6e  pairs %llu  cutoff %.6e\n", ++count,
               c.epsilon, s, r.J, l1, static_cast<unsigned long long>(r.candidate_pairs), tr.cutoff);
  std::fflush(stderr);
  return r;
}
