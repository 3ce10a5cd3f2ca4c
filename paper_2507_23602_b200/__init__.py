"""B200-native evaluator of the entropy-regularized semi-discrete OT dual.

Drop-in for rsot::evaluate_dual of arXiv 2507.23602's reference artifact
(proj/src/evaluate.cpp:86-174): hand-written sm_100a CUDA behind the C ABI
in include/rsot_cuda.h, with a Python mirror of the reference interface in
``paper_2507_23602_b200.rsot``.
"""
from . import _lib  # noqa: F401
from .rsot import (  # noqa: F401
    Context,
    CostKind,
    DualPotential,
    EvalResult,
    Gauge,
    MapKind,
    MapSample,
    PlanView,
    barycentric_map,
    modal_map,
    SolverConfig,
    SourceAtoms,
    SpatialIndex,
    TargetMeasure,
    TruncationKind,
    TruncationState,
    ball_radius,
    build_index,
    covering_cost,
    cutoff_bootstrap,
    cutoff_geometric,
    cutoff_integrated,
    cutoff_pointwise,
    evaluate_dual,
    evaluate_dual_debug,
    gauge_fixed,
    refresh_truncation,
    require_finite,
    softmax_refine,
)
