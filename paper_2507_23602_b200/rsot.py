"""Host-side mirror of the reference's C++ evaluation interface.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/rsot/*.hpp so parity tests read like the
reference's own tests (proj/tests/test_core.cpp):

  SourceAtoms, TargetMeasure        measures.hpp:13-32
  DualPotential, require_finite     potential.hpp:13-46
  SolverConfig, TruncationKind      solver_config.hpp:10-45
  TruncationState, cutoff_*,        evaluate.hpp:33-68, evaluate.cpp:11-72
    refresh_truncation
  EvalResult, evaluate_dual         evaluate.hpp:15-28, :79-82
  SpatialIndex, covering_cost       spatial_index.hpp:15-54

evaluate_dual runs only on the GPU through librsot_b200.so (C ABI
include/rsot_cuda.h); there is no CPU path.  The cutoff formulas are host
scalars in the reference too and are restated here.
"""
from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib

# ---------------------------------------------------------------------------
# Types (measures.hpp, potential.hpp, solver_config.hpp, cost.hpp)


class CostKind(enum.Enum):
    SqEuclidean = 0
    SqGeodesicSphere = 1


class TruncationKind(enum.Enum):
    None_ = 0
    Pointwise = 1
    Integrated = 2
    Geometric = 3


class Gauge(enum.Enum):
    Raw = 0
    MeanZero = 1


def _points3(points) -> np.ndarray:
    """Point lists are zero-padded to 3 components (point.hpp:10-13)."""
    p = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    if p.ndim == 1:
        p = p.reshape(-1, 1)
    if p.shape[1] < 3:
        p = np.ascontiguousarray(np.hstack([p, np.zeros((p.shape[0], 3 - p.shape[1]))]))
    return p


@dataclass
class TargetMeasure:
    dim: int = 0
    points: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    weights: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def size(self) -> int:
        return int(len(self.points))


@dataclass
class SourceAtoms:
    dim: int = 0
    points: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    quad_weights: np.ndarray = field(default_factory=lambda: np.zeros(0))
    densities: np.ndarray = field(default_factory=lambda: np.zeros(0))
    masses: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def size(self) -> int:
        return int(len(self.points))


@dataclass
class DualPotential:
    values: np.ndarray
    gauge: Gauge = Gauge.Raw

    def size(self) -> int:
        return int(len(self.values))


def require_finite(psi) -> None:
    """potential.hpp:42-46."""
    if not np.all(np.isfinite(np.asarray(psi, dtype=np.float64))):
        raise ValueError("potential has non-finite entries")


def weighted_mean(psi, nu) -> float:
    psi = np.asarray(psi, dtype=np.float64)
    nu = np.asarray(nu, dtype=np.float64)
    if psi.shape != nu.shape:
        raise ValueError("gauge: psi/nu size mismatch")
    mean = 0.0
    for p, w in zip(psi.tolist(), nu.tolist()):  # sequential, potential.hpp:26-28
        mean += p * w
    return mean


def gauge_fixed(psi: DualPotential, nu) -> DualPotential:
    """potential.hpp:32-40."""
    mean = weighted_mean(psi.values, nu)
    return DualPotential(np.asarray(psi.values, dtype=np.float64) - mean, Gauge.MeanZero)


@dataclass
class SolverConfig:
    epsilon: float = 1e-2
    delta_tol: float = 1e-3
    truncation: TruncationKind = TruncationKind.None_
    tau: float = 1e-4
    delta_thr: float = 1e-12
    lbfgs_memory: int = 10
    max_iterations: int = 1000
    wolfe_c1: float = 1e-4
    wolfe_c2: float = 0.9
    scaling_steps: int = 0
    cost_kind: CostKind = CostKind.SqEuclidean
    workers: int = 1

    def validate(self) -> None:
        """solver_config.hpp:34-44."""
        if not self.epsilon > 0.0:
            raise ValueError("epsilon must be > 0")
        if not self.delta_tol > 0.0:
            raise ValueError("tolerance must be > 0")
        if not (0.0 < self.tau < 1.0):
            raise ValueError("tau must be in (0,1)")
        if not (0.0 < self.delta_thr < 1.0):
            raise ValueError("delta_thr must be in (0,1)")
        if self.lbfgs_memory < 1:
            raise ValueError("lbfgs memory must be >= 1")
        if self.max_iterations < 0:
            raise ValueError("max_iterations must be >= 0")
        if self.scaling_steps < 0:
            raise ValueError("scaling_steps must be >= 0")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")


def ball_radius(kind: CostKind, cutoff: float) -> Optional[float]:
    """cost.hpp:38-42."""
    if cutoff < 0.0:
        return 0.0
    if kind == CostKind.SqEuclidean:
        return math.sqrt(2.0 * cutoff)
    return None


# ---------------------------------------------------------------------------
# Truncation bookkeeping (evaluate.hpp:33-68, evaluate.cpp:11-72)


@dataclass
class TruncationState:
    cutoff: float = math.inf
    cached_D: float = 0.0
    cached_absJ: float = 0.0
    has_cache: bool = False
    psi_max: float = 0.0
    psi_min: float = 0.0
    psi_range: float = 0.0
    nu_max: float = 0.0
    nu_min: float = 0.0
    covering: float = 0.0

    def set_psi_stats(self, psi) -> None:
        psi = np.asarray(psi, dtype=np.float64)
        self.psi_max = float(psi.max())
        self.psi_min = float(psi.min())
        self.psi_range = self.psi_max - self.psi_min

    def set_weight_stats(self, nu) -> None:
        nu = np.asarray(nu, dtype=np.float64)
        self.nu_max = float(nu.max())
        self.nu_min = float(nu.min())


def cutoff_pointwise(t: TruncationState, eps: float, delta_thr: float) -> float:
    return t.psi_max + eps * math.log(t.nu_max / delta_thr)


def cutoff_integrated(t: TruncationState, eps: float, tau: float) -> float:
    absJ = max(t.cached_absJ, 1e-30)
    if absJ <= 1e-30:
        raise RuntimeError("functional estimate degenerate")
    c = t.psi_max + eps * math.log(eps * t.cached_D / (tau * absJ))
    return max(c, t.covering)


def cutoff_geometric(t: TruncationState, eps: float, tau: float) -> float:
    absJ = max(t.cached_absJ, 1e-30)
    if absJ <= 1e-30:
        raise RuntimeError("functional estimate degenerate")
    c = t.covering + t.psi_range + eps * math.log(eps / (t.nu_min * tau * absJ))
    return max(c, t.covering)


def cutoff_bootstrap(t: TruncationState, eps: float, tau: float) -> float:
    c = t.covering + t.psi_range + eps * math.log(eps / (t.nu_min * tau))
    return max(c, t.covering)


def refresh_truncation(t: TruncationState, psi, cfg: SolverConfig) -> None:
    t.set_psi_stats(psi)
    if cfg.truncation == TruncationKind.None_:
        t.cutoff = math.inf
    elif cfg.truncation == TruncationKind.Pointwise:
        t.cutoff = cutoff_pointwise(t, cfg.epsilon, cfg.delta_thr)
    elif cfg.truncation == TruncationKind.Integrated:
        t.cutoff = (cutoff_integrated(t, cfg.epsilon, cfg.tau) if t.has_cache
                    else cutoff_bootstrap(t, cfg.epsilon, cfg.tau))
    else:
        t.cutoff = (cutoff_geometric(t, cfg.epsilon, cfg.tau) if t.has_cache
                    else cutoff_bootstrap(t, cfg.epsilon, cfg.tau))


@dataclass
class EvalResult:
    J: float = 0.0
    gradient: np.ndarray = field(default_factory=lambda: np.zeros(0))
    D: float = 0.0
    atoms_visited: int = 0
    candidate_pairs: int = 0
    empty_candidate_atoms: int = 0

    def grad_l1(self) -> float:
        return float(np.abs(self.gradient).sum())


# ---------------------------------------------------------------------------
# Device context and resident data


class Context:
    """One CUDA context per GPU (one process per GPU)."""

    _default = {}

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(self.lib.rsot_cuda_ctx_create(int(device), ctypes.byref(h)))
        self.handle = h
        self.device = int(device)
        self.rank = 0
        self.world = 1
        self.vworld = 1

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = cls(device)
        return cls._default[device]

    @staticmethod
    def unique_id() -> bytes:
        lib = _lib.load()
        buf = (ctypes.c_uint8 * 128)()
        _lib.check(lib.rsot_cuda_comm_unique_id(buf))
        return bytes(buf)

    def set_comm(self, rank: int, world: int, uid: bytes) -> None:
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _lib.check(self.lib.rsot_cuda_ctx_set_comm(self.handle, int(rank), int(world), buf))
        self.rank, self.world = int(rank), int(world)

    def set_virtual_rank(self, rank: int, world: int) -> None:
        """Testing / diagnostics without a communicator: evaluate partitioned
        atoms as rank `rank` of `world` (the result is that rank's partial,
        finalised alone; include/rsot_cuda.h)."""
        _lib.check(self.lib.rsot_cuda_ctx_set_virtual_rank(self.handle, int(rank), int(world)))
        self.vworld = int(world)

    def shard_range(self, nq: int):
        lo, hi = ctypes.c_size_t(), ctypes.c_size_t()
        self.lib.rsot_cuda_shard_range(nq, self.rank, self.world, ctypes.byref(lo), ctypes.byref(hi))
        return lo.value, hi.value

    @property
    def stream(self) -> int:
        return self.lib.rsot_cuda_ctx_stream(self.handle)

    def synchronize(self) -> None:
        _lib.check(self.lib.rsot_cuda_ctx_synchronize(self.handle))

    def set_precision(self, precision: str) -> None:
        """"fp64" (default, reference-exact) or "fp32" (mixed: FP32 exponent
        + hardware ex2 for truncated evaluations; observed <= 1.5e-8 relative on J)."""
        code = {"fp64": 0, "fp32": 1}.get(precision)
        if code is None:
            raise ValueError(f"unknown precision {precision!r}")
        _lib.check(self.lib.rsot_cuda_ctx_set_precision(self.handle, code))
        self.precision = precision

    def set_timing(self, on: bool) -> None:
        _lib.check(self.lib.rsot_cuda_ctx_set_timing(self.handle, 1 if on else 0))

    def last_kernel_ms(self):
        a, b, t = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        _lib.check(self.lib.rsot_cuda_last_kernel_ms(self.handle, ctypes.byref(a), ctypes.byref(b),
                                                     ctypes.byref(t)))
        return a.value, b.value, t.value

    def fp32_rates(self):
        """(FFMA lane-ops/s, MUFU ex2 lane-ops/s) measured on the device."""
        a, b = ctypes.c_double(), ctypes.c_double()
        _lib.check(self.lib.rsot_cuda_measure_fp32_peaks(self.handle, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def fp64_dfma_rate(self) -> float:
        v = ctypes.c_double()
        _lib.check(self.lib.rsot_cuda_measure_fp64_peak(self.handle, ctypes.byref(v)))
        return v.value


def _ptr(a: Optional[np.ndarray]) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data if a is not None else None)


class DeviceTargets:
    """Resident TargetMeasure (+ cell list) on one context."""

    def __init__(self, ctx: Context, points, weights):
        self.ctx = ctx
        pts = _points3(points)
        nu = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        if len(pts) != len(nu):
            raise ValueError("target measure: point/weight size mismatch")
        h = ctypes.c_void_p()
        _lib.check(ctx.lib.rsot_cuda_targets_create(ctx.handle, _ptr(pts), _ptr(nu), len(pts),
                                                    ctypes.byref(h)))
        self.handle = h
        self.n = len(pts)

    def __del__(self):
        try:
            if self.handle:
                self.ctx.lib.rsot_cuda_targets_destroy(self.handle)
        except Exception:
            pass


class DeviceAtoms:
    """Resident SourceAtoms (points, masses) on one context.

    shard=True on a multi-rank context: balanced=True (default) keeps every
    atom on every rank and lets each evaluation split the work (truncated:
    work-balanced Hilbert chunk ranges; rsot_cuda_atoms_create_partitioned),
    balanced=False uploads only this rank's contiguous parallel_blocks range
    (parallel.hpp:14-31).  shard=False: every rank evaluates every atom."""

    def __init__(self, ctx: Context, points, masses, shard: bool = True, balanced: bool = True):
        self.ctx = ctx
        pts = _points3(points)
        m = np.ascontiguousarray(np.asarray(masses, dtype=np.float64))
        multi = ctx.world > 1 or getattr(ctx, "vworld", 1) > 1
        partitioned = shard and balanced and multi
        lo, hi = ctx.shard_range(len(pts)) if shard and not partitioned else (0, len(pts))
        pts = np.ascontiguousarray(pts[lo:hi])
        m = np.ascontiguousarray(m[lo:hi])
        h = ctypes.c_void_p()
        create = ctx.lib.rsot_cuda_atoms_create_partitioned if partitioned else ctx.lib.rsot_cuda_atoms_create
        _lib.check(create(ctx.handle, _ptr(pts), _ptr(m), len(pts), ctypes.byref(h)))
        self.partitioned = partitioned
        self.handle = h
        self.nq = len(pts)
        self.lo, self.hi = lo, hi

    def __del__(self):
        try:
            if self.handle:
                self.ctx.lib.rsot_cuda_atoms_destroy(self.handle)
        except Exception:
            pass


class SpatialIndex:
    """Per-stage index over the target points (spatial_index.hpp:15-40).

    The device-side state is the target cell list; it lives with the
    resident targets used by evaluate_dual.  Throws ValueError on an empty
    point set like the reference ctor (spatial_index.cpp:31-32).
    """

    def __init__(self, points, ctx: Optional[Context] = None):
        pts = _points3(points) if len(points) else np.zeros((0, 3))
        if len(pts) == 0:
            raise ValueError("spatial index: empty point set")
        self.ctx = ctx or Context.default()
        self.points = pts
        self._dev = DeviceTargets(self.ctx, pts, np.ones(len(pts)))

    def size(self) -> int:
        return len(self.points)

    def nearest(self, center) -> int:
        c = _points3(np.asarray(center, dtype=np.float64).reshape(1, -1))
        out = np.zeros(1, dtype=np.uint64)
        _lib.check(self.ctx.lib.rsot_cuda_nearest(self.ctx.handle, self._dev.handle, _ptr(c), 1,
                                                  _ptr(out)))
        return int(out[0])

    def nearest_many(self, centers) -> np.ndarray:
        c = _points3(centers)
        out = np.zeros(len(c), dtype=np.uint64)
        _lib.check(self.ctx.lib.rsot_cuda_nearest(self.ctx.handle, self._dev.handle, _ptr(c), len(c),
                                                  _ptr(out)))
        return out.astype(np.int64)


def build_index(points, ctx: Optional[Context] = None) -> SpatialIndex:
    return SpatialIndex(points, ctx)


def _resident(obj, ctx: Context, arrays, extra, make):
    """Device copy of `obj`'s arrays on `ctx`, reused only while the arrays
    hold exactly the uploaded values: a host shadow copy is compared in full
    (np.array_equal) on every call, so in-place edits of any entry (e.g. the
    barycenter loop's `nu.points = points`, barycenter.cpp:55) are seen."""
    arrays = [np.ascontiguousarray(np.asarray(a, dtype=np.float64)) for a in arrays]
    dev = getattr(obj, "_rsot_dev", None)
    if (dev is not None and dev[0] is ctx and dev[1] == extra and len(dev[2]) == len(arrays)
            and all(a.shape == b.shape and np.array_equal(a, b) for a, b in zip(arrays, dev[2]))):
        return dev[3]
    handle = make(*arrays)
    object.__setattr__(obj, "_rsot_dev", (ctx, extra, [a.copy() for a in arrays], handle))
    return handle


def _device_targets(target: TargetMeasure, ctx: Context) -> DeviceTargets:
    return _resident(target, ctx, [target.points, target.weights], (),
                     lambda p, w: DeviceTargets(ctx, p, w))


def _device_atoms(atoms: SourceAtoms, ctx: Context) -> DeviceAtoms:
    return _resident(atoms, ctx, [atoms.points, atoms.masses], (ctx.world, getattr(ctx, "vworld", 1)),
                     lambda p, m: DeviceAtoms(ctx, p, m))


def covering_cost(atoms: SourceAtoms, target: TargetMeasure, kind: CostKind = CostKind.SqEuclidean,
                  ctx: Optional[Context] = None) -> float:
    """spatial_index.cpp:101-121 on the GPU, both cost kinds."""
    if atoms.size() == 0 or target.size() == 0:
        raise ValueError("covering cost: empty input")
    ctx = ctx or Context.default()
    out = ctypes.c_double()
    _lib.check(ctx.lib.rsot_cuda_covering_cost_kind(ctx.handle, _device_atoms(atoms, ctx).handle,
                                                    _device_targets(target, ctx).handle, _cost_code(kind),
                                                    ctypes.byref(out)))
    return out.value


def evaluate_dual(atoms: SourceAtoms, target: TargetMeasure, psi: DualPotential,
                  cfg: SolverConfig, trunc: TruncationState, index: Optional[SpatialIndex] = None,
                  ctx: Optional[Context] = None) -> EvalResult:
    """rsot::evaluate_dual (evaluate.hpp:79-82, evaluate.cpp:86-174) on the GPU."""
    values = np.ascontiguousarray(np.asarray(psi.values, dtype=np.float64))
    if len(values) != target.size():
        raise ValueError("evaluate_dual: psi length != target count")
    require_finite(values)
    ctx = ctx or (index.ctx if index is not None else Context.default())
    dev_t = _device_targets(target, ctx)
    dev_a = _device_atoms(atoms, ctx)
    g = np.empty(target.size(), dtype=np.float64)
    sc = _lib.RsotCudaScalars()
    if cfg.cost_kind == CostKind.SqEuclidean:
        _lib.check(ctx.lib.rsot_cuda_eval(ctx.handle, dev_a.handle, dev_t.handle, _ptr(values),
                                          float(cfg.epsilon), float(trunc.cutoff), _ptr(g),
                                          ctypes.byref(sc)))
    else:  # cost.hpp:27-30, full-scan truncation (evaluate.cpp:124-128)
        _lib.check(ctx.lib.rsot_cuda_eval_cost(ctx.handle, dev_a.handle, dev_t.handle, _ptr(values),
                                               float(cfg.epsilon), float(trunc.cutoff), 1, _ptr(g),
                                               ctypes.byref(sc)))
    return EvalResult(J=sc.J, gradient=g, D=sc.D, atoms_visited=int(sc.atoms_visited),
                      candidate_pairs=int(sc.candidate_pairs),
                      empty_candidate_atoms=int(sc.empty_candidate_atoms))


def softmax_refine(coarse: TargetMeasure, coarse_psi, fine_points, atoms: SourceAtoms, eps: float,
                   kind: CostKind = CostKind.SqEuclidean, cutoff: float = math.inf, workers: int = 1,
                   ctx: Optional[Context] = None) -> np.ndarray:
    """rsot::softmax_refine (solve.hpp, solve.cpp:62-142) on the GPU: the
    initial fine-level potential from a coarse one (multilevel prolongation).
    `workers` (a CPU thread count in the reference) is ignored."""
    cpsi = np.ascontiguousarray(np.asarray(coarse_psi, dtype=np.float64))
    if len(cpsi) != coarse.size():
        raise ValueError("softmax refine: psi/coarse size mismatch")
    require_finite(cpsi)
    if kind != CostKind.SqEuclidean:
        raise NotImplementedError("SqGeodesicSphere is out of scope for the B200 evaluator")
    ctx = ctx or Context.default()
    fine = _points3(fine_points)
    out = np.empty(len(fine), dtype=np.float64)
    dev_t = _device_targets(coarse, ctx)
    dev_a = _device_atoms(atoms, ctx) if ctx.world == 1 else DeviceAtoms(ctx, atoms.points, atoms.masses,
                                                                          shard=False)
    _lib.check(ctx.lib.rsot_cuda_softmax_refine(ctx.handle, dev_t.handle, _ptr(cpsi), _ptr(fine), len(fine),
                                                dev_a.handle, float(eps), float(cutoff), _ptr(out)))
    return out


def _cost_code(kind: CostKind) -> int:
    return 1 if kind == CostKind.SqGeodesicSphere else 0


def evaluate_dual_debug(atoms: SourceAtoms, target: TargetMeasure, psi, eps: float, cutoff: float,
                        ctx: Optional[Context] = None, kind: CostKind = CostKind.SqEuclidean):
    """evaluate_dual plus per-atom candidate counts, candidate hashes and ln S_q
    (for selection parity against the oracle)."""
    ctx = ctx or Context.default()
    values = np.ascontiguousarray(np.asarray(psi, dtype=np.float64))
    dev_t = _device_targets(target, ctx)
    dev_a = _device_atoms(atoms, ctx)
    g = np.empty(target.size(), dtype=np.float64)
    cnt = np.zeros(dev_a.nq, dtype=np.uint32)
    hsh = np.zeros(dev_a.nq, dtype=np.uint64)
    logs = np.zeros(dev_a.nq, dtype=np.float64)
    sc = _lib.RsotCudaScalars()
    _lib.check(ctx.lib.rsot_cuda_eval_debug_cost(ctx.handle, dev_a.handle, dev_t.handle, _ptr(values),
                                                 float(eps), float(cutoff), _cost_code(kind), _ptr(g),
                                                 ctypes.byref(sc), _ptr(cnt), _ptr(hsh), _ptr(logs)))
    res = EvalResult(J=sc.J, gradient=g, D=sc.D, atoms_visited=int(sc.atoms_visited),
                     candidate_pairs=int(sc.candidate_pairs),
                     empty_candidate_atoms=int(sc.empty_candidate_atoms))
    return res, cnt, hsh, logs


# ---- PlanView (proj/include/rsot/plan.hpp, proj/src/plan.cpp) --------------

class MapKind(enum.Enum):
    Barycentric = 0
    Modal = 1


@dataclass
class MapSample:
    kind: MapKind
    mapped: np.ndarray                  # (nq, 3) T(x_q)
    target_index: Optional[np.ndarray]  # modal only
    displacement: np.ndarray            # ||T(x_q) - x_q||


class PlanView:
    """The plan induced by a potential (plan.hpp:17-73).  The constructor
    computes log_S_q and the candidate sets on the GPU (plan.cpp:12-59); the
    reductions over the plan density run on the GPU over those sets."""

    def __init__(self, atoms: SourceAtoms, target: TargetMeasure, psi: DualPotential, eps: float,
                 kind: CostKind = CostKind.SqEuclidean, cutoff: float = math.inf, workers: int = 1,
                 ctx: Optional[Context] = None):
        values = np.ascontiguousarray(np.asarray(psi.values, dtype=np.float64))
        if len(values) != target.size():
            raise ValueError("plan view: psi length != target count")
        require_finite(values)
        self.ctx = ctx or Context.default()
        self.atoms, self.target, self.psi, self.eps, self.kind = atoms, target, values, float(eps), kind
        self._dt = DeviceTargets(self.ctx, target.points, target.weights)
        self._da = DeviceAtoms(self.ctx, atoms.points, atoms.masses, shard=False)
        _, cnt, _, logs = evaluate_dual_debug(atoms, target, values, eps, cutoff, ctx=self.ctx, kind=kind)
        self.log_S = logs
        self.offsets = np.zeros(len(cnt) + 1, dtype=np.uint64)
        np.cumsum(cnt.astype(np.uint64), out=self.offsets[1:])
        self.idx = np.zeros(max(int(self.offsets[-1]), 1), dtype=np.uint64)
        _lib.check(self.ctx.lib.rsot_cuda_plan_candidates(self.ctx.handle, self._da.handle, self._dt.handle,
                                                          float(cutoff), _cost_code(kind), _ptr(self.offsets),
                                                          _ptr(self.idx)))
        self.converged_known = False
        self.converged = False

    def set_convergence(self, grad_l1: float, delta_tol: float) -> None:
        self.converged_known = True
        self.converged = grad_l1 <= delta_tol

    def candidates(self, q: int) -> np.ndarray:
        return self.idx[int(self.offsets[q]):int(self.offsets[q + 1])].astype(np.int64)

    def psi_value(self, j: int) -> float:
        return float(self.psi[j])

    def _moments(self, marginal=False, moment=False, bary_map=False, modal=False):
        n, nq = self.target.size(), self.atoms.size()
        out = dict(marginal=np.zeros(n) if marginal else None, moment=np.zeros((n, 3)) if moment else None,
                   map=np.zeros((nq, 3)) if bary_map else None,
                   modal=np.zeros(nq, dtype=np.uint64) if modal else None)
        _lib.check(self.ctx.lib.rsot_cuda_plan_moments(
            self.ctx.handle, self._da.handle, self._dt.handle, _ptr(self.psi), self.eps, _cost_code(self.kind),
            _ptr(self.log_S),
            _ptr(self.offsets), _ptr(self.idx), _ptr(out["marginal"]), _ptr(out["moment"]), _ptr(out["map"]),
            _ptr(out["modal"])))
        return out

    def plan_density(self, q: int):
        """(target index, probability) pairs of atom q (plan.cpp:70-83)."""
        x = _points3(self.atoms.points)[q]
        cand = self.candidates(q)
        y = _points3(self.target.points)[cand]
        if self.kind == CostKind.SqGeodesicSphere:
            c = np.arccos(np.clip((x[0] * y[:, 0] + x[1] * y[:, 1]) + x[2] * y[:, 2], -1.0, 1.0)) ** 2
        else:
            c = 0.5 * (((x[0] - y[:, 0]) ** 2 + (x[1] - y[:, 1]) ** 2) + (x[2] - y[:, 2]) ** 2)
        e = (self.psi[cand] - c) / self.eps + np.log(np.asarray(self.target.weights)[cand])
        return list(zip(cand.tolist(), np.exp(e - self.log_S[q]).tolist()))

    def target_marginals(self) -> np.ndarray:
        return self._moments(marginal=True)["marginal"]

    def all_conditional_barycenters(self) -> np.ndarray:
        r = self._moments(marginal=True, moment=True)
        tilde = r["marginal"]
        bad = np.nonzero(tilde < 1e-30)[0]
        if len(bad):
            raise RuntimeError(f"target starved: index {int(bad[0])}")
        return (1.0 / tilde)[:, None] * r["moment"]

    def conditional_barycenter(self, j: int) -> np.ndarray:
        return self.all_conditional_barycenters()[j]


def barycentric_map(plan: PlanView) -> MapSample:
    """T(x_q) = sum_j p_j(x_q) y_j (plan.cpp:142-156)."""
    m = plan._moments(bary_map=True)["map"]
    x = _points3(plan.atoms.points)
    return MapSample(MapKind.Barycentric, m, None, np.sqrt(((m - x) ** 2).sum(axis=1)))


def modal_map(plan: PlanView) -> MapSample:
    """argmax_j (psi_j - c + eps ln nu_j), lowest index on ties (plan.cpp:158-182)."""
    idx = plan._moments(modal=True)["modal"].astype(np.int64)
    y = _points3(plan.target.points)[idx]
    x = _points3(plan.atoms.points)
    return MapSample(MapKind.Modal, y, idx, np.sqrt(((y - x) ** 2).sum(axis=1)))
