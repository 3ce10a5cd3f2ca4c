"""evaluate_dual with CostKind::SqGeodesicSphere on the GPU (SURVEY.md
§8(f) #4; cost.hpp:19-33, evaluate.cpp:119-133): dense and full-scan
truncated, Euclidean-nearest fallback for empty sets, against the geodesic
oracle (pinned bitwise to the reference build in tests/test_oracle.py).
Tolerance as the Euclidean evaluator (1e-10); counters and candidate sets
exact: the device decides acos(t)^2 < cutoff as t >= t_min, with t_min found
on the host by bisection under the reference's own libm acos
(geo_dot_threshold), so the selection is the reference's bit for bit even
where libdevice's acos differs from glibc's in the last ulp
(test_geodesic_selection_at_the_cutoff)."""
import math

import numpy as np
import pytest

from conftest import assert_parity, marginal_scale
import paper_2507_23602_b200 as rs
from oracle.oracle import COracle

pytestmark = pytest.mark.gpu

C = COracle()


def sphere(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


@pytest.fixture(scope="module")
def ctx():
    return rs.Context.default(0)


@pytest.mark.parametrize("n,nq,eps,cutoff", [(300, 2000, 0.05, math.inf), (300, 2000, 0.05, 0.05),
                                              (100, 500, 0.02, 0.0005), (50, 400, 0.1, -1.0),
                                              (2000, 7000, 0.01, 0.02), (1, 100, 0.1, math.inf)])
def test_geodesic_matches_oracle(ctx, n, nq, eps, cutoff):
    rng = np.random.default_rng(n * 3 + nq)
    T, A = sphere(rng, n), sphere(rng, nq)
    M = rng.uniform(size=nq) + 0.1
    M /= M.sum()
    W = rng.uniform(size=n) + 0.1
    W /= W.sum()
    psi = rng.normal(0, 0.01, size=n)
    atoms = rs.SourceAtoms(dim=3, points=A, masses=M)
    tgt = rs.TargetMeasure(dim=3, points=T, weights=W)
    cfg = rs.SolverConfig(epsilon=eps, cost_kind=rs.CostKind.SqGeodesicSphere)
    r = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), cfg, rs.TruncationState(cutoff=cutoff), ctx=ctx)
    got = dict(J=r.J, D=r.D, gradient=r.gradient, atoms_visited=r.atoms_visited,
               candidate_pairs=r.candidate_pairs, empty_candidate_atoms=r.empty_candidate_atoms)
    want = C.evaluate_dual_geodesic(A, M, T, W, psi, eps, cutoff)
    assert_parity(got, want, marginal_scale(W, want["gradient"]), 1e-10)


@pytest.mark.parametrize("n,nq", [(1, 50), (300, 2000), (4000, 3000)])
def test_geodesic_covering_cost_matches_reference(ctx, n, nq):
    """covering_cost(SqGeodesicSphere) on the GPU (rsot_cuda_covering_cost_kind:
    min_q max_j clamped unfused dot, then one host acos) equals the
    reference's brute-force max_q min_j acos(clamp(x . y))^2
    (spatial_index.cpp:113-119, reference build oracle/_ref) bit for bit; the
    SqEuclidean kind through the same entry point too."""
    from oracle.oracle import RefLib
    rng = np.random.default_rng(900 + n)
    A, T = sphere(rng, nq), sphere(rng, n)
    M = np.full(nq, 1.0 / nq)
    W = np.full(n, 1.0 / n)
    ref = RefLib().problem(3, A, M, T, W)
    atoms = rs.SourceAtoms(dim=3, points=A, masses=M)
    tgt = rs.TargetMeasure(dim=3, points=T, weights=W)
    assert rs.covering_cost(atoms, tgt, kind=rs.CostKind.SqGeodesicSphere, ctx=ctx) == ref.covering_cost(1)
    assert rs.covering_cost(atoms, tgt, ctx=ctx) == ref.covering_cost(0)


def test_geodesic_selection_at_the_cutoff(ctx):
    """Cutoffs placed exactly on pair costs (and one ulp either side), with
    the cost computed as the reference does -- unfused dot, clamp, libm acos,
    square (Python floats call the same libm) -- so a device acos one ulp off
    glibc's would flip those pairs: the candidate counts must still equal
    the geodesic oracle's."""
    import math as m
    rng = np.random.default_rng(4242)
    T, A = sphere(rng, 400), sphere(rng, 300)
    M = np.full(len(A), 1.0 / len(A))
    W = np.full(len(T), 1.0 / len(T))
    psi = rng.normal(0, 0.01, size=len(T))
    atoms = rs.SourceAtoms(dim=3, points=A, masses=M)
    tgt = rs.TargetMeasure(dim=3, points=T, weights=W)
    cfg = rs.SolverConfig(epsilon=0.05, cost_kind=rs.CostKind.SqGeodesicSphere)

    def cost(x, y):
        d = (x[0] * y[0] + x[1] * y[1]) + x[2] * y[2]
        g = m.acos(-1.0 if d < -1.0 else (1.0 if d > 1.0 else d))
        return g * g

    for q, j in ((0, 0), (5, 17), (100, 3), (299, 399)):
        c = cost(A[q], T[j])
        for cut in (c, m.nextafter(c, 0.0), m.nextafter(c, 10.0)):
            r = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), cfg, rs.TruncationState(cutoff=cut), ctx=ctx)
            want = C.evaluate_dual_geodesic(A, M, T, W, psi, 0.05, cut)
            assert r.candidate_pairs == want["candidate_pairs"]
            assert r.empty_candidate_atoms == want["empty_candidate_atoms"]
            assert abs(r.J - want["J"]) <= 1e-10 * abs(want["J"])
