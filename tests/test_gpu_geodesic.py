"""evaluate_dual with CostKind::SqGeodesicSphere on the GPU (SURVEY.md
§8(f) #4; cost.hpp:19-33, evaluate.cpp:119-133): dense and full-scan
truncated, Euclidean-nearest fallback for empty sets, against the geodesic
oracle (pinned bitwise to the reference build in tests/test_oracle.py).
Tolerance as the Euclidean evaluator (1e-10); counters exact (the candidate
predicate acos(t)^2 < cutoff can only differ for a pair whose cost lies
within an ulp of the cutoff -- libdevice vs glibc acos -- none in these
seeded cases)."""
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
