"""PlanView on the GPU (proj/src/plan.cpp): candidate
sets bitwise equal to the oracle's (= the reference's, test_oracle.py),
target marginals / conditional barycentres / barycentric map within 1e-12
relative, modal map indices exact, starved targets reported like the
reference."""
import math

import numpy as np
import pytest

from conftest import random_instance
import paper_2507_23602_b200 as rs
from oracle.oracle import COracle

pytestmark = pytest.mark.gpu

C = COracle()
TOL = 1e-12


@pytest.fixture(scope="module")
def ctx():
    return rs.Context.default(0)


def _plan(ctx, dim, A, M, T, W, psi, eps, cutoff):
    atoms = rs.SourceAtoms(dim=dim, points=A, masses=M)
    tgt = rs.TargetMeasure(dim=dim, points=T, weights=W)
    return rs.PlanView(atoms, tgt, rs.DualPotential(psi), eps, cutoff=cutoff, ctx=ctx)


CASES = [(3, 300, 2000, 0.02, math.inf), (3, 300, 2000, 0.02, 0.01), (2, 200, 1500, 0.01, 0.002),
         (3, 50, 800, 0.05, -1.0), (3, 2000, 5000, 1e-3, 0.004), (1, 40, 300, 0.05, 0.01)]


@pytest.mark.parametrize("dim,n,nq,eps,cutoff", CASES)
def test_plan_view_matches_oracle(ctx, dim, n, nq, eps, cutoff):
    rng = np.random.default_rng(n + nq + dim)
    A, M, T, W, psi = random_instance(rng, dim, n, nq, 0.05)
    plan = _plan(ctx, dim, A, M, T, W, psi, eps, cutoff)
    want = C.plan_view(A, M, T, W, psi, eps, cutoff)
    assert np.array_equal(np.diff(plan.offsets), want["count"])
    # candidate lists (ascending) equal the oracle's ball query
    radius = math.sqrt(2 * cutoff) if math.isfinite(cutoff) and cutoff > 0 else 0.0
    for q in range(0, nq, max(1, nq // 50)):
        cand = plan.candidates(q)
        if math.isfinite(cutoff):
            ref = C.ball_query(T, A[q], radius) if radius > 0 else np.array([], dtype=np.int64)
            if len(ref) == 0:
                ref = C.nearest(T, A[q:q + 1])
            assert np.array_equal(cand, ref)
        else:
            assert np.array_equal(cand, np.arange(n))
    assert np.max(np.abs(plan.log_S - want["log_s"]) / np.maximum(1, np.abs(want["log_s"]))) <= 1e-12
    marg = plan.target_marginals()
    assert np.max(np.abs(marg - want["marginal"])) <= TOL * np.max(want["marginal"])
    if want["starved"] >= 0:  # e.g. cutoff < 0: only nearest targets receive mass
        with pytest.raises(RuntimeError, match=f"target starved: index {want['starved']}$"):
            plan.all_conditional_barycenters()
    else:
        bary = plan.all_conditional_barycenters()
        scale = np.max(np.abs(want["bary"]))
        assert np.max(np.abs(bary - want["bary"])) <= TOL * scale
    m = rs.barycentric_map(plan)
    assert np.max(np.abs(m.mapped - want["map"])) <= TOL * max(1.0, np.max(np.abs(want["map"])))
    assert np.array_equal(rs.modal_map(plan).target_index, want["modal"].astype(np.int64))
    # plan_density rows sum to one (plan.hpp:37-39)
    for q in (0, nq // 2, nq - 1):
        assert abs(sum(p for _, p in plan.plan_density(q)) - 1.0) <= 1e-12


def test_plan_view_starved_target(ctx):
    rng = np.random.default_rng(5)
    A, M, T, W, psi = random_instance(rng, 3, 300, 2000, 0.05)
    T[17] = [5, 5, 5]
    T[40] = [6, 6, 6]
    psi[17] = -10
    for cutoff in (math.inf, 0.01):
        plan = _plan(ctx, 3, A, M, T, W, psi, 0.02, cutoff)
        want = C.plan_view(A, M, T, W, psi, 0.02, cutoff)
        assert want["starved"] == 17
        with pytest.raises(RuntimeError, match="target starved: index 17"):
            plan.all_conditional_barycenters()


def test_plan_view_rejects_bad_psi(ctx):
    rng = np.random.default_rng(6)
    A, M, T, W, psi = random_instance(rng, 3, 20, 100, 0.05)
    atoms = rs.SourceAtoms(dim=3, points=A, masses=M)
    tgt = rs.TargetMeasure(dim=3, points=T, weights=W)
    bad = psi.copy()
    bad[3] = np.nan
    with pytest.raises(ValueError):
        rs.PlanView(atoms, tgt, rs.DualPotential(bad), 0.1, ctx=ctx)
    with pytest.raises(ValueError):
        rs.PlanView(atoms, tgt, rs.DualPotential(psi[:-1]), 0.1, ctx=ctx)


@pytest.mark.parametrize("cutoff", [math.inf, 0.05])
def test_plan_view_geodesic(ctx, cutoff):
    """PlanView with CostKind::SqGeodesicSphere (the blue-noise plan,
    sphere.cpp:139): candidate counts and log_S from the geodesic oracle,
    marginals = g + nu of the geodesic evaluation, maps against a numpy
    restatement of plan.cpp over the same candidate sets."""
    rng = np.random.default_rng(17)
    v = rng.normal(size=(200, 3))
    T = v / np.linalg.norm(v, axis=1, keepdims=True)
    v = rng.normal(size=(1500, 3))
    A = v / np.linalg.norm(v, axis=1, keepdims=True)
    M = np.full(1500, 1 / 1500)
    W = np.full(200, 1 / 200)
    psi = rng.normal(0, 0.01, size=200)
    eps = 0.05
    atoms = rs.SourceAtoms(dim=3, points=A, masses=M)
    tgt = rs.TargetMeasure(dim=3, points=T, weights=W)
    plan = rs.PlanView(atoms, tgt, rs.DualPotential(psi), eps, kind=rs.CostKind.SqGeodesicSphere,
                       cutoff=cutoff, ctx=ctx)
    want = C.evaluate_dual_geodesic(A, M, T, W, psi, eps, cutoff, per_atom=True)
    assert np.array_equal(np.diff(plan.offsets), want["count"])
    assert np.max(np.abs(plan.log_S - want["log_s"])) <= 1e-12 * np.max(np.abs(want["log_s"]))
    marg = plan.target_marginals()
    assert np.max(np.abs(marg - (want["gradient"] + W))) <= 1e-12
    dots = np.clip(A @ T.T, -1.0, 1.0)
    cost = np.arccos(dots) ** 2
    e = (psi[None, :] - cost) / eps + np.log(W)[None, :]
    mask = np.zeros_like(e, dtype=bool)
    for q in range(len(A)):
        mask[q, plan.candidates(q)] = True
    p = np.where(mask, np.exp(e - plan.log_S[:, None]), 0.0)
    bary_map = p @ T
    assert np.max(np.abs(rs.barycentric_map(plan).mapped - bary_map)) <= 1e-12
    score = np.where(mask, psi[None, :] - cost + eps * np.log(W)[None, :], -np.inf)
    assert np.array_equal(rs.modal_map(plan).target_index, np.argmax(score, axis=1))
    if np.all((p * M[:, None]).sum(axis=0) >= 1e-30):
        first = (p * M[:, None]).T @ A / (p * M[:, None]).sum(axis=0)[:, None]
        assert np.max(np.abs(plan.all_conditional_barycenters() - first)) <= 1e-10
