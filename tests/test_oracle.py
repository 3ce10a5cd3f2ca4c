"""CPU tests: the oracle pinned against the reference's frozen values, its
own tests, the golden vectors and (when built here) the reference library
compiled from /root/reference.  No GPU."""
import math
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, assert_parity, load_golden, marginal_scale, random_instance
from oracle.oracle import COracle, REF_LIB, candidate_hash

C = COracle()
REF_BIN = os.path.join(ROOT, "oracle", "_ref")
have_ref = os.path.exists(REF_LIB)


def two_by_two(weights=(0.75, 0.25)):
    A = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    return A, np.array([0.5, 0.5]), A.copy(), np.array(weights)


def test_frozen_2x2_values():
    """proj/tests/test_core.cpp:65-73."""
    A, M, T, W = two_by_two()
    r = C.evaluate_dual(A, M, T, W, np.zeros(2), 1.0)
    assert r["J"] == pytest.approx(-0.226625130922122, rel=1e-12)
    assert r["gradient"][0] == pytest.approx(-0.011418450214431, rel=1e-10)
    assert r["gradient"][1] == pytest.approx(+0.011418450214431, rel=1e-10)


def test_symmetric_zero_gradient():
    """test_core.cpp:75-81."""
    A, M, T, _ = two_by_two()
    r = C.evaluate_dual(A, M, T, np.array([0.5, 0.5]), np.zeros(2), 1.0)
    assert np.all(np.abs(r["gradient"]) <= 1e-15)


def test_single_target_closed_form():
    """test_core.cpp:45-63: J = -sum c m for any psi shift, g = 0."""
    xs = (np.arange(16) + 0.5) / 16
    A = np.zeros((16, 3))
    A[:, 0] = xs
    M = np.full(16, 1 / 16)
    T = np.array([[0.4, 0, 0]])
    expected = -np.sum(0.5 * (xs - 0.4) ** 2 * M)
    for shift in (0.0, -3.0, 11.0):
        r = C.evaluate_dual(A, M, T, np.array([1.0]), np.array([shift]), 0.5)
        assert r["J"] == pytest.approx(expected, rel=1e-12)
        assert abs(r["gradient"][0]) < 1e-15


def test_nonfinite_psi_rejected():
    A, M, T, W = two_by_two()
    with pytest.raises(ValueError):
        C.evaluate_dual(A, M, T, W, np.array([np.nan, 0.0]), 1.0)


def test_gradient_sums_to_zero_and_fd():
    """test_core.cpp:91-116."""
    rng = np.random.default_rng(23)
    for _ in range(5):
        A, M, T, W, psi = random_instance(rng, 2, 15, 120)
        r = C.evaluate_dual(A, M, T, W, psi, 0.3)
        assert abs(r["gradient"].sum()) <= 1e-10
    A, M, T, W, psi = random_instance(rng, 1, 8, 60)
    r = C.evaluate_dual(A, M, T, W, psi, 0.1)
    for k in range(8):
        h = 1e-6 * (1 + abs(psi[k]))
        p, m = psi.copy(), psi.copy()
        p[k] += h
        m[k] -= h
        fd = (C.evaluate_dual(A, M, T, W, p, 0.1)["J"] - C.evaluate_dual(A, M, T, W, m, 0.1)["J"]) / (2 * h)
        assert abs(r["gradient"][k] - fd) <= 1e-5 * max(1e-10, abs(fd))


def test_determinism_and_workers():
    """test_core.cpp:152-164."""
    rng = np.random.default_rng(41)
    A, M, T, W, psi = random_instance(rng, 2, 30, 500)
    a1 = C.evaluate_dual(A, M, T, W, psi, 0.1, workers=3)
    a2 = C.evaluate_dual(A, M, T, W, psi, 0.1, workers=3)
    assert a1["J"] == a2["J"] and np.array_equal(a1["gradient"], a2["gradient"])
    b = C.evaluate_dual(A, M, T, W, psi, 0.1, workers=1)
    assert abs(a1["J"] - b["J"]) <= 1e-12 * abs(b["J"])
    assert np.max(np.abs(a1["gradient"] - b["gradient"])) <= 1e-12


def test_golden_vectors_bitwise():
    """Oracle vs the reference library's outputs stored in tests/golden."""
    for c in load_golden():
        r = C.evaluate_dual(c["A"], c["M"], c["T"], c["W"], c["psi"], c["eps"], c["cutoff"], c["workers"])
        assert r["J"] == c["J"], c["name"]
        assert r["D"] == c["D"], c["name"]
        assert np.array_equal(r["gradient"], c["g"]), c["name"]
        assert [r["atoms_visited"], r["candidate_pairs"], r["empty_candidate_atoms"]] == c["counts"]


def test_ball_query_and_nearest_match_brute_force():
    """test_geometry.cpp:228-268 (strict <, ascending; lowest index ties)."""
    rng = np.random.default_rng(7)
    for dim in (1, 2, 3):
        P = np.zeros((1000, 3))
        P[:, :dim] = rng.uniform(size=(1000, dim))
        for _ in range(30):
            c = np.zeros(3)
            c[:dim] = rng.uniform(size=dim)
            cutoff = 0.25 * rng.uniform()
            radius = math.sqrt(2 * cutoff)
            got = C.ball_query(P, c, radius)
            d2 = ((P - c) ** 2).sum(axis=1)
            want = np.nonzero(np.sqrt(d2) < radius)[0]
            assert np.array_equal(got, want)
    Q = rng.uniform(size=(100, 3))
    got = C.nearest(P, Q)
    want = np.array([np.argmin(((P - q) ** 2).sum(axis=1)) for q in Q])
    assert np.array_equal(got, want)
    # line example and strict inequality (test_geometry.cpp:205-218)
    L = np.array([[0.0, 0, 0], [1.0, 0, 0], [3.0, 0, 0]])
    assert list(C.ball_query(L, [0, 0, 0], math.sqrt(2.0))) == [0, 1]
    assert list(C.ball_query(L, [0, 0, 0], 0.0)) == []
    assert list(C.ball_query(L, [1, 0, 0], math.sqrt(2e-12))) == [1]
    # ties resolve to the lowest index
    Tt = np.array([[1.0, 0, 0], [-1.0, 0, 0], [0, 1.0, 0]])
    assert C.nearest(Tt, [[0, 0, 0]])[0] == 0


def test_covering_cost_worked_example():
    """test_geometry.cpp:270-304."""
    A = np.array([[0.0, 0, 0], [0.5, 0, 0], [1.0, 0, 0]])
    T = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    assert C.covering_cost(A, T) == pytest.approx(0.125)
    assert C.covering_cost(A, A) == 0.0


def test_cutoff_frozen_values():
    """test_core.cpp:166-213."""
    L = C.L
    import ctypes
    assert L.oracle_cutoff_pointwise(0.0, 1.0, 0.01, 1e-12) == pytest.approx(0.276310211159286, rel=1e-12)
    out = ctypes.c_double()
    assert L.oracle_cutoff_integrated(0.0, 0.0, 1.0, 1.0, 0.01, 1e-4, ctypes.byref(out)) == 0
    assert out.value == pytest.approx(0.046051701859881, rel=1e-12)
    assert L.oracle_cutoff_geometric(1.0, 0.0, 0.5, 1.0, 0.01, 1e-4, ctypes.byref(out)) == 0
    assert out.value == pytest.approx(1.052983173665480, rel=1e-12)
    assert L.oracle_cutoff_geometric(1.0, 0.25, 0.5, 1.0, 0.01, 1e-4, ctypes.byref(out)) == 0
    assert out.value == pytest.approx(1.302983173665480, rel=1e-12)
    assert L.oracle_cutoff_integrated(0.0, 0.0, 1.0, 0.0, 0.01, 1e-4, ctypes.byref(out)) == -2


def test_per_atom_outputs_consistent():
    rng = np.random.default_rng(5)
    A, M, T, W, psi = random_instance(rng, 3, 300, 500, 0.05)
    r = C.evaluate_dual(A, M, T, W, psi, 0.02, 0.01, per_atom=True)
    assert int(r["count"].sum()) == r["candidate_pairs"]
    radius = math.sqrt(0.02)
    for q in range(0, 500, 37):
        cand = C.ball_query(T, A[q], radius)
        if len(cand) == 0:
            cand = C.nearest(T, A[q:q + 1])
        assert candidate_hash(cand) == int(r["hash"][q])
        assert len(cand) == r["count"][q]


@pytest.mark.skipif(not have_ref, reason="reference library not built here")
def test_oracle_matches_reference_build_bitwise():
    from oracle.oracle import RefLib
    ref = RefLib()
    rng = np.random.default_rng(11)
    for k, (dim, n, nq, eps, cutoff, w) in enumerate([
            (3, 400, 3000, 0.02, math.inf, 1), (3, 400, 3000, 0.02, 0.01, 3), (2, 300, 2000, 0.005, 0.004, 4),
            (3, 400, 1000, 0.02, -1.0, 1), (1, 40, 500, 0.1, 0.02, 2), (3, 2000, 3000, 1e-3, 2e-3, 8)]):
        A, M, T, W, psi = random_instance(rng, dim, n, nq, 0.05)
        o = C.evaluate_dual(A, M, T, W, psi, eps, cutoff, w)
        r = ref.problem(dim, A, M, T, W).evaluate_dual(psi, eps, cutoff, w)
        assert o["J"] == r["J"] and o["D"] == r["D"], k
        assert np.array_equal(o["gradient"], r["gradient"]), k
        assert o["candidate_pairs"] == r["candidate_pairs"]
        assert o["empty_candidate_atoms"] == r["empty_candidate_atoms"]


KNOWN_REFERENCE_FAILURES = {
    # A solver-iteration heuristic of the reference itself (L-BFGS on a 1D
    # instance: 30 fine-level iterations with the hierarchy vs 39 cold, the
    # test wants 4x).  Reproduced with the reference's own evaluate.cpp; it
    # does not involve the index or the evaluator (dense, no truncation).
    "solve_multilevel: target hierarchy cuts fine-level iterations",
}


@pytest.mark.parametrize("suite", ["core", "geometry", "measures"])
def test_reference_doctest_suites(suite):
    """proj/tests/test_{core,geometry,measures}.cpp compiled unmodified
    against the reference library with the Boost-free index."""
    exe = os.path.join(REF_BIN, f"test_{suite}")
    if not os.path.exists(exe):
        pytest.skip("reference suites not built here")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600, cwd="/tmp")
    failed = [ln.split('TEST_CASE("', 1)[1].rstrip('")') for ln in p.stderr.splitlines() if "in TEST_CASE(" in ln]
    assert set(failed) <= KNOWN_REFERENCE_FAILURES, p.stderr[-2000:]


@pytest.mark.skipif(not have_ref, reason="reference library not built here")
def test_softmax_refine_oracle_matches_reference_bitwise():
    """rsot::softmax_refine (solve.cpp:62-142): C restatement vs the reference."""
    from oracle.oracle import RefLib
    ref = RefLib()
    rng = np.random.default_rng(17)
    for (nc, nf, nq, eps, cut) in [(50, 120, 1500, 0.05, math.inf), (80, 150, 2000, 0.02, 0.01),
                                   (40, 60, 800, 0.01, 0.001), (30, 40, 500, 0.02, -1.0)]:
        cy = rng.uniform(size=(nc, 3))
        cnu = rng.uniform(size=nc) + 0.1
        cnu /= cnu.sum()
        cpsi = rng.normal(0, 0.02, nc)
        fy = rng.uniform(size=(nf, 3))
        ax = rng.uniform(size=(nq, 3))
        am = rng.uniform(size=nq) + 0.1
        am /= am.sum()
        o = C.softmax_refine(cy, cnu, cpsi, fy, ax, am, eps, cut)
        r = ref.problem(3, ax, am, cy, cnu).softmax_refine(cpsi, fy, eps, cut, 1)
        assert np.array_equal(o, r)


def test_softmax_refine_identity_cases():
    """test_core.cpp:370-397 analogue: a single coarse target refines to a
    potential whose gauge-fixed values are the closed form."""
    rng = np.random.default_rng(2)
    ax = rng.uniform(size=(300, 3))
    am = np.full(300, 1 / 300)
    fy = rng.uniform(size=(20, 3))
    out = C.softmax_refine(np.array([[0.5, 0.5, 0.5]]), np.array([1.0]), np.array([0.3]), fy, ax, am, 0.1)
    # ln S_q = (0.3 - c(x_q, y0)) / eps  ->  psi_k = -eps LSE_q(-c_qk/eps - ln S_q + ln m_q)
    c0 = 0.5 * ((ax - 0.5) ** 2).sum(axis=1)
    logS = (0.3 - c0) / 0.1
    for k in range(5):
        t = -0.5 * ((ax - fy[k]) ** 2).sum(axis=1) / 0.1 - logS + np.log(am)
        m = t.max()
        assert out[k] == pytest.approx(-0.1 * (m + np.log(np.exp(t - m).sum())), rel=1e-12, abs=1e-14)


def _ref_or_skip():
    if not have_ref:
        pytest.skip("reference library not built here")
    from oracle.oracle import RefLib
    return RefLib()


@pytest.mark.parametrize("dim,n,nq,eps,cutoff", [(3, 300, 2000, 0.02, math.inf), (3, 300, 2000, 0.02, 0.01),
                                                 (2, 200, 1500, 0.01, 0.002), (3, 50, 800, 0.05, -1.0)])
def test_plan_view_oracle_equals_reference(dim, n, nq, eps, cutoff):
    """PlanView restatement (oracle_plan_view) vs the reference plan.cpp
    compiled from its sources: candidate counts, marginals, conditional
    barycentres, barycentric and modal maps bit for bit."""
    ref = _ref_or_skip()
    rng = np.random.default_rng(5)
    A, M, T, W, psi = random_instance(rng, dim, n, nq, 0.05)
    o = C.plan_view(A, M, T, W, psi, eps, cutoff)
    r = ref.problem(dim, A, M, T, W).plan_view(psi, eps, cutoff)
    for k in ("count", "marginal", "bary", "map", "modal"):
        assert np.array_equal(o[k], r[k]), k
    assert o["starved"] == r["starved"] == -1


def test_plan_view_oracle_starved_equals_reference():
    ref = _ref_or_skip()
    rng = np.random.default_rng(5)
    A, M, T, W, psi = random_instance(rng, 3, 300, 2000, 0.05)
    T[17] = [5, 5, 5]
    T[40] = [6, 6, 6]
    psi[17] = -10
    for cutoff in (math.inf, 0.01):
        o = C.plan_view(A, M, T, W, psi, 0.02, cutoff)
        r = ref.problem(3, A, M, T, W).plan_view(psi, 0.02, cutoff)
        assert o["starved"] == r["starved"] == 17
        assert np.array_equal(o["marginal"], r["marginal"]) and np.array_equal(o["map"], r["map"])


@pytest.mark.parametrize("n,nq,eps,cutoff", [(300, 2000, 0.05, math.inf), (300, 2000, 0.05, 0.05),
                                              (100, 500, 0.02, 0.0005), (50, 400, 0.1, -1.0)])
def test_geodesic_oracle_equals_reference(n, nq, eps, cutoff):
    """SqGeodesicSphere restatement vs the reference evaluate.cpp (cost kind
    switched in SolverConfig), bit for bit."""
    ref = _ref_or_skip()
    rng = np.random.default_rng(n + nq)
    v = rng.normal(size=(n, 3))
    T = v / np.linalg.norm(v, axis=1, keepdims=True)
    v = rng.normal(size=(nq, 3))
    A = v / np.linalg.norm(v, axis=1, keepdims=True)
    M = rng.uniform(size=nq) + 0.1
    M /= M.sum()
    W = rng.uniform(size=n) + 0.1
    W /= W.sum()
    psi = rng.normal(0, 0.01, size=n)
    o = C.evaluate_dual_geodesic(A, M, T, W, psi, eps, cutoff)
    r = ref.problem(3, A, M, T, W).evaluate_dual_geodesic(psi, eps, cutoff)
    assert o["J"] == r["J"] and o["D"] == r["D"] and np.array_equal(o["gradient"], r["gradient"])
    assert o["candidate_pairs"] == r["candidate_pairs"]
    assert o["empty_candidate_atoms"] == r["empty_candidate_atoms"]
