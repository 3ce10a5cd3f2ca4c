"""GPU parity tests: the sm_100a evaluator through the C ABI
(include/rsot_cuda.h via paper_2507_23602_b200) against the CPU oracle and
the golden vectors of the reference library.

Tolerance (fp64, SURVEY.md §8d / north star): |dJ| <= 1e-10 |J|,
||dg||_inf <= 1e-10 * max_k(nu~_k + nu_k), |dD| <= 1e-10 D; counters and
per-atom candidate sets (size + hash) exact."""
import ctypes
import math

import numpy as np
import pytest

from conftest import assert_parity, load_golden, marginal_scale, random_instance
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import _lib, synth
from oracle.oracle import COracle

pytestmark = pytest.mark.gpu

TOL = 1e-10
C = COracle()


@pytest.fixture(scope="module")
def ctx():
    return rs.Context.default(0)


def gpu_eval(ctx, A, M, T, W, psi, eps, cutoff, dim=3):
    atoms = rs.SourceAtoms(dim=dim, points=A, masses=M)
    tgt = rs.TargetMeasure(dim=dim, points=T, weights=W)
    r = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), rs.SolverConfig(epsilon=eps),
                         rs.TruncationState(cutoff=cutoff), ctx=ctx)
    return dict(J=r.J, D=r.D, gradient=r.gradient, atoms_visited=r.atoms_visited,
                candidate_pairs=r.candidate_pairs, empty_candidate_atoms=r.empty_candidate_atoms)


def test_loaded_native_library(ctx):
    lib = _lib.load()
    assert lib.rsot_cuda_ctx_num_sms(ctx.handle) >= 100


# ---- reference frozen tests (proj/tests/test_core.cpp) through the API ----

def test_frozen_2x2_values(ctx):
    A = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    r = gpu_eval(ctx, A, np.array([0.5, 0.5]), A.copy(), np.array([0.75, 0.25]), np.zeros(2), 1.0, math.inf)
    assert r["J"] == pytest.approx(-0.226625130922122, rel=1e-12)
    assert r["gradient"][0] == pytest.approx(-0.011418450214431, rel=1e-10)
    assert r["gradient"][1] == pytest.approx(+0.011418450214431, rel=1e-10)


def test_symmetric_instance_zero_gradient(ctx):
    A = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    r = gpu_eval(ctx, A, np.array([0.5, 0.5]), A.copy(), np.array([0.5, 0.5]), np.zeros(2), 1.0, math.inf)
    assert np.all(np.abs(r["gradient"]) <= 1e-15)


def test_single_target_short_circuit(ctx):
    xs = (np.arange(16) + 0.5) / 16
    A = np.zeros((16, 3))
    A[:, 0] = xs
    M = np.full(16, 1 / 16)
    T = np.array([[0.4, 0, 0]])
    expected = -np.sum(0.5 * (xs - 0.4) ** 2 * M)
    for shift in (0.0, -3.0, 11.0):
        r = gpu_eval(ctx, A, M, T, np.array([1.0]), np.array([shift]), 0.5, math.inf)
        assert r["J"] == pytest.approx(expected, rel=1e-12)
        # reference: doctest::Approx(0.0) (tolerance 1.2e-5); our exp2 is
        # within a few ulp of 1 for the single target
        assert abs(r["gradient"][0]) <= 1e-13


def test_input_validation(ctx):
    atoms = rs.SourceAtoms(dim=1, points=np.array([[0.0, 0, 0], [1.0, 0, 0]]), masses=np.array([.5, .5]))
    tgt = rs.TargetMeasure(dim=1, points=atoms.points.copy(), weights=np.array([.75, .25]))
    with pytest.raises(ValueError):
        rs.evaluate_dual(atoms, tgt, rs.DualPotential(np.zeros(1)), rs.SolverConfig(epsilon=1.0),
                         rs.TruncationState(), ctx=ctx)
    with pytest.raises(ValueError):
        rs.evaluate_dual(atoms, tgt, rs.DualPotential(np.array([np.nan, 0.0])), rs.SolverConfig(epsilon=1.0),
                         rs.TruncationState(), ctx=ctx)
    # the C ABI itself also refuses non-finite psi (device-side check)
    lib = _lib.load()
    g = np.zeros(2)
    sc = _lib.RsotCudaScalars()
    dev_a = rs.rsot._device_atoms(atoms, ctx)
    dev_t = rs.rsot._device_targets(tgt, ctx)
    bad = np.array([np.inf, 0.0])
    rc = lib.rsot_cuda_eval(ctx.handle, dev_a.handle, dev_t.handle, rs.rsot._ptr(bad), 1.0, math.inf,
                            rs.rsot._ptr(g), sc)
    assert rc == _lib.RSOT_CUDA_INVALID_ARGUMENT
    with pytest.raises(ValueError):
        rs.SpatialIndex(np.zeros((0, 3)), ctx=ctx)


def test_handle_validation_and_mass_range(ctx):
    """Handles are validated from the first element (a non-finite target
    point 0 used to slip through and poison the grid's bounding box); masses
    must be finite and >= 0.  Unnormalised masses whose single contributions
    exceed 2^10 (they used to lose the high limb of the fixed-point gradient
    accumulator) match the oracle; a total mass >= 2^40 is refused instead of
    overflowing the accumulator."""
    lib = _lib.load()
    h = ctypes.c_void_p()
    pts = np.array([[np.nan, 0.0, 0.0], [1.0, 0.0, 0.0]])
    assert lib.rsot_cuda_targets_create(ctx.handle, rs.rsot._ptr(pts), rs.rsot._ptr(np.array([.5, .5])), 2,
                                        ctypes.byref(h)) == _lib.RSOT_CUDA_INVALID_ARGUMENT
    assert lib.rsot_cuda_atoms_create(ctx.handle, rs.rsot._ptr(pts), rs.rsot._ptr(np.array([.5, .5])), 2,
                                      ctypes.byref(h)) == _lib.RSOT_CUDA_INVALID_ARGUMENT
    ok = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    assert lib.rsot_cuda_atoms_create(ctx.handle, rs.rsot._ptr(ok), rs.rsot._ptr(np.array([.5, -.5])), 2,
                                      ctypes.byref(h)) == _lib.RSOT_CUDA_INVALID_ARGUMENT
    rng = np.random.default_rng(2026)
    A, M, T, W, psi = random_instance(rng, 3, 3000, 4000)
    eps, cutoff = 0.01, 0.02
    for scale in (1e7, 3e9):  # atoms of mass ~ 2.5e3 .. 7.5e5 (>= 2^10)
        want = C.evaluate_dual(A, M * scale, T, W, psi, eps, cutoff, workers=8)
        got = gpu_eval(ctx, A, M * scale, T, W, psi, eps, cutoff)
        assert got["candidate_pairs"] == want["candidate_pairs"]
        assert abs(got["J"] - want["J"]) <= TOL * abs(want["J"])
        ref = np.abs(want["gradient"] + W).max()
        assert np.abs(got["gradient"] - want["gradient"]).max() <= TOL * ref
    with pytest.raises(ValueError, match="2\\^40"):
        gpu_eval(ctx, A, M * 2.0 ** 41, T, W, psi, eps, cutoff)


def test_gradient_sums_to_zero_gauge_invariance(ctx):
    rng = np.random.default_rng(31)
    A, M, T, W, psi = random_instance(rng, 2, 12, 80)
    base = gpu_eval(ctx, A, M, T, W, psi, 0.25, math.inf, dim=2)
    assert abs(base["gradient"].sum()) <= 1e-10
    for c in (1.0, -1.0, 100.0, -100.0):
        r = gpu_eval(ctx, A, M, T, W, psi + c, 0.25, math.inf, dim=2)
        assert abs(r["J"] - base["J"]) <= 1e-10
        assert np.max(np.abs(r["gradient"] - base["gradient"])) <= 1e-10


def test_empty_atom_set(ctx):
    """N_q = 0: J = -sum psi nu, g = -nu (parallel.hpp:16-19 n<2 path)."""
    rng = np.random.default_rng(3)
    T = rng.uniform(size=(50, 3))
    W = np.full(50, 1 / 50)
    psi = rng.normal(0, 0.1, 50)
    for cutoff in (math.inf, 0.01):
        r = gpu_eval(ctx, np.zeros((0, 3)), np.zeros(0), T, W, psi, 0.1, cutoff)
        want = C.evaluate_dual(np.zeros((0, 3)), np.zeros(0), T, W, psi, 0.1, cutoff)
        assert r["J"] == pytest.approx(want["J"], rel=1e-14)
        assert np.allclose(r["gradient"], -W, rtol=0, atol=1e-18)
        assert r["atoms_visited"] == 0 and r["candidate_pairs"] == 0


# ---- golden vectors of the reference library (tests/golden) ---------------

@pytest.mark.parametrize("case", load_golden(), ids=lambda c: c["name"])
def test_golden_vectors(ctx, case):
    got = gpu_eval(ctx, case["A"], case["M"], case["T"], case["W"], case["psi"], case["eps"], case["cutoff"],
                   dim=case["dim"])
    want = dict(J=case["J"], D=case["D"], gradient=case["g"], atoms_visited=case["counts"][0],
                candidate_pairs=case["counts"][1], empty_candidate_atoms=case["counts"][2])
    assert_parity(got, want, marginal_scale(case["W"], case["g"]), TOL)


# ---- random instances with per-atom selection parity ----------------------

CASES = [
    (3, 3000, 400, 0.02, math.inf), (3, 3000, 400, 0.02, 0.01), (3, 3000, 400, 0.02, 0.03),
    (3, 3000, 400, 0.02, -1.0), (3, 3000, 400, 0.02, 0.0), (3, 3000, 400, 0.02, 0.002),
    (2, 5000, 300, 0.05, math.inf), (2, 5000, 300, 0.005, 0.004), (1, 700, 50, 0.1, 0.02),
    (3, 20000, 5000, 1e-3, 0.01), (3, 2, 2, 1.0, math.inf), (3, 100, 1, 0.5, math.inf),
    (3, 100, 1, 0.5, 0.001), (3, 2000, 300, 1e-4, math.inf), (3, 2000, 3000, 1e-4, 1e-3),
    (2, 3000, 500, 1e-3, math.inf), (3, 1000, 200, 0.05, 50.0), (3, 129, 257, 0.03, 0.02),
]


@pytest.mark.parametrize("dim,nq,n,eps,cutoff", CASES)
def test_random_instances_with_selection_parity(ctx, dim, nq, n, eps, cutoff):
    rng = np.random.default_rng(hash((dim, nq, n, eps, cutoff)) % (2 ** 32))
    A, M, T, W, psi = random_instance(rng, dim, n, nq, 0.05)
    atoms = rs.SourceAtoms(dim=dim, points=A, masses=M)
    tgt = rs.TargetMeasure(dim=dim, points=T, weights=W)
    res, cnt, hsh, logs = rs.evaluate_dual_debug(atoms, tgt, psi, eps, cutoff, ctx=ctx)
    want = C.evaluate_dual(A, M, T, W, psi, eps, cutoff, per_atom=True)
    got = dict(J=res.J, D=res.D, gradient=res.gradient, atoms_visited=res.atoms_visited,
               candidate_pairs=res.candidate_pairs, empty_candidate_atoms=res.empty_candidate_atoms)
    assert_parity(got, want, marginal_scale(W, want["gradient"]), TOL)
    assert np.array_equal(cnt, want["count"])
    assert np.array_equal(hsh, want["hash"])
    assert np.max(np.abs(logs - want["log_s"]) / np.maximum(1.0, np.abs(want["log_s"]))) <= 1e-12


def test_all_covering_cutoff_equals_dense(ctx):
    """A finite cutoff covering every target selects every target (same
    set as dense, evaluate.cpp:119-128)."""
    rng = np.random.default_rng(8)
    A, M, T, W, psi = random_instance(rng, 3, 300, 1000, 0.05)
    d = gpu_eval(ctx, A, M, T, W, psi, 0.05, math.inf)
    t = gpu_eval(ctx, A, M, T, W, psi, 0.05, 10.0)
    assert t["candidate_pairs"] == d["candidate_pairs"] == 300 * 1000
    assert abs(t["J"] - d["J"]) <= 1e-13 * abs(d["J"])
    assert np.max(np.abs(t["gradient"] - d["gradient"])) <= 1e-14


def test_bitwise_determinism(ctx):
    rng = np.random.default_rng(41)
    A, M, T, W, psi = random_instance(rng, 3, 2000, 20000, 0.05)
    for cutoff in (math.inf, 0.005):
        a = gpu_eval(ctx, A, M, T, W, psi, 0.01, cutoff)
        b = gpu_eval(ctx, A, M, T, W, psi, 0.01, cutoff)
        assert a["J"] == b["J"] and a["D"] == b["D"]
        assert np.array_equal(a["gradient"], b["gradient"])


def test_nearest_and_covering_cost(ctx):
    rng = np.random.default_rng(12)
    T = rng.uniform(size=(5000, 3))
    Q = np.vstack([rng.uniform(size=(500, 3)), rng.uniform(-1, 2, size=(100, 3))])
    idx = rs.SpatialIndex(T, ctx=ctx)
    got = idx.nearest_many(Q)
    assert np.array_equal(got, C.nearest(T, Q))
    assert idx.nearest([5.0, 5.0, 5.0]) == int(np.argmin(((T - 5.0) ** 2).sum(axis=1)))
    A = rng.uniform(size=(3000, 3))
    atoms = rs.SourceAtoms(dim=3, points=A, masses=np.full(3000, 1 / 3000))
    tgt = rs.TargetMeasure(dim=3, points=T, weights=np.full(5000, 1 / 5000))
    assert rs.covering_cost(atoms, tgt, ctx=ctx) == C.covering_cost(A, T)
    # worked example (test_geometry.cpp:270-290)
    a1 = rs.SourceAtoms(dim=1, points=np.array([[0.0, 0, 0], [0.5, 0, 0], [1.0, 0, 0]]),
                        masses=np.full(3, 1 / 3))
    t1 = rs.TargetMeasure(dim=1, points=np.array([[0.0, 0, 0], [1.0, 0, 0]]), weights=np.array([.5, .5]))
    assert rs.covering_cost(a1, t1, ctx=ctx) == pytest.approx(0.125)


# ---- BASELINE configs -------------------------------------------------------

def test_cfg1_full_parity(ctx):
    """cfg1 (2D dense, 16384 x 1024): full-size parity vs the oracle."""
    p = synth.make("cfg1")
    psi = p.psi(0)
    got = gpu_eval(ctx, p.atoms, p.masses, p.targets, p.nu, psi, p.eps, math.inf, dim=2)
    want = C.evaluate_dual(p.atoms, p.masses, p.targets, p.nu, psi, p.eps, math.inf, workers=8)
    assert_parity(got, want, marginal_scale(p.nu, want["gradient"]), TOL)


@pytest.mark.parametrize("name,count", [("cfg2", 8192), ("cfg3", 4096), ("cfg5", 4096)])
def test_config_subsample_parity(ctx, name, count):
    """Seeded atom subsets of the BASELINE configs (full targets) vs the
    oracle, including per-atom candidate sets for the truncated ones."""
    p = synth.make(name)
    psi = p.psi(0)
    cut = p.cutoff(psi)
    sub = synth.subsample_atoms(p, count)
    atoms = rs.SourceAtoms(dim=p.dim, points=sub.atoms, masses=sub.masses)
    tgt = rs.TargetMeasure(dim=p.dim, points=p.targets, weights=p.nu)
    res, cnt, hsh, _ = rs.evaluate_dual_debug(atoms, tgt, psi, p.eps, cut, ctx=ctx)
    want = C.evaluate_dual(sub.atoms, sub.masses, p.targets, p.nu, psi, p.eps, cut, workers=8, per_atom=True)
    got = dict(J=res.J, D=res.D, gradient=res.gradient, atoms_visited=res.atoms_visited,
               candidate_pairs=res.candidate_pairs, empty_candidate_atoms=res.empty_candidate_atoms)
    assert_parity(got, want, marginal_scale(p.nu, want["gradient"]), TOL)
    assert np.array_equal(cnt, want["count"]) and np.array_equal(hsh, want["hash"])


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg5"])
def test_full_size_properties(ctx, name):
    """Full BASELINE sizes: size-independent properties (gradient sums to
    zero, counters consistent, determinism, J finite)."""
    p = synth.make(name)
    atoms = rs.SourceAtoms(dim=p.dim, points=p.atoms, masses=p.masses)
    tgt = rs.TargetMeasure(dim=p.dim, points=p.targets, weights=p.nu)
    psi = p.psi(0)
    cfg = rs.SolverConfig(epsilon=p.eps)
    tr = rs.TruncationState(cutoff=p.cutoff(psi))
    r1 = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), cfg, tr, ctx=ctx)
    r2 = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), cfg, tr, ctx=ctx)
    assert r1.J == r2.J and np.array_equal(r1.gradient, r2.gradient)
    assert abs(r1.gradient.sum()) <= 1e-10
    assert np.all(r1.gradient >= -p.nu)  # nu~ = g + nu >= 0
    assert r1.atoms_visited == p.nq
    if p.truncation == "none":
        assert r1.candidate_pairs == p.nq * p.n and r1.empty_candidate_atoms == 0
    else:
        assert p.nq <= r1.candidate_pairs < p.nq * p.n
    assert math.isfinite(r1.J) and r1.D > 0


# ---- softmax_refine -------------------------------------

@pytest.mark.parametrize("nc,nf,nq,eps,cut", [(50, 300, 4000, 0.05, math.inf), (80, 500, 6000, 0.02, 0.01),
                                              (40, 200, 3000, 0.01, 0.001), (30, 100, 2000, 0.02, -1.0),
                                              (600, 900, 20000, 0.005, 0.002)])
def test_softmax_refine_parity(ctx, nc, nf, nq, eps, cut):
    rng = np.random.default_rng(nc * 7 + nf)
    cy = rng.uniform(size=(nc, 3))
    cnu = rng.uniform(size=nc) + 0.1
    cnu /= cnu.sum()
    cpsi = rng.normal(0, 0.02, nc)
    fy = rng.uniform(size=(nf, 3))
    ax = rng.uniform(size=(nq, 3))
    am = rng.uniform(size=nq) + 0.1
    am /= am.sum()
    want = C.softmax_refine(cy, cnu, cpsi, fy, ax, am, eps, cut)
    coarse = rs.TargetMeasure(dim=3, points=cy, weights=cnu)
    atoms = rs.SourceAtoms(dim=3, points=ax, masses=am)
    got = rs.softmax_refine(coarse, cpsi, fy, atoms, eps, cutoff=cut, ctx=ctx)
    scale = np.max(np.abs(want))
    assert np.max(np.abs(got - want)) <= 1e-10 * scale


def test_softmax_refine_cfg4_subsample(ctx):
    """cfg4 shapes: coarse 8192 mixture targets, fine points, fine atoms (subset)."""
    co = synth.make("cfg4_coarse")
    fi = synth.make("cfg4_fine")
    sub = synth.subsample_atoms(fi, 3000)
    cpsi = np.random.default_rng(5).normal(0, 1e-3, co.n)
    fine_pts = fi.targets[:400]
    cut = float(np.max(cpsi)) + 1e-3 * math.log(float(np.max(co.nu)) / 1e-12)
    want = C.softmax_refine(co.targets, co.nu, cpsi, fine_pts, sub.atoms, sub.masses, 1e-3, cut)
    got = rs.softmax_refine(rs.TargetMeasure(dim=3, points=co.targets, weights=co.nu), cpsi, fine_pts,
                            rs.SourceAtoms(dim=3, points=sub.atoms, masses=sub.masses), 1e-3, cutoff=cut, ctx=ctx)
    assert np.max(np.abs(got - want)) <= 1e-10 * np.max(np.abs(want))


def test_nccl_collective_path_single_rank():
    """The multi-GPU reduction (ncclAllGather + rank-ordered sum, NCCL bound
    with dlopen) on a 1-rank communicator: must reproduce the no-comm result
    bit for bit, dense and truncated.  (Only one GPU is available here; the
    2-rank host logic is tests/test_distributed.py.)"""
    ctx1 = rs.Context(0)
    ctx1.set_comm(0, 1, rs.Context.unique_id())
    rng = np.random.default_rng(91)
    A, M, T, W, psi = random_instance(rng, 3, 3000, 20000, 0.05)
    for cutoff in (math.inf, 0.005):
        a = gpu_eval(ctx1, A, M, T, W, psi, 0.01, cutoff)
        b = gpu_eval(rs.Context.default(0), A, M, T, W, psi, 0.01, cutoff)
        assert a["J"] == b["J"] and a["D"] == b["D"] and a["candidate_pairs"] == b["candidate_pairs"]
        assert np.array_equal(a["gradient"], b["gradient"])
    atoms = rs.SourceAtoms(dim=3, points=A, masses=M)
    tgt = rs.TargetMeasure(dim=3, points=T, weights=W)
    assert rs.covering_cost(atoms, tgt, ctx=ctx1) == rs.covering_cost(atoms, tgt)  # max-allreduce path


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_full_in_split_parity(precision):
    """Dense atom cluster with a ball much larger than a warp's atom box
    (r ~ 8 half-diagonals): most culled targets are full-in for the whole
    warp and skip the per-pair pre-test (truncated.cu fused_cull2); counts,
    hashes and values must still match the oracle."""
    ctx = rs.Context(0)
    ctx.set_precision(precision)
    rng = np.random.default_rng(2024)
    A = 0.45 + 0.1 * rng.uniform(size=(60000, 3))  # warp boxes ~0.01 wide, r = 0.15
    M = rng.uniform(size=60000) + 0.1
    M /= M.sum()
    T = rng.uniform(size=(5000, 3))
    W = np.full(5000, 1 / 5000)
    psi = rng.normal(0, 1e-3, size=5000)
    eps, cutoff = 2e-3, 0.01125
    atoms = rs.SourceAtoms(dim=3, points=A, masses=M)
    tgt = rs.TargetMeasure(dim=3, points=T, weights=W)
    res, cnt, hsh, _ = rs.evaluate_dual_debug(atoms, tgt, psi, eps, cutoff, ctx=ctx)
    r = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), rs.SolverConfig(epsilon=eps),
                         rs.TruncationState(cutoff=cutoff), ctx=ctx)  # non-debug kernel (split active)
    want = C.evaluate_dual(A, M, T, W, psi, eps, cutoff, per_atom=True, workers=8)
    assert np.array_equal(cnt, want["count"]) and np.array_equal(hsh, want["hash"])
    tol = TOL if precision == "fp64" else 2e-5
    for got in (res, r):
        g = dict(J=got.J, D=got.D, gradient=got.gradient, atoms_visited=got.atoms_visited,
                 candidate_pairs=got.candidate_pairs, empty_candidate_atoms=got.empty_candidate_atoms)
        assert_parity(g, want, marginal_scale(W, want["gradient"]), tol)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_edge_geometries(precision):
    """Duplicate targets (nearest ties -> lowest index), atoms far outside the
    target box (clamped cells), a cutoff that empties most candidate sets,
    and a 2D instance: selection and values against the oracle."""
    ctx = rs.Context(0)
    ctx.set_precision(precision)
    tol = TOL if precision == "fp64" else 2e-5
    rng = np.random.default_rng(77)
    T = rng.uniform(size=(800, 3))
    T[400:] = T[:400]  # every target duplicated
    A = np.vstack([rng.uniform(size=(3000, 3)), rng.uniform(-2.0, 3.0, size=(500, 3))])
    M = rng.uniform(size=3500) + 0.1
    M /= M.sum()
    W = rng.uniform(size=800) + 0.1
    W /= W.sum()
    psi = rng.normal(0, 0.02, size=800)
    for eps, cutoff in ((0.01, 0.002), (0.01, 1e-5), (0.05, 0.05)):
        atoms = rs.SourceAtoms(dim=3, points=A, masses=M)
        tgt = rs.TargetMeasure(dim=3, points=T, weights=W)
        res, cnt, hsh, _ = rs.evaluate_dual_debug(atoms, tgt, psi, eps, cutoff, ctx=ctx)
        want = C.evaluate_dual(A, M, T, W, psi, eps, cutoff, per_atom=True)
        assert np.array_equal(cnt, want["count"]) and np.array_equal(hsh, want["hash"])
        got = dict(J=res.J, D=res.D, gradient=res.gradient, atoms_visited=res.atoms_visited,
                   candidate_pairs=res.candidate_pairs, empty_candidate_atoms=res.empty_candidate_atoms)
        assert_parity(got, want, marginal_scale(W, want["gradient"]), tol)
    # 2D, larger
    A2 = np.zeros((40000, 3))
    A2[:, :2] = rng.uniform(size=(40000, 2))
    T2 = np.zeros((6000, 3))
    T2[:, :2] = rng.uniform(size=(6000, 2)) ** 2  # skewed
    M2 = np.full(40000, 1 / 40000)
    W2 = np.full(6000, 1 / 6000)
    psi2 = rng.normal(0, 1e-3, size=6000)
    atoms = rs.SourceAtoms(dim=2, points=A2, masses=M2)
    tgt = rs.TargetMeasure(dim=2, points=T2, weights=W2)
    res, cnt, hsh, _ = rs.evaluate_dual_debug(atoms, tgt, psi2, 1e-3, 0.004, ctx=ctx)
    want = C.evaluate_dual(A2, M2, T2, W2, psi2, 1e-3, 0.004, per_atom=True, workers=8)
    assert np.array_equal(cnt, want["count"]) and np.array_equal(hsh, want["hash"])
    got = dict(J=res.J, D=res.D, gradient=res.gradient, atoms_visited=res.atoms_visited,
               candidate_pairs=res.candidate_pairs, empty_candidate_atoms=res.empty_candidate_atoms)
    assert_parity(got, want, marginal_scale(W2, want["gradient"]), tol)


def test_dense_graph_replay_matches_direct_launches():
    """Dense evaluations without per-kernel timing replay a captured CUDA
    graph (capi.cu eval_dense_graph); with timing on the same kernels launch
    directly.  Both must agree bit for bit across psi / eps changes, on the
    host and the device entry points, and count the same kernel launches."""
    ctx1 = rs.Context(0)
    lib = _lib.load()
    rng = np.random.default_rng(123)
    A, M, T, W, _ = random_instance(rng, 3, 2500, 9000, 0.05)
    for eps in (0.02, 0.005, 0.02):
        for k in range(3):
            psi = rng.normal(scale=0.01, size=len(T))
            ctx1.set_timing(True)
            l0 = lib.rsot_cuda_kernel_launches()
            d = gpu_eval(ctx1, A, M, T, W, psi, eps, math.inf)
            direct_launches = lib.rsot_cuda_kernel_launches() - l0
            ctx1.set_timing(False)
            l0 = lib.rsot_cuda_kernel_launches()
            g = gpu_eval(ctx1, A, M, T, W, psi, eps, math.inf)
            graph_launches = lib.rsot_cuda_kernel_launches() - l0
            assert g["J"] == d["J"] and g["D"] == d["D"]
            assert np.array_equal(g["gradient"], d["gradient"])
            assert graph_launches == direct_launches > 0
            if k == 0:
                want = C.evaluate_dual(A, M, T, W, psi, eps, math.inf)
                assert_parity(g, want, marginal_scale(W, want["gradient"]), TOL)
    # device entry point: outputs copied out of the replayed graph
    import torch
    dev_t = rs.rsot.DeviceTargets(ctx1, T, W)
    dev_a = rs.rsot.DeviceAtoms(ctx1, A, M)
    psis = torch.tensor(rng.normal(scale=0.01, size=(2, len(T))), dtype=torch.float64, device="cuda")
    outs = []
    for timing in (False, True, False):
        ctx1.set_timing(timing)
        res = []
        for k in range(2):
            d_g = torch.empty(len(T), dtype=torch.float64, device="cuda")
            d_sc = torch.empty(8, dtype=torch.float64, device="cuda")
            _lib.check(lib.rsot_cuda_eval_device(ctx1.handle, dev_a.handle, dev_t.handle,
                                                 ctypes.c_void_p(psis[k].data_ptr()), 0.01, math.inf,
                                                 ctypes.c_void_p(d_g.data_ptr()),
                                                 ctypes.c_void_p(d_sc.data_ptr())))
            ctx1.synchronize()
            res.append((d_g.cpu().numpy(), d_sc.cpu().numpy()[:5]))
        outs.append(res)
    ctx1.set_timing(False)
    for k in range(2):
        for o in outs[1:]:
            assert np.array_equal(outs[0][k][0], o[k][0]) and np.array_equal(outs[0][k][1], o[k][1])


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("mode", ["all", "default", "off"])
def test_heavy_chunk_split_parity(mode, precision, monkeypatch):
    """Heavy chunks run split across a cluster of 8 CTAs (truncated.cu
    trunc_fused_split: every 8th target row per CTA, phase-1 sums / counts /
    hashes combined through distributed shared memory in rank order).  A dense
    atom cluster over a dense target cluster makes the heavy chunks; `all`
    forces every chunk (up to one per SM) through the split kernel.  Candidate
    sets exact, values within 1e-10, bitwise deterministic."""
    if mode == "all":
        monkeypatch.setenv("RSOT_CUDA_SPLIT_ALPHA", "0")
        monkeypatch.setenv("RSOT_CUDA_SPLIT_FLOOR", "0")
    elif mode == "off":
        monkeypatch.setenv("RSOT_CUDA_SPLIT_ALPHA", "-1")
    ctx = rs.Context(0)
    ctx.set_precision(precision)
    tol = TOL if precision == "fp64" else 2e-5
    rng = np.random.default_rng(3031)
    A = np.vstack([0.48 + 0.04 * rng.uniform(size=(3000, 3)), rng.uniform(size=(20000, 3))])
    T = np.vstack([0.45 + 0.1 * rng.uniform(size=(120000, 3)), rng.uniform(size=(30000, 3))])
    M = rng.uniform(size=len(A)) + 0.1
    M /= M.sum()
    W = rng.uniform(size=len(T)) + 0.1
    W /= W.sum()
    psi = rng.normal(0, 2e-3, size=len(T))
    eps, cutoff = 2e-3, 0.004
    atoms = rs.SourceAtoms(dim=3, points=A, masses=M)
    tgt = rs.TargetMeasure(dim=3, points=T, weights=W)
    res, cnt, hsh, _ = rs.evaluate_dual_debug(atoms, tgt, psi, eps, cutoff, ctx=ctx)
    want = C.evaluate_dual(A, M, T, W, psi, eps, cutoff, per_atom=True, workers=8)
    assert np.array_equal(cnt, want["count"]) and np.array_equal(hsh, want["hash"])
    runs = [gpu_eval(ctx, A, M, T, W, psi, eps, cutoff) for _ in range(2)]
    assert runs[0]["J"] == runs[1]["J"] and np.array_equal(runs[0]["gradient"], runs[1]["gradient"])
    dbg = dict(J=res.J, D=res.D, gradient=res.gradient, atoms_visited=res.atoms_visited,
               candidate_pairs=res.candidate_pairs, empty_candidate_atoms=res.empty_candidate_atoms)
    for got in (dbg, runs[0]):
        assert_parity(got, want, marginal_scale(W, want["gradient"]), tol)


def _clustered_instance(rng, nq_side=40, n=30000, background=0):
    g = (np.arange(nq_side) + 0.5) / nq_side
    A = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    means = rng.uniform(0.3, 0.7, size=(3, 3))
    T = np.concatenate([m + 0.06 * rng.standard_normal((n // 3, 3)) for m in means] +
                       [rng.uniform(size=(background, 3))])
    M = rng.uniform(size=len(A)) + 0.1
    M /= M.sum()
    W = np.full(len(T), 1.0 / len(T))
    psi = rng.normal(0, 1e-3, size=len(T))
    return A, M, T, W, psi


def _virtual_rank_sum(A, M, T, W, psi, eps, cutoff, world, precision):
    ctx = rs.Context(0)
    ctx.set_precision(precision)
    parts = []
    for r in range(world):
        ctx.set_virtual_rank(r, world)
        parts.append(gpu_eval(ctx, A, M, T, W, psi, eps, cutoff))
    psinu = float(np.dot(psi, W))
    got = dict(J=sum(p["J"] for p in parts) + (world - 1) * psinu, D=sum(p["D"] for p in parts),
               gradient=sum(p["gradient"] for p in parts) + (world - 1) * W,
               atoms_visited=sum(p["atoms_visited"] for p in parts),
               candidate_pairs=sum(p["candidate_pairs"] for p in parts),
               empty_candidate_atoms=sum(p["empty_candidate_atoms"] for p in parts))
    return ctx, parts, got


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_partitioned_atoms_virtual_ranks(precision):
    """Partitioned atoms (rsot_cuda_atoms_create_partitioned): every rank
    holds all atoms and a truncated evaluation takes the work-balanced
    Hilbert chunk range chunk_role_kernel assigns it (dense: equal atom
    ranges).  On one GPU the ranks are virtual (rsot_cuda_ctx_set_virtual_rank):
    the per-rank partials, summed as the collective would, must reproduce the
    oracle (candidate counts exact) and cover every atom once; each rank's
    partial is bitwise reproducible."""
    rng = np.random.default_rng(555)
    A, M, T, W, psi = _clustered_instance(rng)
    tol = TOL if precision == "fp64" else 2e-5
    for eps, cutoff in ((2e-3, 0.004), (0.01, math.inf)):
        want = C.evaluate_dual(A, M, T, W, psi, eps, cutoff, workers=8)
        for world in (2, 3, 8):
            ctx, parts, got = _virtual_rank_sum(A, M, T, W, psi, eps, cutoff, world, precision)
            assert got["atoms_visited"] == len(A)
            assert all(p["atoms_visited"] > 0 for p in parts)
            assert_parity(got, want, marginal_scale(W, want["gradient"]), tol)
            if math.isfinite(cutoff):
                ctx.set_virtual_rank(world - 1, world)
                again = gpu_eval(ctx, A, M, T, W, psi, eps, cutoff)
                assert again["J"] == parts[-1]["J"] and np.array_equal(again["gradient"], parts[-1]["gradient"])


def _virtual_world_eval(ctx, A, M, T, W, psi, eps, cutoff, world):
    lib = _lib.load()
    dev_t = rs.rsot.DeviceTargets(ctx, T, W)
    h = ctypes.c_void_p()  # partitioned atom handle (every rank holds every atom)
    _lib.check(lib.rsot_cuda_atoms_create_partitioned(ctx.handle, rs.rsot._ptr(np.ascontiguousarray(A)),
                                                      rs.rsot._ptr(np.ascontiguousarray(M)), len(A),
                                                      ctypes.byref(h)))
    g = np.empty(len(T))
    sc = _lib.RsotCudaScalars()
    try:
        _lib.check(lib.rsot_cuda_eval_virtual_world(ctx.handle, h, dev_t.handle,
                                                    rs.rsot._ptr(np.ascontiguousarray(psi)), eps, cutoff, world,
                                                    rs.rsot._ptr(g), ctypes.byref(sc)))
    finally:
        lib.rsot_cuda_atoms_destroy(h)
    return dict(J=sc.J, D=sc.D, gradient=g, atoms_visited=sc.atoms_visited, candidate_pairs=sc.candidate_pairs,
                empty_candidate_atoms=sc.empty_candidate_atoms)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_virtual_world_collective_path(precision):
    """The multi-GPU combination code on one GPU (rsot_cuda_eval_virtual_world):
    W virtual ranks' packed partial buffers land in the gather buffer where
    ncclAllGather would put them, then the same rank_sum_kernel +
    finalize_kernel launches that follow the collective produce the result.
    Dense and truncated, W = 1, 2, 3, 8: oracle parity (counters exact),
    bitwise reproducible, and W = 1 bitwise equal to the plain evaluation."""
    rng = np.random.default_rng(556)
    A, M, T, W, psi = _clustered_instance(rng, nq_side=32, n=20000, background=3000)
    tol = TOL if precision == "fp64" else 2e-5
    ctx = rs.Context(0)
    ctx.set_precision(precision)
    for eps, cutoff in ((2e-3, 0.004), (0.01, math.inf)):
        want = C.evaluate_dual(A, M, T, W, psi, eps, cutoff, workers=8)
        plain = gpu_eval(ctx, A, M, T, W, psi, eps, cutoff)
        for world in (1, 2, 3, 8):
            got = _virtual_world_eval(ctx, A, M, T, W, psi, eps, cutoff, world)
            assert got["atoms_visited"] == len(A)
            assert_parity(got, want, marginal_scale(W, want["gradient"]), tol)
            again = _virtual_world_eval(ctx, A, M, T, W, psi, eps, cutoff, world)
            assert again["J"] == got["J"] and np.array_equal(again["gradient"], got["gradient"])
            if world == 1 and precision == "fp64":
                assert got["J"] == plain["J"] and np.array_equal(got["gradient"], plain["gradient"])


def test_partitioned_atoms_balance():
    """Without empty candidate sets the chunk weights track the accepted
    pairs: 8 virtual ranks stay within 1.5x of the mean pairs on a clustered
    instance (with a uniform background: no empty sets) where equal atom
    ranges reach 2.5x."""
    rng = np.random.default_rng(555)
    A, M, T, W, psi = _clustered_instance(rng, background=8000)
    eps, cutoff = 5e-3, 0.008
    want = C.evaluate_dual(A, M, T, W, psi, eps, cutoff, per_atom=True, workers=8)
    assert want["empty_candidate_atoms"] == 0
    _, parts, got = _virtual_rank_sum(A, M, T, W, psi, eps, cutoff, 8, "fp64")
    assert_parity(got, want, marginal_scale(W, want["gradient"]), TOL)
    pairs = np.array([p["candidate_pairs"] for p in parts], dtype=float)
    assert pairs.max() / pairs.mean() < 1.5, pairs
    cnt = want["count"].astype(float)
    contiguous = np.array([cnt[len(A) * r // 8:len(A) * (r + 1) // 8].sum() for r in range(8)])
    assert contiguous.max() / contiguous.mean() > 2.0


@pytest.mark.parametrize("cutoff", [0.004, 0.02])
def test_pair_mask_replay_and_fallbacks(cutoff, monkeypatch):
    """Phase 2 of the fp64 truncated kernel runs target-major over phase 1's
    pair masks and item-index streams (truncated.cu phase2_tm); CTAs whose
    masks or streams overflow (forced here with RSOT_CUDA_MASK_WORDS) or that
    hold no slot (RSOT_CUDA_PAIR_MASKS=0) run the tiled phase 2 and recompute
    the masks.  Phase 1 is common: J, D and the counters are bitwise identical
    in all three modes; the gradients differ only in the summation order of a
    target's column (<= 1e-13 of the marginal scale); every mode is
    reproducible run to run and within 1e-10 of the oracle."""
    rng = np.random.default_rng(977)
    A = np.vstack([0.45 + 0.1 * rng.uniform(size=(4000, 3)), rng.uniform(size=(12000, 3))])
    T = np.vstack([0.4 + 0.2 * rng.uniform(size=(60000, 3)), rng.uniform(size=(20000, 3))])
    M = rng.uniform(size=len(A)) + 0.1
    M /= M.sum()
    W = np.full(len(T), 1.0 / len(T))
    psi = rng.normal(0, 1e-3, size=len(T))
    eps = 2e-3
    runs = {}
    for mode, env in (("replay", {}), ("overflow", {"RSOT_CUDA_MASK_WORDS": "3"}),
                      ("recompute", {"RSOT_CUDA_PAIR_MASKS": "0"})):
        for k in ("RSOT_CUDA_MASK_WORDS", "RSOT_CUDA_PAIR_MASKS"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        ctx = rs.Context(0)
        runs[mode] = gpu_eval(ctx, A, M, T, W, psi, eps, cutoff)
        again = gpu_eval(ctx, A, M, T, W, psi, eps, cutoff)
        assert again["J"] == runs[mode]["J"] and np.array_equal(again["gradient"], runs[mode]["gradient"]), mode
    want = C.evaluate_dual(A, M, T, W, psi, eps, cutoff, workers=8)
    scale = marginal_scale(W, want["gradient"])
    for mode in ("overflow", "recompute"):
        assert runs[mode]["J"] == runs["replay"]["J"] and runs[mode]["D"] == runs["replay"]["D"], mode
        assert np.max(np.abs(runs[mode]["gradient"] - runs["replay"]["gradient"])) <= 1e-13 * scale, mode
        assert runs[mode]["candidate_pairs"] == runs["replay"]["candidate_pairs"], mode
        assert_parity(runs[mode], want, scale, TOL)
    assert_parity(runs["replay"], want, scale, TOL)


@pytest.mark.parametrize("mass_scale", [1.0, 1e-280, 1e-305])
def test_target_major_phase2_range_fallback(ctx, mass_scale):
    """The target-major phase 2 (truncated.cu phase2_tm) folds log2(m_q / S_q)
    into the exponents and is taken only when that stays within +-1000 for
    every atom of the CTA; tiny masses push it out of range, and those CTAs
    run the tiled phase 2 instead.  Either way the result matches the oracle
    (relative to the masses' scale), with empty-set atoms, a partial last
    chunk and a wide psi range in the instance."""
    rng = np.random.default_rng(4242)
    nq, n = 3 * 256 + 77, 6000            # partial last chunk
    A = rng.uniform(size=(nq, 3))
    A[:40] += 3.0                          # atoms far from every target: empty candidate sets
    T = rng.uniform(size=(n, 3))
    M = (rng.uniform(size=nq) + 0.1)
    M = M / M.sum() * mass_scale
    W = rng.uniform(size=n) + 0.5
    W /= W.sum()
    psi = rng.normal(0, 0.05, size=n)      # exponents spread over ~ +-30 at eps = 2e-3
    eps, cutoff = 2e-3, 0.012
    got = gpu_eval(ctx, A, M, T, W, psi, eps, cutoff)
    want = C.evaluate_dual(A, M, T, W, psi, eps, cutoff, workers=4)
    assert got["candidate_pairs"] == want["candidate_pairs"]
    assert got["empty_candidate_atoms"] == want["empty_candidate_atoms"] >= 40
    assert abs(got["J"] - want["J"]) <= TOL * abs(want["J"])
    # (D = sum m_q exp(-L_q) overflows in the reference as well: the far atoms)
    assert got["D"] == want["D"] or abs(got["D"] - want["D"]) <= TOL * abs(want["D"])
    gm = got["gradient"] + W                # nu~ (the transported marginal), scale of the masses
    wm = want["gradient"] + W
    assert np.max(np.abs(gm - wm)) <= TOL * np.max(wm)
    again = gpu_eval(ctx, A, M, T, W, psi, eps, cutoff)
    assert again["J"] == got["J"] and np.array_equal(again["gradient"], got["gradient"])
