"""Mixed-precision (RSOT_CUDA_PRECISION_FP32) truncated evaluation: BASELINE
cfg5 asks for fp64 and fp32.  The FP32 path keeps the reference's candidate
sets exactly (same FP32 pre-test + exact fp64 band predicate), so counters,
per-atom candidate counts and hashes must match the oracle bit for bit;
J, the gradient and D are held to the stated FP32 tolerance

    |dJ| <= 2e-5 |J|,  ||dg||_inf <= 2e-5 max_k(nu~_k + nu_k),  |dD| <= 2e-5 D

against the fp64 oracle (observed 1e-9 - 1e-7 at the BASELINE sizes: FP32 rounding of the local
coordinates and of the exponent, hardware ex2 with 2^-22 relative error)."""
import math

import numpy as np
import pytest

from conftest import assert_parity, marginal_scale, random_instance
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import synth
from oracle.oracle import COracle

pytestmark = pytest.mark.gpu

TOL32 = 2e-5
C = COracle()


@pytest.fixture(scope="module")
def ctx32():
    c = rs.Context(0)
    c.set_precision("fp32")
    return c


def _debug(ctx, A, M, T, W, psi, eps, cutoff, dim=3):
    atoms = rs.SourceAtoms(dim=dim, points=A, masses=M)
    tgt = rs.TargetMeasure(dim=dim, points=T, weights=W)
    res, cnt, hsh, logs = rs.evaluate_dual_debug(atoms, tgt, psi, eps, cutoff, ctx=ctx)
    got = dict(J=res.J, D=res.D, gradient=res.gradient, atoms_visited=res.atoms_visited,
               candidate_pairs=res.candidate_pairs, empty_candidate_atoms=res.empty_candidate_atoms)
    return got, cnt, hsh, logs


CASES32 = [
    (3, 3000, 400, 0.02, 0.01), (3, 3000, 400, 0.02, 0.03), (3, 3000, 400, 0.02, -1.0),
    (3, 3000, 400, 0.02, 0.002), (2, 5000, 300, 0.005, 0.004), (1, 700, 50, 0.1, 0.02),
    (3, 20000, 5000, 1e-3, 0.01), (3, 100, 1, 0.5, 0.001), (3, 2000, 3000, 1e-4, 1e-3),
    (3, 1000, 200, 0.05, 50.0), (3, 129, 257, 0.03, 0.02),
]


@pytest.mark.parametrize("dim,nq,n,eps,cutoff", CASES32)
def test_fp32_random_instances(ctx32, dim, nq, n, eps, cutoff):
    rng = np.random.default_rng(hash((dim, nq, n, eps, cutoff, 32)) % (2 ** 32))
    A, M, T, W, psi = random_instance(rng, dim, n, nq, 0.05)
    got, cnt, hsh, logs = _debug(ctx32, A, M, T, W, psi, eps, cutoff, dim)
    want = C.evaluate_dual(A, M, T, W, psi, eps, cutoff, per_atom=True)
    assert_parity(got, want, marginal_scale(W, want["gradient"]), TOL32)
    assert np.array_equal(cnt, want["count"])
    assert np.array_equal(hsh, want["hash"])
    assert np.max(np.abs(logs - want["log_s"]) / np.maximum(1.0, np.abs(want["log_s"]))) <= 1e-5


@pytest.mark.parametrize("spread,shift", [(1.0, 0.0), (0.3, 100.0), (5.0, -100.0)])
def test_fp32_wide_potential_range(ctx32, spread, shift):
    """psi spread of many epsilon (late-solve potentials) and gauge shifts of
    +-100 (test_core.cpp:118-130): the per-CTA running shift keeps the FP32
    sums in range; atoms whose sum underflows take the exact fp64 path."""
    rng = np.random.default_rng(int(spread * 10 + shift + 1000))
    A, M, T, W, _ = random_instance(rng, 3, 3000, 6000, 0.05)
    eps = 1e-3
    psi = rng.normal(0.0, spread * eps * 40, size=3000) + shift
    cutoff = float(np.max(psi) + eps * math.log(np.max(W) / 1e-12))
    got, cnt, hsh, _ = _debug(ctx32, A, M, T, W, psi, eps, cutoff)
    want = C.evaluate_dual(A, M, T, W, psi, eps, cutoff, per_atom=True)
    assert_parity(got, want, marginal_scale(W, want["gradient"]), TOL32)
    assert np.array_equal(cnt, want["count"]) and np.array_equal(hsh, want["hash"])


@pytest.mark.parametrize("name,count", [("cfg3", 4096), ("cfg5", 4096)])
def test_fp32_config_subsample(ctx32, name, count):
    p = synth.make(name)
    psi = p.psi(0)
    cut = p.cutoff(psi)
    sub = synth.subsample_atoms(p, count)
    got, cnt, hsh, _ = _debug(ctx32, sub.atoms, sub.masses, p.targets, p.nu, psi, p.eps, cut)
    want = C.evaluate_dual(sub.atoms, sub.masses, p.targets, p.nu, psi, p.eps, cut, workers=8,
                           per_atom=True)
    assert_parity(got, want, marginal_scale(p.nu, want["gradient"]), TOL32)
    assert np.array_equal(cnt, want["count"]) and np.array_equal(hsh, want["hash"])


def test_fp32_vs_fp64_full_cfg5(ctx32):
    """Full cfg5 (16.7 M atoms x 1 M targets): fp32 against the parity-pinned
    fp64 GPU path; identical counters, values within the FP32 tolerance,
    bitwise deterministic."""
    p = synth.make("cfg5")
    atoms = rs.SourceAtoms(dim=3, points=p.atoms, masses=p.masses)
    tgt = rs.TargetMeasure(dim=3, points=p.targets, weights=p.nu)
    psi = p.psi(0)
    cfg = rs.SolverConfig(epsilon=p.eps)
    tr = rs.TruncationState(cutoff=p.cutoff(psi))
    r32 = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), cfg, tr, ctx=ctx32)
    r32b = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), cfg, tr, ctx=ctx32)
    r64 = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), cfg, tr, ctx=rs.Context.default(0))
    assert r32.J == r32b.J and np.array_equal(r32.gradient, r32b.gradient)
    assert r32.candidate_pairs == r64.candidate_pairs
    assert r32.empty_candidate_atoms == r64.empty_candidate_atoms
    assert abs(r32.J - r64.J) <= TOL32 * abs(r64.J)
    scale = float(np.max(r64.gradient + 2 * p.nu))
    assert np.max(np.abs(r32.gradient - r64.gradient)) <= TOL32 * scale
    assert abs(r32.D - r64.D) <= TOL32 * r64.D
    ctx64 = rs.Context.default(0)
    for k in (1, 2, 3):
        psi = p.psi(k)
        tr = rs.TruncationState(cutoff=p.cutoff(psi))
        a = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), cfg, tr, ctx=ctx32)
        b = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), cfg, tr, ctx=ctx64)
        assert a.candidate_pairs == b.candidate_pairs and a.empty_candidate_atoms == b.empty_candidate_atoms
        assert abs(a.J - b.J) <= TOL32 * abs(b.J)
