import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU; parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running")


GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def load_golden():
    z = np.load(GOLDEN)
    cases = []
    for i in range(int(z["ncases"])):
        p = f"c{i:02d}_"
        eps, cutoff, workers, dim = z[p + "scal"].tolist()
        cases.append(dict(name=str(z[p + "name"]), A=z[p + "A"], M=z[p + "M"], T=z[p + "T"], W=z[p + "W"],
                          psi=z[p + "psi"], eps=eps, cutoff=cutoff, workers=int(workers), dim=int(dim),
                          J=float(z[p + "J"]), D=float(z[p + "D"]), g=z[p + "g"],
                          counts=[int(v) for v in z[p + "counts"]]))
    return cases


def random_instance(rng, dim, n, nq, psi_scale=0.1):
    """proj/tests/test_util.hpp:103-135 (numpy RNG instead of mt19937_64)."""
    A = np.zeros((nq, 3))
    A[:, :dim] = rng.uniform(size=(nq, dim))
    M = rng.uniform(size=nq) + 0.1
    M /= M.sum()
    T = np.zeros((n, 3))
    T[:, :dim] = rng.uniform(size=(n, dim))
    W = rng.uniform(size=n) + 0.1
    W /= W.sum()
    psi = rng.normal(0.0, psi_scale, size=n)
    return A, M, T, W, psi


def assert_parity(got, want, n_marginal_scale, tol=1e-10, exact_counts=True):
    """SURVEY.md §8(d) parity metric: |dJ| <= tol |J|; ||dg||_inf <= tol *
    max_k(nu~_k + nu_k) (cancellation-safe scale); |dD| <= tol D; counters
    exact."""
    J, Jw = got["J"], want["J"]
    assert abs(J - Jw) <= tol * abs(Jw) + 1e-300, (J, Jw)
    g, gw = np.asarray(got["gradient"]), np.asarray(want["gradient"])
    assert np.max(np.abs(g - gw)) <= tol * n_marginal_scale, np.max(np.abs(g - gw))
    D, Dw = got["D"], want["D"]
    if np.isfinite(Dw):
        assert abs(D - Dw) <= tol * abs(Dw), (D, Dw)
    else:
        assert D == Dw
    if exact_counts:
        assert got["atoms_visited"] == want["atoms_visited"]
        assert got["candidate_pairs"] == want["candidate_pairs"]
        assert got["empty_candidate_atoms"] == want["empty_candidate_atoms"]


def marginal_scale(nu, g=None):
    """max_k (nu~_k + nu_k) with nu~ = g + nu."""
    nu = np.asarray(nu)
    if g is None:
        return float(np.max(2 * nu))
    return float(np.max(np.asarray(g) + 2 * nu))
