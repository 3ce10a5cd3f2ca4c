"""Generates tests/golden/golden.npz from the REFERENCE library compiled from
/root/reference/proj/src (oracle/_ref/librsot_ref.so, built by
`make -C oracle ref`).  Run in the build container (the reference is not on
the GPU box); the committed .npz is what travels.

Each case stores the inputs (atoms, masses, targets, nu, psi, eps, cutoff,
workers) and the reference outputs (J, D, gradient, atoms_visited,
candidate_pairs, empty_candidate_atoms) of rsot::evaluate_dual
(proj/src/evaluate.cpp:86-174).  Cases mirror the fixtures of
proj/tests/test_util.hpp (random_instance: U[0,1]^d points, masses/weights
U+0.1 normalised, psi ~ N(0, scale)) and the frozen 2x2 instance of
proj/tests/test_core.cpp:14-28, plus truncated cases covering empty-set
fallbacks, negative / zero cutoffs and all-covering cutoffs.
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import RefLib  # noqa: E402


def random_instance(rng, dim, n, nq, psi_scale=0.1):
    A = np.zeros((nq, 3))
    M = np.empty(nq)
    for q in range(nq):
        A[q, :dim] = rng.uniform(size=dim)
        M[q] = rng.uniform() + 0.1
    M /= M.sum()
    T = np.zeros((n, 3))
    W = np.empty(n)
    for j in range(n):
        T[j, :dim] = rng.uniform(size=dim)
        W[j] = rng.uniform() + 0.1
    W /= W.sum()
    psi = rng.normal(0.0, psi_scale, size=n)
    return A, M, T, W, psi


def main():
    ref = RefLib()
    rng = np.random.default_rng(20250731)
    cases = []
    # frozen 2x2 asymmetric instance (test_core.cpp:14-28), eps = 1
    cases.append(dict(name="two_by_two", dim=1, A=np.array([[0., 0, 0], [1, 0, 0]]), M=np.array([.5, .5]),
                      T=np.array([[0., 0, 0], [1, 0, 0]]), W=np.array([.75, .25]), psi=np.zeros(2),
                      eps=1.0, cutoff=math.inf, workers=1))
    specs = [
        (1, 8, 60, 1.0, math.inf, 1), (1, 8, 60, 0.1, math.inf, 1), (2, 15, 120, 0.3, math.inf, 1),
        (2, 30, 500, 0.1, math.inf, 3), (3, 40, 800, 0.05, math.inf, 2), (3, 1, 50, 0.5, math.inf, 1),
        (2, 200, 2000, 0.01, 0.02, 4), (3, 300, 1500, 0.02, 0.01, 3), (3, 300, 1500, 0.02, 0.002, 1),
        (3, 100, 400, 0.05, -0.5, 1), (3, 100, 400, 0.05, 0.0, 1), (2, 50, 300, 0.1, 10.0, 2),
        (1, 64, 256, 1e-3, 1e-3, 1), (3, 500, 3000, 1e-3, 4e-3, 4),
    ]
    for k, (dim, n, nq, eps, cutoff, workers) in enumerate(specs):
        A, M, T, W, psi = random_instance(rng, dim, n, nq, 0.05 if k % 2 else 0.1)
        cases.append(dict(name=f"rand{k}", dim=dim, A=A, M=M, T=T, W=W, psi=psi, eps=eps, cutoff=cutoff,
                          workers=workers))
    out = {}
    for i, c in enumerate(cases):
        prob = ref.problem(c["dim"], c["A"], c["M"], c["T"], c["W"])
        r = prob.evaluate_dual(c["psi"], c["eps"], c["cutoff"], c["workers"])
        p = f"c{i:02d}_"
        out[p + "name"] = np.array(c["name"])
        for key in ("A", "M", "T", "W", "psi"):
            out[p + key] = c[key]
        out[p + "scal"] = np.array([c["eps"], c["cutoff"], c["workers"], c["dim"]], dtype=np.float64)
        out[p + "J"] = np.array(r["J"])
        out[p + "D"] = np.array(r["D"])
        out[p + "g"] = r["gradient"]
        out[p + "counts"] = np.array([r["atoms_visited"], r["candidate_pairs"], r["empty_candidate_atoms"]],
                                     dtype=np.uint64)
        print(f"{c['name']:12s} J={r['J']:.17g} pairs={r['candidate_pairs']} empty={r['empty_candidate_atoms']}")
    out["ncases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)


if __name__ == "__main__":
    main()
