"""The reference's own doctest suites (proj/tests/test_{core,geometry,
measures}.cpp), compiled unmodified against the B200 drop-in library
(paper_2507_23602_b200/csrc/dropin: reference headers and host solver
sources, GPU evaluate_dual / covering_cost).  The reference L-BFGS,
epsilon-scaling, softmax_refine and multilevel drivers run on the host and
call the GPU evaluator through the reference's Objective closure."""
import math
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "paper_2507_23602_b200", "lib")
KNOWN_REFERENCE_FAILURES = {
    # fails identically with the reference's own CPU evaluate.cpp
    # (tests/test_oracle.py::test_reference_doctest_suites)
    "solve_multilevel: target hierarchy cuts fine-level iterations",
}


@pytest.mark.parametrize("suite", ["core", "geometry", "measures"])
def test_reference_suite_on_gpu_dropin(suite):
    exe = os.path.join(BIN, f"test_{suite}_cuda")
    assert os.path.exists(exe), "drop-in suites not built (build() in the build container)"
    p = subprocess.run([exe], capture_output=True, text=True, timeout=900, cwd="/tmp")
    failed = [ln.split('TEST_CASE("', 1)[1].rstrip('")') for ln in p.stderr.splitlines() if "in TEST_CASE(" in ln]
    summary = [ln for ln in p.stdout.splitlines() if "test cases" in ln]
    print(summary)
    assert set(failed) <= KNOWN_REFERENCE_FAILURES, p.stderr[-3000:]
    assert summary, p.stdout[-2000:]


def test_cfg4_small_multilevel_solve_matches_reference():
    """Reduced BASELINE cfg4 (8^3 -> 16^3 hexes, 512 -> 4096 mixture targets,
    eps 1e-1 -> 1e-2 | softmax_refine | 1e-3 -> 1e-4, pointwise 1e-12, L1
    tolerance 1e-8): the reference's L-BFGS / solve / softmax_refine driving
    the GPU evaluator vs the same driver on the reference CPU evaluator
    (tests/golden/make_cfg4_small.py).  Iteration counts must agree stage by
    stage and the final gauge-fixed potential to 1e-10 relative."""
    import json
    import sys
    import numpy as np
    golden = os.path.join(ROOT, "tests", "golden")
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "cfg4_prepare.py"), "/tmp/cfg4s_t", "small"],
                   check=True, capture_output=True)
    dump = "/tmp/cfg4s_t_psi.f64"
    env = dict(os.environ, RSOT_DUMP_PSI=dump)
    p = subprocess.run([os.path.join(BIN, "cfg4_solve"), "/tmp/cfg4s_t", "1e-8", "1000"], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    got = json.loads(p.stdout)
    want = json.load(open(os.path.join(golden, "cfg4_small_ref.json")))
    for key in ("coarse_stages", "fine_stages"):
        for a, b in zip(want[key], got[key]):
            assert a["iterations"] == b["iterations"], (key, a, b)
            assert a["status"] == b["status"]
            assert abs(a["final_J"] - b["final_J"]) <= 1e-10 * abs(a["final_J"])
    pr = np.fromfile(os.path.join(golden, "cfg4_small_ref_psi.f64"))
    pg = np.fromfile(dump)
    assert np.max(np.abs(pr - pg)) <= 1e-10 * np.max(np.abs(pr))


@pytest.mark.parametrize("cutoff", [math.inf, 0.01, -1.0])
def test_dropin_plan_view(tmp_path, cutoff):
    """The drop-in PlanView (csrc/dropin/plan_cuda.cpp, unchanged plan.hpp)
    through the reference's C++ interface vs the PlanView oracle (pinned to
    the reference plan.cpp in tests/test_oracle.py)."""
    import numpy as np
    from conftest import random_instance
    from oracle.oracle import COracle
    rng = np.random.default_rng(44)
    A, M, T, W, psi = random_instance(rng, 3, 400, 3000, 0.05)
    for name, arr in (("atoms", A), ("masses", M), ("targets", T), ("nu", W), ("psi", psi)):
        np.ascontiguousarray(arr, dtype=np.float64).tofile(tmp_path / f"{name}.f64")
    exe = os.path.join(BIN, "plan_check")
    assert os.path.exists(exe), "drop-in not built (build() in the build container)"
    p = subprocess.run([exe, str(tmp_path), "0.02", repr(cutoff)], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    want = COracle().plan_view(A, M, T, W, psi, 0.02, cutoff)
    assert np.array_equal(np.fromfile(tmp_path / "count.u64", dtype=np.uint64), want["count"])
    marg = np.fromfile(tmp_path / "marginal.f64")
    assert np.max(np.abs(marg - want["marginal"])) <= 1e-12 * np.max(want["marginal"])
    starved = int(open(tmp_path / "starved.txt").read())
    assert starved == want["starved"]
    if starved < 0:
        bary = np.fromfile(tmp_path / "bary.f64").reshape(-1, 3)
        assert np.max(np.abs(bary - want["bary"])) <= 1e-12 * np.max(np.abs(want["bary"]))
    mp = np.fromfile(tmp_path / "map.f64").reshape(-1, 3)
    assert np.max(np.abs(mp - want["map"])) <= 1e-12
    assert np.array_equal(np.fromfile(tmp_path / "modal.u64", dtype=np.uint64), want["modal"])


def _inplace_data(seed=45):
    import numpy as np
    from conftest import random_instance
    rng = np.random.default_rng(seed)
    A, M, T, W, psi = random_instance(rng, 3, 20000, 3000, 0.01)
    idx = np.array([1, 7, 4099, 12345, 19997])  # off any sampling grid (step 4 for N = 20000)
    T2 = T.copy()
    T2[idx] = rng.uniform(size=(len(idx), 3))
    W2 = W.copy()
    W2[idx] *= 3.0
    M2 = M.copy()
    M2[[3, 1001, 2999]] *= 5.0
    return A, M, M2, T, T2, W, W2, psi


def _check_sequence(outs, A, M, M2, T, T2, W, W2, psi, eps, cutoff):
    import numpy as np
    from conftest import assert_parity, marginal_scale
    from oracle.oracle import COracle
    C = COracle()
    cases = [(M, T, W), (M, T2, W), (M, T2, W2), (M2, T2, W2)]
    prev = None
    for got, (m, t, w) in zip(outs, cases):
        want = C.evaluate_dual(A, m, t, w, psi, eps, cutoff, workers=8)
        assert_parity(got, want, marginal_scale(w, want["gradient"]), 1e-10)
        if prev is not None:
            assert not np.array_equal(got["gradient"], prev)  # every edit changed the result
        prev = got["gradient"]


@pytest.mark.parametrize("cutoff", [0.004, math.inf])
def test_dropin_inplace_edits(tmp_path, cutoff):
    """Exact device caches: the drop-in re-uploads whenever the caller's
    arrays change in place -- target points overwritten in the same vector as
    the reference's barycenter loop does (barycenter.cpp:55), weights and
    masses edited at a few entries no sampled hash would visit -- and every
    result matches the oracle for the edited data (C++ drop-in)."""
    import numpy as np
    A, M, M2, T, T2, W, W2, psi = _inplace_data()
    for name, arr in (("atoms", A), ("masses", M), ("masses2", M2), ("targets", T), ("targets2", T2),
                      ("nu", W), ("nu2", W2), ("psi", psi)):
        np.ascontiguousarray(arr, dtype=np.float64).tofile(tmp_path / f"{name}.f64")
    exe = os.path.join(BIN, "inplace_check")
    assert os.path.exists(exe), "drop-in not built (build() in the build container)"
    p = subprocess.run([exe, str(tmp_path), "0.01", repr(cutoff)], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    outs = []
    for k in range(1, 5):
        v = np.fromfile(tmp_path / f"out{k}.f64")
        outs.append(dict(J=v[0], D=v[1], candidate_pairs=int(v[2]), empty_candidate_atoms=int(v[3]),
                         atoms_visited=int(v[4]), gradient=v[5:]))
    _check_sequence(outs, A, M, M2, T, T2, W, W2, psi, 0.01, cutoff)


@pytest.mark.parametrize("cutoff", [0.004, math.inf])
def test_python_mirror_inplace_edits(cutoff):
    """The same in-place edit sequence through the Python mirror
    (rsot.evaluate_dual): numpy arrays edited in place on the same
    TargetMeasure / SourceAtoms objects."""
    import paper_2507_23602_b200 as rs
    A, M, M2, T, T2, W, W2, psi = _inplace_data()
    ctx = rs.Context(0)
    atoms = rs.SourceAtoms(dim=3, points=A.copy(), masses=M.copy())
    tgt = rs.TargetMeasure(dim=3, points=T.copy(), weights=W.copy())
    outs = []

    def ev():
        r = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), rs.SolverConfig(epsilon=0.01),
                             rs.TruncationState(cutoff=cutoff), ctx=ctx)
        outs.append(dict(J=r.J, D=r.D, gradient=r.gradient, atoms_visited=r.atoms_visited,
                         candidate_pairs=r.candidate_pairs, empty_candidate_atoms=r.empty_candidate_atoms))

    ev()
    tgt.points[...] = T2
    ev()
    tgt.weights[...] = W2
    ev()
    atoms.masses[...] = M2
    ev()
    _check_sequence(outs, A, M, M2, T, T2, W, W2, psi, 0.01, cutoff)
