"""The reference's own doctest suites (proj/tests/test_{core,geometry,
measures}.cpp), compiled unmodified against the B200 drop-in library
(paper_2507_23602_b200/csrc/dropin: reference headers and host solver
sources, GPU evaluate_dual / covering_cost).  The reference L-BFGS,
epsilon-scaling, softmax_refine and multilevel drivers run on the host and
call the GPU evaluator through the reference's Objective closure."""
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
