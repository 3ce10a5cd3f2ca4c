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
