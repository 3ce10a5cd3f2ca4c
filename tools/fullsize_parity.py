"""Full-size parity of the GPU evaluator against the C oracle (test
infrastructure: oracle/ restates the reference evaluate_dual) on the BASELINE
configs, on identical seeded inputs; the oracle runs on every host core.
Prints one JSON object per config (|dJ|/|J|, ||dg||_inf / max(nu~+nu),
|dD|/D, counters) against the 1e-10 bar.
usage: python tools/fullsize_parity.py cfg2 cfg5 [cfg3]"""
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_23602_b200 as rs  # noqa: E402
from paper_2507_23602_b200 import synth  # noqa: E402
from oracle.oracle import COracle  # noqa: E402

ctx = rs.Context.default(0)
C = COracle()
workers = os.cpu_count() or 8
for name in sys.argv[1:] or ["cfg2", "cfg5"]:
    p = synth.make(name)
    psi = p.psi(0)
    cut = p.cutoff(psi)
    atoms = rs.SourceAtoms(dim=p.dim, points=p.atoms, masses=p.masses)
    tgt = rs.TargetMeasure(dim=p.dim, points=p.targets, weights=p.nu)
    t0 = time.perf_counter()
    g = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), rs.SolverConfig(epsilon=p.eps),
                         rs.TruncationState(cutoff=cut), ctx=ctx)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    w = C.evaluate_dual(p.atoms, p.masses, p.targets, p.nu, psi, p.eps, cut, workers=workers)
    t_cpu = time.perf_counter() - t0
    scale = float(np.max(np.asarray(w["gradient"]) + 2 * np.asarray(p.nu)))
    dJ = abs(g.J - w["J"]) / abs(w["J"])
    dg = float(np.max(np.abs(np.asarray(g.gradient) - np.asarray(w["gradient"])))) / scale
    dD = abs(g.D - w["D"]) / w["D"] if math.isfinite(w["D"]) and w["D"] > 0 else 0.0
    same = (g.candidate_pairs == w["candidate_pairs"] and g.empty_candidate_atoms == w["empty_candidate_atoms"]
            and g.atoms_visited == w["atoms_visited"])
    print(json.dumps({"config": name, "nq": p.nq, "n": p.n, "cutoff": cut, "J_gpu": g.J, "J_oracle": w["J"],
                      "rel_dJ": dJ, "rel_dg_marginal": dg, "rel_dD": dD,
                      "candidate_pairs": [g.candidate_pairs, w["candidate_pairs"]],
                      "empty_atoms": [g.empty_candidate_atoms, w["empty_candidate_atoms"]],
                      "counters_equal": bool(same), "pass_1e-10": bool(dJ <= 1e-10 and dg <= 1e-10 and dD <= 1e-10
                                                                          and same),
                      "gpu_s_incl_setup": t_gpu, "oracle_s": t_cpu, "oracle_workers": workers}), flush=True)
