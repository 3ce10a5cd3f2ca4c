"""Observed deviation of the fp32 (mixed) truncated path from the fp64 path
at full BASELINE size (development aid; the tests assert 2e-5)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import synth
c64 = rs.Context(0)
c32 = rs.Context(0)
c32.set_precision("fp32")
for name in sys.argv[1:] or ["cfg5", "cfg3"]:
    p = synth.make(name)
    atoms = rs.SourceAtoms(dim=3, points=p.atoms, masses=p.masses)
    tgt = rs.TargetMeasure(dim=3, points=p.targets, weights=p.nu)
    for k in range(2):
        psi = p.psi(k)
        cfg = rs.SolverConfig(epsilon=p.eps)
        tr = rs.TruncationState(cutoff=p.cutoff(psi))
        a = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), cfg, tr, ctx=c64)
        b = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), cfg, tr, ctx=c32)
        scale = float(np.max(a.gradient + 2 * p.nu))
        print(f"{name} psi{k}: |dJ|/|J| {abs(a.J - b.J) / abs(a.J):.2e}  max|dg|/scale "
              f"{np.max(np.abs(a.gradient - b.gradient)) / scale:.2e}  |dD|/D {abs(a.D - b.D) / a.D:.2e}  "
              f"pairs equal {a.candidate_pairs == b.candidate_pairs}", flush=True)
