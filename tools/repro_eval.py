import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import synth
name = sys.argv[1]; prec = sys.argv[2]; k = int(sys.argv[3])
ctx = rs.Context(0); ctx.set_precision(prec)
if len(sys.argv) > 4: ctx.set_timing(True)
p = synth.make(name)
atoms = rs.SourceAtoms(dim=3, points=p.atoms, masses=p.masses)
tgt = rs.TargetMeasure(dim=3, points=p.targets, weights=p.nu)
for kk in range(k + 1):
    psi = p.psi(kk)
    r = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), rs.SolverConfig(epsilon=p.eps), rs.TruncationState(cutoff=p.cutoff(psi)), ctx=ctx)
    print(prec, kk, r.J, r.candidate_pairs, flush=True)
