"""Runs a few cfg5 (or given config) evaluations for ncu capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import synth
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
nev = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = rs.Context.default(0)
ctx.set_precision(os.environ.get("RSOT_PRECISION", "fp64"))
p = synth.make(name)
atoms = rs.SourceAtoms(dim=p.dim, points=p.atoms, masses=p.masses)
tgt = rs.TargetMeasure(dim=p.dim, points=p.targets, weights=p.nu)
for k in range(nev):
    psi = p.psi(k)
    r = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), rs.SolverConfig(epsilon=p.eps),
                         rs.TruncationState(cutoff=p.cutoff(psi)), ctx=ctx)
print("done", r.candidate_pairs)
