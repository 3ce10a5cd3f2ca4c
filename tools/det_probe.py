"""Run-to-run determinism probe of a truncated config (development aid):
evaluates the same psi several times and reports differing gradient entries."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import synth
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
p = synth.make(name)
ctx = rs.Context.default(0)
atoms = rs.SourceAtoms(dim=p.dim, points=p.atoms, masses=p.masses)
tgt = rs.TargetMeasure(dim=p.dim, points=p.targets, weights=p.nu)
psi = p.psi(0)
cfg = rs.SolverConfig(epsilon=p.eps)
tr = rs.TruncationState(cutoff=p.cutoff(psi))
ref = None
for k in range(4):
    r = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), cfg, tr, ctx=ctx)
    if ref is None:
        ref = r
        continue
    d = np.nonzero(r.gradient != ref.gradient)[0]
    print(name, "run", k, "J equal", r.J == ref.J, "differing", d.size,
          "max abs diff", float(np.max(np.abs(r.gradient - ref.gradient))), "first", d[:5], flush=True)
