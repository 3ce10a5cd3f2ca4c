"""Times the truncated configs (pass A / pass B / total) for the current
RSOT_CELLS_PER_RADIUS; prints one line per config (development aid)."""
import os, sys, time, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import synth

ctx = rs.Context.default(0)
prec = os.environ.get("RSOT_PRECISION", "fp64")
ctx.set_precision(prec)
for name in sys.argv[1:] or ["cfg3", "cfg5"]:
    p = synth.make(name)
    atoms = rs.SourceAtoms(dim=p.dim, points=p.atoms, masses=p.masses)
    tgt = rs.TargetMeasure(dim=p.dim, points=p.targets, weights=p.nu)
    ctx.set_timing(True)
    res = []
    for k in range(4):
        psi = p.psi(k)
        r = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), rs.SolverConfig(epsilon=p.eps),
                             rs.TruncationState(cutoff=p.cutoff(psi)), ctx=ctx)
        res.append(ctx.last_kernel_ms())
    a, b, t = np.median(np.array(res[1:]), axis=0)
    print(f"{prec} cpr={os.environ.get('RSOT_CELLS_PER_RADIUS','default')} {name}: passA {a:.2f} ms passB {b:.2f} ms "
          f"total {t:.2f} ms pairs {r.candidate_pairs} -> {r.candidate_pairs/t/1e-3:.3e} pairs/s", flush=True)
