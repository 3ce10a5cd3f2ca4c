"""Writes the BASELINE cfg4 inputs (seeded synthetic, see synth.py) as raw
float64 files for csrc/dropin/cfg4_solve."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_23602_b200 import synth
out = sys.argv[1] if len(sys.argv) > 1 else "/tmp/cfg4"
small = len(sys.argv) > 2 and sys.argv[2] == "small"
os.makedirs(out, exist_ok=True)
for lvl, name in (("coarse", "cfg4_coarse"), ("fine", "cfg4_fine")):
    p = synth.make(name) if not small else synth.make_cfg4_small(lvl)
    np.ascontiguousarray(p.atoms, dtype=np.float64).tofile(f"{out}/{lvl}_atoms.f64")
    np.ascontiguousarray(p.masses, dtype=np.float64).tofile(f"{out}/{lvl}_masses.f64")
    np.ascontiguousarray(p.targets, dtype=np.float64).tofile(f"{out}/{lvl}_targets.f64")
    np.ascontiguousarray(p.nu, dtype=np.float64).tofile(f"{out}/{lvl}_nu.f64")
    print(lvl, p.nq, p.n)
