"""Distribution of per-CTA work (candidate pairs of 256 Hilbert-near atoms)
for a truncated config: is the fused kernel tail-bound?  (development aid)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import synth
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
p = synth.make(name)
psi = p.psi(0)
atoms = rs.SourceAtoms(dim=3, points=p.atoms, masses=p.masses)
tgt = rs.TargetMeasure(dim=3, points=p.targets, weights=p.nu)
res, cnt, _, _ = rs.evaluate_dual_debug(atoms, tgt, psi, p.eps, p.cutoff(psi))
def morton(pts, bits=10):
    q = np.clip(((pts - pts.min(0)) / np.ptp(pts, 0).max() * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)
    k = np.zeros(len(pts), dtype=np.int64)
    for b in range(bits):
        for d in range(3):
            k |= ((q[:, d] >> b) & 1) << (3 * b + d)
    return k
order = np.argsort(morton(p.atoms[:, :3]))
c = cnt[order].astype(np.float64)
nch = (len(c) + 255) // 256
chunks = np.add.reduceat(c, np.arange(0, len(c), 256))
slots = 148 * 4
print(f"{name}: chunks {nch}, pairs {c.sum():.3e}, max chunk {chunks.max():.3e}, "
      f"mean {chunks.mean():.3e}, total/slots {c.sum() / slots:.3e}, "
      f"max/(total/slots) {chunks.max() / (c.sum() / slots):.2f}")
for qq in (50, 90, 99, 99.9):
    print(f"  p{qq} chunk {np.percentile(chunks, qq):.3e}")
