"""A few evaluations of a config (optionally as virtual rank r of W on
partitioned atoms) for ncu launch lists (development aid).
usage: python tools/eval_once.py cfg5 [rank world] [nev]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import numpy as np
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import _lib, synth
name = sys.argv[1]
rank, world = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 1)
nev = int(sys.argv[4]) if len(sys.argv) > 4 else 3
p = synth.make(name)
ctx = rs.Context(0)
if world > 1:
    ctx.set_virtual_rank(rank, world)
lib = _lib.load()
dev_t = rs.rsot.DeviceTargets(ctx, p.targets, p.nu)
dev_a = rs.rsot.DeviceAtoms(ctx, p.atoms, p.masses)
psi = p.psi(0)
g = np.empty(p.n)
sc = _lib.RsotCudaScalars()
for k in range(nev):
    _lib.check(lib.rsot_cuda_eval(ctx.handle, dev_a.handle, dev_t.handle, rs.rsot._ptr(psi), p.eps, p.cutoff(psi),
                                  rs.rsot._ptr(g), ctypes.byref(sc)))
print("done", sc.candidate_pairs)
