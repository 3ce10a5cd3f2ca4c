"""Single-GPU check of the multi-GPU load balance: evaluates each rank's
contiguous atom shard (rsot_cuda_shard_range) of an N-GPU strong-scaling run
separately and reports the per-shard kernel times and max/mean (the
compute-bound scaling efficiency is mean/max).
usage: python tools/shard_balance.py cfg3 8"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import numpy as np
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import _lib, synth

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
p = synth.make(name)
psi = p.psi(0)
cut = p.cutoff(psi)
ctx = rs.Context(0)
ctx.set_timing(True)
lib = _lib.load()
dev_t = rs.rsot.DeviceTargets(ctx, p.targets, p.nu)
A = np.ascontiguousarray(p.atoms)
for mode in ("contiguous",):
    times = []
    for r in range(world):
        if mode == "contiguous":
            lo, hi = ctypes.c_size_t(), ctypes.c_size_t()
            lib.rsot_cuda_shard_range(p.nq, r, world, ctypes.byref(lo), ctypes.byref(hi))
            sel = np.arange(lo.value, hi.value)
        a = rs.rsot.DeviceAtoms(ctx, p.atoms[sel], p.masses[sel], shard=False)
        g = np.empty(p.n)
        sc = _lib.RsotCudaScalars()
        ms = []
        for k in range(3):
            _lib.check(lib.rsot_cuda_eval(ctx.handle, a.handle, dev_t.handle, rs.rsot._ptr(psi), p.eps, cut,
                                          rs.rsot._ptr(g), ctypes.byref(sc)))
            ms.append(ctx.last_kernel_ms())
        ms = np.array(ms)
        times.append(float(np.median(ms[:, 2])))
        if r in (0, world // 2):
            print(f"  {mode} shard {r}: atoms {len(sel)} fused {np.median(ms[:, 0]):.2f} ms nearest "
                  f"{np.median(ms[:, 1]):.2f} ms total {np.median(ms[:, 2]):.2f} ms", flush=True)
    t = np.array(times)
    print(f"{name} {world} GPUs {mode:10s}: per-shard ms {np.round(t, 2).tolist()}  max/mean {t.max() / t.mean():.3f}",
          flush=True)
