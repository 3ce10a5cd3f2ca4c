"""Median fused-kernel time (CUDA events inside the library) of truncated
evaluations per config, with a result fingerprint (development aid for A/B
runs of kernel variants; the numbers reported in the bench come from
bench.py).  usage: python tools/trunc_timing.py cfg5 cfg3 [--nev 6]
RSOT_PRECISION=fp32 selects the mixed-precision kernel."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import _lib, synth

args = [a for a in sys.argv[1:] if not a.startswith("--")]
nev = 6
if "--nev" in sys.argv:
    nev = int(sys.argv[sys.argv.index("--nev") + 1])
    args.remove(str(nev))
prec = os.environ.get("RSOT_PRECISION", "fp64")
lib = _lib.load()
for name in args or ["cfg5", "cfg3"]:
    p = synth.make(name)
    ctx = rs.Context(0)
    ctx.set_precision(prec)
    dev_t = rs.rsot.DeviceTargets(ctx, p.targets, p.nu)
    dev_a = rs.rsot.DeviceAtoms(ctx, p.atoms, p.masses)
    g = np.empty(p.n)
    sc = _lib.RsotCudaScalars()
    times = []
    for k in range(nev + 2):
        psi = p.psi(k)
        ctx.set_timing(k >= 2)
        _lib.check(lib.rsot_cuda_eval(ctx.handle, dev_a.handle, dev_t.handle, rs.rsot._ptr(psi), p.eps,
                                      p.cutoff(psi), rs.rsot._ptr(g), ctypes.byref(sc)))
        if k >= 2:
            a, b, _ = ctx.last_kernel_ms()
            times.append(a + b)
        if k == 0:
            J0, g0, pairs0 = sc.J, g.copy(), sc.candidate_pairs
    ms = statistics.median(times)
    frac = 25 * 2 * pairs0 / (ms * 1e-3) / (2 * ctx.fp64_dfma_rate()) if prec == "fp64" else float("nan")
    print(f"{name} {prec}: {ms:.3f} ms (min {min(times):.3f})  pairs {pairs0}  frac {frac:.3f}  "
          f"J {J0!r}  gsum {float(np.abs(g0).sum())!r}", flush=True)
    del dev_a, dev_t
    del ctx
