"""Per-shard cost diagnosis (development aid): for each contiguous atom shard
of an N-GPU run, evaluated alone on one GPU, the fused-kernel time, accepted
pairs, empty atoms and ns per accepted pair; also the whole problem.
Mode "balanced" (default) evaluates the partitioned atoms as each virtual
rank (rsot_cuda_ctx_set_virtual_rank: the work-balanced Hilbert chunk
ranges); "contiguous" uploads equal contiguous atom ranges.
usage: python tools/shard_diag.py cfg3 8 [balanced|contiguous]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import numpy as np
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import _lib, synth

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
mode = sys.argv[3] if len(sys.argv) > 3 else "balanced"
p = synth.make(name)
psi = p.psi(0)
cut = p.cutoff(psi)
ctx = rs.Context(0)
ctx.set_timing(True)
ctx.set_precision(os.environ.get("RSOT_PRECISION", "fp64"))
lib = _lib.load()
dev_t = rs.rsot.DeviceTargets(ctx, p.targets, p.nu)


def run(sel, label, a=None):
    a = a or rs.rsot.DeviceAtoms(ctx, p.atoms[sel], p.masses[sel], shard=False)
    g = np.empty(p.n)
    sc = _lib.RsotCudaScalars()
    ms = []
    for k in range(3):
        _lib.check(lib.rsot_cuda_eval(ctx.handle, a.handle, dev_t.handle, rs.rsot._ptr(psi), p.eps, cut,
                                      rs.rsot._ptr(g), ctypes.byref(sc)))
        ms.append(ctx.last_kernel_ms())
    ms = np.median(np.array(ms), axis=0)
    pairs = sc.candidate_pairs
    print(f"{label:>10}: atoms {sc.atoms_visited:8d} fused {ms[0]:7.2f} ms nearest {ms[1]:5.2f} total {ms[2]:7.2f} "
          f"pairs {pairs:.3e} empty {sc.empty_candidate_atoms:7d} ns/pair {1e6 * ms[0] / max(pairs, 1):.4f}",
          flush=True)


run(np.arange(p.nq), "all")
if mode == "balanced" and world > 1:
    ctx.set_virtual_rank(0, world)
    full = rs.rsot.DeviceAtoms(ctx, p.atoms, p.masses)  # partitioned
    for r in range(world):
        ctx.set_virtual_rank(r, world)
        run(None, f"rank {r}", full)
else:
    for r in range(world):
        lo, hi = ctypes.c_size_t(), ctypes.c_size_t()
        lib.rsot_cuda_shard_range(p.nq, r, world, ctypes.byref(lo), ctypes.byref(hi))
        run(np.arange(lo.value, hi.value), f"shard {r}")
