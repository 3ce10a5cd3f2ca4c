"""Per-evaluation overhead at an 8-GPU cfg2 shard size (1/8 of the atoms):
device time of back-to-back eval_device calls vs the hot kernels' event
time (development aid)."""
import os, sys, ctypes, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import _lib, synth
frac = int(sys.argv[1]) if len(sys.argv) > 1 else 8
p = synth.make("cfg2")
ctx = rs.Context(0)
lib = _lib.load()
nq = p.nq // frac
dev_t = rs.rsot.DeviceTargets(ctx, p.targets, p.nu)
dev_a = rs.rsot.DeviceAtoms(ctx, p.atoms[:nq], p.masses[:nq], shard=False)
d_psi = torch.tensor(p.psi(0), dtype=torch.float64, device="cuda")
d_g = torch.empty(p.n, dtype=torch.float64, device="cuda")
d_sc = torch.empty(8, dtype=torch.float64, device="cuda")
stream = torch.cuda.ExternalStream(ctx.stream)
def ev():
    _lib.check(lib.rsot_cuda_eval_device(ctx.handle, dev_a.handle, dev_t.handle, ctypes.c_void_p(d_psi.data_ptr()),
                                         p.eps, float("inf"), ctypes.c_void_p(d_g.data_ptr()),
                                         ctypes.c_void_p(d_sc.data_ptr())))
for _ in range(5):
    ev()
ctx.set_timing(True)
ev(); ctx.synchronize()
a, b, tot = ctx.last_kernel_ms()
ctx.set_timing(False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
K = 50
e0.record(stream)
for _ in range(K):
    ev()
e1.record(stream)
torch.cuda.synchronize()
print(f"cfg2/{frac}: atoms {nq}: per-eval {e0.elapsed_time(e1) / K:.3f} ms, passes {a:.3f}+{b:.3f} ms, "
      f"prologue->finalize {tot:.3f} ms", flush=True)
