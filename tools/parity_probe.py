"""Quick GPU-vs-oracle probe (development aid; prints diagnostics)."""
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_23602_b200 as rs  # noqa: E402
from paper_2507_23602_b200 import synth  # noqa: E402
from oracle.oracle import COracle  # noqa: E402


def compare(tag, got, want, n):
    dJ = abs(got.J - want["J"]) / max(abs(want["J"]), 1e-300)
    scale = 2.0 / n
    dg = np.max(np.abs(got.gradient - want["gradient"])) / scale
    dD = abs(got.D - want["D"]) / max(abs(want["D"]), 1e-300)
    ok = dJ <= 1e-10 and dg <= 1e-10 and (dD <= 1e-10 or not math.isfinite(want["D"]))
    ok = ok and got.candidate_pairs == want["candidate_pairs"] and got.empty_candidate_atoms == want["empty_candidate_atoms"]
    print(f"{tag:40s} dJ={dJ:.2e} dg={dg:.2e} dD={dD:.2e} pairs {got.candidate_pairs}/{want['candidate_pairs']} "
          f"empty {got.empty_candidate_atoms}/{want['empty_candidate_atoms']} {'OK' if ok else 'FAIL'}", flush=True)
    return ok


def main():
    ctx = rs.Context.default(0)
    C = COracle()
    rng = np.random.default_rng(0)
    allok = True
    for trial, (dim, nq, n, eps, cutoff) in enumerate([
            (3, 3000, 400, 0.02, math.inf), (3, 3000, 400, 0.02, 0.01), (3, 3000, 400, 0.02, 0.03),
            (3, 3000, 400, 0.02, -1.0), (3, 3000, 400, 0.02, 0.0), (3, 3000, 400, 0.02, 0.002),
            (2, 5000, 300, 0.05, math.inf), (2, 5000, 300, 0.005, 0.004), (1, 700, 50, 0.1, 0.02),
            (3, 20000, 5000, 1e-3, 0.01), (3, 2, 2, 1.0, math.inf), (3, 100, 1, 0.5, math.inf),
            (3, 2000, 300, 1e-4, math.inf), (3, 2000, 3000, 1e-4, 1e-3), (2, 3000, 500, 1e-3, math.inf)]):
        A = np.zeros((nq, 3)); A[:, :dim] = rng.uniform(size=(nq, dim))
        M = rng.uniform(size=nq) + 0.1; M /= M.sum()
        T = np.zeros((n, 3)); T[:, :dim] = rng.uniform(size=(n, dim))
        NU = rng.uniform(size=n) + 0.1; NU /= NU.sum()
        psi = rng.normal(0, 0.05, n)
        atoms = rs.SourceAtoms(dim=dim, points=A, masses=M)
        tgt = rs.TargetMeasure(dim=dim, points=T, weights=NU)
        got, cnt, hsh, logs = rs.evaluate_dual_debug(atoms, tgt, psi, eps, cutoff, ctx=ctx)
        want = C.evaluate_dual(A, M, T, NU, psi, eps, cutoff, per_atom=True)
        ok = compare(f"rand{trial} d{dim} {nq}x{n} eps{eps} C{cutoff}", got, want, n)
        ok2 = np.array_equal(cnt, want["count"]) and np.array_equal(hsh, want["hash"])
        dl = np.max(np.abs(logs - want["log_s"]) / np.maximum(1, np.abs(want["log_s"])))
        print(f"   per-atom counts/hash equal: {ok2}  max dlogS {dl:.2e}")
        allok &= ok and ok2
    for name in ["cfg1", "cfg2"]:
        p = synth.make(name)
        psi = p.psi(0)
        sub = synth.subsample_atoms(p, 4096 if name == "cfg2" else p.nq)
        atoms = rs.SourceAtoms(dim=p.dim, points=sub.atoms, masses=sub.masses)
        tgt = rs.TargetMeasure(dim=p.dim, points=p.targets, weights=p.nu)
        got = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), rs.SolverConfig(epsilon=p.eps),
                               rs.TruncationState(cutoff=math.inf), ctx=ctx)
        want = C.evaluate_dual(sub.atoms, sub.masses, p.targets, p.nu, psi, p.eps, math.inf, workers=8)
        allok &= compare(name + " (sub)", got, want, p.n)
    for name in ["cfg3", "cfg5"]:
        p = synth.make(name)
        psi = p.psi(0)
        cut = p.cutoff(psi)
        sub = synth.subsample_atoms(p, 2048)
        atoms = rs.SourceAtoms(dim=p.dim, points=sub.atoms, masses=sub.masses)
        tgt = rs.TargetMeasure(dim=p.dim, points=p.targets, weights=p.nu)
        got, cnt, hsh, logs = rs.evaluate_dual_debug(atoms, tgt, psi, p.eps, cut, ctx=ctx)
        want = C.evaluate_dual(sub.atoms, sub.masses, p.targets, p.nu, psi, p.eps, cut, workers=8, per_atom=True)
        allok &= compare(name + " (sub, truncated)", got, want, p.n)
        print("   per-atom counts/hash equal:", np.array_equal(cnt, want["count"]) and np.array_equal(hsh, want["hash"]))
    # timing
    for name in ["cfg1", "cfg2", "cfg3", "cfg5"]:
        p = synth.make(name)
        atoms = rs.SourceAtoms(dim=p.dim, points=p.atoms, masses=p.masses)
        tgt = rs.TargetMeasure(dim=p.dim, points=p.targets, weights=p.nu)
        ctx.set_timing(True)
        for k in range(4):
            psi = p.psi(k)
            t0 = time.perf_counter()
            r = rs.evaluate_dual(atoms, tgt, rs.DualPotential(psi), rs.SolverConfig(epsilon=p.eps),
                                 rs.TruncationState(cutoff=p.cutoff(psi)), ctx=ctx)
            t1 = time.perf_counter()
            a, b, tot = ctx.last_kernel_ms()
            print(f"{name} eval {k}: wall {1e3*(t1-t0):.3f} ms, passA {a:.3f} passB {b:.3f} total {tot:.3f} ms "
                  f"pairs {r.candidate_pairs} empty {r.empty_candidate_atoms} J {r.J:.15e}", flush=True)
    print("ALLOK", allok)


if __name__ == "__main__":
    main()
