"""ctypes bindings of the parity checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) import this module.  The product package never does.

  C       : liboracle.so          C restatement (rsot_oracle.c)
  Ref     : _ref/librsot_ref.so   the reference library compiled from
                                  /root/reference/proj/src (ref_capi.cpp)
"""
from __future__ import annotations

import ctypes
import math
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_size_t, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "librsot_ref.so")


class Scalars(ctypes.Structure):
    _fields_ = [("J", c_double), ("D", c_double), ("atoms_visited", ctypes.c_uint64),
                ("candidate_pairs", ctypes.c_uint64), ("empty_candidate_atoms", ctypes.c_uint64)]


def _p(a):
    return c_void_p(a.ctypes.data) if a is not None else None


def _pts(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if a.shape[1] < 3:
        a = np.ascontiguousarray(np.hstack([a, np.zeros((len(a), 3 - a.shape[1]))]))
    return a


class COracle:
    """The C restatement (rsot_oracle.c)."""

    def __init__(self, path: str = C_LIB):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing (make -C oracle)")
        L = ctypes.CDLL(path)
        L.oracle_last_error.restype = c_char_p
        L.oracle_grid_create.restype = c_void_p
        L.oracle_grid_create.argtypes = [c_void_p, c_size_t]
        L.oracle_grid_destroy.argtypes = [c_void_p]
        L.oracle_grid_ball_query.restype = c_size_t
        L.oracle_grid_ball_query.argtypes = [c_void_p, c_void_p, c_double, c_void_p, c_size_t]
        L.oracle_grid_nearest.restype = ctypes.c_uint64
        L.oracle_grid_nearest.argtypes = [c_void_p, c_void_p]
        L.oracle_candidate_hash_term.restype = ctypes.c_uint64
        L.oracle_candidate_hash_term.argtypes = [ctypes.c_uint64]
        L.oracle_evaluate_dual.restype = c_int
        L.oracle_evaluate_dual.argtypes = [c_size_t, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p,
                                           c_void_p, c_double, c_double, c_int, c_void_p, c_void_p,
                                           POINTER(Scalars), c_void_p, c_void_p, c_void_p]
        L.oracle_covering_cost.restype = c_int
        L.oracle_covering_cost.argtypes = [c_size_t, c_void_p, c_size_t, c_void_p, POINTER(c_double)]
        L.oracle_softmax_refine.restype = c_int
        L.oracle_softmax_refine.argtypes = [c_size_t, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p,
                                            c_size_t, c_void_p, c_void_p, c_double, c_double, c_void_p]
        L.oracle_evaluate_dual_geodesic.restype = c_int
        L.oracle_evaluate_dual_geodesic.argtypes = [c_size_t, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p,
                                                    c_void_p, c_double, c_double, c_void_p, POINTER(Scalars),
                                                    c_void_p, c_void_p]
        L.oracle_plan_view.restype = c_int
        L.oracle_plan_view.argtypes = [c_size_t, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p, c_void_p,
                                       c_double, c_double] + [c_void_p] * 8
        L.oracle_ball_radius.restype = c_double
        L.oracle_ball_radius.argtypes = [c_double]
        L.oracle_cutoff_pointwise.restype = c_double
        L.oracle_cutoff_pointwise.argtypes = [c_double] * 4
        L.oracle_cutoff_integrated.restype = c_int
        L.oracle_cutoff_integrated.argtypes = [c_double] * 6 + [POINTER(c_double)]
        L.oracle_cutoff_geometric.restype = c_int
        L.oracle_cutoff_geometric.argtypes = [c_double] * 6 + [POINTER(c_double)]
        L.oracle_cutoff_bootstrap.restype = c_double
        L.oracle_cutoff_bootstrap.argtypes = [c_double] * 5
        self.L = L

    def evaluate_dual(self, atoms, masses, targets, nu, psi, eps, cutoff=math.inf, workers=1,
                      per_atom=False):
        atoms, targets = _pts(atoms), _pts(targets)
        masses = np.ascontiguousarray(masses, dtype=np.float64)
        nu = np.ascontiguousarray(nu, dtype=np.float64)
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        g = np.empty(len(targets))
        sc = Scalars()
        cnt = np.zeros(len(atoms), dtype=np.uint32) if per_atom else None
        hsh = np.zeros(len(atoms), dtype=np.uint64) if per_atom else None
        logs = np.zeros(len(atoms)) if per_atom else None
        rc = self.L.oracle_evaluate_dual(len(atoms), _p(atoms), _p(masses), len(targets), _p(targets),
                                         _p(nu), _p(psi), float(eps), float(cutoff), int(workers), None,
                                         _p(g), ctypes.byref(sc), _p(cnt), _p(hsh), _p(logs))
        if rc == -1:
            raise ValueError(self.L.oracle_last_error().decode())
        if rc != 0:
            raise RuntimeError(self.L.oracle_last_error().decode())
        out = dict(J=sc.J, D=sc.D, gradient=g, atoms_visited=sc.atoms_visited,
                   candidate_pairs=sc.candidate_pairs, empty_candidate_atoms=sc.empty_candidate_atoms)
        if per_atom:
            out.update(count=cnt, hash=hsh, log_s=logs)
        return out

    def softmax_refine(self, coarse_xyz, coarse_nu, coarse_psi, fine_xyz, atoms, masses, eps,
                       cutoff=math.inf):
        cy, fy, ax = _pts(coarse_xyz), _pts(fine_xyz), _pts(atoms)
        cnu = np.ascontiguousarray(coarse_nu, dtype=np.float64)
        cpsi = np.ascontiguousarray(coarse_psi, dtype=np.float64)
        am = np.ascontiguousarray(masses, dtype=np.float64)
        out = np.empty(len(fy))
        rc = self.L.oracle_softmax_refine(len(cy), _p(cy), _p(cnu), _p(cpsi), len(fy), _p(fy), len(ax), _p(ax),
                                          _p(am), float(eps), float(cutoff), _p(out))
        if rc != 0:
            raise ValueError(self.L.oracle_last_error().decode())
        return out

    def evaluate_dual_geodesic(self, atoms, masses, targets, nu, psi, eps, cutoff=math.inf,
                               per_atom=False):
        atoms, targets = _pts(atoms), _pts(targets)
        masses = np.ascontiguousarray(masses, dtype=np.float64)
        nu = np.ascontiguousarray(nu, dtype=np.float64)
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        g = np.empty(len(targets))
        sc = Scalars()
        cnt = np.zeros(len(atoms), dtype=np.uint32) if per_atom else None
        logs = np.zeros(len(atoms)) if per_atom else None
        rc = self.L.oracle_evaluate_dual_geodesic(len(atoms), _p(atoms), _p(masses), len(targets), _p(targets),
                                                  _p(nu), _p(psi), float(eps), float(cutoff), _p(g),
                                                  ctypes.byref(sc), _p(cnt), _p(logs))
        if rc != 0:
            raise ValueError(self.L.oracle_last_error().decode())
        out = dict(J=sc.J, D=sc.D, gradient=g, atoms_visited=sc.atoms_visited,
                   candidate_pairs=sc.candidate_pairs, empty_candidate_atoms=sc.empty_candidate_atoms)
        if per_atom:
            out.update(count=cnt, log_s=logs)
        return out

    def plan_view(self, atoms, masses, targets, nu, psi, eps, cutoff=math.inf):
        """PlanView (plan.cpp): dict of log_s, count, marginal, moment (n,3),
        bary (n,3), starved (first starved index or -1), map (nq,3), modal."""
        a, t = _pts(atoms), _pts(targets)
        m = np.ascontiguousarray(masses, dtype=np.float64)
        nu = np.ascontiguousarray(nu, dtype=np.float64)
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        nq, n = len(a), len(t)
        out = dict(log_s=np.zeros(nq), count=np.zeros(nq, dtype=np.uint64), marginal=np.zeros(n),
                   moment=np.zeros((n, 3)), bary=np.zeros((n, 3)), map=np.zeros((nq, 3)),
                   modal=np.zeros(nq, dtype=np.uint64))
        st = ctypes.c_int64(-1)
        rc = self.L.oracle_plan_view(nq, _p(a), _p(m), n, _p(t), _p(nu), _p(psi), float(eps), float(cutoff),
                                     _p(out["log_s"]), _p(out["count"]), _p(out["marginal"]),
                                     _p(out["moment"]), _p(out["bary"]), _p(out["map"]), _p(out["modal"]),
                                     ctypes.byref(st))
        if rc != 0:
            raise ValueError(self.L.oracle_last_error().decode())
        out["starved"] = int(st.value)
        return out

    def hash_term(self, j: int) -> int:
        return int(self.L.oracle_candidate_hash_term(j))

    def ball_query(self, points, center, radius):
        pts = _pts(points)
        grid = self.L.oracle_grid_create(_p(pts), len(pts))
        if not grid:
            raise ValueError(self.L.oracle_last_error().decode())
        c = _pts(np.asarray(center, dtype=np.float64).reshape(1, -1))[0].copy()
        n = self.L.oracle_grid_ball_query(grid, _p(c), float(radius), None, 0)
        out = np.zeros(max(n, 1), dtype=np.uint64)
        self.L.oracle_grid_ball_query(grid, _p(c), float(radius), _p(out), n)
        self.L.oracle_grid_destroy(grid)
        return out[:n].astype(np.int64)

    def nearest(self, points, centers):
        pts = _pts(points)
        grid = self.L.oracle_grid_create(_p(pts), len(pts))
        if not grid:
            raise ValueError(self.L.oracle_last_error().decode())
        cs = _pts(centers)
        out = np.array([self.L.oracle_grid_nearest(grid, _p(np.ascontiguousarray(c))) for c in cs],
                       dtype=np.int64)
        self.L.oracle_grid_destroy(grid)
        return out

    def covering_cost(self, atoms, targets):
        a, t = _pts(atoms), _pts(targets)
        v = c_double()
        rc = self.L.oracle_covering_cost(len(a), _p(a), len(t), _p(t), ctypes.byref(v))
        if rc != 0:
            raise ValueError(self.L.oracle_last_error().decode())
        return v.value


class RefLib:
    """The reference library compiled from /root/reference/proj/src."""

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing (make -C oracle ref, needs /root/reference)")
        L = ctypes.CDLL(path)
        L.ref_last_error.restype = c_char_p
        L.ref_problem_create.restype = c_void_p
        L.ref_problem_create.argtypes = [c_int, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p, c_size_t]
        L.ref_problem_destroy.argtypes = [c_void_p]
        L.ref_evaluate_dual.restype = c_int
        L.ref_evaluate_dual.argtypes = [c_void_p, c_void_p, c_size_t, c_double, c_double, c_int,
                                        c_void_p, POINTER(Scalars)]
        L.ref_softmax_refine.restype = c_int
        L.ref_softmax_refine.argtypes = [c_void_p, c_void_p, c_void_p, c_size_t, c_double, c_double, c_int,
                                         c_void_p]
        L.ref_covering_cost.restype = c_int
        L.ref_covering_cost.argtypes = [c_void_p, POINTER(c_double)]
        L.ref_covering_cost_kind.restype = c_int
        L.ref_covering_cost_kind.argtypes = [c_void_p, c_int, POINTER(c_double)]
        L.ref_evaluate_dual_kind.restype = c_int
        L.ref_evaluate_dual_kind.argtypes = [c_void_p, c_void_p, c_size_t, c_double, c_double, c_int, c_void_p,
                                             POINTER(Scalars)]
        L.ref_plan_view.restype = c_int
        L.ref_plan_view.argtypes = [c_void_p, c_void_p, c_double, c_double] + [c_void_p] * 6
        self.L = L

    def problem(self, dim, atoms, masses, targets, nu):
        return RefProblem(self, dim, atoms, masses, targets, nu)


class RefProblem:
    def __init__(self, lib: RefLib, dim, atoms, masses, targets, nu):
        self.lib = lib
        self.atoms, self.targets = _pts(atoms), _pts(targets)
        self.masses = np.ascontiguousarray(masses, dtype=np.float64)
        self.nu = np.ascontiguousarray(nu, dtype=np.float64)
        self.h = lib.L.ref_problem_create(int(dim), _p(self.atoms), _p(self.masses), len(self.atoms),
                                          _p(self.targets), _p(self.nu), len(self.targets))
        if not self.h:
            raise ValueError(lib.L.ref_last_error().decode())

    def evaluate_dual(self, psi, eps, cutoff=math.inf, workers=1):
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        g = np.empty(len(self.targets))
        sc = Scalars()
        rc = self.lib.L.ref_evaluate_dual(self.h, _p(psi), len(psi), float(eps), float(cutoff),
                                          int(workers), _p(g), ctypes.byref(sc))
        if rc == -1:
            raise ValueError(self.lib.L.ref_last_error().decode())
        if rc != 0:
            raise RuntimeError(self.lib.L.ref_last_error().decode())
        return dict(J=sc.J, D=sc.D, gradient=g, atoms_visited=sc.atoms_visited,
                    candidate_pairs=sc.candidate_pairs, empty_candidate_atoms=sc.empty_candidate_atoms)

    def softmax_refine(self, coarse_psi, fine_xyz, eps, cutoff=math.inf, workers=1):
        cpsi = np.ascontiguousarray(coarse_psi, dtype=np.float64)
        fy = _pts(fine_xyz)
        out = np.empty(len(fy))
        rc = self.lib.L.ref_softmax_refine(self.h, _p(cpsi), _p(fy), len(fy), float(eps), float(cutoff),
                                           int(workers), _p(out))
        if rc != 0:
            raise ValueError(self.lib.L.ref_last_error().decode())
        return out

    def evaluate_dual_geodesic(self, psi, eps, cutoff=math.inf):
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        g = np.empty(len(self.targets))
        sc = Scalars()
        rc = self.lib.L.ref_evaluate_dual_kind(self.h, _p(psi), len(psi), float(eps), float(cutoff), 1, _p(g),
                                               ctypes.byref(sc))
        if rc != 0:
            raise ValueError(self.lib.L.ref_last_error().decode())
        return dict(J=sc.J, D=sc.D, gradient=g, atoms_visited=sc.atoms_visited,
                    candidate_pairs=sc.candidate_pairs, empty_candidate_atoms=sc.empty_candidate_atoms)

    def plan_view(self, psi, eps, cutoff=math.inf):
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        nq, n = len(self.atoms), len(self.targets)
        out = dict(count=np.zeros(nq, dtype=np.uint64), marginal=np.zeros(n), bary=np.zeros((n, 3)),
                   map=np.zeros((nq, 3)), modal=np.zeros(nq, dtype=np.uint64))
        st = ctypes.c_int64(-1)
        rc = self.lib.L.ref_plan_view(self.h, _p(psi), float(eps), float(cutoff), _p(out["count"]),
                                      _p(out["marginal"]), _p(out["bary"]), ctypes.byref(st), _p(out["map"]),
                                      _p(out["modal"]))
        if rc != 0:
            raise ValueError(self.lib.L.ref_last_error().decode())
        out["starved"] = int(st.value)
        return out

    def covering_cost(self, kind: int = 0):
        """kind 0 = SqEuclidean, 1 = SqGeodesicSphere."""
        v = c_double()
        if self.lib.L.ref_covering_cost_kind(self.h, kind, ctypes.byref(v)) != 0:
            raise ValueError(self.lib.L.ref_last_error().decode())
        return v.value

    def __del__(self):
        try:
            self.lib.L.ref_problem_destroy(self.h)
        except Exception:
            pass


def candidate_hash(cand_indices) -> int:
    """Wrapping sum of splitmix64(j) (same as rsot_oracle.c / device_math.cuh)."""
    M = (1 << 64) - 1
    tot = 0
    for j in cand_indices:
        z = (int(j) + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        tot = (tot + (z ^ (z >> 31))) & M
    return tot
