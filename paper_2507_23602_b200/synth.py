"""Seeded synthetic inputs with the shapes of BASELINE.json's configs.

No public dataset is involved: the reference artifact ships no data
(proj/.gitignore:1) and the configs are defined by shape.  Atoms are the
tensor 2-point Gauss-Legendre rule on a structured Q1 quad/hex mesh of the
unit square/cube, with the same 1D offsets the reference's rule uses
(proj/src/quadrature.cpp:16-19: 0.5 -/+ 0.5/sqrt(3), weight 1/2 per
factor), masses m_q = rho(x_q) w_q normalised to sum 1
(proj/src/measures.cpp:39-44).  The reference has simplex rules only, so the
atoms are fed directly as SourceAtoms (as atoms_from_point_cloud would,
quadrature.cpp:139-152).  Targets: U[0,1]^d or the Gaussian mixture,
rejection-restricted to the unit cube; nu_j = 1/N.  All randomness is
numpy's PCG64 seeded per config (fixed seeds below).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

GAUSS_OFF = 0.5 / math.sqrt(3.0)  # quadrature.cpp:17


@dataclass
class Problem:
    name: str
    dim: int
    atoms: np.ndarray        # (nq, 3) float64, zero-padded
    masses: np.ndarray       # (nq,)
    targets: np.ndarray      # (n, 3)
    nu: np.ndarray           # (n,)
    eps: float
    psi_sigma: float
    truncation: str          # "none" | "pointwise"
    delta_thr: float = 1e-12
    seed: int = 0

    @property
    def nq(self) -> int:
        return len(self.atoms)

    @property
    def n(self) -> int:
        return len(self.targets)

    def psi(self, k: int = 0) -> np.ndarray:
        """psi_j ~ N(0, sigma^2), fresh per evaluation index k."""
        rng = np.random.default_rng([self.seed, 1000 + k])
        return rng.normal(0.0, self.psi_sigma, size=self.n)

    def cutoff(self, psi: np.ndarray) -> float:
        """Reference cutoff for this config's truncation kind
        (evaluate.cpp:22-25 pointwise; +inf for none)."""
        if self.truncation == "none":
            return math.inf
        nu_max = float(np.max(self.nu))
        return float(np.max(psi)) + self.eps * math.log(nu_max / self.delta_thr)


def gauss_coords(cells: int) -> np.ndarray:
    """1D Gauss points of `cells` uniform cells of [0,1], cell-major."""
    h = 1.0 / cells
    i = np.arange(cells, dtype=np.float64)
    pts = np.stack([(i + (0.5 - GAUSS_OFF)) * h, (i + (0.5 + GAUSS_OFF)) * h], axis=1)
    return pts.reshape(-1)


def tensor_atoms(cells: int, dim: int) -> np.ndarray:
    """Atoms ordered cell by cell (x fastest), Gauss points inside a cell
    x fastest; (cells*2)^dim points."""
    c = gauss_coords(cells).reshape(cells, 2)
    if dim == 2:
        # index (cy, cx, gy, gx)
        X = np.broadcast_to(c[None, :, None, :], (cells, cells, 2, 2))
        Y = np.broadcast_to(c[:, None, :, None], (cells, cells, 2, 2))
        pts = np.zeros((cells * cells * 4, 3))
        pts[:, 0] = X.reshape(-1)
        pts[:, 1] = Y.reshape(-1)
        return pts
    # index (cz, cy, cx, gz, gy, gx)
    shape = (cells, cells, cells, 2, 2, 2)
    X = np.broadcast_to(c[None, None, :, None, None, :], shape)
    Y = np.broadcast_to(c[None, :, None, None, :, None], shape)
    Z = np.broadcast_to(c[:, None, None, :, None, None], shape)
    pts = np.empty((cells ** 3 * 8, 3))
    pts[:, 0] = X.reshape(-1)
    pts[:, 1] = Y.reshape(-1)
    pts[:, 2] = Z.reshape(-1)
    return pts


def mixture_means(seed: int, k: int = 3) -> np.ndarray:
    rng = np.random.default_rng([seed, 7])
    return rng.uniform(0.2, 0.8, size=(k, 3))


def mixture_density(pts: np.ndarray, means: np.ndarray, sigma: float = 0.1) -> np.ndarray:
    rho = np.zeros(len(pts))
    for mu in means:
        d2 = ((pts - mu) ** 2).sum(axis=1)
        rho += np.exp(-d2 / (2.0 * sigma * sigma))
    return rho


def mixture_samples(n: int, means: np.ndarray, seed: int, sigma: float = 0.1) -> np.ndarray:
    """n samples of the equal-weight isotropic mixture, rejected outside [0,1]^3."""
    rng = np.random.default_rng([seed, 11])
    out = np.empty((0, 3))
    while len(out) < n:
        m = 2 * (n - len(out)) + 1024
        comp = rng.integers(0, len(means), size=m)
        s = means[comp] + sigma * rng.standard_normal((m, 3))
        ok = np.all((s >= 0.0) & (s <= 1.0), axis=1)
        out = np.vstack([out, s[ok]])
    return np.ascontiguousarray(out[:n])


def _masses(rho: np.ndarray) -> np.ndarray:
    m = rho.astype(np.float64)
    return m / m.sum()


def make(name: str, seed: Optional[int] = None) -> Problem:
    if name == "cfg1":
        seed = 0 if seed is None else seed
        atoms = tensor_atoms(64, 2)
        rng = np.random.default_rng(seed)
        tg = np.zeros((1024, 3))
        tg[:, :2] = rng.uniform(0.0, 1.0, size=(1024, 2))
        return Problem("cfg1", 2, atoms, _masses(np.ones(len(atoms))), tg,
                       np.full(1024, 1.0 / 1024), 1e-2, 1e-2, "none", seed=seed)
    if name in ("cfg2", "cfg3", "cfg4_coarse", "cfg4_fine"):
        seed = {"cfg2": 2, "cfg3": 3, "cfg4_coarse": 4, "cfg4_fine": 4}[name] if seed is None else seed
        cells, n, eps, sig, trunc = {
            "cfg2": (32, 16384, 1e-2, 1e-3, "none"),
            "cfg3": (64, 262144, 1e-3, 1e-4, "pointwise"),
            "cfg4_coarse": (32, 8192, 1e-1, 0.0, "pointwise"),
            "cfg4_fine": (64, 131072, 1e-3, 0.0, "pointwise"),
        }[name]
        means = mixture_means(seed)
        atoms = tensor_atoms(cells, 3)
        masses = _masses(mixture_density(atoms, means))
        if name == "cfg4_coarse":
            fine = mixture_samples(131072, means, seed)
            sel = np.sort(np.random.default_rng([seed, 13]).choice(131072, size=8192, replace=False))
            tg = np.ascontiguousarray(fine[sel])
        else:
            tg = mixture_samples(n, means, seed)
        return Problem(name, 3, atoms, masses, tg, np.full(len(tg), 1.0 / len(tg)), eps, sig,
                       trunc, seed=seed)
    if name == "cfg5":
        seed = 5 if seed is None else seed
        atoms = tensor_atoms(128, 3)
        two_pi = 2.0 * math.pi
        rho = 1.0 + 0.5 * (np.sin(two_pi * atoms[:, 0]) * np.sin(two_pi * atoms[:, 1])
                           * np.sin(two_pi * atoms[:, 2]))
        rng = np.random.default_rng([seed, 17])
        tg = rng.uniform(0.0, 1.0, size=(1048576, 3))
        return Problem("cfg5", 3, atoms, _masses(rho), tg, np.full(1048576, 1.0 / 1048576), 1e-4,
                       1e-5, "pointwise", seed=seed)
    raise ValueError(f"unknown config {name}")


def make_cfg4_small(level: str, seed: int = 4) -> Problem:
    """cfg4 at reduced size (8^3 -> 16^3 hexes, 512 -> 4096 targets) for
    solve-level comparisons against the CPU reference."""
    cells, n = (8, 512) if level == "coarse" else (16, 4096)
    means = mixture_means(seed)
    atoms = tensor_atoms(cells, 3)
    masses = _masses(mixture_density(atoms, means))
    fine = mixture_samples(4096, means, seed)
    if level == "coarse":
        sel = np.sort(np.random.default_rng([seed, 13]).choice(4096, size=512, replace=False))
        tg = np.ascontiguousarray(fine[sel])
    else:
        tg = fine
    return Problem("cfg4_small_" + level, 3, atoms, masses, tg, np.full(len(tg), 1.0 / len(tg)), 1e-3, 0.0,
                   "pointwise", seed=seed)


def subsample_atoms(p: Problem, count: int, seed: int = 99) -> Problem:
    """A seeded subset of the atoms (masses kept as is) for bounded oracle runs."""
    rng = np.random.default_rng([seed, p.seed])
    idx = np.sort(rng.choice(p.nq, size=min(count, p.nq), replace=False))
    return Problem(p.name + f"_sub{count}", p.dim, np.ascontiguousarray(p.atoms[idx]),
                   np.ascontiguousarray(p.masses[idx]), p.targets, p.nu, p.eps, p.psi_sigma,
                   p.truncation, p.delta_thr, p.seed)
