"""Full-size parity fixtures (BASELINE cfg2 / cfg3 / cfg5): shared helpers.

TEST INFRASTRUCTURE.  `make_fullsize.py` (build container only: it needs the
reference build oracle/_ref) writes tests/golden/fullsize_<cfg>.npz; the
`-m gpu` tests (tests/test_gpu_fullsize.py) regenerate the same seeded inputs
on the GPU box, check their SHA-256 against the fixture, evaluate them through
the C ABI and compare with the stored reference outputs.

Stored per config: J, D, the three counters and the full gradient of the
reference's own evaluate_dual (proj/src/evaluate.cpp:86-174, compiled from
its sources), plus an order-independent digest of the per-atom
(candidate count, candidate hash) pairs of the C restatement (which the
generator checks bit-equal to the reference on J, D, g and counters at this
size), and a seeded sample of the raw per-atom values to localise a mismatch.
"""
from __future__ import annotations

import hashlib
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
CONFIGS = ("cfg2", "cfg3", "cfg5")
PSI_INDEX = 0          # Problem.psi(k) index evaluated
SAMPLE = 1 << 16       # per-atom (count, hash) entries stored verbatim


def path(cfg: str) -> str:
    return os.path.join(HERE, f"fullsize_{cfg}.npz")


def input_sha256(prob, psi) -> str:
    """SHA-256 over the exact input bits (atoms, masses, targets, nu, psi)."""
    h = hashlib.sha256()
    for a in (prob.atoms, prob.masses, prob.targets, prob.nu, psi):
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def atom_digest(count: np.ndarray, hsh: np.ndarray) -> int:
    """Wrapping sum over atoms q of splitmix(hash_q + splitmix(q << 32 | count_q)):
    order independent, position and value sensitive."""
    q = np.arange(len(count), dtype=np.uint64)
    key = (q << np.uint64(32)) | np.asarray(count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        v = _splitmix(np.asarray(hsh, dtype=np.uint64) + _splitmix(key))
        return int(np.sum(v, dtype=np.uint64))


def sample_index(nq: int) -> np.ndarray:
    rng = np.random.default_rng([2025, nq])
    return np.sort(rng.choice(nq, size=min(SAMPLE, nq), replace=False))
