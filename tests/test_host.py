"""CPU tests of the host side: the C-ABI library loads and exports every
symbol include/rsot_cuda.h declares (no compute calls), host mirrors of the
reference's scalar logic, the synthetic config generator."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT
import paper_2507_23602_b200 as rs
from paper_2507_23602_b200 import _lib, synth


def header_symbols():
    src = open(os.path.join(ROOT, "include", "rsot_cuda.h")).read()
    return sorted(set(re.findall(r"\b(rsot_cuda_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED_SYMBOLS)
    assert lib.rsot_cuda_abi_version() == 1


def test_library_is_sm100a_only():
    path = _lib.LIB_PATH
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {path} 2>&1").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_no_cpu_fallback_without_gpu():
    """Without a GPU the product path fails loudly (no silent CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.RsotCudaError) as e:
        rs.Context(0)
    assert e.value.code == _lib.RSOT_CUDA_NO_DEVICE


def test_shard_range_matches_parallel_blocks():
    """rsot_cuda_shard_range == parallel_blocks partition (parallel.hpp:14-31)."""
    lib = _lib.load()
    for nq in (0, 1, 2, 7, 100, 1001, 16777216):
        for world in (1, 2, 3, 4, 8):
            covered = []
            for r in range(world):
                lo, hi = ctypes.c_size_t(), ctypes.c_size_t()
                lib.rsot_cuda_shard_range(nq, r, world, ctypes.byref(lo), ctypes.byref(hi))
                assert lo.value <= hi.value <= nq
                covered.append((lo.value, hi.value))
            # contiguous, in rank order, covering [0, nq)
            pos = 0
            for lo, hi in covered:
                if lo < hi:
                    assert lo == pos
                    pos = hi
            assert pos == nq
            if world > 1 and nq >= 2:
                w = min(world, nq)
                chunk = (nq + w - 1) // w
                assert covered[0] == (0, min(nq, chunk))


def test_cutoff_mirror_frozen_values():
    """rsot.py mirrors evaluate.cpp:22-49 (test_core.cpp:166-213 values)."""
    t = rs.TruncationState(psi_max=0.0, psi_min=0.0, psi_range=0.0, nu_max=1.0, nu_min=0.5, covering=0.0)
    assert rs.cutoff_pointwise(t, 0.01, 1e-12) == pytest.approx(0.276310211159286, rel=1e-12)
    t.cached_D, t.cached_absJ, t.has_cache = 1.0, 1.0, True
    assert rs.cutoff_integrated(t, 0.01, 1e-4) == pytest.approx(0.046051701859881, rel=1e-12)
    t.covering = 1.0
    assert rs.cutoff_geometric(t, 0.01, 1e-4) == pytest.approx(1.052983173665480, rel=1e-12)
    t.psi_range = 0.25
    assert rs.cutoff_geometric(t, 0.01, 1e-4) == pytest.approx(1.302983173665480, rel=1e-12)
    t.psi_range = 0.0
    t.cached_absJ = 1e20
    assert rs.cutoff_geometric(t, 0.01, 1e-4) == pytest.approx(1.0)
    t.cached_absJ = 0.0
    with pytest.raises(RuntimeError, match="degenerate"):
        rs.cutoff_integrated(t, 0.01, 1e-4)
    assert rs.ball_radius(rs.CostKind.SqEuclidean, -1.0) == 0.0
    assert rs.ball_radius(rs.CostKind.SqGeodesicSphere, 1.0) is None


def test_solver_config_validate():
    rs.SolverConfig().validate()
    for kw in (dict(epsilon=0.0), dict(tau=1.0), dict(delta_thr=0.0), dict(workers=0)):
        with pytest.raises(ValueError):
            rs.SolverConfig(**kw).validate()


def test_evaluate_dual_validates_before_device_work():
    """evaluate.cpp:91-93: size and finiteness checks throw invalid_argument
    before any device call (so they work without a GPU)."""
    atoms = rs.SourceAtoms(dim=1, points=np.array([[0.0, 0, 0]]), masses=np.array([1.0]))
    tgt = rs.TargetMeasure(dim=1, points=np.array([[0.0, 0, 0], [1.0, 0, 0]]), weights=np.array([0.5, 0.5]))
    with pytest.raises(ValueError, match="psi length"):
        rs.evaluate_dual(atoms, tgt, rs.DualPotential(np.zeros(1)), rs.SolverConfig(), rs.TruncationState())
    with pytest.raises(ValueError, match="non-finite"):
        rs.evaluate_dual(atoms, tgt, rs.DualPotential(np.array([np.inf, 0.0])), rs.SolverConfig(),
                         rs.TruncationState())


@pytest.mark.parametrize("name,nq,n,dim", [("cfg1", 16384, 1024, 2), ("cfg2", 262144, 16384, 3)])
def test_synth_shapes_and_determinism(name, nq, n, dim):
    p = synth.make(name)
    assert p.nq == nq and p.n == n and p.dim == dim
    assert p.atoms.shape == (nq, 3) and p.targets.shape == (n, 3)
    assert abs(p.masses.sum() - 1.0) < 1e-12 and np.all(p.masses > 0)
    assert np.all(p.nu == 1.0 / n)
    assert np.all((p.atoms >= 0) & (p.atoms <= 1)) and np.all((p.targets >= 0) & (p.targets <= 1))
    if dim == 2:
        assert np.all(p.atoms[:, 2] == 0) and np.all(p.targets[:, 2] == 0)
    q = synth.make(name)
    assert np.array_equal(p.atoms, q.atoms) and np.array_equal(p.targets, q.targets)
    assert np.array_equal(p.psi(3), q.psi(3)) and not np.array_equal(p.psi(3), p.psi(4))


def test_synth_gauss_points_match_reference_rule():
    """quadrature.cpp:16-19: offsets 0.5 -/+ 0.5/sqrt(3) per cell."""
    c = synth.gauss_coords(4)
    off = 0.5 / math.sqrt(3.0)
    assert c[0] == (0 + (0.5 - off)) * 0.25 and c[1] == (0 + (0.5 + off)) * 0.25
    assert len(c) == 8 and np.all(np.diff(c) > 0)


def test_pointwise_cutoff_of_configs():
    p = synth.make("cfg1")
    assert p.cutoff(p.psi(0)) == math.inf
