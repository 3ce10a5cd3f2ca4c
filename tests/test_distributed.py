"""world_size-2 gloo test of the multi-GPU host logic on CPU.

The B200 path shards atoms contiguously (rsot_cuda_shard_range), evaluates
each shard, all-gathers the packed partial buffers [g + nu | J + sum psi nu |
D | pairs | empty | visited], sums them in rank order on every rank and
finalises once.  Here the
shard evaluation is the CPU oracle, the collective is gloo, the rank-ordered
sum and finalisation are the library's (host mirrors of rank_sum_kernel /
finalize_kernel), and the result must equal the single-process evaluation.
The device kernels themselves run in tests/test_gpu_parity.py
(rsot_cuda_eval_virtual_world, W = 2, 3, 8)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import random_instance


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cutoff, q):
    import ctypes
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.oracle import COracle
    from paper_2507_23602_b200 import _lib
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(77)
    A, M, T, W, psi = random_instance(rng, 3, 300, 2001, 0.05)
    lib = _lib.load()
    lo, hi = ctypes.c_size_t(), ctypes.c_size_t()
    lib.rsot_cuda_shard_range(len(A), rank, world, ctypes.byref(lo), ctypes.byref(hi))
    C = COracle()
    part = C.evaluate_dual(A[lo.value:hi.value], M[lo.value:hi.value], T, W, psi, 0.02, cutoff)
    psinu = float(np.sum(psi * W))
    # un-finalise the shard result into the packed partial buffer
    buf = np.concatenate([part["gradient"] + W, [part["J"] + psinu, part["D"], part["candidate_pairs"],
                                                  part["empty_candidate_atoms"], part["atoms_visited"]]])
    t = torch.from_numpy(buf)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    # the library's rank-ordered sum and finalisation (host mirrors of
    # rank_sum_kernel / finalize_kernel: the same element functions)
    gathered = np.ascontiguousarray(np.concatenate([p.numpy() for p in parts]))
    n = len(W)
    red = np.empty(n + 5)
    lib.rsot_cuda_host_rank_sum(gathered.ctypes.data, world, n + 5, red.ctypes.data)
    g = np.empty(n)
    sc = np.empty(5)
    lib.rsot_cuda_host_finalize(red.ctypes.data, np.ascontiguousarray(W).ctypes.data, n, psinu,
                                g.ctypes.data, sc.ctypes.data)
    J = sc[0]
    full = C.evaluate_dual(A, M, T, W, psi, 0.02, cutoff)
    ok = (abs(J - full["J"]) <= 1e-12 * abs(full["J"]) and np.max(np.abs(g - full["gradient"])) <= 1e-14
          and abs(sc[1] - full["D"]) <= 1e-12 * full["D"] and int(sc[2]) == full["candidate_pairs"]
          and int(sc[3]) == full["empty_candidate_atoms"] and int(sc[4]) == len(A))
    q.put((rank, bool(ok), red.tobytes()))
    dist.destroy_process_group()


@pytest.mark.parametrize("cutoff", [math.inf, 0.01])
def test_two_rank_shard_gather_sum_matches_single(cutoff):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cutoff, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted((r, ok) for r, ok, _ in res) == [(0, True), (1, True)]
    assert res[0][2] == res[1][2]  # bitwise identical on every rank
