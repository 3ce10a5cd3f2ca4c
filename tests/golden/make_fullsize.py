"""Writes tests/golden/fullsize_<cfg>.npz (see fullsize.py) from the REFERENCE
library compiled from /root/reference/proj/src (oracle/_ref/librsot_ref.so)
and the C restatement (oracle/liboracle.so) for the per-atom digest.  Build
container only; takes ~40 min on 8 cores for all three configs.

usage: python tests/golden/make_fullsize.py [cfg2 cfg3 cfg5]
"""
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
from fullsize import CONFIGS, PSI_INDEX, atom_digest, input_sha256, path, sample_index  # noqa: E402
from oracle.oracle import COracle, RefLib  # noqa: E402
from paper_2507_23602_b200 import synth  # noqa: E402


def main(cfgs):
    workers = os.cpu_count() or 8
    ref, C = RefLib(), COracle()
    for name in cfgs:
        p = synth.make(name)
        psi = p.psi(PSI_INDEX)
        cut = p.cutoff(psi)
        sha = input_sha256(p, psi)
        t0 = time.perf_counter()
        rp = ref.problem(p.dim, p.atoms, p.masses, p.targets, p.nu)
        w = rp.evaluate_dual(psi, p.eps, cut, workers)
        t_ref = time.perf_counter() - t0
        del rp
        t0 = time.perf_counter()
        c = C.evaluate_dual(p.atoms, p.masses, p.targets, p.nu, psi, p.eps, cut, workers=workers, per_atom=True)
        t_c = time.perf_counter() - t0
        c_equal = bool(c["J"] == w["J"] and (c["D"] == w["D"] or (math.isnan(c["D"]) and math.isnan(w["D"])))
                       and np.array_equal(c["gradient"], w["gradient"])
                       and all(c[k] == w[k] for k in ("atoms_visited", "candidate_pairs", "empty_candidate_atoms")))
        cnt, hsh = c["count"], c["hash"]
        idx = sample_index(p.nq)
        np.savez_compressed(
            path(name), sha256=np.array(sha), cutoff=np.float64(cut), eps=np.float64(p.eps),
            J=np.float64(w["J"]), D=np.float64(w["D"]), gradient=w["gradient"],
            counters=np.array([w["atoms_visited"], w["candidate_pairs"], w["empty_candidate_atoms"]], dtype=np.uint64),
            digest=np.uint64(atom_digest(cnt, hsh)), count_sum=np.uint64(int(np.sum(cnt, dtype=np.uint64))),
            count_max=np.uint64(int(cnt.max())), sample_idx=idx.astype(np.int64), sample_count=cnt[idx],
            sample_hash=hsh[idx], c_oracle_equals_ref=np.bool_(c_equal),
            meta=np.array(json.dumps({"workers": workers, "ref_s": t_ref, "c_oracle_s": t_c, "psi_index": PSI_INDEX,
                                      "generator": "tests/golden/make_fullsize.py"})))
        print(json.dumps({"config": name, "nq": p.nq, "n": p.n, "J": w["J"], "pairs": w["candidate_pairs"],
                          "empty": w["empty_candidate_atoms"], "c_oracle_equals_ref": c_equal, "ref_s": t_ref,
                          "c_s": t_c, "sha256": sha}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CONFIGS))
