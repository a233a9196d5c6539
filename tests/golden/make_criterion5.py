"""One-off golden fixture for the reference's acceptance criterion 5
(reference-resolution rank / compression bands, proj/tests/acceptance.cpp:
244-313; R's captured values proj/test_output.txt:31), computed by the CPU
oracle (oracle/, a restatement of the reference — R itself cannot be built
here: Eigen is absent).  TEST INFRASTRUCTURE ONLY.

Cases, as acceptance.cpp runs them (run() = full rank and low rank with the
preset's solver defaults):
  homogeneous(100,2), seed 1            R: rank 52, iterations FR/LR 6/6
  variable_scattering:full, seed 1      R: rank 317, C-R 40.86 %, it 9/9
  pin_cell:full, FR + LR seeds 1..8     R: FR 17 iterations, mean LR rank 220.00

Each solve runs in its own process (8 at a time).  Writes
tests/golden/criterion5.npz (phi of every seed-1 solve and the pin-cell FR
solve, iterations, factor ranks, rank histories, sampled logs).

Usage: python tests/golden/make_criterion5.py [workers]
"""
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

CASES = [("homogeneous(100,2)", "full", 1), ("homogeneous(100,2)", "lowrank", 1),
         ("variable_scattering:full", "full", 1), ("variable_scattering:full", "lowrank", 1),
         ("pin_cell:full", "full", 1)] + [("pin_cell:full", "lowrank", s) for s in range(1, 9)]


def tag(name, method, seed):
    base = name.replace("(", "_").replace(")", "").replace(",", "_").replace(":", "_")
    return f"{base}__{method}__s{seed}"


def solve(case):
    import _oracle as O
    name, method, seed = case
    p = O.Problem(name, seed=seed, store_psi=0)
    t0 = time.time()
    r = p.solve(method)
    dt = time.time() - t0
    out = {"tag": tag(*case), "iterations": r.iterations, "converged": r.converged, "seconds": dt,
           "n_dofs": p.n, "n_omega": p.n_omega, "phi": r.get("phi", p.n)}
    if method == "lowrank":
        log = r.sampled_log()
        out.update(factor_rank=r.factor_rank, ranks=r.history("rank"),
                   sampled_counts=np.array([len(x) for x in log], dtype=np.int64),
                   sampled_flat=np.array([v for x in log for v in x], dtype=np.int64))
    print(json.dumps({k: (v if not isinstance(v, np.ndarray) else None) for k, v in out.items()
                      if k != "phi"}), flush=True)
    return out


def main():
    workers = int(sys.argv[1]) if len(sys.argv) > 1 else min(8, os.cpu_count() or 1)
    import _oracle as O
    O.build()
    with mp.get_context("spawn").Pool(workers) as pool:
        results = pool.map(solve, CASES, chunksize=1)
    arrays = {}
    for r in results:
        t = r["tag"]
        for k in ("iterations", "converged", "seconds", "n_dofs", "n_omega", "factor_rank"):
            if k in r:
                arrays[f"{t}.{k}"] = np.asarray(r[k])
        for k in ("ranks", "sampled_counts", "sampled_flat"):
            if k in r:
                arrays[f"{t}.{k}"] = np.asarray(r[k])
        if r["tag"].endswith("__s1"):
            arrays[f"{t}.phi"] = r["phi"]
    np.savez_compressed(os.path.join(HERE, "criterion5.npz"), **arrays)
    print("wrote criterion5.npz")


if __name__ == "__main__":
    main()
