"""Generates golden fixtures for the BASELINE configs from the CPU oracle
(oracle/, a restatement of the reference; the reference itself cannot be
built here).  Usage:  python tests/golden/make_golden.py C2 [lowrank|full]

Writes tests/golden/<config>_<method>.npz with phi, the outer history, the
sampled log (low rank) and the wall time.  TEST INFRASTRUCTURE ONLY."""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import _oracle as O  # noqa: E402


def main():
    name = sys.argv[1]
    method = sys.argv[2] if len(sys.argv) > 2 else "lowrank"
    overrides = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
    t0 = time.time()
    p = O.Problem(name, store_psi=0, build_factors=0, **overrides)
    t_asm = time.time() - t0
    t1 = time.time()
    r = p.solve(method)
    t_solve = time.time() - t1
    tag = name + ("_" + "_".join(f"{k}{v}" for k, v in sorted(overrides.items())) if overrides else "")
    out = os.path.join(HERE, f"{tag}_{method}.npz")
    log = r.sampled_log() if method == "lowrank" else []
    np.savez_compressed(
        out, phi=r.get("phi", p.n), iterations=r.iterations, converged=r.converged,
        diff_two_norm=r.history("diff_two_norm"), diff_inf_norm=r.history("diff_inf_norm"),
        rank=r.history("rank"), inner_iterations=r.history("inner_iterations"),
        sampled_counts=np.array([len(x) for x in log], dtype=np.int64),
        sampled_flat=np.array([v for x in log for v in x], dtype=np.int64),
        solve_seconds=t_solve, assembly_seconds=t_asm, overrides=json.dumps(overrides))
    print(json.dumps({"config": tag, "method": method, "iterations": r.iterations, "converged": r.converged,
                      "ranks": [int(x) for x in r.history("rank")], "solve_seconds": t_solve,
                      "assembly_seconds": t_asm, "file": out}))


if __name__ == "__main__":
    main()
