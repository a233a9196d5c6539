#!/usr/bin/env python
"""Runs the BASELINE solver configs (C1-C4) on one GPU through the C ABI and
prints one JSON line per (config, method): time-to-tol (the solver's own
solve_seconds, assembly/upload excluded as in the reference), outer
iterations, ranks, PCG iterations, and parity against the oracle's golden
fixture when one exists (tests/golden/<config>_<method>.npz).

Usage: python tools/run_configs.py C1:full C1:lowrank C2:lowrank ...
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_25233_b200 as P  # noqa: E402


def main():
    jobs = sys.argv[1:] or ["C1:full", "C1:lowrank", "C2:lowrank", "C2:full"]
    for job in jobs:
        name, method = job.split(":")
        ov = {}
        if "@" in method:
            method, extra = method.split("@")
            ov = json.loads(extra)
        t0 = time.time()
        p = P.Problem(name, **ov)
        t_asm = time.time() - t0
        solve = p.solve_full_rank if method == "full" else p.solve_low_rank
        kw = {"store_psi": 0} if method == "full" else {"build_factors": 0}
        r = solve(**kw)
        out = {"config": name, "method": method, "overrides": ov, "n_dofs": p.n, "n_omega": p.n_omega,
               "time_to_tol_s": r.get("solve_seconds", 1)[0], "assembly_upload_s": t_asm,
               "iterations": r.iterations, "converged": r.converged,
               "pcg_iterations": [int(x) for x in r.history("dsa_iterations")],
               "diff_inf_norm": [float(x) for x in r.history("diff_inf_norm")]}
        if method == "lowrank":
            out["ranks"] = [int(x) for x in r.history("rank")]
            out["inner_iterations"] = [int(x) for x in r.history("inner_iterations")]
            out["sampled_counts"] = [int(x) for x in r.history("sampled_count")]
        tag = name + ("_" + "_".join(f"{k}{v}" for k, v in sorted(ov.items())) if ov else "")
        gold = os.path.join(ROOT, "tests", "golden", f"{tag}_{method}.npz")
        if os.path.exists(gold):
            g = np.load(gold)
            phi_ref = g["phi"]
            out["oracle"] = {"iterations": int(g["iterations"]), "solve_seconds_1core": float(g["solve_seconds"]),
                             "phi_rel_l2": float(np.linalg.norm(r.phi - phi_ref) / np.linalg.norm(phi_ref))}
            if method == "lowrank":
                out["oracle"]["ranks"] = [int(x) for x in g["rank"]]
                counts = g["sampled_counts"]
                flat = g["sampled_flat"]
                ref_log, k = [], 0
                for c in counts:
                    ref_log.append([int(v) for v in flat[k:k + c]])
                    k += c
                mine = r.sampled_log()
                out["oracle"]["sampled_jaccard_first_outer"] = (
                    len(set(mine[0]) & set(ref_log[0])) / max(1, len(set(mine[0]) | set(ref_log[0]))))
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
