#!/usr/bin/env python
"""C4 full-rank SI-DSA: time-to-tol and parity against the oracle fixture
(tests/golden/C4_full.npz) as a function of the DSA PCG stopping tolerance
(relative residual) and the multigrid switch.  Usage: python tools/dsa_rtol_sweep.py [C4]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_25233_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
ref = np.load(os.path.join(ROOT, "tests", "golden", f"{name}_full.npz"))["phi"]
p = P.Problem(name)
for rtol in (1e-13, 1e-12, 1e-11, 1e-10, 1e-9):
    p.set_option("pcg_rtol", rtol)
    ts = []
    for _ in range(2):
        r = p.solve_full_rank(store_psi=0)
        ts.append(float(r.get("solve_seconds", 1)[0]))
    print(json.dumps({"config": name, "pcg_rtol": rtol, "time_to_tol_s": min(ts), "iterations": r.iterations,
                      "pcg_iterations": [int(x) for x in r.history("dsa_iterations")],
                      "rel_vs_oracle": float(np.linalg.norm(r.phi - ref) / np.linalg.norm(ref))}), flush=True)
