#!/usr/bin/env python
"""Singular values of an r x N_Omega coefficient block through the
truncation path (svd_values): times the bidiagonalisation (m n >= 3e5) or
QR + Jacobi path.  Usage: python tools/svd_time.py r n_omega [reps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_25233_b200 as P  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 600
nom = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
g = P.Problem("homogeneous(1,1)", nx=16, ny=16, n_theta=nom, n_omega_z=1, use_dsa=0)
rng = np.random.default_rng(1)
k = min(r, nom)
u, _ = np.linalg.qr(rng.standard_normal((r, k)))
v, _ = np.linalg.qr(rng.standard_normal((nom, k)))
C = u @ np.diag(np.logspace(0, -12, k)) @ v.T
X, _ = np.linalg.qr(rng.standard_normal((g.n, r)))
for i in range(reps):
    t0 = time.perf_counter()
    sv = P.svd_values(g, C, X)
    print(f"r {r} n_omega {nom}: {1e3 * (time.perf_counter() - t0):.1f} ms (incl. host copies)", flush=True)
ref = np.linalg.svd(C, compute_uv=False)
k = min(len(ref), len(sv))
err = np.max(np.abs(np.asarray(sv[:k]) - ref[:k])) / ref[0]
print(f"r {r} n_omega {nom}: max |sv - numpy| / sv_max = {err:.2e}", flush=True)
