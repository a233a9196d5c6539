#!/usr/bin/env python
"""One bordered Galerkin finish (dense.cu galerkin_border_kernel) at a given
size, through the test hook: python tools/border_probe.py [r0 k m] (for ncu
captures; also prints the agreement with the full pivoted LU)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_25233_b200 as P  # noqa: E402

r0, k, m = (int(a) for a in (sys.argv[1:4] if len(sys.argv) >= 4 else (600, 8, 16)))
rng = np.random.default_rng(5)
r = r0 + k
proj = []
for _ in range(4):
    g = rng.standard_normal((r, r)) / np.sqrt(r)
    h = rng.standard_normal((r, r)) / np.sqrt(r)
    proj.append(g - g.T + 0.3 * h @ h.T)
h = rng.standard_normal((r, r)) / np.sqrt(r)
proj.append(np.eye(r) + 0.2 * h @ h.T)
th = rng.uniform(0, 2 * np.pi, 64)
dirs = np.stack([np.cos(th), np.sin(th), rng.uniform(0.1, 0.9, 64)], axis=1)
angles = rng.choice(64, size=m, replace=False)
full, bord = P.dense_galerkin_border(r0, k, angles, dirs, proj, rng.standard_normal(r))
print("r0", r0, "k", k, "m", m, "worst rel diff", max(np.linalg.norm(full[:, c] - bord[:, c]) / np.linalg.norm(full[:, c]) for c in range(m)))
