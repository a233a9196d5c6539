#!/usr/bin/env python
"""A/B of environment-switch variants on low-rank solves: every (variant,
config) in a fresh process (one warm solve, then R timed solves), variants
interleaved.  python tools/lr_ab.py C2,C3,C4 'A:RTLR_X=0' 'B:' [--reps R]
prints time-to-tol, iterations, ranks per run and whether phi is bitwise
equal across variants."""
import os
import subprocess
import sys

import numpy as np

args = sys.argv[1:]
reps = 2
if "--reps" in args:
    i = args.index("--reps")
    reps = int(args[i + 1])
    del args[i:i + 2]
cfgs = args[0].split(",")
variants = []
for spec in args[1:]:
    name, _, envs = spec.partition(":")
    env = dict(kv.split("=", 1) for kv in envs.split(",") if kv)
    variants.append((name, env))
code = r'''
import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2603_25233_b200 as P
p = P.Problem(sys.argv[2])
p.solve_low_rank(build_factors=0)
for k in range(int(sys.argv[3])):
    r = p.solve_low_rank(build_factors=0)
    ranks = [int(x) for x in r.history("rank")]
    inner = int(sum(r.history("inner_iterations")))
    print(f"{r.get('solve_seconds', 1)[0]:.4f} s it {r.iterations} inner {inner} ranks {ranks}", flush=True)
np.save(sys.argv[1], r.phi)
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for cfg in cfgs:
    for k in range(2):
        for name, env in (variants if k == 0 else variants[::-1]):
            out = subprocess.run([sys.executable, "-c", code, f"/tmp/phi_ab_{name}_{cfg}.npy", cfg, str(reps)],
                                 env=dict(os.environ, **env), capture_output=True, text=True, cwd=root)
            lines = out.stdout.strip().splitlines()
            print(cfg, name, " | ".join(lines), out.stderr[-300:] if out.returncode else "", flush=True)
    phis = [np.load(f"/tmp/phi_ab_{n}_{cfg}.npy") for n, _ in variants]
    for (n, _), ph in zip(variants[1:], phis[1:]):
        print(cfg, f"phi {variants[0][0]} vs {n}: bitwise {np.array_equal(phis[0], ph)}, rel "
              f"{np.linalg.norm(ph - phis[0]) / np.linalg.norm(phis[0]):.2e}", flush=True)
