#!/usr/bin/env python
"""Per-phase roofline of the low-rank solver (bench.py's lowrank_phases) for
the given configs: python tools/lr_phases.py C2 C3 C4"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2603_25233_b200 as P  # noqa: E402

for name in sys.argv[1:] or ["C2"]:
    sp = P.Problem(name)
    sp.solve_low_rank(build_factors=0)  # warm (one-time costs)
    ph = bench.lowrank_phases(sp)
    print(json.dumps({"config": name, "phases": ph}), flush=True)
    for k, v in ph.items():
        if isinstance(v, dict) and "seconds" in v:
            f = lambda x: "-" if x is None else f"{x:.3f}"
            print(f"  {k:12s} {v['seconds']:.3f} s  {v['GB']:9.1f} GB {v['GFLOP']:10.1f} GFLOP  "
                  f"hbm {f(v['frac_hbm'])}  dmma {f(v['frac_fp64_tensor'])}", flush=True)
