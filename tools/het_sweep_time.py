#!/usr/bin/env python
"""Times the heterogeneous many-direction sweep at the solver configs: the
unique directions of C3 / C4 with one shared right-hand side (the full-rank
SI sweep), per kernel (sweep_kernel 1 = skewed wavefront, 5 = direction
groups), psi written; and si_step (sweep + scalar flux) per kernel.
CUDA events on the problem's stream.  Usage: python tools/het_sweep_time.py [C4 C3]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_25233_b200 as P  # noqa: E402


def main():
    for name in sys.argv[1:] or ["C4", "C3"]:
        g = P.Problem(name, use_dsa=0)
        s = torch.cuda.Stream()
        torch.cuda.set_stream(s)
        g.set_stream(s.cuda_stream)
        nz = g.n_omega_z
        reps = np.array([j1 * nz + j2 for j1 in range(g.n_theta) for j2 in range(nz // 2)], dtype=np.int32)
        n = g.n
        rhs = torch.rand(n, dtype=torch.float64, device="cuda")
        psi = torch.empty(len(reps) * n, dtype=torch.float64, device="cuda")
        out = {"config": name, "directions": len(reps), "cells": n // 4}
        ref = None
        for k in (1, 5):
            g.set_option("sweep_kernel", k)
            for _ in range(2):
                g.sweep_device(reps.ctypes.data, len(reps), rhs.data_ptr(), 0, psi.data_ptr(), n)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            reps_n = 5
            for _ in range(reps_n):
                g.sweep_device(reps.ctypes.data, len(reps), rhs.data_ptr(), 0, psi.data_ptr(), n)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps_n
            cur = psi.view(len(reps), n).cpu().numpy()
            if ref is None:
                ref = cur
            out[f"sweep_ms_k{k}"] = ms
            out[f"upd_per_s_k{k}"] = len(reps) * (n // 4) / (ms * 1e-3)
            out[f"rel_vs_k1_k{k}"] = float(np.linalg.norm(cur - ref) / np.linalg.norm(ref))
            phi = np.linspace(0, 1, n)
            g.si_step(phi)
            torch.cuda.synchronize()
            import time
            t0 = time.perf_counter()
            for _ in range(3):
                g.si_step(phi)
            out[f"si_step_ms_k{k}"] = (time.perf_counter() - t0) / 3 * 1e3
        print(json.dumps(out), flush=True)
        del psi
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
