#!/usr/bin/env python
"""Few-direction sweeps (the low-rank inner loop's p sampled directions) on a
config's own medium: ms per launch for each K1 kernel (sweep_kernel 0 auto, 1 skew,
2 scan, 3 prefactored scan, 4 cluster wavefront), CUDA events on the problem's stream.
Usage: python tools/few_dir_sweep.py C4 [p ...]"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2603_25233_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
ps = [int(a) for a in sys.argv[2:]] or [1, 8, 16]
prob = P.Problem(name)
st = torch.cuda.Stream()
prob.set_stream(st.cuda_stream)
n, nom = prob.n, prob.n_omega
rhs = torch.rand(n, dtype=torch.float64, device="cuda")
for p in ps:
    ang = torch.arange(0, nom, max(1, nom // p), dtype=torch.int32, device="cuda")[:p].contiguous()
    psi = torch.empty(n * p, dtype=torch.float64, device="cuda")
    row = []
    for k in (0, 1, 2, 3, 4):
        prob.set_option("sweep_kernel", k)
        with torch.cuda.stream(st):
            for _ in range(3):
                prob.sweep_async(ang.data_ptr(), p, rhs.data_ptr(), 0, psi.data_ptr(), n)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            reps = 20
            for _ in range(reps):
                prob.sweep_async(ang.data_ptr(), p, rhs.data_ptr(), 0, psi.data_ptr(), n)
            e1.record(st)
        st.synchronize()
        prob.check()
        row.append(f"k{k} {e0.elapsed_time(e1) / reps:.3f} ms")
    print(f"{name} p={p}: " + "  ".join(row), flush=True)
