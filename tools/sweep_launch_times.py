#!/usr/bin/env python
"""Per-launch sweep durations (CUDA events between back-to-back launches) at
the bench workload, plus isolated launches after idle gaps: shows whether
back-to-back launches run slower than isolated ones (clocks / power)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2603_25233_b200 as P  # noqa: E402

grid, nt, nz = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (512, 128, 32)))
prob = P.Problem("C5", nx=grid, ny=grid, n_theta=nt, n_omega_z=nz, use_dsa=0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
prob.set_stream(s.cuda_stream)
D, n = prob.n_omega, prob.n
rhs = torch.empty(D * n, dtype=torch.float64, device="cuda")
psi = torch.empty(D * n, dtype=torch.float64, device="cuda")
ang = torch.arange(D, dtype=torch.int32, device="cuda")
prob.c5_fill(rhs.data_ptr(), D, 0, 12345)


def step():
    prob.sweep_async(ang.data_ptr(), D, rhs.data_ptr(), n, psi.data_ptr(), n)


for _ in range(3):
    step()
torch.cuda.synchronize()
K = 30
ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
ev[0].record(s)
for i in range(K):
    step()
    ev[i + 1].record(s)
torch.cuda.synchronize()
bb = [ev[i].elapsed_time(ev[i + 1]) for i in range(K)]
print("back-to-back ms:", " ".join(f"{x:.2f}" for x in bb))
iso = []
for gap in (0.001, 0.01, 0.05, 0.2, 0.5):
    time.sleep(gap)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    step()
    b.record(s)
    torch.cuda.synchronize()
    iso.append((gap, a.elapsed_time(b)))
print("isolated (gap s, ms):", " ".join(f"{g}:{x:.2f}" for g, x in iso))

# Long back-to-back run with clocks sampled alongside (nvidia-smi, 20 ms).
import subprocess  # noqa: E402
q = "timestamp,clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active,temperature.gpu,temperature.memory"
smi = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader", "-lms", "20"],
                       stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
K = 120
ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
ev[0].record(s)
for i in range(K):
    step()
    ev[i + 1].record(s)
torch.cuda.synchronize()
time.sleep(0.2)
smi.terminate()
lines = smi.communicate()[0].strip().splitlines()
bb = [ev[i].elapsed_time(ev[i + 1]) for i in range(K)]
print("long run ms (every 10th):", " ".join(f"{x:.2f}" for x in bb[::10]))
for ln in lines[::5]:
    print("  smi:", ln)
