"""One direction-group sweep at C4 (1024 unique directions, shared rhs,
psi written) for ncu: python tools/het_profile.py [config] [kernel]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_25233_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
kern = int(sys.argv[2]) if len(sys.argv) > 2 else 5
g = P.Problem(name, use_dsa=0)
g.set_option("sweep_kernel", kern)
nz = g.n_omega_z
reps = np.array([j1 * nz + j2 for j1 in range(g.n_theta) for j2 in range(nz // 2)], dtype=np.int32)
n = g.n
rhs = torch.rand(n, dtype=torch.float64, device="cuda")
psi = torch.empty(len(reps) * n, dtype=torch.float64, device="cuda")
mode = sys.argv[3] if len(sys.argv) > 3 else "psi"
for _ in range(3):
    if mode == "psi":
        g.sweep_device(reps.ctypes.data, len(reps), rhs.data_ptr(), 0, psi.data_ptr(), n)
    else:  # si_step: the scalar flux in the sweep epilogue, no psi
        g.si_step(np.linspace(0.0, 1.0, n))
torch.cuda.synchronize()
print("ok")
