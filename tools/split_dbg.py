import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np
import paper_2603_25233_b200 as P
g = P.Problem("homogeneous(1,1)", use_dsa=0, nx=1000, ny=24, n_theta=8, n_omega_z=2)
g.set_option("sweep_kernel", 2)
rhs = np.random.default_rng(1).standard_normal((g.n, g.n_omega))
psi = g.sweep(np.arange(g.n_omega), rhs)
print("ok", np.abs(psi).max())
