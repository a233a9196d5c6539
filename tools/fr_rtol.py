import numpy as np, sys, time
sys.path.insert(0, '.')
import paper_2603_25233_b200 as P
g = np.load('tests/golden/C4_full.npz')
p = P.Problem("C4")
for rt in (1e-13, 1e-14, 1e-15, 3e-16):
    p.set_option("pcg_rtol", rt)
    r = p.solve_full_rank(store_psi=0)
    err = np.linalg.norm(r.phi - g["phi"]) / np.linalg.norm(g["phi"])
    print(rt, r.iterations, "%.3e" % err, [int(x) for x in r.history("dsa_iterations")], "%.4f" % r.get("solve_seconds", 1)[0], flush=True)
