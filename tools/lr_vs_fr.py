"""|phi_LR - phi_FR| of the GPU solvers on the BASELINE configs (the reference's
LR-vs-FR bar is 1e-6 absolute, proj/tests/test_low_rank.cpp:472-498)."""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2603_25233_b200 as P
for name in ("C2", "C3", "C4"):
    p = P.Problem(name)
    fr = p.solve_full_rank(store_psi=0)
    lr = p.solve_low_rank(build_factors=0)
    d = np.linalg.norm(lr.phi - fr.phi)
    print(name, "FR it", fr.iterations, "LR it", lr.iterations, "|phi_LR - phi_FR|_2 =", d, "rel", d / np.linalg.norm(fr.phi), "|phi|", np.linalg.norm(fr.phi))
