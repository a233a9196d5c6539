"""A/B check of a device-path switch on the C2 low-rank solve: runs it with
ENV=1 and ENV=0 in fresh processes and reports time-to-tol and whether phi is
bitwise equal.  Usage: python tools/cgs_ab.py [ENV] (default RTLR_CGS_COOP)."""
import os, sys, subprocess
import numpy as np
sys.path.insert(0, '.')
VAR = sys.argv[1] if len(sys.argv) > 1 else "RTLR_CGS_COOP"
code = r'''
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2603_25233_b200 as P
p = P.Problem("C2")
r = p.solve_low_rank(build_factors=1)
np.save(sys.argv[1], np.concatenate([r.phi, r.get("S", 0) if False else []]))
print(r.get("solve_seconds", 1)[0], r.iterations)
'''
for v in ["1", "0"]:
    env = dict(os.environ, **{VAR: v})
    out = subprocess.run([sys.executable, "-c", code, f"/tmp/phi_{v}.npy"], env=env, capture_output=True, text=True)
    print(VAR, v, out.stdout.strip(), out.stderr[-300:])
a, b = np.load("/tmp/phi_1.npy"), np.load("/tmp/phi_0.npy")
print("bitwise equal:", np.array_equal(a, b), "max diff", np.max(np.abs(a - b)))
