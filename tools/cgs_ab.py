import os, sys, subprocess, json
import numpy as np
sys.path.insert(0, '.')
code = r'''
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2603_25233_b200 as P
p = P.Problem("C2")
r = p.solve_low_rank()
np.save(sys.argv[1], r.phi)
print(r.get("solve_seconds", 1)[0], r.iterations)
'''
for v in ["1", "0"]:
    env = dict(os.environ, RTLR_CGS_COOP=v)
    out = subprocess.run([sys.executable, "-c", code, f"/tmp/phi_{v}.npy"], env=env, capture_output=True, text=True)
    print("coop", v, out.stdout.strip(), out.stderr[-300:])
a, b = np.load("/tmp/phi_1.npy"), np.load("/tmp/phi_0.npy")
print("bitwise equal:", np.array_equal(a, b), "max diff", np.max(np.abs(a - b)))
