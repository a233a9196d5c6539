"""Same-process-free A/B of one environment switch on a low-rank solve:
python tools/env_ab.py CONFIG VAR v1 v2 ... [--rounds R].  Each value runs in a
fresh process, values interleaved over R rounds; prints time-to-tol per run,
the per-value minimum, and whether phi is bitwise equal across values."""
import os, sys, subprocess
import numpy as np

args = sys.argv[1:]
rounds = 2
if "--rounds" in args:
    i = args.index("--rounds")
    rounds = int(args[i + 1])
    del args[i:i + 2]
cfg, var, vals = args[0], args[1], args[2:]
code = r'''
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2603_25233_b200 as P
p = P.Problem(sys.argv[2])
r = p.solve_low_rank(build_factors=0)
np.save(sys.argv[1], r.phi)
print(r.get("solve_seconds", 1)[0], r.iterations)
'''
times = {v: [] for v in vals}
for k in range(rounds):
    for v in (vals if k % 2 == 0 else vals[::-1]):
        env = dict(os.environ, **{var: v})
        out = subprocess.run([sys.executable, "-c", code, f"/tmp/phi_ab_{v}.npy", cfg], env=env,
                             capture_output=True, text=True)
        print(var, v, out.stdout.strip(), out.stderr[-300:], flush=True)
        times[v].append(float(out.stdout.split()[0]))
base = np.load(f"/tmp/phi_ab_{vals[0]}.npy")
for v in vals:
    print(f"{var}={v}: min {min(times[v]):.3f} s  runs {times[v]}  bitwise-equal-to-{vals[0]}:",
          np.array_equal(base, np.load(f"/tmp/phi_ab_{v}.npy")))
