import sys, numpy as np
sys.path.insert(0, '.')
import paper_2603_25233_b200 as P
name = sys.argv[1]
p = P.Problem(name)
r = p.solve_low_rank(build_factors=0)
np.save(sys.argv[2], np.concatenate([[r.iterations], r.history("rank"), r.phi]))
print(name, r.iterations, list(map(int, r.history("rank"))), r.get("solve_seconds", 1)[0])
