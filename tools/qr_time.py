#!/usr/bin/env python
"""Times the blocked Householder QR (basis rebuild) at C3/C4 sizes through
rtlr_cu_dense_qr (host buffers; the transfers are inside the time)."""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2603_25233_b200 as P  # noqa: E402

sizes = [(262144, 400), (1048576, 600)] if len(sys.argv) < 3 else [(int(sys.argv[1]), int(sys.argv[2]))]
for m, n in sizes:
    a = np.asfortranarray(np.random.default_rng(0).standard_normal((m, n)))
    P.dense_qr(a[:4096, :64].copy(order="F"))
    t = time.time()
    q, r = P.dense_qr(a)
    dt = time.time() - t
    print(m, n, f"{dt:.3f} s incl. transfers", np.linalg.norm(q[:, :5].T @ q[:, :5] - np.eye(5)))
