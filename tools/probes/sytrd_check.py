import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1012_0365_b200 as B
rs = np.random.default_rng(1)
for n in (64, 65, 100, 200):
    g = rs.standard_normal((n, n)); t = 0.5 * (g + g.T)
    vals, vecs = B.sym_evd_small(t)
    ref = np.linalg.eigvalsh(t)[::-1]
    print(os.environ.get("BLWS_SYTRD", "cluster"), n, "max eig err", np.abs(vals - ref).max(), flush=True)
