"""Time sym_evd_top (all n pairs) on random symmetric T at the orders BLWS
produces (C2 ~200, C3 ~202-230, C5 ~810) through the library's region timer."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1012_0365_b200 as B  # noqa: E402

ctx = B.Context(0)
for n in [int(x) for x in (sys.argv[1:] or ["200", "222", "230", "260", "420", "810"])]:
    g = np.random.default_rng(n).standard_normal((n, n))
    t = 0.5 * (g + g.T)
    for _ in range(2):
        B.api.sym_evd_small(t, ctx=ctx)
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        B.api.sym_evd_small(t, ctx=ctx)
    print(f"n={n}: {1e3 * (time.perf_counter() - t0) / reps:.2f} ms per full sym_evd_small (incl. H2D/D2H)", flush=True)
