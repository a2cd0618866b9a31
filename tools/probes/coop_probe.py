"""One m = 2000 cold Lanczos reseed (r = 100) for profiling the cooperative kernel."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1012_0365_b200 as B  # noqa: E402

rs = np.random.default_rng(0)
m = 2000
w = rs.standard_normal((m, 200)) @ rs.standard_normal((200, m)) + 1e-3 * rs.standard_normal((m, m))
op = B.DenseOperator(np.asfortranarray(w))
for _ in range(2):
    c0 = op.application_count()
    t = time.perf_counter()
    _, s, _, st = B.lanczos_partial_svd(op, 100, tol=1e-8)
    op.ctx.synchronize()
    dt = time.perf_counter() - t
    steps = op.application_count() - c0
    print(f"{steps} steps {1e3 * dt:.1f} ms = {1e6 * dt / steps:.1f} us/step", flush=True)
