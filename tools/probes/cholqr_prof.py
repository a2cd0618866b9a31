"""Phase clocks of cholqr_factor_k (run with BLWS_LIB_PATH=tools/probes/prof_lib/libblws_cuda.so)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_1012_0365_b200 as B  # noqa: E402

ctx = B.Context(0)
L = B.api.lib()
L.blws_debug_cholqr_prof.argtypes = [C.c_void_p]
names = {0: "start", 1: "load+trace+off", 16: "chol done", 17: "inverse done", 18: "outputs (rinv, product, rank)",
         19: "write R"}
for which, n in ((7, 100), (6, 100), (5, 100), (5, 112), (5, 32)):
    det = ctx.microbench(which, n, 0, 3, detail=True)
    us = det[0]
    print("status", det[1])
    p = np.zeros(24, dtype=np.int64)
    L.blws_debug_cholqr_prof(p.ctypes.data)
    print(f"mode {which} n={n}: {us:.1f} us (event)")
    t0 = p[0]
    prev = t0
    for k in [1] + list(range(2, 16)) + [16, 17, 18, 19]:
        if p[k] == 0 or p[k] < t0:
            continue
        nm = names.get(k, f"block {(k - 2) // 2} {'factor' if k % 2 == 0 else 'diag done'}")
        print(f"   {k:2d} {nm:32s} +{p[k] - prev:7d}  @{p[k] - t0:7d}")
        prev = p[k]
    L.blws_debug_cholqr_prof  # keep
    # clear for the next mode
