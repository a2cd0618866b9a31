"""Gram X^T X: split-K GEMM + reduce (mode 8) against the cluster gram16 (mode
10, BLWS_GRAM_CL picks the cluster size), event-timed eager launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_0365_b200 as B  # noqa: E402

ctx = B.Context(0)
print("BLWS_GRAM_V", os.environ.get("BLWS_GRAM_V", "0"))
for rows, b in ((4000, 100), (4000, 50), (8000, 100), (2000, 111), (10000, 50), (40000, 100), (1000, 30), (500, 25)):
    g = ctx.microbench(8, rows, b, 30)
    d = ctx.microbench(10, rows, b, 30, detail=True)
    print(f"{rows:6d} x {b:3d}: gemm {g:7.1f} us   gram16 {d[0]:7.1f} us   rel diff {d[1]:.2e}", flush=True)
