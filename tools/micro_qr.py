"""Microbenchmarks of the CholQR pieces (event-timed, eager, warm)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_0365_b200 as B  # noqa: E402

ctx = B.Context(0)
for n in (32, 64, 100, 112):
    d0 = ctx.microbench(0, n, 0, 20)
    d5, d6, d7 = (ctx.microbench(w, n, 0, 20) for w in (5, 6, 7))
    print(f"n={n}: chol_inv {d0:7.1f} us | cholqr full {d5:7.1f}  near-id {d6:7.1f}  skip {d7:7.1f} us", flush=True)
for rows, b in ((8000, 100), (4000, 100), (2000, 111), (1000, 30)):
    print(f"{rows}x{b}: gram {ctx.microbench(8, rows, b, 20):7.1f} us  apply {ctx.microbench(9, rows, b, 20):7.1f} us"
          f"  thin_qr {ctx.microbench(2, rows, b, 10):7.1f} us", flush=True)
