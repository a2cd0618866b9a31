import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1012_0365_b200 as B  # noqa: E402
ctx = B.Context(0)
for n in (112, 200, 300, 400, 411):
    d = ctx.microbench(0, n, 0, 5, detail=True)
    print(f"chol_inv n={n}: {d[0]:8.1f} us", flush=True)
for rows, b in ((80000, 400), (40000, 400), (8000, 400), (4000, 200)):
    print(f"thin_qr {rows}x{b}: {ctx.microbench(2, rows, b, 3):8.1f} us", flush=True)
    print(f"gram TN {rows}x{b}: {ctx.microbench(4, rows, b, 3):8.1f} us", flush=True)
