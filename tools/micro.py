"""Microbenchmarks of the small hot-path kernels (event-timed, warm)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_0365_b200 as B  # noqa: E402

ctx = B.Context(0)
ctx.fp64_peak(0)
for n in (32, 64, 100, 111, 200):
    d = ctx.microbench(0, n, 0, 20, detail=True)
    print(f"chol_inv n={n}: {d[0]:8.1f} us   diag {d[1]:.0f} chol {d[2]:.0f} inv {d[3]:.0f} "
          f"panel {int(d[4] // 1e6)} syrk {d[4] % 1e6:.0f}", flush=True)
for n in (60, 110, 200, 222):
    print(f"sym_evd_top n={n} (want n/2): {ctx.microbench(1, n, 0, 5):8.1f} us", flush=True)
for rows, b in ((8000, 100), (4000, 100), (1000, 30)):
    print(f"thin_qr {rows}x{b}: {ctx.microbench(2, rows, b, 10):8.1f} us", flush=True)
for n, b in ((4000, 100), (4000, 104), (4000, 128), (2000, 105)):
    us = ctx.microbench(3, n, b, 10)
    print(f"gemm NN {n}x{n}*{n}x{b}: {us:8.1f} us  {2*n*n*b/us/1e6:6.2f} TF/s", flush=True)
for n, b in ((8000, 100), (4000, 100)):
    us = ctx.microbench(4, n, b, 10)
    print(f"gemm TN gram {n}x{b}: {us:8.1f} us  {2*n*b*b/us/1e6:6.2f} TF/s", flush=True)
