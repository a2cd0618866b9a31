"""sym_evd_top microbenchmark at the BLWS orders (T of order 2b)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1012_0365_b200 as B  # noqa: E402
ctx = B.Context(0)
for n in (60, 110, 200, 222, 260, 820):
    print(f"sym_evd_top n={n} want={n//2}: {ctx.microbench(1, n, 0, 10):8.1f} us", flush=True)
