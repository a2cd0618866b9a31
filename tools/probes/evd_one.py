"""One sym_evd_top call (n from argv) for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1012_0365_b200 as B  # noqa: E402
ctx = B.Context(0)
print(ctx.microbench(1, int(sys.argv[1]) if len(sys.argv) > 1 else 200, 0, 2))
