"""One cholqr_factor launch per mode (for ncu): argv[1] in {5 full, 6 near-id, 7 skip}, n = argv[2]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_0365_b200 as B  # noqa: E402

ctx = B.Context(0)
which, n = int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 100
print(which, n, ctx.microbench(which, n, 0, 1))
