import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_0365_b200 as B
ctx = B.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
print(ctx.microbench(0, n, 0, 3, detail=True))
