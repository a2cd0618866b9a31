import os, sys
sys.path.insert(0, "/root/repo")
import paper_1012_0365_b200 as B
ctx = B.Context(0)
for rows, b in ((40000, 100), (4000, 100), (8000, 100), (10000, 50)):
    worst = 0.0
    bad = 0
    for it in range(15):
        d = ctx.microbench(10, rows, b, 3, detail=True)
        worst = max(worst, d[1]); bad += d[1] > 1e-12
    print(rows, b, "worst", worst, "bad", bad, flush=True)
