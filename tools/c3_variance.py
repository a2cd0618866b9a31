import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1012_0365_b200 as B
from paper_1012_0365_b200 import synth
ctx = B.Context(0)
d, a0, _, _ = synth.rpca_lowrank_sparse(2000, 100, 400000, 1, B.Rng, B.sample_distinct)
bseed = 1 ^ 0x5BDBEEF
out = []
for rep in range(5):
    ctx.set_profiling(True); ctx.region_reset()
    t = time.perf_counter()
    _, _, st, _ = B.rpca_adm(d, B.SvdBackend.blws(seed=bseed, ctx=ctx), truth=a0, want_outputs=False)
    dt = time.perf_counter() - t
    regs = {n: round(ctx.region_stats(i)["ms"], 1) for i, n in ((3, "reseed"), (5, "blws_svd"), (6, "svt"), (8, "setup"), (9, "epilogue"))}
    ctx.set_profiling(False)
    out.append(dict(rep=rep, solve_s=round(dt, 4), iterations=st.iterations, **regs))
    print(json.dumps(out[-1]), flush=True)
