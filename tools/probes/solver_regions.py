"""Where an RPCA solve spends its time: region timers (K1, EVD, thin_qr, Lanczos
reseed, Ritz checkpoints, whole blws_svd calls) over one solve."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1012_0365_b200 as B  # noqa: E402
from paper_1012_0365_b200 import synth  # noqa: E402


def main(m=2000, rank=100, frac=0.10, mc=False):
    ctx = B.Context(0)
    if mc:  # C4-style MC: m x m, frac * m^2 observed, tol 1e-6
        colptr, rowidx, vals, ml, mr = synth.mc_lowrank(m, rank, int(round(frac * m * m)), 1, B.Rng,
                                                       B.sample_distinct)

        def solve():
            u, s_, v, st = B.mc_svt(m, m, colptr, rowidx, vals, B.SvdBackend.blws(seed=1 ^ 0x5BDBEEF, ctx=ctx),
                                    tol_outer=1e-6, truth_ml=ml, truth_mr=mr, cap=512)
            return u, s_, st, v

        t = time.perf_counter()
        solve()
        print(f"MC m={m}: profiling off: {time.perf_counter() - t:.3f} s", flush=True)
    elif m > 8000:  # C5-size: D formed on the device (solve_configs.rpca_device), one profiled solve
        import torch

        dt, a0t, _, _ = synth.rpca_lowrank_sparse_device(m, rank, int(round(frac * m * m)), 1, B.Rng,
                                                         B.sample_distinct, torch.device("cuda:0"))
        B.rpca_adm(np.ascontiguousarray(dt[:64, :64].cpu().numpy().T), B.SvdBackend.blws(seed=1 ^ 0x5BDBEEF, ctx=ctx))

        def solve():
            return B.rpca_adm(dt, B.SvdBackend.blws(seed=1 ^ 0x5BDBEEF, ctx=ctx), truth=a0t, device=True, m=m, ld=m)
    else:
        d, a0, _, _ = synth.rpca_lowrank_sparse(m, rank, int(round(frac * m * m)), 1, B.Rng, B.sample_distinct)
        B.rpca_adm(d[:64, :64].copy(order="F"), B.SvdBackend.blws(seed=1 ^ 0x5BDBEEF, ctx=ctx))

        def solve():
            return B.rpca_adm(d, B.SvdBackend.blws(seed=1 ^ 0x5BDBEEF, ctx=ctx), truth=a0, want_outputs=False)

        t = time.perf_counter()
        solve()
        print(f"m={m}: profiling off: {time.perf_counter() - t:.3f} s", flush=True)
    ctx.set_profiling(True)
    ctx.region_reset()
    t = time.perf_counter()
    _, _, st, _ = solve()
    tot = time.perf_counter() - t
    print(f"m={m}: {tot:.3f} s, {st.iterations} iterations, {st.matvec_count} matvecs", flush=True)
    names = {0: "K1 paired products", 1: "EVD of T", 2: "thin_qr", 3: "Lanczos reseed (whole)", 4: "Ritz checkpoints",
             5: "blws_svd (whole)", 6: "svt (whole)", 7: "MC loop outside svt",
             8: "solver set-up", 9: "solver epilogue"}
    for i, nm in names.items():
        r = ctx.region_stats(i)
        print(f"  {nm:26s} {r['ms']:9.1f} ms over {r['count']:5d}", flush=True)


if __name__ == "__main__":
    mc = "--mc" in sys.argv
    args = [a for a in sys.argv[1:] if a != "--mc"]
    main(*(int(x) if i < 2 else float(x) for i, x in enumerate(args)), mc=mc)
