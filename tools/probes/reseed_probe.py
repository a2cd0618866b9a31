"""One C5-scale cold Lanczos reseed (r = 400): steps, time, time per step vs the
2.2 ms pass over W (the rest is CGS2 reorthogonalisation + checkpoints)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1012_0365_b200 as B  # noqa: E402


def main(m=40000, r=400):
    import torch

    torch.manual_seed(0)
    ctx = B.Context(0)
    k = 2 * r
    u0 = torch.linalg.qr(torch.randn(m, k, dtype=torch.float64, device="cuda"))[0]
    v0 = torch.linalg.qr(torch.randn(m, k, dtype=torch.float64, device="cuda"))[0]
    s = 100.0 * 0.995 ** torch.arange(k, dtype=torch.float64, device="cuda")
    wt = (v0 * s) @ u0.T + 1e-3 * torch.randn(m, m, dtype=torch.float64, device="cuda")
    del u0, v0
    op = B.DenseOperator(wt, ctx=ctx, device=True, shape=(m, m), ld=m)
    for rr, tol in ((40, 1e-8), (r, 1e-8)):
        c0 = op.application_count()
        ctx.synchronize()
        t = time.perf_counter()
        _, sig, _, stats = B.lanczos_partial_svd(op, rr, tol=tol)
        ctx.synchronize()
        dt = time.perf_counter() - t
        steps = op.application_count() - c0
        print(f"reseed r={rr}: {steps} steps in {dt:.2f} s = {1e3 * dt / steps:.2f} ms/step; stats {list(stats)}",
              flush=True)


if __name__ == "__main__":
    main()
