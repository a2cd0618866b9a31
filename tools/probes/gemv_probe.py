"""Paired GEMV (Lanczos step, K10) at C5 scale: time per W x, W^T y pair vs the
HBM roofline of one (fused) or two reads of W."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1012_0365_b200 as B  # noqa: E402


def main(m=40000):
    import torch

    torch.manual_seed(0)
    ctx = B.Context(0)
    wt = torch.randn(m, m, dtype=torch.float64, device="cuda")
    op = B.DenseOperator(wt, ctx=ctx, device=True, shape=(m, m), ld=m)
    B.spectral_norm(op)  # warm
    for tol in (1e-6, 1e-10):
        c0 = op.application_count()
        ctx.synchronize()
        t = time.perf_counter()
        B.spectral_norm(op, tol=tol)
        ctx.synchronize()
        dt = time.perf_counter() - t
        steps = op.application_count() - c0
        print(f"spectral_norm tol={tol}: {steps} pair applies in {1e3 * dt:.1f} ms -> {1e3 * dt / steps:.3f} ms/step; "
              f"one W read = {m * m * 8 / 6.55e12 * 1e3:.3f} ms at 6.55 TB/s", flush=True)


if __name__ == "__main__":
    main()
