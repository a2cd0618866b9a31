"""Run the C2 partial SVT a few times (for ncu launch lists / quick timing)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1012_0365_b200 as B  # noqa: E402


def main(calls=2):
    import torch

    W, U, V, s, _ = bench.make_instance(B.Rng)
    ctx = B.Context(0)
    Wd = torch.from_numpy(np.ascontiguousarray(W.T)).cuda()
    op = B.DenseOperator(Wd, ctx=ctx, device=True, shape=(bench.M, bench.N), ld=bench.M)
    warm = B.DeviceWarmStart.from_host(U, V, s, ctx)
    ctx.set_profiling(True)
    for i in range(calls):
        ctx.region_reset()
        t = time.perf_counter()
        res = B.blws_svd(op, warm, 2, bench.R, B.Rng(1), keep_device=True)
        ctx.synchronize()
        print(f"call {i}: {1e3 * (time.perf_counter() - t):.2f} ms, launches {ctx.launches}, "
              f"achieved {int(np.sum(res.warm.sigma() > bench.threshold_for(res.warm.sigma())))}", flush=True)
        for reg, name in ((0, "K1 W products"), (1, "EVD"), (2, "thin_qr"), (5, "blws_svd")):
            st = ctx.region_stats(reg)
            print(f"   {name:14s} {st['ms']:8.3f} ms over {st['count']} calls", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
