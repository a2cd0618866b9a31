"""Do the C2 kernels slow down while a large H2D copy runs on another stream?"""
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_1012_0365_b200 as B  # noqa: E402


def main(steps=10):
    import torch

    W, U, V, s, eps = bench.make_instance(B.Rng)
    ctx = B.Context(0)
    Wd = torch.from_numpy(np.ascontiguousarray(W.T)).cuda()
    op = B.DenseOperator(Wd, ctx=ctx, device=True, shape=(bench.M, bench.N), ld=bench.M)
    warm = B.DeviceWarmStart.from_host(U, V, s, ctx)
    big_h = torch.empty(128 * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
    big_d = torch.empty_like(big_h, device="cuda")
    small_h = torch.empty(8 * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
    small_d = torch.empty_like(small_h, device="cuda")
    side = torch.cuda.Stream()
    for label, bg in (("quiet", False), ("H2D 128MB target", True), ("H2D 8MB target", "small"), ("quiet", False)):
        for _ in range(2):
            B.blws_svd(op, warm, 2, bench.R, B.Rng(7), keep_device=True)
        ctx.synchronize()
        ctx.set_profiling(True)
        ctx.region_reset()
        times = []
        for _ in range(steps):
            if bg:
                with torch.cuda.stream(side):
                    if bg == "small":
                        for _ in range(48):
                            small_d.copy_(small_h, non_blocking=True)
                    else:
                        for _ in range(3):
                            big_d.copy_(big_h, non_blocking=True)
            t = time.perf_counter()
            B.blws_svd(op, warm, 2, bench.R, B.Rng(7), keep_device=True)
            ctx.synchronize()
            times.append(time.perf_counter() - t)
            torch.cuda.synchronize()
        st = [ctx.region_stats(i) for i in range(3)]
        ctx.set_profiling(False)
        # the same with the captured graph (profiling off)
        gt = []
        for _ in range(steps):
            if bg:
                with torch.cuda.stream(side):
                    for _ in range(3):
                        big_d.copy_(big_h, non_blocking=True)
            t = time.perf_counter()
            B.blws_svd(op, warm, 2, bench.R, B.Rng(7), keep_device=True)
            ctx.synchronize()
            gt.append(time.perf_counter() - t)
            torch.cuda.synchronize()
        print(f"{label:18s} graph svd {1e3 * np.median(gt):6.2f} ms", flush=True)
        print(f"{label:18s} svd {1e3 * np.median(times):6.2f} ms  K1 {st[0]['ms'] / steps:6.3f}  "
              f"EVD {st[1]['ms'] / steps:6.3f}  thin_qr {st[2]['ms'] / steps:6.3f} ms/call", flush=True)


if __name__ == "__main__":
    main()
