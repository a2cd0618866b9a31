"""Break down the e2e step (bench.py e2e leg): where the time beyond the
device step goes with the async double-buffered W upload."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1012_0365_b200 as B  # noqa: E402


def pinned_f(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a.T)).pin_memory()


def main(steps=10):
    import torch

    W, U, V, s, eps = bench.make_instance(B.Rng)
    M, N, R = bench.M, bench.N, bench.R
    ctx = B.Context(0)
    Wh = pinned_f(W)
    Ut, Vt = pinned_f(U), pinned_f(V)
    Up, Vp = Ut.numpy().T, Vt.numpy().T  # F-ordered views of pinned memory
    ops = [B.DenseOperator(W, ctx=ctx), B.DenseOperator(W, ctx=ctx)]
    out_h = B.WarmStart(torch.empty((R, M), dtype=torch.float64).pin_memory().numpy().T,
                        torch.empty((R, N), dtype=torch.float64).pin_memory().numpy().T,
                        torch.empty(R, dtype=torch.float64).pin_memory().numpy())

    def run(label, async_w, pinned_warm, overlap=True):
        ctx.synchronize()
        t0 = time.perf_counter()
        tw = tc = td = 0.0
        if async_w:
            ops[0].assign_async(Wh.data_ptr(), M)
        for i in range(steps):
            if not async_w:
                ops[0].assign_ptr(Wh.data_ptr(), M, B.api.HOST)
            a = time.perf_counter()
            w_in = B.DeviceWarmStart.from_host(Up if pinned_warm else U, Vp if pinned_warm else V, s, ctx)
            # same-direction copies share the DMA queue: the next W goes behind this step's warm start
            if async_w and overlap and i + 1 < steps:
                ops[(i + 1) % 2].assign_async(Wh.data_ptr(), M)
            b = time.perf_counter()
            r = B.blws_svd(ops[i % 2] if async_w else ops[0], w_in, 2, R, B.Rng(7), keep_device=True)
            c = time.perf_counter()
            out = r.warm.to_host(M, N, out=out_h if pinned_warm else None)
            d = time.perf_counter()
            tw += b - a
            tc += c - b
            td += d - c
            if async_w and not overlap and i + 1 < steps:
                ops[(i + 1) % 2].assign_async(Wh.data_ptr(), M)
        ctx.synchronize()
        tot = time.perf_counter() - t0
        print(f"{label:40s} {1e3 * tot / steps:7.2f} ms/step  warm-up {1e3 * tw / steps:6.2f}  "
              f"svd {1e3 * tc / steps:6.2f}  download {1e3 * td / steps:6.2f}", flush=True)

    for _ in range(2):
        run("sync assign, pageable warm", False, False)
        run("async assign overlapped, pageable warm", True, False)
        run("async assign overlapped, pinned warm", True, True)
        run("async assign not overlapped, pinned warm", True, True, overlap=False)
    # device-only reference
    Wd = torch.from_numpy(np.ascontiguousarray(W.T)).cuda()
    op = B.DenseOperator(Wd, ctx=ctx, device=True, shape=(M, N), ld=M)
    warm = B.DeviceWarmStart.from_host(U, V, s, ctx)
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        B.blws_svd(op, warm, 2, R, B.Rng(7), keep_device=True)
    ctx.synchronize()
    print(f"{'device-resident':40s} {1e3 * (time.perf_counter() - t0) / steps:7.2f} ms/step", flush=True)


if __name__ == "__main__":
    main()
