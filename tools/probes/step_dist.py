"""Per-step time distribution of the C2 call (CUDA events on the library stream)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_1012_0365_b200 as B  # noqa: E402


def main(steps=40):
    import torch

    W, U, V, s, eps = bench.make_instance(B.Rng)
    ctx = B.Context(0)
    dev = torch.device("cuda:0")
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    Wd = torch.from_numpy(np.ascontiguousarray(W.T)).to(dev)
    op = B.DenseOperator(Wd, ctx=ctx, device=True, shape=(bench.M, bench.N), ld=bench.M)
    warm = B.DeviceWarmStart.from_host(U, V, s, ctx)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for label in ("graph", "graph-noflush"):
        for _ in range(4):
            B.blws_svd(op, warm, 2, bench.R, B.Rng(7), keep_device=True)
        ctx.synchronize()
        ts = []
        for _ in range(steps):
            with torch.cuda.stream(stream):
                if label == "graph":
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            B.blws_svd(op, warm, 2, bench.R, B.Rng(7), keep_device=True)
            with torch.cuda.stream(stream):
                e1.record(stream)
            ts.append((e0, e1))
        ctx.synchronize()
        torch.cuda.synchronize()
        ms = np.array([a.elapsed_time(b) for a, b in ts])
        print(f"{label:14s} min {ms.min():.3f} p10 {np.percentile(ms, 10):.3f} med {np.median(ms):.3f} "
              f"p90 {np.percentile(ms, 90):.3f} max {ms.max():.3f} mean {ms.mean():.3f}", flush=True)
        print("   ", " ".join(f"{x:.2f}" for x in ms[:40]), flush=True)


if __name__ == "__main__":
    main()
