"""Tiny-kernel throughput with/without a concurrent H2D stream, eager vs CUDA graph."""
import time

import torch

x = torch.ones(1024, device="cuda", dtype=torch.float64)
big_h = torch.empty(128 * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
big_d = torch.empty_like(big_h, device="cuda")
side = torch.cuda.Stream()
main = torch.cuda.Stream()
N = 400
with torch.cuda.stream(main):
    for _ in range(3):
        x.mul_(1.0)
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=main):
        for _ in range(N):
            x.mul_(1.0)
torch.cuda.synchronize()


def run(kind, bg):
    torch.cuda.synchronize()
    if bg:
        with torch.cuda.stream(side):
            for _ in range(4):
                big_d.copy_(big_h, non_blocking=True)
    time.sleep(0.0003)
    with torch.cuda.stream(main):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if kind == "graph":
            g.replay()
        else:
            for _ in range(N):
                x.mul_(1.0)
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / N


for kind in ("eager", "graph"):
    for bg in (False, True, False, True):
        r = sorted(run(kind, bg) for _ in range(5))[2]
        print(f"{kind:6s} {'H2D busy' if bg else 'quiet   '} {r:6.2f} us/kernel", flush=True)
