"""Does a small D2H (or H2D) on stream B wait for a large H2D on stream A?"""
import time

import torch

dev = torch.device("cuda:0")
big_h = torch.empty(128 * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
big_d = torch.empty_like(big_h, device=dev)
small_d = torch.ones(16, dtype=torch.float64, device=dev)
small_h = torch.empty(16, dtype=torch.float64).pin_memory()
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
for kind in ("d2h", "h2d", "kernel"):
    for trial in range(3):
        torch.cuda.synchronize()
        with torch.cuda.stream(sa):
            big_d.copy_(big_h, non_blocking=True)
        time.sleep(0.0002)
        t = time.perf_counter()
        with torch.cuda.stream(sb):
            if kind == "d2h":
                small_h.copy_(small_d, non_blocking=True)
            elif kind == "h2d":
                small_d.copy_(small_h, non_blocking=True)
            else:
                small_d.mul_(1.0)
        sb.synchronize()
        lat = time.perf_counter() - t
        sa.synchronize()
        tot = time.perf_counter() - t
        print(f"{kind:6s} small op latency {1e3 * lat:7.3f} ms (big copy finished after {1e3 * tot:6.3f} ms)", flush=True)
