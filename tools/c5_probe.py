"""C5-scale building blocks on one GPU: EVD of order 2b, CholQR at b, one
blws_svd on a 40000^2 W synthesised on the device (timing only)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_0365_b200 as B  # noqa: E402


def timed(f, reps=3):
    f()
    t = time.perf_counter()
    for _ in range(reps):
        f()
    return (time.perf_counter() - t) / reps


def main(m=40000, r=400, seed=0, evd=True):
    import torch

    torch.manual_seed(seed)
    ctx = B.Context(0)
    rs = np.random.default_rng(0)
    for n in ((200, 410, 810) if evd else ()):
        g = rs.standard_normal((n, n))
        t = 0.5 * (g + g.T)
        dt = timed(lambda: B.sym_evd_small(t))
        print(f"sym_evd_small n={n}: {1e3 * dt:.2f} ms (host round trip incl.)", flush=True)
    dev = torch.device("cuda:0")
    # W = U0 diag(s) V0^T + 1e-3 N on the device (column-major = row-major W^T)
    k = 2 * r
    u0 = torch.linalg.qr(torch.randn(m, k, dtype=torch.float64, device=dev))[0]
    v0 = torch.linalg.qr(torch.randn(m, k, dtype=torch.float64, device=dev))[0]
    s = 100.0 * 0.995 ** torch.arange(k, dtype=torch.float64, device=dev)
    wt = (v0 * s) @ u0.T  # = W^T (row-major) = W column-major
    wt += 1e-3 * torch.randn(m, m, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    print(f"W ready: {wt.numel() * 8 / 1e9:.1f} GB", flush=True)
    op = B.DenseOperator(wt, ctx=ctx, device=True, shape=(m, m), ld=m)
    uw = torch.linalg.qr(u0[:, :r] + 1e-2 * torch.randn(m, r, dtype=torch.float64, device=dev))[0]
    vw = torch.linalg.qr(v0[:, :r] + 1e-2 * torch.randn(m, r, dtype=torch.float64, device=dev))[0]
    warm = B.DeviceWarmStart.from_host(uw.cpu().numpy(), vw.cpu().numpy(), s[:r].cpu().numpy(), ctx)
    ctx.set_profiling(True)
    for i in range(4):
        ctx.region_reset()
        t = time.perf_counter()
        res = B.blws_svd(op, warm, 2, r, B.Rng(1), keep_device=True)
        ctx.synchronize()
        dt = time.perf_counter() - t
        st = [ctx.region_stats(j) for j in range(3)]
        print(f"blws_svd m={m} r={r}: {1e3 * dt:.1f} ms; K1 {st[0]['ms']:.1f} ms ({st[0]['flops'] / st[0]['ms'] / 1e9:.1f} "
              f"TF/s), EVD {st[1]['ms']:.1f} ms, thin_qr {st[2]['ms']:.1f} ms / {st[2]['count']}", flush=True)
    sig = res.warm.sigma()
    print("sigma[:3]", sig[:3], "fallbacks", B.deferred_fallbacks(), "graphs", B.graph_launches(), flush=True)


if __name__ == "__main__":
    evd = os.environ.get("C5_EVD", "0") == "1"
    for sd in [int(x) for x in (sys.argv[1:] or ["0"])]:
        print("seed", sd, flush=True)
        main(seed=sd, evd=evd)
