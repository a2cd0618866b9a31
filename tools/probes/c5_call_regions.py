"""Region breakdown of one C5-scale standalone blws_svd call (bench.py --mode
sharded's call at N = 1): K1, the EVD of T, thin_qr, whole call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1012_0365_b200 as B  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
r = int(sys.argv[2]) if len(sys.argv) > 2 else 400
dev = torch.device("cuda:0")
Wt, Uw, Vw, sigma, U0, V0 = bench.c5_inputs(m, r, 0, m, dev)
ctx = B.Context(0)
op = B.DenseOperator(Wt, ctx=ctx, device=True, shape=(m, m), ld=m)
warm = B.DeviceWarmStart.from_host(np.asfortranarray(Uw.cpu().numpy()), np.asfortranarray(Vw.cpu().numpy()),
                                   sigma[:r].cpu().numpy(), ctx)
for _ in range(2):
    B.blws_svd(op, warm, 2, r, B.Rng(1), keep_device=True)
ctx.synchronize()
ctx.set_profiling(True)
ctx.region_reset()
for _ in range(2):
    B.blws_svd(op, warm, 2, r, B.Rng(1), keep_device=True)
ctx.synchronize()
names = {0: "K1 paired products", 1: "EVD of T", 2: "thin_qr", 5: "blws_svd (whole)"}
for i, nm in names.items():
    st = ctx.region_stats(i)
    print(f"  {nm:22s} {st['ms'] / 2:9.2f} ms per call over {st['count'] // 2} per call", flush=True)
