"""One C5-size cold Lanczos reseed (m = n = 40000, r = 400) on a device-resident
operator: steps, time, us/step. Under ncu with --launch-skip it samples the
per-step kernels at mid basis sizes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1012_0365_b200 as B  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
r = int(sys.argv[2]) if len(sys.argv) > 2 else 400
g = torch.Generator(device="cuda:0").manual_seed(0)
dev = torch.device("cuda:0")
lw = torch.randn(m, r + 20, device=dev, dtype=torch.float64, generator=g)
rw = torch.randn(r + 20, m, device=dev, dtype=torch.float64, generator=g)
w = lw @ rw  # column-major view = transpose of this row-major tensor; any W will do
w += 1e-3 * torch.randn(m, m, device=dev, dtype=torch.float64, generator=g)
del lw, rw
torch.cuda.synchronize()
op = B.DenseOperator(w, device=True, shape=(m, m), ld=m)
c0 = op.application_count()
t = time.perf_counter()
_, s, _, st = B.lanczos_partial_svd(op, r, tol=1e-8)
op.ctx.synchronize()
dt = time.perf_counter() - t
steps = op.application_count() - c0
print(f"m={m} r={r}: {steps} steps {dt:.2f} s = {1e3 * dt / steps:.3f} ms/step", flush=True)
