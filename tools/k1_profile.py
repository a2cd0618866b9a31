"""One K1 paired product (W V, W^T U at b = 100 on the C2 W) between
cudaProfilerStart/Stop, for `ncu --profile-from-start off --set full`.

Gives the DRAM traffic of one K1 launch group (NN GEMM + TN GEMM + split-K
reduces) that bench.py's roofline.traffic reports (profiles/r01_k1.md).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1012_0365_b200 as B  # noqa: E402


def main(b=100):
    import torch

    W, U, V, s, eps = bench.make_instance(B.Rng)
    ctx = B.Context(0)
    Wd = torch.from_numpy(np.ascontiguousarray(W.T)).cuda()
    op = B.DenseOperator(Wd, ctx=ctx, device=True, shape=(bench.M, bench.N), ld=bench.M)
    left, right = U[:, :b].copy(order="F"), V[:, :b].copy(order="F")
    top, bot = op.apply_pair_block(left, right)  # warm (plans, pool)
    ctx.synchronize()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    top2, bot2 = op.apply_pair_block(left, right)
    ctx.synchronize()
    torch.cuda.profiler.stop()
    err = max(np.abs(top2 - W @ right).max(), np.abs(bot2 - W.T @ left).max())
    print(f"K1 b={b}: max err vs numpy {err:.3e}", flush=True)


if __name__ == "__main__":
    main()
