"""The --mode sharded instance at a small order: device blws_svd vs the CPU oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1012_0365_b200 as B  # noqa: E402
from oracle import oracle as O  # noqa: E402

m, r = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda:0")
Wt, Uw, Vw, sigma, _, _ = bench.c5_inputs(m, r, 0, m, dev)
W = np.asfortranarray(Wt.cpu().numpy().T)
U, V, s = np.asfortranarray(Uw.cpu().numpy()), np.asfortranarray(Vw.cpu().numpy()), sigma[:r].cpu().numpy()
g = B.blws_svd(B.DenseOperator(W), B.WarmStart(U, V, s), 2, r, B.Rng(1 ^ 0x5BDBEEF))
O.set_threads(os.cpu_count() or 1)
o = O.blws_svd(O.DenseOperator(W), O.WarmStart(U, V, s), 2, r, O.Rng(1 ^ 0x5BDBEEF))
print("flags gpu", g.padded, g.k_raised, g.terminated_early, "oracle", o.padded, o.k_raised, o.terminated_early)
print("gpu   ", g.warm.sigma[:3], g.warm.sigma[-3:])
print("oracle", o.warm.sigma[:3], o.warm.sigma[-3:])
print("max |diff| / sigma1", np.abs(g.warm.sigma - o.warm.sigma).max() / o.warm.sigma.max())
