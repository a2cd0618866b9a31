import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import bench, paper_1012_0365_b200 as B
m = int(sys.argv[1]); r = int(sys.argv[2])
dev = torch.device('cuda:0')
Wt, Uw, Vw, sigma, U0, V0 = bench.c5_inputs(m, r, 0, m, dev)
print('W finite', bool(torch.isfinite(Wt).all()), 'sigma head', sigma[:3].tolist(), flush=True)
ctx = B.Context(0)
op = B.DenseOperator(Wt, ctx=ctx, device=True, shape=(m, m), ld=m)
w = B.DeviceWarmStart.from_host(np.asfortranarray(Uw.cpu().numpy()), np.asfortranarray(Vw.cpu().numpy()), sigma[:r].cpu().numpy(), ctx)
res = B.blws_svd(op, w, 2, r, B.Rng(1 ^ 0x5BDBEEF), keep_device=True)
s = res.warm.sigma()
print('flags', res.padded, res.k_raised, res.terminated_early, 'sigma', s[:4], s[-4:], 'n', s.size, 'finite', np.isfinite(s).all(), flush=True)
print('true', sigma[:4].tolist(), sigma[r-4:r].tolist())
