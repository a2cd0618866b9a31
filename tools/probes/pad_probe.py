import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1012_0365_b200 as G
from oracle import oracle as O
for (m, r) in [(600, 30), (800, 40), (1200, 60), (1600, 80)]:
    rng = O.Rng(m)
    u0 = O.thin_qr(rng.gaussian_matrix(m, 2 * r)).q
    v0 = O.thin_qr(rng.gaussian_matrix(m, 2 * r)).q
    sig = 100 * 0.97 ** (100 * np.arange(2 * r) / r)
    w = (u0 * sig) @ v0.T + 1e-3 * rng.gaussian_matrix(m, m)
    eps = 1e-2 * np.sqrt(4000 / m)
    wu = O.thin_qr(u0[:, :r] + eps * rng.gaussian_matrix(m, r)).q
    wv = O.thin_qr(v0[:, :r] + eps * rng.gaussian_matrix(m, r)).q
    res = G.blws_svd(G.DenseOperator(w), G.WarmStart(wu, wv, sig[:r].copy()), 2, r, G.Rng(1))
    print(m, r, "padded", res.padded, flush=True)
