"""1-rank NCCL sharded blws_svd vs unsharded at several r (n-side sharding debug)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1012_0365_b200 as G  # noqa: E402
m = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
rng = np.random.default_rng(1)
for r in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "100,112,113,200").split(",")]:
    u0, _ = np.linalg.qr(rng.standard_normal((m, 2 * r)))
    v0, _ = np.linalg.qr(rng.standard_normal((m, 2 * r)))
    w = np.asfortranarray((u0 * (100 * 0.97 ** (100 * np.arange(2 * r) / r))) @ v0.T + 1e-3 * rng.standard_normal((m, m)))
    wu, _ = np.linalg.qr(u0[:, :r] + 1e-2 * rng.standard_normal((m, r)))
    wv, _ = np.linalg.qr(v0[:, :r] + 1e-2 * rng.standard_normal((m, r)))
    s = 100 * 0.97 ** (100 * np.arange(r) / r)
    ctx = G.Context(0)
    ctx.init_comm(1, 0, G.api.nccl_unique_id())
    op = G.DenseOperator(w, ctx=ctx)
    op.set_row_shard(m, 0)
    a = G.blws_svd(op, G.WarmStart(np.asfortranarray(wu), np.asfortranarray(wv), s), 2, r, G.Rng(1))
    b = G.blws_svd(G.DenseOperator(w), G.WarmStart(np.asfortranarray(wu), np.asfortranarray(wv), s), 2, r, G.Rng(1))
    err = np.abs(a.warm.sigma - b.warm.sigma) / b.warm.sigma
    print(f"m={m} r={r}: max rel sigma err {err.max():.3e} at {err.argmax()}, padded {a.padded} {b.padded}", flush=True)
