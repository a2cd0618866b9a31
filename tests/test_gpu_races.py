"""Race detection without compute-sanitizer (closed on this pool:
profiles/r02_sanitizer_closed.txt).

Every hot path here is deterministic by construction (fixed reduction orders,
no float atomics), so
  * a run with CUDA_LAUNCH_BLOCKING=1 (every launch serialised, streams and
    fork/join overlap removed) must give BITWISE the same outputs as a normal
    run -- a missing stream / event dependency, a buffer freed or reused while
    another stream still reads it, or a collective racing a kernel shows up as
    a difference (this is how the n-side sharding race of r02 was found);
  * repeated runs in one process must agree bitwise -- an intra-kernel race on
    shared memory or an mbarrier ring would perturb some of them.
The cases cover the TMA/mbarrier GEMMs, the CholQR factor, both
tridiagonalisations, the grid-synchronised Lanczos, K7, K8 / K9 and the sharded
collectives (one-rank NCCL, column sharding forced).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import paper_1012_0365_b200 as G
from oracle import oracle as O
from paper_1012_0365_b200 import synth
out = {}
def inst(m, n, r, seed):
    rng = O.Rng(seed)
    u0 = O.thin_qr(rng.gaussian_matrix(m, 2 * r)).q
    v0 = O.thin_qr(rng.gaussian_matrix(n, 2 * r)).q
    w = (u0 * (10.0 * 0.97 ** np.arange(2 * r))) @ v0.T + 1e-3 * rng.gaussian_matrix(m, n)
    wu = O.thin_qr(u0[:, :r] + 1e-2 * rng.gaussian_matrix(m, r)).q
    wv = O.thin_qr(v0[:, :r] + 1e-2 * rng.gaussian_matrix(n, r)).q
    return w, wu, wv, 10.0 * 0.97 ** np.arange(r)
for (m, n, r) in [(2000, 1800, 100), (900, 800, 130)]:  # fused sytrd + CholQR factor; cluster sytrd + chol_inv
    w, wu, wv, s = inst(m, n, r, m)
    op = G.DenseOperator(w)
    for it in range(4):  # eager, eager, graph capture, replay
        res = G.blws_svd(op, G.WarmStart(wu, wv, s), 2, r, G.Rng(1))
        out[f"blws{m}_{it}"] = np.concatenate([res.warm.sigma, res.warm.u.ravel(), res.warm.v.ravel()])
w, wu, wv, s = inst(1200, 1000, 110, 7)
ctx = G.Context(0)
ctx.init_comm(1, 0, G.api.nccl_unique_id())
op = G.DenseOperator(w, ctx=ctx)
op.set_row_shard(1200, 0)
for it in range(4):
    res = G.blws_svd(op, G.WarmStart(wu, wv, s), 2, 110, G.Rng(1))
    out[f"shard_{it}"] = np.concatenate([res.warm.sigma, res.warm.u.ravel(), res.warm.v.ravel()])
d, a0, _, _ = synth.rpca_lowrank_sparse(400, 12, 8000, 3, O.Rng, O.sample_distinct)
a, e, st, _ = G.rpca_adm(d, G.SvdBackend.blws(seed=5), truth=a0)
out["rpca"] = np.concatenate([a.ravel(), e.ravel(), [st.iterations, st.rank_hat]])
colptr, rowidx, vals, ml, mr = synth.mc_lowrank(600, 6, 54000, 2, O.Rng, O.sample_distinct)
u, sg, v, st = G.mc_svt(600, 600, colptr, rowidx, vals, G.SvdBackend.blws(seed=8), truth_ml=ml, truth_mr=mr)
out["mc"] = np.concatenate([u.ravel(), sg, v.ravel(), [st.iterations]])
np.savez(sys.argv[1], **out)
'''


def _run(tmp_path, name, extra_env):
    env = dict(os.environ, BLWS_NSHARD="force", **extra_env)
    path = tmp_path / f"{name}.npz"
    r = subprocess.run([sys.executable, "-c", CASES, str(path)], env=env, cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(path))


def test_launch_blocking_and_repeats_agree_bitwise(tmp_path):
    normal = _run(tmp_path, "normal", {})
    blocking = _run(tmp_path, "blocking", {"CUDA_LAUNCH_BLOCKING": "1"})
    assert normal.keys() == blocking.keys()
    for k in normal:
        assert np.array_equal(normal[k], blocking[k]), k
    for base in ("blws2000", "blws900", "shard"):  # eager, graph capture and replays: identical
        for it in range(1, 4):
            assert np.array_equal(normal[f"{base}_0"], normal[f"{base}_{it}"]), (base, it)
