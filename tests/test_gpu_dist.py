"""Row-sharded path on the device with a one-rank NCCL
communicator: every sharded code path runs (panel reductions split into an
allreduced top and a local bottom, the sharded paired apply, the shared
non-finite flag, NCCL calls captured in the blws_svd graph) and must agree
with the oracle and with the unsharded device path. Multi-rank runs need one
GPU per rank; the decomposition itself is checked with gloo in
test_dist_cpu.py.
"""
import numpy as np
import pytest

from conftest import principal_angle

pytestmark = pytest.mark.gpu


def _instance(O, m=700, n=500, r=24, seed=123):
    rng = O.Rng(seed)
    u0, _, v0 = O.full_svd_small(rng.gaussian_matrix(m, n))
    w = (u0[:, :2 * r] * (50.0 * 0.9 ** np.arange(2 * r))) @ v0[:, :2 * r].T + 1e-3 * rng.gaussian_matrix(m, n)
    su, ss, sv = O.full_svd_small(w + 1e-2 * rng.gaussian_matrix(m, n))
    return w, su[:, :r].copy(order="F"), sv[:, :r].copy(order="F"), ss[:r].copy()


@pytest.mark.parametrize("exact", [False, True])
def test_sharded_single_rank_matches_oracle_and_unsharded(G, O, exact, monkeypatch):
    if exact:
        monkeypatch.setenv("BLWS_EXACT", "1")
    else:
        monkeypatch.delenv("BLWS_EXACT", raising=False)
    w, u, v, s = _instance(O)
    m, n = w.shape
    r = u.shape[1]
    ctx = G.Context(0)
    ctx.init_comm(1, 0, G.api.nccl_unique_id())
    assert ctx.comm_info() == (1, 0)
    op = G.DenseOperator(w, ctx=ctx)
    op.set_row_shard(m, 0)
    warm = G.DeviceWarmStart.from_host(u, v, s, ctx)
    g0 = G.graph_launches()
    outs = [G.blws_svd(op, warm, 2, r, G.Rng(1)) for _ in range(4)]  # eager, eager, capture, replay
    if not exact:
        assert G.graph_launches() == g0 + 2  # NCCL allreduces captured in the graph
    ref = O.blws_svd(O.DenseOperator(w), O.WarmStart(u, v, s), 2, r, O.Rng(1))
    plain = G.blws_svd(G.DenseOperator(w), G.WarmStart(u, v, s), 2, r, G.Rng(1))
    for o in outs:
        assert np.abs(o.warm.sigma - ref.warm.sigma).max() <= 1e-10 * ref.warm.sigma.max()
        assert principal_angle(o.warm.u, ref.warm.u) <= 1e-8 and principal_angle(o.warm.v, ref.warm.v) <= 1e-8
        assert np.abs(o.warm.sigma - plain.warm.sigma).max() <= 1e-12 * plain.warm.sigma.max()
        assert np.array_equal(o.warm.sigma, outs[0].warm.sigma)  # eager and graph replays agree bitwise
    assert op.application_count() == 4 * 2 * r


def test_sharded_operator_guards(G, O):
    w, u, v, s = _instance(O, m=200, n=150, r=6)
    ctx = G.Context(0)
    ctx.init_comm(1, 0, G.api.nccl_unique_id())
    op = G.DenseOperator(w, ctx=ctx)
    with pytest.raises(ValueError):
        op.set_row_shard(100, 0)  # fewer global rows than local


def test_sharded_lanczos_and_svt_single_rank(G, O):
    # the cold Lanczos reseed (lanczos.hpp:85-329) and svt (svt.hpp:216-254)
    # on a row-sharded operator: dot / norm / Q^T r reductions and the W^T x
    # half of the paired GEMV go through the allreduce
    w, u, v, s = _instance(O, m=600, n=450, r=12, seed=5)
    ctx = G.Context(0)
    ctx.init_comm(1, 0, G.api.nccl_unique_id())
    op = G.DenseOperator(w, ctx=ctx)
    op.set_row_shard(w.shape[0], 0)
    plain = G.DenseOperator(w)
    assert abs(G.spectral_norm(op) - G.spectral_norm(plain)) <= 1e-12 * G.spectral_norm(plain)
    us, ss, vs, _ = G.lanczos_partial_svd(op, 8, tol=1e-10)
    up, sp, vp, _ = G.lanczos_partial_svd(plain, 8, tol=1e-10)
    assert np.abs(ss - sp).max() <= 1e-10 * sp[0]
    assert principal_angle(us, up) <= 1e-8 and principal_angle(vs, vp) <= 1e-8
    eps = 0.5 * (O.full_svd_small(w)[1][14] + O.full_svd_small(w)[1][15])
    b1 = G.SvdBackend.blws(seed=3, ctx=ctx)
    b2 = G.SvdBackend.blws(seed=3)
    p1, p2 = G.RankPredictor(10, 5, 450), G.RankPredictor(10, 5, 450)
    for _ in range(4):  # reseed (rank growth), then BLWS steps
        r1 = G.svt(op, eps, b1, p1)
        r2 = G.svt(plain, eps, b2, p2)
        assert r1.achieved_rank == r2.achieved_rank and p1.history == p2.history
        assert np.abs(r1.sigma - r2.sigma).max() <= 1e-9 * r2.sigma.max()
