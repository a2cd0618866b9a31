"""Row-sharded path on the device with a one-rank NCCL
communicator: every sharded code path runs (panel reductions split into an
allreduced top and a local bottom, the sharded paired apply, the shared
non-finite flag, NCCL calls captured in the blws_svd graph) and must agree
with the oracle and with the unsharded device path. Multi-rank runs need one
GPU per rank; the decomposition itself is checked with gloo in
test_dist_cpu.py.
"""
import os

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
    _sharded_single_rank(G, O, exact)


def test_col_sharded_single_rank_nccl(G, O):
    # the column-sharded panels on a one-rank NCCL communicator (BLWS_NSHARD=force,
    # set in a subprocess: the switch is read once per process): NCCL all-gather /
    # reduce-scatter, eager and captured in the blws_svd graph
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, 'tests'); import conftest, test_gpu_dist as t; "
            "import paper_1012_0365_b200 as G; from oracle import oracle as O; t._sharded_single_rank(G, O, False); "
            "t.test_sharded_lanczos_and_svt_single_rank(G, O)")
    env = dict(os.environ, BLWS_NSHARD="force")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-3000:]


def _sharded_single_rank(G, O, exact):
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


def test_sharded_rpca_single_rank(G, O):
    # rpca_adm (solvers.hpp:72-157) row-sharded over a one-rank NCCL communicator:
    # the allreduced scalars, the sharded operator / SVT and the row-local ALM
    # kernel agree with the unsharded device solve and with the oracle
    from paper_1012_0365_b200 import synth

    d, a0, _, _ = synth.rpca_lowrank_sparse(160, 8, 1280, 4, O.Rng, O.sample_distinct)
    ctx = G.Context(0)
    ctx.init_comm(1, 0, G.api.nccl_unique_id())
    a_s, e_s, st_s, _ = G.rpca_adm_sharded(d, 160, 0, G.SvdBackend.blws(seed=11, ctx=ctx), truth_rows=a0)
    a_p, e_p, st_p, _ = G.rpca_adm(d, G.SvdBackend.blws(seed=11), truth=a0)
    a_o, e_o, st_o, _ = O.rpca_adm(d, O.SvdBackend.blws(seed=11), truth=a0)
    assert st_s.converged and st_s.iterations == st_p.iterations
    assert abs(st_s.iterations - st_o.iterations) <= 1
    assert st_s.rank_hat == st_p.rank_hat == 8 and st_s.predicted_ranks == st_p.predicted_ranks
    assert st_s.e_l0 == st_p.e_l0 and st_s.matvec_count == st_p.matvec_count
    assert np.linalg.norm(a_s - a_p) <= 1e-10 * np.linalg.norm(a_p)
    assert np.linalg.norm(a_s - a_o) <= 1e-6 * np.linalg.norm(a_o)
    assert abs(st_s.rel_err - st_p.rel_err) <= 1e-12 + 1e-9 * st_p.rel_err


def test_sharded_mc_single_rank(G, O):
    # mc_svt (solvers.hpp:202-270) row-sharded over a one-rank communicator: the
    # sparse operator's W^T halves go through the allreduce, K9 runs on the local
    # rows, nnz / norms are summed over the ranks
    from paper_1012_0365_b200 import dist, synth

    colptr, rowidx, vals, ml, mr = synth.mc_lowrank(200, 5, 11850, 13, O.Rng, O.sample_distinct)
    lp, lr, lv, pos = dist.shard_csc(colptr, rowidx, vals, 0, 200)
    assert len(pos) == len(vals)
    ctx = G.Context(0)
    ctx.init_comm(1, 0, G.api.nccl_unique_id())
    us, ss, vs, st_s = G.mc_svt_sharded(200, 0, 200, 200, lp, lr, lv, G.SvdBackend.blws(seed=8, ctx=ctx),
                                        truth_ml_rows=ml, truth_mr=mr)
    up, sp, vp, st_p = G.mc_svt(200, 200, colptr, rowidx, vals, G.SvdBackend.blws(seed=8), truth_ml=ml, truth_mr=mr)
    assert st_s.converged and st_s.iterations == st_p.iterations and st_s.rank_hat == st_p.rank_hat
    assert st_s.predicted_ranks == st_p.predicted_ranks and st_s.matvec_count == st_p.matvec_count
    a_s, a_p = (us * ss) @ vs.T, (up * sp) @ vp.T
    assert np.linalg.norm(a_s - a_p) <= 1e-9 * np.linalg.norm(a_p)
    assert st_s.rel_err <= 2e-4


def test_sharded_solver_guards(G, O):
    ctx = G.Context(0)
    ctx.init_comm(1, 0, G.api.nccl_unique_id())
    d = np.eye(20)
    with pytest.raises(ValueError):
        G.rpca_adm_sharded(d[:12], 20, 10, G.SvdBackend.blws(ctx=ctx))  # rows past m
    with pytest.raises(ValueError):
        G.mc_svt_sharded(20, 0, 10, 20, np.zeros(21, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0),
                         G.SvdBackend.blws(ctx=ctx))  # empty observation on every rank
