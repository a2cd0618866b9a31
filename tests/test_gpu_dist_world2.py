"""Row-sharded path executed by TWO ranks: two processes on the
same GPU, each with its own context, joined by host-staged collectives over a
gloo process group (Context.init_host_comm: every reduction syncs the stream,
copies its buffer to the host and all-reduces it with torch.distributed). The
sharded device code runs for real with world size 2 -- rows split between
the ranks, the W^T x halves summed across them -- and is compared with the
unsharded device path and the oracle. NCCL needs one GPU per rank; these
tests exercise the same library calls with the collective swapped, and make
no timing claims.
"""
import os
import socket
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from conftest import principal_angle  # noqa: E402

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _instance(O, m=700, n=500, r=24, seed=123):
    rng = O.Rng(seed)
    u0, _, v0 = O.full_svd_small(rng.gaussian_matrix(m, n))
    w = (u0[:, :2 * r] * (50.0 * 0.9 ** np.arange(2 * r))) @ v0[:, :2 * r].T + 1e-3 * rng.gaussian_matrix(m, n)
    su, ss, sv = O.full_svd_small(w + 1e-2 * rng.gaussian_matrix(m, n))
    return w, su[:, :r].copy(order="F"), sv[:, :r].copy(order="F"), ss[:r].copy()


def _worker(rank, port, outdir, case, shape=(700, 500, 24)):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_1012_0365_b200 as G
        from oracle import oracle as O
        from paper_1012_0365_b200 import dist as gd
        from paper_1012_0365_b200 import synth

        ctx = G.Context(0)
        gd.init_host_comm(ctx)
        out = {}
        if case == "blws":
            w, u, v, s = _instance(O, *shape)
            m, r = w.shape[0], u.shape[1]
            row0, rows = gd.row_partition(m, WORLD, rank)
            op = G.DenseOperator(np.asfortranarray(w[row0:row0 + rows]), ctx=ctx)
            op.set_row_shard(m, row0)
            warm = G.WarmStart(np.asfortranarray(u[row0:row0 + rows]), v, s)
            for it in range(3):
                res = G.blws_svd(op, warm, 2, r, G.Rng(1))
                out[f"u{it}"], out[f"v{it}"], out[f"s{it}"] = res.warm.u, res.warm.v, res.warm.sigma
            out["row0"], out["count"] = row0, op.application_count()
        elif case == "svt":
            w, _, _, _ = _instance(O, m=600, n=450, r=12, seed=5)
            m = w.shape[0]
            row0, rows = gd.row_partition(m, WORLD, rank)
            op = G.DenseOperator(np.asfortranarray(w[row0:row0 + rows]), ctx=ctx)
            op.set_row_shard(m, row0)
            out["snorm"] = G.spectral_norm(op)
            us, ss, vs, _ = G.lanczos_partial_svd(op, 8, tol=1e-10)
            out["lz_u"], out["lz_s"], out["lz_v"] = us, ss, vs
            sv = O.full_svd_small(w)[1]
            eps = 0.5 * (sv[14] + sv[15])
            b = G.SvdBackend.blws(seed=3, ctx=ctx)
            p = G.RankPredictor(10, 5, 450)
            for it in range(4):
                res = G.svt(op, eps, b, p)
                out[f"svt_rank{it}"], out[f"svt_s{it}"] = res.achieved_rank, res.sigma
            out["hist"] = np.array(p.history)
            out["row0"] = row0
        elif case == "rpca":
            d, a0, _, _ = synth.rpca_lowrank_sparse(160, 8, 1280, 4, O.Rng, O.sample_distinct)
            row0, rows = gd.row_partition(160, WORLD, rank)
            a, e, st, _ = G.rpca_adm_sharded(np.asfortranarray(d[row0:row0 + rows]), 160, row0,
                                             G.SvdBackend.blws(seed=11, ctx=ctx),
                                             truth_rows=np.asfortranarray(a0[row0:row0 + rows]))
            out.update(a=a, e=e, it=st.iterations, rank=st.rank_hat, e_l0=st.e_l0, mv=st.matvec_count,
                       rel=st.rel_err, pred=np.array(st.predicted_ranks), row0=row0)
        elif case == "mc":
            colptr, rowidx, vals, ml, mr = synth.mc_lowrank(200, 5, 11850, 13, O.Rng, O.sample_distinct)
            row0, rows = gd.row_partition(200, WORLD, rank)
            lp, lr, lv, _ = gd.shard_csc(colptr, rowidx, vals, row0, rows)
            us, ss, vs, st = G.mc_svt_sharded(200, row0, rows, 200, lp, lr, lv, G.SvdBackend.blws(seed=8, ctx=ctx),
                                              truth_ml_rows=np.asfortranarray(ml[row0:row0 + rows]), truth_mr=mr)
            out.update(u=us, s=ss, v=vs, it=st.iterations, rank=st.rank_hat, mv=st.matvec_count, rel=st.rel_err,
                       pred=np.array(st.predicted_ranks), row0=row0)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), **out)
    finally:
        dist.destroy_process_group()


def _run(case, tmp_path, *extra):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(_free_port(), str(tmp_path), case, *extra), nprocs=WORLD, join=True)
    return [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(WORLD)]


def _stack_rows(parts, key):
    return np.concatenate([p[key] for p in sorted(parts, key=lambda p: int(p["row0"]))], axis=0)


@pytest.mark.parametrize("nshard,shape", [("1", (700, 500, 24)), ("1", (300, 251, 20)), ("0", (700, 500, 24))])
def test_world2_blws_svd_matches_oracle(G, O, tmp_path, monkeypatch, nshard, shape):
    # nshard 1: V and the bottom rows of every panel split over the ranks (the
    # default; n = 251 leaves a zero padding row on rank 1); 0: replicated
    monkeypatch.setenv("BLWS_NSHARD", nshard)
    parts = _run("blws", tmp_path, shape)
    w, u, v, s = _instance(O, *shape)
    r = u.shape[1]
    ref = O.blws_svd(O.DenseOperator(w), O.WarmStart(u, v, s), 2, r, O.Rng(1))
    plain = G.blws_svd(G.DenseOperator(w), G.WarmStart(u, v, s), 2, r, G.Rng(1))
    for it in range(3):
        uu = _stack_rows(parts, f"u{it}")
        for p in parts:
            assert np.array_equal(p[f"s{it}"], parts[0][f"s{it}"])  # both ranks hold the same sigma and V
            assert np.array_equal(p[f"v{it}"], parts[0][f"v{it}"])
        sg = parts[0][f"s{it}"]
        assert np.abs(sg - ref.warm.sigma).max() <= 1e-10 * ref.warm.sigma.max()
        assert np.abs(sg - plain.warm.sigma).max() <= 1e-12 * plain.warm.sigma.max()
        assert principal_angle(uu, ref.warm.u) <= 1e-8
        assert principal_angle(parts[0][f"v{it}"], ref.warm.v) <= 1e-8
    assert all(int(p["count"]) == 3 * 2 * r for p in parts)


def test_world2_lanczos_svt(G, O, tmp_path):
    parts = _run("svt", tmp_path)
    w, _, _, _ = _instance(O, m=600, n=450, r=12, seed=5)
    plain = G.DenseOperator(w)
    sn = G.spectral_norm(plain)
    assert all(abs(float(p["snorm"]) - sn) <= 1e-12 * sn for p in parts)
    up, sp, vp, _ = G.lanczos_partial_svd(plain, 8, tol=1e-10)
    assert np.abs(parts[0]["lz_s"] - sp).max() <= 1e-10 * sp[0]
    assert principal_angle(_stack_rows(parts, "lz_u"), up) <= 1e-8
    assert principal_angle(parts[0]["lz_v"], vp) <= 1e-8
    sv = O.full_svd_small(w)[1]
    eps = 0.5 * (sv[14] + sv[15])
    b = G.SvdBackend.blws(seed=3)
    p = G.RankPredictor(10, 5, 450)
    for it in range(4):
        res = G.svt(plain, eps, b, p)
        assert all(int(q[f"svt_rank{it}"]) == res.achieved_rank for q in parts)
        assert np.abs(parts[0][f"svt_s{it}"] - res.sigma).max() <= 1e-9 * res.sigma.max()
    assert list(parts[0]["hist"]) == list(p.history)


def test_world2_rpca(G, O, tmp_path):
    from paper_1012_0365_b200 import synth

    parts = _run("rpca", tmp_path)
    d, a0, _, _ = synth.rpca_lowrank_sparse(160, 8, 1280, 4, O.Rng, O.sample_distinct)
    a_p, e_p, st_p, _ = G.rpca_adm(d, G.SvdBackend.blws(seed=11), truth=a0)
    a_o, _, st_o, _ = O.rpca_adm(d, O.SvdBackend.blws(seed=11), truth=a0)
    a_s, e_s = _stack_rows(parts, "a"), _stack_rows(parts, "e")
    for q in parts:
        assert int(q["it"]) == st_p.iterations and int(q["rank"]) == st_p.rank_hat == 8
        assert int(q["e_l0"]) == st_p.e_l0 and int(q["mv"]) == st_p.matvec_count
        assert list(q["pred"]) == list(st_p.predicted_ranks)
        assert abs(float(q["rel"]) - st_p.rel_err) <= 1e-12 + 1e-9 * st_p.rel_err
    assert abs(st_p.iterations - st_o.iterations) <= 1
    assert np.linalg.norm(a_s - a_p) <= 1e-10 * np.linalg.norm(a_p)
    assert np.linalg.norm(a_s - a_o) <= 1e-6 * np.linalg.norm(a_o)
    assert np.linalg.norm(e_s - e_p) <= 1e-9 * np.linalg.norm(e_p)


def test_world2_mc(G, O, tmp_path):
    from paper_1012_0365_b200 import synth

    parts = _run("mc", tmp_path)
    colptr, rowidx, vals, ml, mr = synth.mc_lowrank(200, 5, 11850, 13, O.Rng, O.sample_distinct)
    up, sp, vp, st_p = G.mc_svt(200, 200, colptr, rowidx, vals, G.SvdBackend.blws(seed=8), truth_ml=ml, truth_mr=mr)
    for q in parts:
        assert int(q["it"]) == st_p.iterations and int(q["rank"]) == st_p.rank_hat
        assert int(q["mv"]) == st_p.matvec_count and list(q["pred"]) == list(st_p.predicted_ranks)
    us = _stack_rows(parts, "u")
    a_s, a_p = (us * parts[0]["s"]) @ parts[0]["v"].T, (up * sp) @ vp.T
    assert np.linalg.norm(a_s - a_p) <= 1e-9 * np.linalg.norm(a_p)
