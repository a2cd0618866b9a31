"""Row-sharded multi-GPU path, host side, on CPU with gloo.

The device path (csrc/host_core.cu: RowSplit, panel_tn, panel_sumsq, the
sharded paired apply) allreduces every reduction over the rows of a stacked
panel. Here the same decomposition is restated in numpy with gloo allreduces
(world_size 2) and checked against the oracle's unsharded blws_svd
(block_lanczos.hpp:204-261); plus the row partition and the NCCL unique-id
rendezvous of paper_1012_0365_b200/dist.py.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, fn, *args):
    import torch.multiprocessing as mp

    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(r, world, port, fn, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, res = q.get(timeout=240)
        out[rank] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [out[r] for r in range(world)]


def _entry(rank, world, port, fn, args, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world, *args)))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------ restatement
def _allreduce(x):
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _panel_gram(top, bot):
    # rows [0, mp) sharded (allreduced), rows of the V side replicated
    return _allreduce(top.T @ top) + bot.T @ bot


def _cholqr2(top, bot, sharded_top=True):
    # CholQR2 of the stacked panel [top; bot]; returns Q parts and R
    rs = []
    for _ in range(2):
        g = _panel_gram(top, bot) if sharded_top else top.T @ top + bot.T @ bot
        r = np.linalg.cholesky(g).T
        rinv = np.linalg.inv(r)
        top, bot = top @ rinv, bot @ rinv
        rs.append(r)
    return top, bot, rs[1] @ rs[0]


def _cholqr2_rows(x, sharded):
    g = _allreduce(x.T @ x) if sharded else x.T @ x
    r1 = np.linalg.cholesky(g).T
    x = x @ np.linalg.inv(r1)
    g = _allreduce(x.T @ x) if sharded else x.T @ x
    return x @ np.linalg.inv(np.linalg.cholesky(g).T)


def sharded_blws(w_loc, u_loc, v, k, r):
    """blws_svd with W and U row-sharded, V replicated (k = 2 blocks)."""
    b = u_loc.shape[1]
    xt, xb, _ = _cholqr2(u_loc.copy(), v.copy())  # X1 = qr([U; V] / sqrt(2)).q
    qs, ms, bs_ = [(xt, xb)], [], []
    zt, zb = w_loc @ xb, _allreduce(w_loc.T @ xt)  # augmented apply: W^T X_top summed over ranks
    ms.append(_allreduce(xt.T @ zt) + xb.T @ zb)
    for _ in range(1, k):
        m1 = 0.5 * (ms[-1] + ms[-1].T)
        rt, rb = zt - qs[-1][0] @ m1, zb - qs[-1][1] @ m1
        if len(qs) > 1:
            rt, rb = rt - qs[-2][0] @ bs_[-1].T, rb - qs[-2][1] @ bs_[-1].T
        nt, nb, rr = _cholqr2(rt, rb)
        bs_.append(rr)
        qs.append((nt, nb))
        zt, zb = w_loc @ nb, _allreduce(w_loc.T @ nt)
        ms.append(_allreduce(nt.T @ zt) + nb.T @ zb)
    d = k * b
    t = np.zeros((d, d))
    for l in range(k):
        t[l * b:(l + 1) * b, l * b:(l + 1) * b] = 0.5 * (ms[l] + ms[l].T)
        if l + 1 < k:
            t[(l + 1) * b:(l + 2) * b, l * b:(l + 1) * b] = bs_[l]
            t[l * b:(l + 1) * b, (l + 1) * b:(l + 2) * b] = bs_[l].T
    vals, vecs = np.linalg.eigh(t)
    vals, vecs = vals[::-1][:r], vecs[:, ::-1][:, :r]
    qt = np.hstack([q[0] for q in qs])
    qb = np.hstack([q[1] for q in qs])
    u_new = np.sqrt(2.0) * qt @ vecs
    v_new = np.sqrt(2.0) * qb @ vecs
    return _cholqr2_rows(u_new, True), _cholqr2_rows(v_new, False), vals


def _case(seed=7, m=120, n=90, r=6):  # noqa: E302
    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    rng = O.Rng(seed)
    u0, _, v0 = O.full_svd_small(rng.gaussian_matrix(m, n))
    s = 10.0 * 0.8 ** np.arange(2 * r)
    w = (u0[:, :2 * r] * s) @ v0[:, :2 * r].T + 1e-3 * rng.gaussian_matrix(m, n)
    uw = O.thin_qr(u0[:, :r] + 1e-2 * rng.gaussian_matrix(m, r)).q
    vw = O.thin_qr(v0[:, :r] + 1e-2 * rng.gaussian_matrix(n, r)).q
    return O, w, uw, vw, s[:r].copy()


def _worker_blws(rank, world):
    from paper_1012_0365_b200.dist import row_partition

    O, w, uw, vw, s = _case()
    row0, rows = row_partition(w.shape[0], world, rank)
    un, vn, vals = sharded_blws(w[row0:row0 + rows], uw[row0:row0 + rows], vw, 2, uw.shape[1])
    return row0, rows, un, vn, vals


def test_row_partition_covers_rows_once():
    from paper_1012_0365_b200.dist import row_partition

    for m, world in [(10, 3), (4000, 8), (7, 7), (40000, 6)]:
        parts = [row_partition(m, world, r) for r in range(world)]
        assert parts[0][0] == 0 and sum(p[1] for p in parts) == m
        for (a0, an), (b0, _) in zip(parts, parts[1:]):
            assert a0 + an == b0
        assert max(p[1] for p in parts) - min(p[1] for p in parts) <= 1
    with pytest.raises(ValueError):
        row_partition(3, 4, 0)


def _worker_uid(rank, world):
    from paper_1012_0365_b200.dist import broadcast_unique_id

    return broadcast_unique_id()


def test_unique_id_rendezvous_gloo():
    ids = _run(2, _worker_uid)
    assert all(isinstance(i, bytes) and len(i) == 128 for i in ids), ids
    assert ids[0] == ids[1]


def test_sharded_blws_decomposition_matches_oracle():
    res = _run(2, _worker_blws)
    assert not any(isinstance(r, str) for r in res), res
    O, w, uw, vw, s = _case()
    ref = O.blws_svd(O.DenseOperator(w), O.WarmStart(uw, vw, s), 2, uw.shape[1], O.Rng(3))
    for row0, rows, un, vn, vals in res:
        assert np.abs(vals - ref.warm.sigma).max() <= 1e-10 * ref.warm.sigma.max()
        assert un.shape == (rows, uw.shape[1])
        assert np.allclose(np.abs(vn), np.abs(ref.warm.v), atol=1e-8)
    # the row panels of U assemble into the oracle's U (columns up to sign)
    u_all = np.vstack([r[2] for r in res])
    assert np.allclose(np.abs(u_all), np.abs(ref.warm.u), atol=1e-8)
    # both ranks computed identical replicated parts
    assert np.array_equal(res[0][3], res[1][3]) and np.array_equal(res[0][4], res[1][4])


# ---- column (n-side) sharding: the bottom rows of every panel split too
def _allgather_rows(x_loc):
    """rows of every rank's block in rank order (NCCL all-gather of the chunks)."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(x_loc, dtype=np.float64))
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return np.concatenate([q.numpy() for q in parts], axis=0)


def _reduce_scatter_rows(x_full, rank, chunk):
    """this rank's rows of the sum over the ranks (NCCL reduce-scatter)."""
    return _allreduce(x_full)[rank * chunk:(rank + 1) * chunk]


def sharded2_blws(w_loc, u_loc, v_loc, rank, chunk, n, k, r):
    """blws_svd with W and U row-sharded AND V / the panel bottoms split into
    chunks (csrc/host_core.cu col_sharded: gather_cols before W X_bot,
    scatter_cols after W^T X_top); every Gram / norm allreduced over all rows."""
    b = u_loc.shape[1]
    npad = chunk * 2

    def apply(xt, xb):
        xfull = _allgather_rows(xb)[:n]
        part = np.zeros((npad, xt.shape[1]))
        part[:n] = w_loc.T @ xt
        return w_loc @ xfull, _reduce_scatter_rows(part, rank, chunk)

    def gram(top, bot):
        return _allreduce(top.T @ top + bot.T @ bot)

    def cholqr2(top, bot):
        rs = []
        for _ in range(2):
            rr = np.linalg.cholesky(gram(top, bot)).T
            ri = np.linalg.inv(rr)
            top, bot = top @ ri, bot @ ri
            rs.append(rr)
        return top, bot, rs[1] @ rs[0]

    xt, xb, _ = cholqr2(u_loc.copy(), v_loc.copy())
    qs, ms, bs_ = [(xt, xb)], [], []
    zt, zb = apply(xt, xb)
    ms.append(_allreduce(xt.T @ zt + xb.T @ zb))
    for _ in range(1, k):
        m1 = 0.5 * (ms[-1] + ms[-1].T)
        rt, rb = zt - qs[-1][0] @ m1, zb - qs[-1][1] @ m1
        nt, nb, rr = cholqr2(rt, rb)
        bs_.append(rr)
        qs.append((nt, nb))
        zt, zb = apply(nt, nb)
        ms.append(_allreduce(nt.T @ zt + nb.T @ zb))
    d = k * b
    t = np.zeros((d, d))
    for l in range(k):
        t[l * b:(l + 1) * b, l * b:(l + 1) * b] = 0.5 * (ms[l] + ms[l].T)
        if l + 1 < k:
            t[(l + 1) * b:(l + 2) * b, l * b:(l + 1) * b] = bs_[l]
            t[l * b:(l + 1) * b, (l + 1) * b:(l + 2) * b] = bs_[l].T
    vals, vecs = np.linalg.eigh(t)
    vals, vecs = vals[::-1][:r], vecs[:, ::-1][:, :r]
    u_new = np.sqrt(2.0) * np.hstack([q[0] for q in qs]) @ vecs
    v_new = np.sqrt(2.0) * np.hstack([q[1] for q in qs]) @ vecs
    return _cholqr2_rows(u_new, True), _cholqr2_rows(v_new, True), vals


def _worker_blws_cols(rank, world):
    from paper_1012_0365_b200.dist import row_partition

    O, w, uw, vw, s = _case(n=91)  # odd n: rank 1 carries a zero padding row
    m, n = w.shape
    row0, rows = row_partition(m, world, rank)
    chunk = -(-n // world)
    v_loc = np.zeros((chunk, vw.shape[1]))
    take = max(0, min(n, (rank + 1) * chunk) - rank * chunk)
    v_loc[:take] = vw[rank * chunk:rank * chunk + take]
    un, vn, vals = sharded2_blws(w[row0:row0 + rows], uw[row0:row0 + rows], v_loc, rank, chunk, n, 2, uw.shape[1])
    return row0, rows, un, vn, vals, take


def test_col_sharded_blws_decomposition_matches_oracle():
    res = _run(2, _worker_blws_cols)
    assert not any(isinstance(r, str) for r in res), res
    O, w, uw, vw, s = _case(n=91)
    ref = O.blws_svd(O.DenseOperator(w), O.WarmStart(uw, vw, s), 2, uw.shape[1], O.Rng(3))
    for row0, rows, un, vn, vals, take in res:
        assert np.abs(vals - ref.warm.sigma).max() <= 1e-10 * ref.warm.sigma.max()
        assert np.abs(vn[take:]).max(initial=0.0) == 0.0  # padding rows stay exactly zero
    u_all = np.vstack([r[2] for r in res])
    v_all = np.vstack([r[3][:r[5]] for r in res])
    assert np.allclose(np.abs(u_all), np.abs(ref.warm.u), atol=1e-8)
    assert np.allclose(np.abs(v_all), np.abs(ref.warm.v), atol=1e-8)
    assert np.array_equal(res[0][4], res[1][4])  # the same T and Ritz values on both ranks


def _lanczos(apply, dot, reorth_coef, q1t, q1b, steps):
    qt, qb = [q1t], [q1b]
    alphas, betas = [], []
    for l in range(steps):
        zt, zb = apply(qt[-1], qb[-1])
        a = dot(qt[-1], qb[-1], zt, zb)
        alphas.append(a)
        zt, zb = zt - a * qt[-1], zb - a * qb[-1]
        if l > 0:
            zt, zb = zt - betas[-1] * qt[-2], zb - betas[-1] * qb[-2]
        for _ in range(2):  # full CGS2 (lanczos.hpp:123-126)
            c = reorth_coef(np.array(qt).T, np.array(qb).T, zt, zb)
            zt, zb = zt - np.array(qt).T @ c, zb - np.array(qb).T @ c
        b = np.sqrt(dot(zt, zb, zt, zb))
        betas.append(b)
        qt.append(zt / b)
        qb.append(zb / b)
    return np.array(alphas), np.array(betas)


def _worker_lanczos(rank, world):
    from paper_1012_0365_b200.dist import row_partition

    _, w, _, _, _ = _case()
    m, n = w.shape
    row0, rows = row_partition(m, world, rank)
    wl = w[row0:row0 + rows]
    q = np.random.default_rng(0).standard_normal(m + n)
    q /= np.linalg.norm(q)
    return _lanczos(lambda xt, xb: (wl @ xb, _allreduce(wl.T @ xt)),
                    lambda at, ab, bt, bb: float(_allreduce(np.array([at @ bt]))[0] + ab @ bb),
                    lambda qt, qb, zt, zb: _allreduce(qt.T @ zt) + qb.T @ zb,
                    q[row0:row0 + rows], q[m:], 12)


def test_sharded_lanczos_decomposition_matches_unsharded():
    res = _run(2, _worker_lanczos)
    assert not any(isinstance(r, str) for r in res), res
    _, w, _, _, _ = _case()
    m, n = w.shape
    q = np.random.default_rng(0).standard_normal(m + n)
    q /= np.linalg.norm(q)
    ref = _lanczos(lambda xt, xb: (w @ xb, w.T @ xt), lambda at, ab, bt, bb: at @ bt + ab @ bb,
                   lambda qt, qb, zt, zb: qt.T @ zt + qb.T @ zb, q[:m], q[m:], 12)
    for alphas, betas in res:
        assert np.abs(alphas - ref[0]).max() <= 1e-12 * np.abs(ref[0]).max()
        assert np.abs(betas - ref[1]).max() <= 1e-12 * ref[1].max()


# ---------------------------------------------- solver loops (row-sharded)
def _allreduce_max(x):
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.numpy()


def _gather_rows(x, m, row0):
    # exact all-gather of row panels: zeros elsewhere, summed
    full = np.zeros((m,) + x.shape[1:])
    full[row0:row0 + x.shape[0]] = x
    return _allreduce(full)


def _shrink(x, t):
    return np.where(x > t, x - t, np.where(x < -t, x + t, 0.0))


def _rpca_instance():
    from oracle import oracle as O
    from paper_1012_0365_b200 import synth

    return synth.rpca_lowrank_sparse(72, 4, 260, 2, O.Rng, O.sample_distinct)


def _worker_rpca(rank, world):
    # rpca_adm (solvers.hpp:72-157) as host_solvers.cu runs it row-sharded: D / Y /
    # E / W row panels, the scalars (||D||_F, max|D|, ||R||_F) allreduced, the
    # ALM update row-local on this rank's rows of U diag(s) V^T. The SVT itself is
    # the oracle's on the gathered W (the sharded SVT is checked above).
    from oracle import oracle as O
    from paper_1012_0365_b200.dist import row_partition

    d, _, _, _ = _rpca_instance()
    m = d.shape[0]
    row0, rows = row_partition(m, world, rank)
    D = d[row0:row0 + rows]
    lam = 1.0 / np.sqrt(m)
    norm_fro = np.sqrt(_allreduce(np.array([np.sum(D * D)]))[0])
    norm2 = O.spectral_norm(O.DenseOperator(_gather_rows(D, m, row0)))
    mu = 1.25 / norm2
    mu_max = mu * 1e7
    dmax = _allreduce_max(np.array([np.abs(D).max()]))[0]
    Y = D / max(norm2, dmax / lam)
    E = np.zeros_like(D)
    backend = O.SvdBackend.blws(seed=11)
    pred = O.RankPredictor(10, 5, m)
    it_done, A = 0, np.zeros_like(D)
    for it in range(1, 1001):
        W = D - E + Y / mu
        prox = O.svt(O.DenseOperator(_gather_rows(W, m, row0)), 1.0 / mu, backend, pred)
        A = (prox.u[row0:row0 + rows] * prox.sigma) @ prox.v.T
        E = _shrink(D - A + Y / mu, lam / mu)
        res = D - A - E
        Y = Y + mu * res
        mu = min(1.5 * mu, mu_max)
        feas = np.sqrt(_allreduce(np.array([np.sum(res * res)]))[0]) / norm_fro
        it_done = it
        if feas <= 1e-7:
            break
    e_l0 = int(_allreduce(np.array([float(np.sum(np.abs(E) > 1e-8 * dmax))]))[0])
    return it_done, A, list(pred.history), e_l0


def test_sharded_rpca_loop_matches_oracle():
    from oracle import oracle as O

    res = _run(2, _worker_rpca)
    assert not any(isinstance(r, str) for r in res), res
    d, a0, _, _ = _rpca_instance()
    a_ref, _, st, _ = O.rpca_adm(d, O.SvdBackend.blws(seed=11), truth=a0)
    a = np.vstack([r[1] for r in res])
    for it, _, hist, e_l0 in res:
        assert it == st.iterations and hist == st.predicted_ranks and e_l0 == st.e_l0
    assert np.linalg.norm(a - a_ref) <= 1e-9 * np.linalg.norm(a_ref)


def _mc_instance():
    from oracle import oracle as O
    from paper_1012_0365_b200 import synth

    return synth.mc_lowrank(120, 4, 5664, 9, O.Rng, O.sample_distinct)  # 6x oversampled (test_solvers.cpp:110)


def _worker_mc(rank, world):
    # mc_svt (solvers.hpp:202-270) row-sharded: this rank's observed rows as a
    # local CSC (dist.shard_csc), nnz / ||P_Ω D|| / the residual norm summed over
    # the ranks, the sampled evaluation on the local rows of U diag(s). The
    # SVT is the oracle's on the gathered iterate.
    from oracle import oracle as O
    from paper_1012_0365_b200.dist import row_partition, shard_csc

    colptr, rowidx, vals, _, _ = _mc_instance()
    m = n = 120
    row0, rows = row_partition(m, world, rank)
    lp, lr, lv, pos = shard_csc(colptr, rowidx, vals, row0, rows)
    nnz = _allreduce(np.array([float(len(lv))]))[0]
    tau, delta = 5.0 * m, 1.2 * m * n / nnz
    full_idx = np.zeros(len(vals))
    full_idx[pos] = 1.0
    assert np.array_equal(_allreduce(full_idx), np.ones(len(vals)))  # the shards cover every position once

    def gathered(local_vals):
        g = np.zeros(len(vals))
        g[pos] = local_vals
        return _allreduce(g)

    norm2 = O.spectral_norm(O.SparseOperator(m, n, colptr, rowidx, gathered(lv)))
    k0 = np.ceil(tau / (delta * norm2))
    obs_norm = np.sqrt(_allreduce(np.array([np.sum(lv * lv)]))[0])
    y = (k0 * delta) * lv
    col_of = np.repeat(np.arange(n), np.diff(lp))
    backend = O.SvdBackend.blws(seed=8)
    pred = O.RankPredictor(10, 5, min(m, n))
    it_done = 0
    for it in range(1, 501):
        prox = O.svt(O.SparseOperator(m, n, colptr, rowidx, gathered(y)), tau, backend, pred)
        us = prox.u[row0:row0 + rows] * prox.sigma
        a_vals = np.einsum("ij,ij->i", us[lr], prox.v[col_of])
        resid = lv - a_vals
        rel = np.sqrt(_allreduce(np.array([np.sum(resid * resid)]))[0]) / obs_norm
        it_done = it
        if rel <= 1e-4:
            break
        y = y + delta * resid
    return it_done, list(pred.history), prox.sigma


def test_sharded_mc_loop_matches_oracle():
    from oracle import oracle as O

    res = _run(2, _worker_mc)
    assert not any(isinstance(r, str) for r in res), res
    colptr, rowidx, vals, _, _ = _mc_instance()
    _, s_ref, _, st = O.mc_svt(120, 120, colptr, rowidx, vals, O.SvdBackend.blws(seed=8))
    for it, hist, s in res:
        assert it == st.iterations and hist == st.predicted_ranks
        assert np.abs(s - s_ref).max() <= 1e-8 * s_ref.max()


def test_shard_csc_roundtrip():
    from paper_1012_0365_b200.dist import row_partition, shard_csc

    colptr, rowidx, vals, _, _ = _mc_instance()
    seen = np.zeros(len(vals), dtype=int)
    for r in range(3):
        row0, rows = row_partition(120, 3, r)
        lp, lr, lv, pos = shard_csc(colptr, rowidx, vals, row0, rows)
        seen[pos] += 1
        assert lp[-1] == len(lv) and np.all((lr >= 0) & (lr < rows))
        assert np.array_equal(lv, vals[pos]) and np.array_equal(lr + row0, rowidx[pos])
        assert np.all(np.diff(lp) >= 0)
    assert np.all(seen == 1)


def test_bench_sharded_inputs_are_rank_count_independent():
    # bench.py --mode sharded generates W per rank in 512-row chunks: the
    # shards of any rank count concatenate to the whole matrix
    import torch

    import bench
    from paper_1012_0365_b200 import dist as D

    m, n = 1300, 40
    full = bench._chunked_noise(0, m, n, 7, torch.device("cpu"))
    for world in (1, 2, 3, 8):
        parts = [bench._chunked_noise(*D.row_partition(m, world, r), n, 7, torch.device("cpu")) for r in range(world)]
        assert torch.equal(torch.cat(parts), full)
