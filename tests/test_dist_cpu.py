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


def _case(seed=7, m=120, n=90, r=6):
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
