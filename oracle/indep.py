"""TEST INFRASTRUCTURE ONLY — a second, independent restatement of the
reference path in pure numpy (numpy.linalg for QR / EVD / SVD, a Python
mt19937_64), written from the reference sources without reusing the C++
oracle. Its job is to cross-check the C++ oracle (oracle/blws_oracle.cpp) and
to decide whether the reference's own pins that the oracle misses are
reachable by the reference's algorithm at all:

* ``test_solvers.cpp:25-67`` (RPCA 80², rank_hat == 8, rel_err <= 1e-5,
  e_l0 = 640 +- 10) — run with the dense ExactFull prox, which has no Krylov
  approximation in it, so a miss here is the instance, not the restatement;
* ``test_svt.cpp:127-153`` / ``bench/checks.hpp:91-139`` (Blws prox vs the
  exact prox to 1e-5).

Only tests/ and tools/pin_reference_tests.py import this module.

Reference map: Rng ``core/rng.hpp:17-90``; thin_qr ``core/qr.hpp:24-47``;
sym_evd ``core/small_dense.hpp:24-62``; LanczosRun ``lanczos.hpp:85-175``;
ritz_checkpoint ``:191-207``; partial_evd_impl ``:209-252``;
lanczos_partial_svd ``:289-329``; spectral_norm ``:332-340``;
block_lanczos_procedure ``block_lanczos.hpp:70-126``; bl_evd ``:139-152``;
adapt_subspace ``:157-187``; blws_svd ``:204-261``; SvdBackend ``svt.hpp:84-196``;
svt ``:216-254``; predict_rank ``:58-64``; rpca_adm ``solvers.hpp:72-157``;
gen_rpca ``synth.hpp:53-96``; sample_distinct ``:23-33``.
"""
from __future__ import annotations

import math

import numpy as np

_M64 = (1 << 64) - 1


class MT64:
    """std::mt19937_64 (C++ [rand.predef]: 10000th output 9981545732273789042)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _M64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _M64
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            y = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            v = mt[(i + 156) % 312] ^ (y >> 1)
            if y & 1:
                v ^= 0xB5026F5AA96619E9
            mt[i] = v
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M64


class Rng:
    """core/rng.hpp:17-90."""

    def __init__(self, seed: int):
        self.seed = seed & _M64
        self.eng = MT64(self.seed)
        self.spare = None

    def split(self, tag: int) -> "Rng":
        return Rng(self.seed ^ ((0x9E3779B97F4A7C15 * (tag + 1)) & _M64))

    def next_u64(self) -> int:
        return self.eng()

    def uniform(self, lo=None, hi=None) -> float:
        u = float(self.eng() >> 11) * 2.0 ** -53
        return u if lo is None else lo + (hi - lo) * u

    def uniform_index(self, n: int) -> int:
        limit = _M64 - _M64 % n
        while True:
            x = self.eng()
            if x < limit:
                return x % n

    def normal(self) -> float:
        if self.spare is not None:
            s, self.spare = self.spare, None
            return s
        while True:
            u1 = self.uniform()
            if u1 > 0.0:
                break
        u2 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        th = 6.283185307179586476925287 * u2
        self.spare = r * math.sin(th)
        return r * math.cos(th)

    def gaussian_matrix(self, rows: int, cols: int) -> np.ndarray:
        return np.array([self.normal() for _ in range(rows * cols)]).reshape(cols, rows).T.copy()

    def gaussian_vector(self, n: int) -> np.ndarray:
        return np.array([self.normal() for _ in range(n)])

    def unit_vector(self, n: int) -> np.ndarray:
        v = self.gaussian_vector(n)
        return v / np.linalg.norm(v)


def sample_distinct(n: int, s: int, rng: Rng) -> np.ndarray:
    """synth.hpp:23-33 (Floyd)."""
    chosen = set()
    for j in range(n - s, n):
        t = rng.uniform_index(j + 1)
        if t in chosen:
            chosen.add(j)
        else:
            chosen.add(t)
    return np.array(sorted(chosen), dtype=np.int64)


def thin_qr(a):
    """qr.hpp:24-47: Q with diag(R) >= 0; rank = #diag(R) > 1e-12 ||A||_F."""
    tau = 1e-12 * np.linalg.norm(a)
    q, r = np.linalg.qr(a)
    s = np.where(np.diag(r) < 0, -1.0, 1.0)
    q, r = q * s, r * s[:, None]
    return q, r, int((np.diag(r) > tau).sum())


def sym_evd(t):
    """small_dense.hpp:24-43 (descending)."""
    t = 0.5 * (t + t.T)
    w, v = np.linalg.eigh(t)
    return w[::-1].copy(), v[:, ::-1].copy()


def full_svd(a):
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    return u, s, vt.T


class Dense:
    """DenseOperator + counter (linear_operator.hpp:57-61,102-131)."""

    def __init__(self, w):
        self.w = np.asarray(w, dtype=np.float64)
        self.count = 0

    def pair(self, left, right):  # (W right, W^T left)
        self.count += right.shape[1] if right.ndim == 2 else 1
        return self.w @ right, self.w.T @ left


def aug_apply(op, x, m):
    """augmented_operator.hpp:39-57: (x; y) -> (W y; W^T x)."""
    zt, zb = op.pair(x[:m], x[m:])
    return np.concatenate([zt, zb], axis=0)


def lanczos_partial_svd(op, m, n, r, tol=1e-8, max_k=0, seed=0x1A2C705):
    """lanczos.hpp:289-329 over partial_evd_impl (:209-252) and LanczosRun (:85-175)."""
    dim = m + n
    q1 = np.zeros(dim)
    q1[:m] = Rng(seed).split(13).unit_vector(m)
    mk = min(max_k, dim) if max_k > 0 else min(dim, 10 * r + 20)
    mk = max(mk, min(dim, r))
    rng = Rng(seed).split(11)
    Q = np.zeros((dim, 0))
    alpha, beta = [], []
    nxt, coup, last_beta, tau, brk = q1, 0.0, 0.0, 0.0, False

    def step():
        nonlocal Q, nxt, coup, last_beta, tau, brk
        l = Q.shape[1]
        Q = np.concatenate([Q, nxt[:, None]], axis=1)
        if l > 0:
            beta.append(coup)
        r_ = aug_apply(op, Q[:, l], m)
        a = Q[:, l] @ r_
        r_ = r_ - a * Q[:, l]
        if l > 0:
            r_ = r_ - beta[-1] * Q[:, l - 1]
        r_ = r_ - Q @ (Q.T @ r_)
        r_ = r_ - Q @ (Q.T @ r_)
        alpha.append(a)
        if len(alpha) == 1:
            tau = 1e-12 * abs(a)
        last_beta = np.linalg.norm(r_)
        if last_beta <= tau or Q.shape[1] >= dim:
            brk = True
        else:
            brk, nxt, coup = False, r_ / last_beta, last_beta

    def restart():
        nonlocal nxt, coup, brk
        if Q.shape[1] >= dim:
            return False
        for _ in range(3):
            v = rng.gaussian_vector(dim)
            v /= np.linalg.norm(v)
            v = v - Q @ (Q.T @ v)
            v = v - Q @ (Q.T @ v)
            nv = np.linalg.norm(v)
            if nv > 1e-8:
                nxt, coup, brk = v / nv, 0.0, False
                return True
        return False

    k_target = min(mk, max(2 * r, 10))
    while True:
        if not brk and Q.shape[1] < k_target:
            step()
            continue
        k = Q.shape[1]
        T = np.diag(alpha) + np.diag(beta, 1) + np.diag(beta, -1)
        vals, vecs = sym_evd(T)
        lim = tol * abs(vals[0])
        conv = 0
        for j in range(k):
            if last_beta * abs(vecs[k - 1, j]) <= lim:
                conv += 1
            else:
                break
        done = conv >= r or k >= mk
        if not done:
            if brk:
                if not restart():
                    done = True
            else:
                k_target = min(mk, 2 * k_target)
        if done:
            avail = min(r, k)
            vals, U = vals[:avail], Q @ vecs[:, :avail]
            keep = 0
            while keep < avail and vals[keep] > 0:
                keep += 1
            s2 = math.sqrt(2.0)
            return (s2 * U[:m, :keep], vals[:keep].copy(), s2 * U[m:, :keep],
                    min(conv, avail, keep), avail == r and conv >= r and keep == r)


def spectral_norm(op, m, n):
    """lanczos.hpp:332-340."""
    _, s, _, _, _ = lanczos_partial_svd(op, m, n, 1, tol=1e-6, seed=0xB1F)
    return s[0] if len(s) else 0.0


def adapt_subspace(warm, r_new, m, n, rng):
    """block_lanczos.hpp:157-187."""
    if warm is None or warm[1].size == 0:
        u = thin_qr(rng.gaussian_matrix(m, r_new))[0]
        v = thin_qr(rng.gaussian_matrix(n, r_new))[0]
        return u, np.zeros(r_new), v
    u, s, v = warm
    r_old = s.size
    if r_new == r_old:
        return warm
    if r_new < r_old:
        return u[:, :r_new], s[:r_new], v[:, :r_new]
    add = r_new - r_old
    ue = np.concatenate([u, rng.gaussian_matrix(m, add)], axis=1)
    ve = np.concatenate([v, rng.gaussian_matrix(n, add)], axis=1)
    s2 = np.zeros(r_new)
    s2[:r_old] = s
    return thin_qr(ue)[0], s2, thin_qr(ve)[0]


def blws_svd(op, warm, k, r, rng, m, n):
    """block_lanczos.hpp:204-261 (block_lanczos_procedure :70-126, bl_evd :139-152)."""
    u, s, v = warm
    bs = s.size
    k_eff = k
    if r > k_eff * bs:
        k_eff = (r + bs - 1) // bs
    k_eff = max(min(k_eff, (m + n) // bs), 1)
    x = thin_qr(np.concatenate([u, v], axis=0) / math.sqrt(2.0))[0]
    blocks, Ms, Bs = [x], [], []
    z = aug_apply(op, x, m)
    scale = np.linalg.norm(z)
    M = x.T @ z
    Ms.append(0.5 * (M + M.T))
    for l in range(1, k_eff):
        R = z - blocks[-1] @ Ms[-1]
        if l > 1:
            R -= blocks[-2] @ Bs[-1].T
        if np.linalg.norm(R) <= 1e-10 * scale:
            break
        q, rr, rank = thin_qr(R)
        if rank < bs:
            break
        blocks.append(q)
        Bs.append(rr)
        z = aug_apply(op, q, m)
        scale = max(scale, np.linalg.norm(z))
        M = q.T @ z
        Ms.append(0.5 * (M + M.T))
    nb = len(blocks)
    T = np.zeros((nb * bs, nb * bs))
    for i in range(nb):
        T[i * bs:(i + 1) * bs, i * bs:(i + 1) * bs] = Ms[i]
        if i + 1 < nb:
            T[(i + 1) * bs:(i + 2) * bs, i * bs:(i + 1) * bs] = Bs[i]
            T[i * bs:(i + 1) * bs, (i + 1) * bs:(i + 2) * bs] = Bs[i].T
    vals, vecs = sym_evd(T)
    Q = np.concatenate(blocks, axis=1)
    floor = 1e-12 * abs(vals[0]) if vals.size else 0.0
    keep = 0
    while keep < vals.size and keep < r and vals[keep] > floor:
        keep += 1
    X = Q @ vecs[:, :keep] * math.sqrt(2.0)
    nu, nv = X[:m], X[m:]
    if keep > 0:
        nu, nv = thin_qr(nu)[0], thin_qr(nv)[0]
    nxt = (nu, vals[:keep].copy(), nv)
    padded = keep < r
    if padded:
        nxt = adapt_subspace(nxt if keep > 0 else None, r, m, n, rng)
    return nxt, padded


class Backend:
    """SvdBackend (svt.hpp:84-196): kind 'exact' or 'blws'."""

    def __init__(self, kind="blws", seed=0xB10C, block_steps=2, ritz_tol=1e-8, seed_margin=5):
        self.kind, self.rng, self.k, self.tol, self.margin = kind, Rng(seed), block_steps, ritz_tol, seed_margin
        self.warm, self.streak = None, 0

    def compute(self, op, m, n, r):
        p = min(m, n)
        if self.kind == "exact":
            u, s, v = full_svd(op.w)
            return u[:, :r], s[:r], v[:, :r], r, False
        held = self.warm[1].size if self.warm is not None else 0
        if held < r:
            margin = self.margin * (1 << min(self.streak, 5))
            self.streak += 1
            r_seed = min(p, r + margin)
            u, s, v, conv, allc = lanczos_partial_svd(op, m, n, r_seed, tol=self.tol, seed=self.rng.next_u64())
            ws = (u, s, v)
            if s.size < r_seed:
                ws = adapt_subspace(ws if s.size > 0 else None, r_seed, m, n, self.rng)
            self.warm = ws
            return ws[0], ws[1], ws[2], conv, not allc
        if r < held:
            self.streak = 0
        if held > r + 2 * self.margin:
            self.warm = adapt_subspace(self.warm, r + self.margin, m, n, self.rng)
        self.warm, padded = blws_svd(op, self.warm, self.k, self.warm[1].size, self.rng, m, n)
        conv = min(r, self.warm[1].size) if padded else self.warm[1].size
        return self.warm[0], self.warm[1], self.warm[2], conv, False


class Predictor:
    def __init__(self, r=10, increment=5, max_rank=1):
        self.r, self.inc, self.max_rank, self.history = r, increment, max_rank, []


def svt(op, m, n, eps, backend, pred):
    """svt.hpp:216-254 with predict_rank (:58-64)."""
    p = min(m, n)
    r = min(max(pred.r, 1), p)
    while True:
        u, s, v, conv, cap = backend.compute(op, m, n, r)
        have = s.size
        above = have > 0 and s[have - 1] > eps
        if not above or max(r, have) >= p:
            all_above = above
            break
        r = min(max(r, have) + pred.inc, p)
    ach = 0
    while ach < s.size and s[ach] > eps:
        ach += 1
    nxt = ach + (pred.inc if all_above else 1)
    pred.r = min(max(nxt, 1), pred.max_rank)
    pred.history.append(pred.r)
    return u[:, :ach], s[:ach] - eps, v[:, :ach], ach


def shrink(x, eps):
    return np.where(x > eps, x - eps, np.where(x < -eps, x + eps, 0.0))


def rpca_adm(d, backend, lam=0.0, tol=1e-7, max_iter=1000, rho=1.5, mu_max_factor=1e7, truth=None):
    """solvers.hpp:72-157. Returns a dict of the stats the reference reports."""
    m = d.shape[0]
    lam = lam if lam > 0 else 1.0 / math.sqrt(m)
    nd = np.linalg.norm(d)
    op = Dense(d)
    n2 = spectral_norm(op, m, m)
    mu = 1.25 / n2
    mu_max = mu * mu_max_factor
    y = d / max(n2, np.abs(d).max() / lam)
    e = np.zeros_like(d)
    a = np.zeros_like(d)
    pred = Predictor(10, 5, m)
    it, conv, rank, feas_hist = 0, False, 0, []
    for it in range(1, max_iter + 1):
        op.w = d - e + y / mu
        u, s, v, rank = svt(op, m, m, 1.0 / mu, backend, pred)
        a = (u * s) @ v.T
        e = shrink(d - a + y / mu, lam / mu)
        res = d - a - e
        y = y + mu * res
        mu = min(rho * mu, mu_max)
        feas = np.linalg.norm(res) / nd
        feas_hist.append(feas)
        if feas <= tol:
            conv = True
            break
    out = dict(iterations=it, converged=conv, rank_hat=rank, a=a, e=e, residual_history=feas_hist,
               e_l0=int((np.abs(e) > 1e-8 * np.abs(d).max()).sum()), predicted_ranks=list(pred.history))
    if truth is not None:
        out["rel_err"] = float(np.linalg.norm(a - truth) / np.linalg.norm(truth))
    return out


def gen_rpca(m, rank_frac, corrupt_frac, seed):
    """synth.hpp:53-96 (orthogonal model). Returns d, a_true, planted sigma."""
    r = int(round(rank_frac * m))
    base = Rng(seed)
    ru, rv, rs, rp, rval = (base.split(t) for t in (1, 2, 3, 4, 5))
    u = thin_qr(ru.gaussian_matrix(m, r))[0]
    v = thin_qr(rv.gaussian_matrix(m, r))[0]
    sig = (m / math.sqrt(r)) * np.array([abs(rs.normal()) for _ in range(r)])
    a = (u * sig) @ v.T
    nnz = int(round(corrupt_frac * m * m))
    e = np.zeros((m, m))
    for pos in sample_distinct(m * m, nnz, rp):
        e[pos % m, pos // m] = rval.uniform(-500.0, 500.0)
    return a + e, a, sig
