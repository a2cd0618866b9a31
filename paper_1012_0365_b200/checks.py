"""Reference correctness gates on the GPU path.

Restates bench/checks.hpp:38-139 of the reference (same Rng draws, sizes,
tolerances and control flow) with every computation on the device:
  * theorem1_suite: the spectrum of the explicit symmetric embedding
    [[0, W], [W^T, 0]] (device sym_evd_small) is {+sigma} u {-sigma} u {0}
    with sigma from the device full_svd_small; the operator's paired apply
    reproduces the explicit embedding exactly; a Lanczos partial SVD unpacks
    orthonormal U, V;
  * prox_agreement_suite: after 5 warm-up steps on a drifting sequence, the
    Blws and Lanczos evaluations of the prox (svt) match the exact singular
    value threshold to 1e-5 relative Frobenius norm.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import api


@dataclass
class CheckReport:
    total: int = 0
    failed: int = 0
    failures: list = field(default_factory=list)
    values: list = field(default_factory=list)  # per-trial measured errors

    def ok(self) -> bool:
        return self.failed == 0

    def record(self, passed: bool, what: str) -> None:
        self.total += 1
        if not passed:
            self.failed += 1
            self.failures.append(what)


def _explicit_aug(w):
    m, n = w.shape
    t = np.zeros((m + n, m + n))
    t[:m, m:] = w
    t[m:, :m] = w.T
    return t


def _kw(mod, ctx):
    # the device API takes the context; the oracle module (same names) does not
    return {"ctx": ctx} if mod is api else {}


def singular_value_threshold(w, eps, ctx=None, mod=api):
    """Exact prox of eps ||.||_* (svt.hpp:20-35 applied to a full SVD)."""
    u, s, v = mod.full_svd_small(w, **_kw(mod, ctx))
    d = np.maximum(s - eps, 0.0)
    return (u * d) @ v.T


def theorem1_suite(trials: int, seed: int, ctx: api.Context | None = None, mod=api) -> CheckReport:
    rep = CheckReport()
    rng = mod.Rng(seed)
    ctx = ctx or (api.default_context() if mod is api else None)
    kw = _kw(mod, ctx)
    for t in range(trials):
        m = 2 + rng.uniform_index(39)
        n = 2 + rng.uniform_index(39)
        w = rng.gaussian_matrix(m, n)
        _, sig, _ = mod.full_svd_small(w, **kw)
        p = min(m, n)
        expected = np.zeros(m + n)
        expected[:p] = sig
        expected[m + n - p:] = -sig[::-1]
        expected = np.sort(expected)[::-1]
        aug = _explicit_aug(w)
        vals, _ = mod.sym_evd_small(aug, **kw)
        scale = max(sig[0], 1.0)
        what = f"theorem1 trial {t} ({m}x{n})"
        rep.record(np.abs(vals - expected).max() <= 1e-10 * scale, what + ": spectrum")
        op = mod.DenseOperator(w, **kw)
        left = np.hstack([np.eye(m), np.zeros((m, n))])
        right = np.hstack([np.zeros((n, m)), np.eye(n)])
        top, bot = op.apply_pair_block(left, right)
        rep.record(np.array_equal(np.vstack([top, bot]), aug), what + ": operator action")
        r = min(3, p)
        u, s, v, _ = mod.lanczos_partial_svd(op, r, tol=1e-9, seed=rng.next_u64())
        got = len(s)
        u_orth = np.linalg.norm(u.T @ u - np.eye(got))
        v_orth = np.linalg.norm(v.T @ v - np.eye(got))
        rep.record(got >= 1 and u_orth <= 1e-8 and v_orth <= 1e-8, what + ": unpacked orthonormality")
    return rep


def prox_agreement_suite(trials: int, seed: int, ctx: api.Context | None = None, mod=api,
                         tol: float = 1e-5) -> CheckReport:
    rep = CheckReport()
    rng = mod.Rng(seed)
    ctx = ctx or (api.default_context() if mod is api else None)
    kw = _kw(mod, ctx)
    m, true_rank, warm_steps = 200, 30, 5
    for t in range(trials):
        base = rng.gaussian_matrix(m, true_rank) @ rng.gaussian_matrix(m, true_rank).T
        drift = rng.gaussian_matrix(m, m)
        drift *= 1e-3 * np.linalg.norm(base) / np.linalg.norm(drift)
        final_w = base + float(warm_steps) * drift
        _, sig, _ = mod.full_svd_small(final_w, **kw)
        eps = 0.5 * (sig[9] + sig[10])
        a_exact = singular_value_threshold(final_w, eps, ctx, mod)

        blws = mod.SvdBackend.blws(block_steps=2, seed=rng.next_u64(), **kw)
        pred = mod.RankPredictor(10, 5, m)
        op = mod.DenseOperator(base, **kw)
        res = None
        for i in range(warm_steps + 1):
            op.assign(base + float(i) * drift)
            res = mod.svt(op, eps, blws, pred)
        blws_err = np.linalg.norm(res.dense() - a_exact) / np.linalg.norm(a_exact)

        lan = mod.SvdBackend.lanczos(ritz_tol=1e-9, seed=rng.next_u64(), **kw)
        lpred = mod.RankPredictor(10, 5, m)
        op.assign(final_w)
        lres = mod.svt(op, eps, lan, lpred)
        lan_err = np.linalg.norm(lres.dense() - a_exact) / np.linalg.norm(a_exact)
        what = f"prox agreement trial {t} blws={blws_err:.3e} lanczos={lan_err:.3e}"
        rep.values.append((blws_err, lan_err))
        rep.record(blws_err <= tol, what + ": blws")
        rep.record(lan_err <= tol, what + ": lanczos")
    return rep
