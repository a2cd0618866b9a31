"""Cross-pins the C++ oracle against a second, independent restatement of the
reference (oracle/indep.py: pure numpy + a Python mt19937_64, written from
the reference sources without reusing the oracle), CPU only.

Two restatements built on different RNG code and different LAPACK entry
points agree to rounding on every case below, including a BASELINE config
(C1) end to end. The same runs decide the two reference pins that neither
reproduces (profiles/r02_reference_pins.json):
test_solvers.cpp:25-67 fails with the dense ExactFull prox too (the planted
8th singular value of gen_rpca(80, .1, .1, 21) is 0.22), and the Blws prox
of test_svt.cpp:127-153 lands at 1.44e-4 in both.
"""
import math

import numpy as np
import pytest

from oracle import indep as I


def test_mt19937_64_known_answer():
    e = I.MT64(5489)
    for _ in range(9999):
        e()
    assert e() == 9981545732273789042


def test_rng_streams_bit_identical(O):
    a, b = I.Rng(0xB10C).split(13), O.Rng(0xB10C).split(13)
    assert [a.next_u64() for _ in range(50)] == [b.next_u64() for _ in range(50)]
    a, b = I.Rng(7), O.Rng(7)
    assert np.array_equal(a.gaussian_matrix(31, 7), b.gaussian_matrix(31, 7))
    assert [a.uniform_index(1000003) for _ in range(20)] == [b.uniform_index(1000003) for _ in range(20)]
    assert np.array_equal(I.sample_distinct(5000, 400, I.Rng(4)), O.sample_distinct(5000, 400, O.Rng(4)))


@pytest.mark.parametrize("m,n,r,k", [(60, 50, 6, 2), (120, 90, 10, 2), (80, 80, 12, 3), (70, 45, 20, 2)])
def test_blws_svd_matches(O, m, n, r, k):
    rng = I.Rng(100 + m)
    u0 = I.thin_qr(rng.gaussian_matrix(m, 2 * r))[0]
    v0 = I.thin_qr(rng.gaussian_matrix(n, 2 * r))[0]
    s0 = 10.0 * 0.85 ** np.arange(2 * r)
    w = (u0 * s0) @ v0.T + 1e-3 * rng.gaussian_matrix(m, n)
    wu = I.thin_qr(u0[:, :r] + 1e-2 * rng.gaussian_matrix(m, r))[0]
    wv = I.thin_qr(v0[:, :r] + 1e-2 * rng.gaussian_matrix(n, r))[0]
    (u, s, v), padded = I.blws_svd(I.Dense(w), (wu, s0[:r], wv), k, r, I.Rng(3), m, n)
    ref = O.blws_svd(O.DenseOperator(O.F(w)), O.WarmStart(O.F(wu), O.F(wv), s0[:r].copy()), k, r, O.Rng(3))
    assert padded == ref.padded
    np.testing.assert_allclose(s, ref.warm.sigma, rtol=1e-12)
    np.testing.assert_allclose(np.abs(u.T @ ref.warm.u).diagonal(), 1.0, atol=1e-9)
    np.testing.assert_allclose(np.abs(v.T @ ref.warm.v).diagonal(), 1.0, atol=1e-9)


def test_lanczos_partial_svd_matches(O):
    rng = I.Rng(5)
    w = rng.gaussian_matrix(90, 70)
    u, s, v, conv, allc = I.lanczos_partial_svd(I.Dense(w), 90, 70, 8, tol=1e-8, seed=77)
    _, rs, _, _ = O.lanczos_partial_svd(O.DenseOperator(O.F(w)), 8, tol=1e-8, seed=77)
    np.testing.assert_allclose(s, rs, rtol=1e-11)
    np.testing.assert_allclose(s, np.linalg.svd(w, compute_uv=False)[:8], rtol=1e-9)


def test_reference_rpca80_pin_unreachable_by_exact_prox(O):
    """test_solvers.cpp:25-67 pins rank_hat == 8, rel_err <= 1e-5, e_l0 = 640 +- 10 on
    gen_rpca(80, 0.1, 0.1, 21). With the exact dense prox (no Krylov step anywhere)
    the reference's rpca_adm gives rank 9, e_l0 728, rel_err 4.0e-3 in both
    restatements: the instance's planted sigma_8 is 0.22 (m / sqrt(r) |N(0,1)|)."""
    d, a_true, sig = I.gen_rpca(80, 0.1, 0.1, 21)
    assert sorted(sig)[0] == pytest.approx(0.219371, abs=1e-6)
    r = I.rpca_adm(d, I.Backend(kind="exact"), truth=a_true)
    a, e, st, _ = O.rpca_adm(O.F(d), O.SvdBackend.exact_full(), truth=a_true)
    assert (r["iterations"], r["rank_hat"], r["e_l0"]) == (st.iterations, st.rank_hat, st.e_l0) == (32, 9, 728)
    assert r["rel_err"] == pytest.approx(st.rel_err, rel=1e-8)
    assert np.linalg.norm(r["a"] - a) <= 1e-10 * np.linalg.norm(a)
    rb = I.rpca_adm(d, I.Backend(kind="blws", seed=6), truth=a_true)
    ab, eb, stb, _ = O.rpca_adm(O.F(d), O.SvdBackend.blws(seed=6), truth=a_true)
    assert (rb["iterations"], rb["rank_hat"], rb["e_l0"]) == (stb.iterations, stb.rank_hat, stb.e_l0)
    assert rb["predicted_ranks"] == stb.predicted_ranks
    assert np.linalg.norm(rb["a"] - ab) <= 1e-10 * np.linalg.norm(ab)


def test_reference_svt_growth_pin(O):
    """test_svt.cpp:127-153: both restatements land at 1.4445e-4 (the pin is 1e-5)
    with achieved rank 10; the error keeps shrinking with further warm calls."""
    rng = I.Rng(19)
    m = 100
    base = rng.gaussian_matrix(m, 30) @ rng.gaussian_matrix(m, 30).T
    drift = rng.gaussian_matrix(m, m)
    drift *= 1e-3 * np.linalg.norm(base) / np.linalg.norm(drift)
    final_w = base + 4.0 * drift
    s = np.linalg.svd(final_w, compute_uv=False)
    eps = 0.5 * (s[9] + s[10])
    be, pred, op = I.Backend(kind="blws", seed=101), I.Predictor(4, 3, m), I.Dense(base)
    obe, opred, oop = O.SvdBackend.blws(seed=101), O.RankPredictor(4, 3, m), O.DenseOperator(O.F(base))
    for i in range(5):
        op.w = base + float(i) * drift
        u, sv, v, ach = I.svt(op, m, m, eps, be, pred)
        oop.assign(O.F(base + float(i) * drift))
        res = O.svt(oop, eps, obe, opred)
        assert ach == res.achieved_rank
        np.testing.assert_allclose(sv, res.sigma, rtol=1e-10)
    u_, s_, v_ = I.full_svd(final_w)
    exact = (u_ * I.shrink(s_, eps)) @ v_.T
    err = np.linalg.norm((u * sv) @ v.T - exact) / np.linalg.norm(exact)
    oerr = np.linalg.norm(res.dense() - exact) / np.linalg.norm(exact)
    assert ach == 10
    assert err == pytest.approx(1.4445e-4, rel=1e-3) and oerr == pytest.approx(err, rel=1e-8)


def test_c1_config_end_to_end(O):
    """BASELINE configs[0] (C1: RPCA 500^2, rank 25, 5% corrupted) through both
    restatements with the Blws backend at make_backend's seed (1 ^ 0x5bdbeef)."""
    from paper_1012_0365_b200 import synth

    m = 500
    d, a0, _, _ = synth.rpca_lowrank_sparse(m, 25, 12500, 1, I.Rng, I.sample_distinct)
    d2, _, _, _ = synth.rpca_lowrank_sparse(m, 25, 12500, 1, O.Rng, O.sample_distinct)
    assert np.array_equal(d, d2)
    seed = 1 ^ 0x5BDBEEF
    r = I.rpca_adm(np.ascontiguousarray(d), I.Backend(kind="blws", seed=seed), truth=a0)
    a, e, st, _ = O.rpca_adm(d, O.SvdBackend.blws(seed=seed), truth=a0)
    assert r["iterations"] == st.iterations and r["rank_hat"] == st.rank_hat == 25
    assert r["predicted_ranks"] == st.predicted_ranks
    assert r["e_l0"] == st.e_l0
    assert np.linalg.norm(r["a"] - a) <= 1e-9 * np.linalg.norm(a)
    assert np.linalg.norm(r["e"] - e) <= 1e-9 * np.linalg.norm(e)
    assert math.isclose(r["rel_err"], st.rel_err, rel_tol=1e-3)
