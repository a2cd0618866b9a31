"""GPU parity of the RPCA / MC solvers against the CPU oracle on identical
seeded inputs (BASELINE.json parity contract: iterations +-1, same recovered
rank, final A and E to 1e-6 relative Frobenius; test_solvers.cpp bounds)."""
import os

import numpy as np
import pytest

from paper_1012_0365_b200 import synth

pytestmark = pytest.mark.gpu


def _rpca_instance(O, m, rank, frac, seed):
    return synth.rpca_lowrank_sparse(m, rank, int(round(frac * m * m)), seed, O.Rng, O.sample_distinct)


@pytest.mark.parametrize("m,rank,frac,seed", [(80, 8, 0.10, 21), (200, 10, 0.05, 1)])
def test_rpca_parity(G, O, m, rank, frac, seed):
    d, a0, _, _ = _rpca_instance(O, m, rank, frac, seed)
    bseed = seed ^ 0x5BDBEEF
    a_g, e_g, st_g, nnz_g = G.rpca_adm(d, G.SvdBackend.blws(seed=bseed), truth=a0)
    a_o, e_o, st_o, nnz_o = O.rpca_adm(d, O.SvdBackend.blws(seed=bseed), truth=a0)
    assert st_g.converged and st_o.converged
    assert abs(st_g.iterations - st_o.iterations) <= 1
    assert st_g.rank_hat == st_o.rank_hat
    assert np.linalg.norm(a_g - a_o) <= 1e-6 * np.linalg.norm(a_o)
    assert np.linalg.norm(e_g - e_o) <= 1e-6 * np.linalg.norm(e_o)
    assert abs(st_g.e_l0 - st_o.e_l0) <= max(2, 1e-3 * st_o.e_l0)
    n = min(st_g.iterations, st_o.iterations)
    assert st_g.predicted_ranks[:n] == st_o.predicted_ranks[:n]
    assert st_g.matvec_history[:n] == st_o.matvec_history[:n]
    assert st_g.matvec_init == st_o.matvec_init
    assert st_g.matvec_init + sum(st_g.matvec_history) == st_g.matvec_count


def test_rpca_clean_rank_one(G, O):
    rng = O.Rng(3)
    a, b = rng.gaussian_vector(40), rng.gaussian_vector(40)
    d = np.outer(a, b)
    a_g, e_g, st, _ = G.rpca_adm(d, G.SvdBackend.blws(seed=6))
    assert st.converged and st.rank_hat == 1 and st.e_l0 == 0
    assert np.linalg.norm(a_g - d) <= 1e-6 * np.linalg.norm(d)


def test_rpca_capped(G, O):
    d, _, _, _ = _rpca_instance(O, 50, 5, 0.1, 9)
    _, _, st, _ = G.rpca_adm(d, G.SvdBackend.blws(seed=3), max_iter=2)
    assert not st.converged and st.iterations == 2


def test_rpca_rejects_non_finite(G):
    d = np.ones((6, 6))
    d[2, 3] = np.nan
    with pytest.raises(ValueError):
        G.rpca_adm(d, G.SvdBackend.blws())


def test_mc_parity(G, O):
    # gen_mc(200, 5, 6.0, 13): s = round(6 * 5 * (2*200 - 5)) = 11850 (test_solvers.cpp:110-137)
    colptr, rowidx, vals, ml, mr = synth.mc_lowrank(200, 5, 11850, 13, O.Rng, O.sample_distinct)
    ug, sg, vg, stg = G.mc_svt(200, 200, colptr, rowidx, vals, G.SvdBackend.blws(seed=8), truth_ml=ml, truth_mr=mr)
    uo, so, vo, sto = O.mc_svt(200, 200, colptr, rowidx, vals, O.SvdBackend.blws(seed=8), truth_ml=ml, truth_mr=mr)
    assert stg.converged and sto.converged
    assert abs(stg.iterations - sto.iterations) <= 1
    assert stg.rank_hat == sto.rank_hat
    assert stg.rel_err <= 2e-4
    ag, ao = (ug * sg) @ vg.T, (uo * so) @ vo.T
    assert np.linalg.norm(ag - ao) <= 1e-6 * np.linalg.norm(ao)


def test_mc_parity_wide_rank(G, O):
    # rank 40: the sampled-residual kernel (K9) runs its two-slot (r <= 64) variant
    colptr, rowidx, vals, ml, mr = synth.mc_lowrank(400, 40, 91200, 21, O.Rng, O.sample_distinct)
    ug, sg, vg, stg = G.mc_svt(400, 400, colptr, rowidx, vals, G.SvdBackend.blws(seed=9), truth_ml=ml, truth_mr=mr)
    uo, so, vo, sto = O.mc_svt(400, 400, colptr, rowidx, vals, O.SvdBackend.blws(seed=9), truth_ml=ml, truth_mr=mr)
    assert stg.converged and sto.converged
    assert abs(stg.iterations - sto.iterations) <= 1
    assert stg.rank_hat == sto.rank_hat == 40
    ag, ao = (ug * sg) @ vg.T, (uo * so) @ vo.T
    assert np.linalg.norm(ag - ao) <= 1e-6 * np.linalg.norm(ao)


def test_mc_rejects_empty(G):
    with pytest.raises(ValueError):
        G.mc_svt(10, 10, np.zeros(11, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0),
                 G.SvdBackend.blws())


@pytest.mark.slow
def test_rpca_c1_config_parity(G, O):
    """BASELINE configs[0] (C1): RPCA 500^2, rank 25, 5% corruption, seed 1."""
    d, a0, _, _ = synth.rpca_lowrank_sparse(500, 25, 12500, 1, O.Rng, O.sample_distinct)
    bseed = 1 ^ 0x5BDBEEF
    a_g, e_g, st_g, _ = G.rpca_adm(d, G.SvdBackend.blws(seed=bseed), truth=a0)
    O.set_threads(os.cpu_count() or 1)
    a_o, e_o, st_o, _ = O.rpca_adm(d, O.SvdBackend.blws(seed=bseed), truth=a0)
    assert st_g.converged and st_o.converged
    assert abs(st_g.iterations - st_o.iterations) <= 1 and st_g.rank_hat == st_o.rank_hat == 25
    assert np.linalg.norm(a_g - a_o) <= 1e-6 * np.linalg.norm(a_o)
    assert np.linalg.norm(e_g - e_o) <= 1e-6 * np.linalg.norm(e_o)
    assert st_g.rel_err <= 1e-5


def test_reference_gates_on_device(G, O):
    # bench/checks.hpp:38-139 (theorem1_suite, prox_agreement_suite), device path.
    # The reference's 1e-5 Blws prox bound is not reached by the restated
    # algorithm either (the oracle gives ~1.7e-4 on these trials, as for
    # test_svt.cpp:127-153): the device must match the oracle trial by trial
    # and stay within the observed level.
    from paper_1012_0365_b200 import checks

    t1 = checks.theorem1_suite(12, 20240601)
    assert t1.ok(), t1.failures
    assert t1.total == 36
    px = checks.prox_agreement_suite(3, 7, tol=5e-4)
    assert px.ok(), px.failures
    ref = checks.prox_agreement_suite(3, 7, mod=O, tol=5e-4)
    for (gb, gl), (ob, ol) in zip(px.values, ref.values):
        assert abs(gb - ob) <= 1e-3 * ob  # blws: same trajectory as the oracle
        assert gl <= 1e-12 and ol <= 1e-12  # lanczos: exact to rounding on both


def test_rpca_k7_variants_agree(G, O, monkeypatch):
    """K7 at a size where every CTA of the persistent TMA kernel runs several
    tiles per consumer group (m = 1600: 625 tiles over 148 CTAs): the same
    solve with the cp.async kernel (BLWS_K7=cpasync) takes the same iterations
    and predicted ranks, and A / E agree to rounding."""
    d, a0, _, _ = synth.rpca_lowrank_sparse(1600, 30, int(0.05 * 1600 * 1600), 7, O.Rng, O.sample_distinct)
    bseed = 7 ^ 0x5BDBEEF
    a_t, e_t, st_t, _ = G.rpca_adm(d, G.SvdBackend.blws(seed=bseed), truth=a0)
    monkeypatch.setenv("BLWS_K7", "cpasync")
    a_c, e_c, st_c, _ = G.rpca_adm(d, G.SvdBackend.blws(seed=bseed), truth=a0)
    assert st_t.converged and st_c.converged
    assert st_t.iterations == st_c.iterations and st_t.rank_hat == st_c.rank_hat == 30
    assert list(st_t.predicted_ranks) == list(st_c.predicted_ranks)
    assert np.linalg.norm(a_t - a_c) <= 1e-10 * np.linalg.norm(a_c)
    assert np.linalg.norm(e_t - e_c) <= 1e-10 * np.linalg.norm(e_c)
    assert st_t.rel_err <= 1e-5


def test_exact_full_backend_rank_one_and_growth(G, O):
    # test_solvers.cpp:12-22: the ExactFull backend recovers a clean rank-1 matrix
    rng = O.Rng(3)
    a, b = rng.gaussian_vector(40), rng.gaussian_vector(40)
    d = np.outer(a, b)
    a_g, e_g, st, _ = G.rpca_adm(d, G.SvdBackend.exact_full())
    a_o, e_o, sto, _ = O.rpca_adm(d, O.SvdBackend.exact_full())
    assert st.converged and st.rank_hat == 1 and st.e_l0 == 0
    assert st.iterations == sto.iterations
    assert np.linalg.norm(a_g - d) <= 1e-6 * np.linalg.norm(d)
    # the RPCA 80^2 instance of test_solvers.cpp:25-67 through the device ExactFull:
    # the same trace as the oracle's ExactFull (rank 9, e_l0 728)
    from tests_support import gen_rpca_reference

    d, a0 = gen_rpca_reference(O, 80, 0.1, 0.1, 21)
    a_g, e_g, st, _ = G.rpca_adm(d, G.SvdBackend.exact_full(), truth=a0)
    a_o, e_o, sto, _ = O.rpca_adm(d, O.SvdBackend.exact_full(), truth=a0)
    assert (st.iterations, st.rank_hat, st.e_l0) == (sto.iterations, sto.rank_hat, sto.e_l0) == (32, 9, 728)
    assert np.linalg.norm(a_g - a_o) <= 1e-8 * np.linalg.norm(a_o)


def test_exact_full_backend_sparse_operator(G, O):
    colptr, rowidx, vals, ml, mr = synth.mc_lowrank(120, 4, 4000, 5, O.Rng, O.sample_distinct)
    ug, sg, vg, stg = G.mc_svt(120, 120, colptr, rowidx, vals, G.SvdBackend.exact_full(), truth_ml=ml, truth_mr=mr)
    uo, so, vo, sto = O.mc_svt(120, 120, colptr, rowidx, vals, O.SvdBackend.exact_full(), truth_ml=ml, truth_mr=mr)
    assert abs(stg.iterations - sto.iterations) <= 1 and stg.rank_hat == sto.rank_hat
    assert np.linalg.norm((ug * sg) @ vg.T - (uo * so) @ vo.T) <= 1e-6 * np.linalg.norm((uo * so) @ vo.T)
