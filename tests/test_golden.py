"""Golden fixtures (tests/golden/oracle_small.npz, made by
tests/golden/make_golden.py from the oracle): the oracle must keep
reproducing them (CPU), and the GPU path must match them (gpu)."""
import os

import numpy as np
import pytest

from conftest import principal_angle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_small.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def test_oracle_reproduces_golden(O, gold):
    r = O.Rng(42)
    assert np.array_equal(np.array([r.next_u64() for _ in range(8)], dtype=np.uint64), gold["rng_u64_seed42"])
    r = O.Rng(7).split(3)
    assert np.array_equal(np.array([r.normal() for _ in range(9)]), gold["rng_normal_seed7_split3"])
    assert np.array_equal(O.sample_distinct(1000, 50, O.Rng(5)), gold["sample_distinct_1000_50_seed5"])
    qr = O.thin_qr(gold["qr_in"])
    assert np.abs(qr.q - gold["qr_q"]).max() <= 1e-13 and np.abs(qr.r - gold["qr_r"]).max() <= 1e-13
    assert np.abs(O.sym_evd_small(gold["evd_in"])[0] - gold["evd_vals"]).max() <= 1e-12


def test_capi_rng_matches_golden(G, gold):
    r = G.Rng(42)
    assert np.array_equal(np.array([r.next_u64() for _ in range(8)], dtype=np.uint64), gold["rng_u64_seed42"])
    r = G.Rng(7).split(3)
    assert np.array_equal(np.array([r.normal() for _ in range(9)]), gold["rng_normal_seed7_split3"])
    assert np.array_equal(G.sample_distinct(1000, 50, G.Rng(5)), gold["sample_distinct_1000_50_seed5"])


@pytest.mark.gpu
def test_gpu_matches_golden(G, gold):
    q, r, rank = G.thin_qr(gold["qr_in"])
    assert np.abs(q - gold["qr_q"]).max() <= 1e-10 and rank == 4
    vals, _ = G.sym_evd_small(gold["evd_in"])
    assert np.abs(vals - gold["evd_vals"]).max() <= 1e-12 * np.abs(gold["evd_vals"]).max()
    w0, d = gold["blws_w0"], gold["blws_delta"]
    warm = G.WarmStart(gold["blws_warm_u"], gold["blws_warm_v"], gold["blws_warm_s"])
    op = G.DenseOperator(w0)
    rng = G.Rng(99)
    for i in range(1, 6):
        op.assign(w0 + i * 0.01 * d)
        warm = G.blws_svd(op, warm, 2, 8, rng).warm
        ref = gold["blws_sigma"][i - 1]
        assert np.abs(warm.sigma - ref).max() <= 1e-10 * ref.max()
    a, e, st, _ = G.rpca_adm(gold["rpca_d"], G.SvdBackend.blws(seed=3 ^ 0x5BDBEEF))
    it, rank_hat, e_l0, mv = gold["rpca_iters"]
    assert abs(st.iterations - it) <= 1 and st.rank_hat == rank_hat
    assert np.linalg.norm(a - gold["rpca_a"]) <= 1e-6 * np.linalg.norm(gold["rpca_a"])
    assert np.linalg.norm(e - gold["rpca_e"]) <= 1e-6 * np.linalg.norm(gold["rpca_e"])
