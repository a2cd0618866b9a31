"""Regenerates tests/golden/*.npz from the CPU oracle (test infrastructure).

The reference ships no golden vectors; these fixtures freeze
the oracle's outputs on small seeded cases so (a) the oracle cannot drift
silently and (b) the GPU parity tests have committed expected values that do
not need the oracle at run time. Run: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import oracle as O  # noqa: E402
from paper_1012_0365_b200 import synth  # noqa: E402


def main():
    out = {}
    # rng known answers (core/rng.hpp)
    r = O.Rng(42)
    out["rng_u64_seed42"] = np.array([r.next_u64() for _ in range(8)], dtype=np.uint64)
    r = O.Rng(7).split(3)
    out["rng_normal_seed7_split3"] = np.array([r.normal() for _ in range(9)])
    out["sample_distinct_1000_50_seed5"] = O.sample_distinct(1000, 50, O.Rng(5))
    # thin_qr / sym_evd
    a = O.Rng(17).gaussian_matrix(20, 4)
    qr = O.thin_qr(a)
    out["qr_in"], out["qr_q"], out["qr_r"] = a, qr.q, qr.r
    g = O.Rng(23).gaussian_matrix(12, 12)
    t = 0.5 * (g + g.T)
    out["evd_in"], out["evd_vals"] = t, O.sym_evd_small(t)[0]
    # BLWS drifting sequence (test_block_lanczos.cpp:216-241): sigma per call
    rng = O.Rng(37)
    m, rr = 120, 8
    u0 = O.thin_qr(rng.gaussian_matrix(m, 12)).q
    v0 = O.thin_qr(rng.gaussian_matrix(m, 12)).q
    s0 = 100.0 * 0.7 ** np.arange(12)
    w0 = (u0 * s0) @ v0.T
    d = rng.gaussian_matrix(m, m)
    d *= 0.01 * np.linalg.norm(w0) / np.linalg.norm(d)
    uu, ss, vv = O.full_svd_small(w0)
    warm = O.WarmStart(uu[:, :rr].copy(order="F"), vv[:, :rr].copy(order="F"), ss[:rr].copy())
    op = O.DenseOperator(w0)
    brng = O.Rng(99)
    sig = []
    for i in range(1, 6):
        op.assign(w0 + i * 0.01 * d)
        warm = O.blws_svd(op, warm, 2, rr, brng).warm
        sig.append(warm.sigma.copy())
    out["blws_w0"], out["blws_delta"] = w0, d
    out["blws_warm_u"], out["blws_warm_v"], out["blws_warm_s"] = uu[:, :rr], vv[:, :rr], ss[:rr]
    out["blws_sigma"] = np.array(sig)
    # RPCA on a small C1-recipe instance
    dd, a0, _, _ = synth.rpca_lowrank_sparse(60, 4, 180, 3, O.Rng, O.sample_distinct)
    a_o, e_o, st, _ = O.rpca_adm(dd, O.SvdBackend.blws(seed=3 ^ 0x5BDBEEF), truth=a0)
    out["rpca_d"], out["rpca_a"], out["rpca_e"] = dd, a_o, e_o
    out["rpca_iters"] = np.array([st.iterations, st.rank_hat, st.e_l0, st.matvec_count])
    out["rpca_residuals"] = np.array(st.residual_history)
    out["rpca_predicted"] = np.array(st.predicted_ranks)
    np.savez_compressed(os.path.join(HERE, "oracle_small.npz"), **out)
    print("wrote", os.path.join(HERE, "oracle_small.npz"), sorted(out))


if __name__ == "__main__":
    main()
