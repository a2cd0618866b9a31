"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck) that
cover the hand-rolled synchronisation: the TMA + mbarrier GEMM
(dgemm_tma_kernel), the CholQR factor (cholqr_factor_k), the one-CTA and
cluster tridiagonalisations (sytrd_fused_k, sytrd_cluster_k, DSMEM), the
grid-synchronised Lanczos (lanczos_rows_k), the fused ALM kernel (alm_tma_k)
and the MC kernels (csr_spmm_k, mc_sampled_k). Each case is checked against
the oracle so a silent corruption also fails."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1012_0365_b200 as B  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1012_0365_b200 import synth  # noqa: E402


def blws_case(m, n, r):
    rng = O.Rng(5 + m)
    u0 = O.thin_qr(rng.gaussian_matrix(m, 2 * r)).q
    v0 = O.thin_qr(rng.gaussian_matrix(n, 2 * r)).q
    w = (u0 * (10.0 * 0.9 ** np.arange(2 * r))) @ v0.T + 1e-3 * rng.gaussian_matrix(m, n)
    wu = O.thin_qr(u0[:, :r] + 1e-2 * rng.gaussian_matrix(m, r)).q
    wv = O.thin_qr(v0[:, :r] + 1e-2 * rng.gaussian_matrix(n, r)).q
    s = 10.0 * 0.9 ** np.arange(r)
    g = B.blws_svd(B.DenseOperator(w), B.WarmStart(wu, wv, s), 2, r, B.Rng(3))
    o = O.blws_svd(O.DenseOperator(w), O.WarmStart(wu, wv, s), 2, r, O.Rng(3))
    err = np.abs(g.warm.sigma - o.warm.sigma).max() / o.warm.sigma.max()
    assert err <= 1e-10, err
    return err


def main():
    print("blws 600x500 r=24 (fused sytrd, b <= 112 CholQR)", blws_case(600, 500, 24), flush=True)
    print("blws 700x600 r=130 (cluster sytrd order 260, chol_inv path)", blws_case(700, 600, 130), flush=True)
    d, a0, _, _ = synth.rpca_lowrank_sparse(160, 6, 1280, 1, O.Rng, O.sample_distinct)
    ag, eg, stg, _ = B.rpca_adm(d, B.SvdBackend.blws(seed=9), truth=a0)
    ao, eo, sto, _ = O.rpca_adm(d, O.SvdBackend.blws(seed=9), truth=a0)
    assert stg.iterations == sto.iterations and np.linalg.norm(ag - ao) <= 1e-6 * np.linalg.norm(ao)
    print("rpca 160^2 (alm_tma_k, lanczos_rows_k)", stg.iterations, flush=True)
    colptr, rowidx, vals, ml, mr = synth.mc_lowrank(150, 4, 6000, 2, O.Rng, O.sample_distinct)
    ug, sg, vg, stg = B.mc_svt(150, 150, colptr, rowidx, vals, B.SvdBackend.blws(seed=8), truth_ml=ml, truth_mr=mr)
    uo, so, vo, sto = O.mc_svt(150, 150, colptr, rowidx, vals, O.SvdBackend.blws(seed=8), truth_ml=ml, truth_mr=mr)
    assert abs(stg.iterations - sto.iterations) <= 1
    print("mc 150^2 (csr_spmm_k, mc_sampled_k, csr_spmv_pair_k)", stg.iterations, flush=True)
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
