"""One solve of a BASELINE config with no warm-up solve before it, so that an
`ncu -k regex:... -c N` capture sees the full-size launches (K7 alm_fused_k,
the reseed Lanczos kernel, K8 csr_spmm_k, K9 mc_sampled_k).

usage: python tools/probes/solver_kernels.py C3|C4
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1012_0365_b200 as B  # noqa: E402
from paper_1012_0365_b200 import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
if cfg == "C3":
    d, a0, _, _ = synth.rpca_lowrank_sparse(2000, 100, 400000, 1, B.Rng, B.sample_distinct)
    _, _, st, _ = B.rpca_adm(d, B.SvdBackend.blws(seed=1 ^ 0x5BDBEEF), truth=a0, want_outputs=False)
else:
    colptr, rowidx, vals, ml, mr = synth.mc_lowrank(10000, 50, 10_000_000, 1, B.Rng, B.sample_distinct)
    _, _, _, st = B.mc_svt(10000, 10000, colptr, rowidx, vals, B.SvdBackend.blws(seed=1 ^ 0x5BDBEEF),
                           tol_outer=1e-6, truth_ml=ml, truth_mr=mr, cap=512)
print(cfg, st.iterations, st.rank_hat, st.rel_err, flush=True)
