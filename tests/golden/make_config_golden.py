#!/usr/bin/env python
"""TEST INFRASTRUCTURE — golden traces of the CPU oracle on BASELINE configs
C3 (RPCA 2000², rank 100, 10 %) and C4 (MC 10⁴², rank 50, 10⁷ observed).

The oracle takes minutes here (C3 ~8 min, C4 longer on 8 cores), too long
for a pytest run or for the GPU box, so its trace is committed as a small
fixture and `tests/test_gpu_configs.py` compares the device solve against it.
Inputs are regenerated from the seed on both sides (the reference's RNG
recipe), so only the oracle's outputs are stored:

* iterations, converged, rank_hat, e_l0, rel_err, the predicted-rank and
  matvec histories, the per-iteration feasibility residuals;
* final singular values (MC) and, instead of the m x m A and E, Gaussian
  sketches A·G and E·G with G = Rng(0x5EED).gaussian_matrix(m, 16): the
  relative sketch error estimates the relative Frobenius error
  ||A - A_ref||_F / ||A_ref||_F (an unbiased JL estimate), plus the exact
  Frobenius norms.

Usage: python tests/golden/make_config_golden.py C3 C4 C5S
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1012_0365_b200 import synth  # noqa: E402

SEED = 1
SKETCH_SEED = 0x5EED
SKETCH_COLS = 16


def sketch(m):
    return O.Rng(SKETCH_SEED).gaussian_matrix(m, SKETCH_COLS)


def _hist(st):
    return dict(iterations=st.iterations, converged=bool(st.converged), rank_hat=st.rank_hat, e_l0=st.e_l0,
                rel_err=st.rel_err, matvec_count=st.matvec_count, matvec_init=st.matvec_init,
                predicted_ranks=np.array(st.predicted_ranks, dtype=np.int64),
                matvec_history=np.array(st.matvec_history, dtype=np.int64),
                residual_history=np.array(st.residual_history))


def c3():
    m, rank, frac = 2000, 100, 0.10
    d, a0, _, _ = synth.rpca_lowrank_sparse(m, rank, int(round(frac * m * m)), SEED, O.Rng, O.sample_distinct)
    O.set_threads(os.cpu_count() or 1)
    t = time.perf_counter()
    a, e, st, _ = O.rpca_adm(d, O.SvdBackend.blws(seed=SEED ^ 0x5BDBEEF), truth=a0)
    secs = time.perf_counter() - t
    g = sketch(m)
    out = _hist(st)
    out.update(a_sketch=a @ g, e_sketch=e @ g, a_fro=np.linalg.norm(a), e_fro=np.linalg.norm(e),
               d_fro=np.linalg.norm(d), oracle_seconds=secs, oracle_threads=os.cpu_count() or 1)
    return out


def c5s():
    """The C5 recipe (RPCA, rank = m / 100, 5 % corrupted, lambda = 1/sqrt(m))
    at m = 4000: the 40000^2 config itself needs ~100 GB of host memory in the
    oracle, so its recipe is pinned at a tenth of the order. Its
    cold Lanczos reseeds reach Ritz checkpoints above the reference's
    kSmallDenseLimit (4096, small_dense.hpp:13), where the reference throws
    std::invalid_argument; the trace is made with ORC_LIFT_SMALL_DENSE_LIMIT=1
    (the device path has no such limit) and records the largest order met."""
    os.environ["ORC_LIFT_SMALL_DENSE_LIMIT"] = "1"
    m, rank, frac = 4000, 40, 0.05
    d, a0, _, _ = synth.rpca_lowrank_sparse(m, rank, int(round(frac * m * m)), SEED, O.Rng, O.sample_distinct)
    O.set_threads(os.cpu_count() or 1)
    t = time.perf_counter()
    a, e, st, _ = O.rpca_adm(d, O.SvdBackend.blws(seed=SEED ^ 0x5BDBEEF), truth=a0)
    secs = time.perf_counter() - t
    g = sketch(m)
    out = _hist(st)
    out.update(a_sketch=a @ g, e_sketch=e @ g, a_fro=np.linalg.norm(a), e_fro=np.linalg.norm(e),
               d_fro=np.linalg.norm(d), oracle_seconds=secs, oracle_threads=os.cpu_count() or 1,
               max_evd_order=O.small_dense_max_order())
    return out


def c4():
    m, rank, nobs = 10000, 50, 10_000_000
    colptr, rowidx, vals, ml, mr = synth.mc_lowrank(m, rank, nobs, SEED, O.Rng, O.sample_distinct)
    O.set_threads(os.cpu_count() or 1)
    t = time.perf_counter()
    u, s, v, st = O.mc_svt(m, m, colptr, rowidx, vals, O.SvdBackend.blws(seed=SEED ^ 0x5BDBEEF), tol_outer=1e-6,
                           truth_ml=ml, truth_mr=mr, cap=512)
    secs = time.perf_counter() - t
    g = sketch(m)
    out = _hist(st)
    out.update(sigma=s, a_sketch=(u * s) @ (v.T @ g), a_fro=float(np.linalg.norm(s)), oracle_seconds=secs,
               oracle_threads=os.cpu_count() or 1)
    return out


def main(names):
    for name in names:
        out = {"C3": c3, "C4": c4, "C5S": c5s}[name]()
        path = os.path.join(HERE, f"{name.lower()}_oracle_trace.npz")
        np.savez_compressed(path, **{k: np.asarray(v) for k, v in out.items()})
        print(json.dumps({k: (v if np.isscalar(v) else f"array{np.shape(v)}") for k, v in out.items()},
                         default=str), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C3", "C4"])
