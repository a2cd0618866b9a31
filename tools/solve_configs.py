"""Solver configs of BASELINE.json on the GPU, with the CPU oracle beside them.

C1: RPCA 500^2, rank 25, 5% corruption, tol 1e-7       (parity + timing)
C3: RPCA 2000^2, rank 100, 10% corruption, tol 1e-7    (parity + timing)
C4: MC 10^4^2, rank 50, 10^7 observed, tol 1e-6        (GPU; oracle skipped: its
    sparse products are naive single-thread loops, hours at this size)
C5: RPCA 40000^2, rank 400, 5% corruption, tol 1e-7    (GPU only, D formed on the
    device from the same host draws: 12.8 GB per m x m matrix; the CPU oracle
    cannot hold the ~100 GB working set)
Prints one JSON line per config.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1012_0365_b200 as B  # noqa: E402
from paper_1012_0365_b200 import report, synth  # noqa: E402

SEED = 1
ROWS = {}  # config -> [ReportRow] (bench/report.hpp schema)


def _row(problem, m, method, st, t, r=0, s_dr=0.0, s_m2=0.0):
    return report.ReportRow(problem=problem, m=m, method=method, rel_err=st.rel_err, rank_hat=st.rank_hat,
                            e_l0=max(st.e_l0, 0), iters=st.iterations, time_s=t, matvecs=st.matvec_count, r=r,
                            s_dr=s_dr, s_m2=s_m2, converged=bool(st.converged))


def rpca(name, m, rank, frac, oracle=True, baseline=False):
    from oracle import oracle as O
    d, a0, _, _ = synth.rpca_lowrank_sparse(m, rank, int(round(frac * m * m)), SEED, B.Rng, B.sample_distinct)
    bseed = SEED ^ 0x5BDBEEF
    ctx = B.Context(0)
    B.rpca_adm(d[:64, :64].copy(order="F"), B.SvdBackend.blws(seed=bseed, ctx=ctx))  # warm-up (module load)
    t = time.perf_counter()
    a, e, st, _ = B.rpca_adm(d, B.SvdBackend.blws(seed=bseed, ctx=ctx), truth=a0)
    gpu_s = time.perf_counter() - t
    ROWS.setdefault(name, [])
    if baseline:  # the paper's ADM row: the same solver with the cold Lanczos backend
        t = time.perf_counter()
        _, _, sl, _ = B.rpca_adm(d, B.SvdBackend.lanczos(seed=bseed, ctx=ctx), truth=a0, want_outputs=False)
        ROWS[name].append(_row(report.RPCA, m, "ADM", sl, time.perf_counter() - t))
    ROWS[name].append(_row(report.RPCA, m, "BLWS-ADM", st, gpu_s))
    line = dict(config=name, m=m, rank=rank, corrupt=frac, gpu_solve_s=gpu_s, iterations=st.iterations,
                rank_hat=st.rank_hat, rel_err=st.rel_err, e_l0=st.e_l0, matvecs=st.matvec_count,
                converged=st.converged)
    if oracle:
        cores = os.cpu_count() or 1
        O.set_threads(cores)
        t = time.perf_counter()
        ao, eo, so, _ = O.rpca_adm(d, O.SvdBackend.blws(seed=bseed), truth=a0)
        line.update(cpu_solve_s=time.perf_counter() - t, cpu_cores=cores, cpu_iterations=so.iterations,
                    cpu_rank_hat=so.rank_hat, cpu_rel_err=so.rel_err,
                    a_rel_diff=float(np.linalg.norm(a - ao) / np.linalg.norm(ao)),
                    e_rel_diff=float(np.linalg.norm(e - eo) / np.linalg.norm(eo)),
                    same_predicted_ranks=st.predicted_ranks[:min(st.iterations, so.iterations)]
                    == so.predicted_ranks[:min(st.iterations, so.iterations)])
    print(json.dumps(line), flush=True)


def mc(name, m, rank, nobs, baseline=False):
    colptr, rowidx, vals, ml, mr = synth.mc_lowrank(m, rank, nobs, SEED, B.Rng, B.sample_distinct)
    ctx = B.Context(0)
    t = time.perf_counter()
    u, s, v, st = B.mc_svt(m, m, colptr, rowidx, vals, B.SvdBackend.blws(seed=SEED ^ 0x5BDBEEF, ctx=ctx),
                           tol_outer=1e-6, truth_ml=ml, truth_mr=mr, cap=512)
    gpu_s = time.perf_counter() - t
    s_dr = nobs / (rank * (2 * m - rank))
    ROWS.setdefault(name, [])
    if baseline:
        t = time.perf_counter()
        _, _, _, sl = B.mc_svt(m, m, colptr, rowidx, vals, B.SvdBackend.lanczos(seed=SEED ^ 0x5BDBEEF, ctx=ctx),
                               tol_outer=1e-6, truth_ml=ml, truth_mr=mr, cap=512)
        ROWS[name].append(_row(report.MC, m, "SVT", sl, time.perf_counter() - t, rank, s_dr, nobs / (m * m)))
    ROWS[name].append(_row(report.MC, m, "BLWS-SVT", st, gpu_s, rank, s_dr, nobs / (m * m)))
    print(json.dumps(dict(config=name, m=m, rank=rank, nobs=nobs, gpu_solve_s=gpu_s, iterations=st.iterations,
                          rank_hat=st.rank_hat, rel_err=st.rel_err, matvecs=st.matvec_count,
                          converged=st.converged)), flush=True)


def rpca_device(name, m, rank, frac, max_iter=1000):
    import torch

    dev = torch.device("cuda:0")
    t = time.perf_counter()
    dt, a0t, _, _ = synth.rpca_lowrank_sparse_device(m, rank, int(round(frac * m * m)), SEED, B.Rng,
                                                     B.sample_distinct, dev)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t
    ctx = B.Context(0)
    B.rpca_adm(np.ascontiguousarray(dt[:64, :64].cpu().numpy().T), B.SvdBackend.blws(seed=SEED ^ 0x5BDBEEF, ctx=ctx))
    t = time.perf_counter()
    _, _, st, e_nnz = B.rpca_adm(dt, B.SvdBackend.blws(seed=SEED ^ 0x5BDBEEF, ctx=ctx), truth=a0t, device=True,
                                 m=m, ld=m, max_iter=max_iter)
    gpu_s = time.perf_counter() - t
    print(json.dumps(dict(config=name, m=m, rank=rank, corrupt=frac, gen_s=gen_s, gpu_solve_s=gpu_s,
                          iterations=st.iterations, rank_hat=st.rank_hat, rel_err=st.rel_err, e_l0=st.e_l0,
                          matvecs=st.matvec_count, converged=st.converged,
                          data=f"D formed on the device ({m * m * 8 / 1e9:.1f} GB per m x m matrix)")),
          flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C1", "C3", "C4"])
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--baseline", action="store_true", help="also run the Lanczos-backend solver (ADM / SVT rows)")
    ap.add_argument("--report", choices=["csv", "markdown"], help="emit the bench/report.hpp table(s) at the end")
    a = ap.parse_args()
    for c in a.configs:
        if c == "C1":
            rpca("C1", 500, 25, 0.05, not a.no_oracle, a.baseline)
        elif c == "C3":
            rpca("C3", 2000, 100, 0.10, not a.no_oracle, a.baseline)
        elif c == "C4":
            mc("C4", 10000, 50, 10_000_000, a.baseline)
        elif c == "C5":
            rpca_device("C5", 40000, 400, 0.05)
        elif c == "C5s":  # reduced C5 (same recipe) to check the device path quickly
            rpca_device("C5s", 8000, 80, 0.05)
    if a.report:
        for name, rows in ROWS.items():
            print(f"# {name}")
            print(report.emit_table(rows, a.report), end="")
