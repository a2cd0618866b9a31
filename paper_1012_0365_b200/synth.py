"""Seeded synthetic instances for the BASELINE.json configs (harness code).

Reuses the reference's generator recipe (proj/include/blws/synth.hpp): RNG
split tags, column-major Gaussian fills, Floyd sampling of distinct positions
(synth.hpp:23-33, :53-96, :121-150). `rng_cls` / `sample` are injected so the
same recipe can run on the product's Rng (C ABI) or the oracle's Rng and
produce bit-identical draws. The dense products (L R^T, Haar QR) use numpy;
inputs are generated once and then handed unchanged to both arms.
"""
from __future__ import annotations

import numpy as np


def _qr_pos(a):
    """Householder QR with diag(R) >= 0 (core/qr.hpp:39-43)."""
    q, r = np.linalg.qr(a)
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return np.asfortranarray(q * s)


def rpca_lowrank_sparse(m, rank, n_corrupt, seed, rng_cls, sample):
    """C1 / C3 / C5 recipe: A0 = L R^T with L, R ~ N(0,1)
    (gen_mc's factor tags 1, 2), E0 on `n_corrupt` Floyd positions (tag 4)
    with values U[-500, 500] (tag 5), D = A0 + E0."""
    base = rng_cls(seed)
    L = base.split(1).gaussian_matrix(m, rank)
    R = base.split(2).gaussian_matrix(m, rank)
    a0 = np.asfortranarray(L @ R.T)
    pos = sample(m * m, n_corrupt, base.split(4))
    rv = base.split(5)
    vals = np.array([rv.uniform(-500.0, 500.0) for _ in range(len(pos))]) if len(pos) < 200000 else \
        _uniform_bulk(rv, len(pos), -500.0, 500.0)
    d = a0.copy(order="F")
    flat = d.reshape(-1, order="F")
    flat[pos] += vals
    return np.asfortranarray(flat.reshape((m, m), order="F")), a0, pos, vals


def _uniform_bulk(rng, n, lo, hi):
    if hasattr(rng, "uniform_fill"):
        return rng.uniform_fill(n, lo, hi)
    return np.array([rng.uniform(lo, hi) for _ in range(n)])


def blws_standalone(m, n, k_signal, r, seed, rng_cls, noise=1e-3, decay=0.97, top=100.0, perturb=1e-2):
    """C2: W = U0 diag(sigma) V0^T + noise * N(0,1), U0/V0 Haar (QR of
    Gaussians), sigma_i = top * decay^i; warm start = QR(U0[:, :r] + perturb * N)
    and likewise V, sigma_warm = sigma[:r]."""
    base = rng_cls(seed)
    U0 = _qr_pos(base.split(1).gaussian_matrix(m, k_signal))
    V0 = _qr_pos(base.split(2).gaussian_matrix(n, k_signal))
    sigma = top * decay ** np.arange(k_signal)
    W = (U0 * sigma) @ V0.T
    W += noise * base.split(3).gaussian_matrix(m, n)
    Uw = _qr_pos(U0[:, :r] + perturb * base.split(4).gaussian_matrix(m, r))
    Vw = _qr_pos(V0[:, :r] + perturb * base.split(5).gaussian_matrix(n, r))
    return np.asfortranarray(W), Uw, Vw, sigma[:r].copy(), sigma


def mc_lowrank(m, rank, n_obs, seed, rng_cls, sample):
    """C4 recipe (gen_mc, synth.hpp:121-150): ML, MR ~ N(0,1) (tags 1, 2),
    Omega = Floyd sample of n_obs positions (tag 3), values ML_i . MR_j.
    Returns CSC (colptr int64, rowidx int32, values)."""
    base = rng_cls(seed)
    ML = base.split(1).gaussian_matrix(m, rank)
    MR = base.split(2).gaussian_matrix(m, rank)
    pos = sample(m * m, n_obs, base.split(3))
    rows = (pos % m).astype(np.int64)
    cols = (pos // m).astype(np.int64)
    vals = np.einsum("ij,ij->i", ML[rows], MR[cols])
    # positions are sorted ascending = column-major order = CSC order
    colptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(colptr, cols + 1, 1)
    colptr = np.cumsum(colptr)
    return colptr, rows.astype(np.int32), vals, ML, MR


def rpca_lowrank_sparse_device(m, rank, n_corrupt, seed, rng_cls, sample, device):
    """C5-scale variant of rpca_lowrank_sparse: the same draws (host Rng, Floyd
    sample), D = L R^T + E0 formed on the GPU (a 40000^2 D is 12.8 GB).
    Returns column-major D and A0 as row-major (m, m) torch tensors holding the
    transposes (i.e. column-major buffers), plus the host positions / values."""
    import torch

    base = rng_cls(seed)
    L = base.split(1).gaussian_matrix(m, rank)
    R = base.split(2).gaussian_matrix(m, rank)
    pos = sample(m * m, n_corrupt, base.split(4))
    vals = _uniform_bulk(base.split(5), len(pos), -500.0, 500.0)
    Ld = torch.from_numpy(np.ascontiguousarray(L)).to(device)
    Rd = torch.from_numpy(np.ascontiguousarray(R)).to(device)
    a0t = Rd @ Ld.T  # row-major (m, m) of A0^T = column-major A0
    dt = a0t.clone()
    flat = dt.view(-1)  # column-major flat index of (i, j) = i + j m = row-major index of A0^T
    flat.index_add_(0, torch.from_numpy(np.asarray(pos, dtype=np.int64)).to(device),
                    torch.from_numpy(np.asarray(vals)).to(device))
    return dt, a0t, pos, vals


def export_rpca_instance(d, a_true, e_true, directory):
    """export_instance (synth.hpp:152-159): d.mtx, a_true.mtx, e_true.mtx (array format)."""
    import os

    from . import api

    os.makedirs(directory, exist_ok=True)
    api.mm_write_dense(os.path.join(directory, "d.mtx"), d)
    api.mm_write_dense(os.path.join(directory, "a_true.mtx"), a_true)
    api.mm_write_dense(os.path.join(directory, "e_true.mtx"), e_true)


def export_mc_instance(m, n, colptr, rowidx, vals, ml, mr, directory):
    """export_instance (synth.hpp:161-168): observed.mtx (coordinate), ml.mtx, mr.mtx."""
    import os

    from . import api

    os.makedirs(directory, exist_ok=True)
    api.mm_write_sparse(os.path.join(directory, "observed.mtx"), m, n, colptr, rowidx, vals)
    api.mm_write_dense(os.path.join(directory, "ml.mtx"), ml)
    api.mm_write_dense(os.path.join(directory, "mr.mtx"), mr)
