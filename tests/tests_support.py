"""Shared test helpers (test infrastructure only)."""
import numpy as np


def gen_rpca_reference(O, m, rank_frac, corrupt_frac, seed):
    """The reference generator gen_rpca (proj/include/blws/synth.hpp:53-96):
    orthogonal model, singular values |N(0,1)| m / sqrt(r), corruption on Floyd
    positions with U[-500, 500] values; RNG tags 1..5."""
    base = O.Rng(seed)
    ru, rv, rs, rp, rval = (base.split(t) for t in (1, 2, 3, 4, 5))
    r = int(round(rank_frac * m))
    u = O.thin_qr(ru.gaussian_matrix(m, r)).q
    v = O.thin_qr(rv.gaussian_matrix(m, r)).q
    scale = m / np.sqrt(r)
    sig = np.array([scale * abs(rs.normal()) for _ in range(r)])
    a = np.asfortranarray((u * sig) @ v.T)
    nnz = int(round(corrupt_frac * m * m))
    pos = O.sample_distinct(m * m, nnz, rp)
    vals = rval.uniform_fill(nnz, -500.0, 500.0)
    d = a.copy(order="F").reshape(-1, order="F")
    d[pos] += vals
    return np.asfortranarray(d.reshape((m, m), order="F")), a
