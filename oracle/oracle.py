"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU oracle.

The oracle is a restatement of the reference BLWS / RPCA / MC algorithm
(/root/reference/proj/include/blws, see oracle/blws_oracle.hpp for the
file:line map). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module; the product
package (paper_1012_0365_b200) never does.

Parity status: the reference cannot be built here (Eigen absent), so the
oracle is pinned against the reference's own known-answer and property
tests (tests/test_oracle_*.py restate them) and against the bit-portable
std::mt19937_64 known answer; see DESIGN.md §3.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import build_oracle

_lib = None

i64 = C.c_int64
u64 = C.c_uint64
dbl = C.c_double
vp = C.c_void_p
P = C.POINTER


def _ptr(a):
    return a.ctypes.data_as(vp) if a is not None else None


def lib():
    global _lib
    if _lib is None:
        path = build_oracle.build()
        L = C.CDLL(path)
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_set_threads": (None, [C.c_int]),
            "orc_small_dense_max_order": (i64, []),
            "orc_rng_new": (vp, [u64]),
            "orc_rng_free": (None, [vp]),
            "orc_rng_split": (vp, [vp, u64]),
            "orc_rng_next_u64": (u64, [vp]),
            "orc_rng_uniform": (dbl, [vp]),
            "orc_rng_uniform_range": (dbl, [vp, dbl, dbl]),
            "orc_rng_normal": (dbl, [vp]),
            "orc_rng_uniform_index": (u64, [vp, u64]),
            "orc_rng_gaussian_matrix": (None, [vp, i64, i64, vp]),
            "orc_rng_unit_vector": (None, [vp, i64, vp]),
            "orc_rng_uniform_fill": (None, [vp, i64, dbl, dbl, vp]),
            "orc_sample_distinct": (i64, [i64, i64, vp, vp]),
            "orc_thin_qr": (C.c_int, [i64, i64, vp, vp, vp, P(i64)]),
            "orc_sym_evd": (C.c_int, [i64, vp, vp, vp]),
            "orc_sym_evd_tridiagonal": (C.c_int, [i64, vp, vp, vp, vp]),
            "orc_full_svd": (C.c_int, [i64, i64, vp, vp, vp, vp]),
            "orc_dense_op_new": (vp, [i64, i64, vp]),
            "orc_dense_op_assign": (C.c_int, [vp, i64, i64, vp]),
            "orc_sparse_op_new": (vp, [i64, i64, i64, vp, vp, vp]),
            "orc_sparse_op_assign_values": (C.c_int, [vp, i64, vp]),
            "orc_aug_op_new": (vp, [vp]),
            "orc_op_count": (i64, [vp]),
            "orc_op_rows": (i64, [vp]),
            "orc_op_cols": (i64, [vp]),
            "orc_op_free": (None, [vp]),
            "orc_op_apply_block": (C.c_int, [vp, i64, vp, vp]),
            "orc_op_apply_pair_block": (C.c_int, [vp, i64, vp, vp, vp, vp]),
            "orc_block_lanczos": (C.c_int, [vp, i64, vp, i64, vp, vp, P(i64), P(C.c_int)]),
            "orc_bl_evd": (C.c_int, [vp, i64, vp, i64, i64, vp, vp, P(i64), P(C.c_int)]),
            "orc_adapt_subspace": (C.c_int, [i64, vp, vp, vp, i64, i64, i64, vp, vp, vp, vp]),
            "orc_blws_svd": (C.c_int, [vp, i64, vp, vp, vp, i64, i64, vp, vp, vp, vp, P(C.c_int)]),
            "orc_lanczos_partial_svd": (C.c_int, [vp, i64, dbl, i64, u64, vp, vp, vp, P(i64), vp]),
            "orc_lanczos_partial_evd": (C.c_int, [vp, i64, dbl, i64, u64, vp, vp, P(i64), vp]),
            "orc_lanczos_procedure": (C.c_int, [vp, vp, i64, vp, vp, vp, P(i64), P(dbl), P(C.c_int)]),
            "orc_spectral_norm": (dbl, [vp, dbl, u64]),
            "orc_backend_new": (vp, [C.c_int, i64, dbl, i64, i64, u64]),
            "orc_backend_free": (None, [vp]),
            "orc_backend_warm_rank": (i64, [vp]),
            "orc_backend_warm_get": (None, [vp, vp, vp, vp]),
            "orc_svt": (C.c_int, [vp, dbl, vp, vp, vp, i64, P(i64), vp, vp, vp, P(i64), P(C.c_int)]),
            "orc_rpca_adm": (C.c_int, [i64, vp, dbl, vp, dbl, i64, dbl, dbl, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp]),
            "orc_mc_svt": (C.c_int, [i64, i64, i64, vp, vp, vp, dbl, dbl, vp, dbl, i64, i64, i64, i64, vp, vp,
                                     vp, vp, vp, i64, vp, vp, vp, vp, vp]),
            "orc_trace_enable": (None, [C.c_int]),
            "orc_trace_clear": (None, []),
            "orc_trace_size": (i64, []),
            "orc_trace_get": (C.c_int, [i64, vp, vp, i64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def F(a, dtype=np.float64):
    return np.asfortranarray(a, dtype=dtype)


def small_dense_max_order() -> int:
    """Largest EVD order met so far (the reference guards it at 4096, small_dense.hpp:13)."""
    return int(lib().orc_small_dense_max_order())


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


# ------------------------------------------------------------------ rng
class Rng:
    """blws::Rng (core/rng.hpp:17-90), bit-exact."""

    def __init__(self, seed: int = 0, _handle=None):
        self._h = _handle if _handle is not None else lib().orc_rng_new(int(seed) & (2**64 - 1))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_rng_free(self._h)
            self._h = None

    def split(self, tag: int) -> "Rng":
        return Rng(_handle=lib().orc_rng_split(self._h, int(tag)))

    def next_u64(self) -> int:
        return int(lib().orc_rng_next_u64(self._h))

    def uniform(self, lo=None, hi=None) -> float:
        if lo is None:
            return float(lib().orc_rng_uniform(self._h))
        return float(lib().orc_rng_uniform_range(self._h, lo, hi))

    def uniform_fill(self, n, lo, hi):
        out = np.empty(n)
        lib().orc_rng_uniform_fill(self._h, n, lo, hi, _ptr(out))
        return out

    def normal(self) -> float:
        return float(lib().orc_rng_normal(self._h))

    def uniform_index(self, n: int) -> int:
        return int(lib().orc_rng_uniform_index(self._h, int(n)))

    def gaussian_matrix(self, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), order="F")
        lib().orc_rng_gaussian_matrix(self._h, rows, cols, _ptr(out))
        return out

    def gaussian_vector(self, n: int) -> np.ndarray:
        return self.gaussian_matrix(n, 1)[:, 0].copy()

    def unit_vector(self, n: int) -> np.ndarray:
        out = np.empty(n)
        lib().orc_rng_unit_vector(self._h, n, _ptr(out))
        return out


def sample_distinct(n: int, s: int, rng: Rng) -> np.ndarray:
    out = np.empty(s, dtype=np.int64)
    got = lib().orc_sample_distinct(n, s, rng._h, _ptr(out))
    return out[:got]


# ------------------------------------------------------- dense kernels
@dataclass
class ThinQr:
    q: np.ndarray
    r: np.ndarray
    rank: int


def thin_qr(m) -> ThinQr:
    m = F(m)
    if m.ndim != 2:
        raise ValueError("thin_qr: 2-D input required")
    rows, cols = m.shape
    q = np.empty((rows, max(cols, 0)), order="F")
    r = np.empty((cols, cols), order="F")
    rank = i64(0)
    _check(lib().orc_thin_qr(rows, cols, _ptr(m), _ptr(q), _ptr(r), C.byref(rank)))
    return ThinQr(q, r, rank.value)


def sym_evd_small(t):
    t = F(t)
    if t.ndim != 2 or t.shape[0] != t.shape[1]:
        raise ValueError("sym_evd_small: not square")
    n = t.shape[0]
    vals = np.empty(n)
    vecs = np.empty((n, n), order="F")
    _check(lib().orc_sym_evd(n, _ptr(t), _ptr(vals), _ptr(vecs)))
    return vals, vecs


def sym_evd_tridiagonal(d, e):
    d = np.ascontiguousarray(d, dtype=np.float64)
    e = np.ascontiguousarray(e, dtype=np.float64)
    if len(d) == 0:
        raise ValueError("sym_evd_tridiagonal: empty")
    if len(e) != len(d) - 1:
        raise ValueError("sym_evd_tridiagonal: size mismatch")
    n = len(d)
    vals = np.empty(n)
    vecs = np.empty((n, n), order="F")
    _check(lib().orc_sym_evd_tridiagonal(n, _ptr(d), _ptr(e), _ptr(vals), _ptr(vecs)))
    return vals, vecs


def full_svd_small(a):
    a = F(a)
    m, n = a.shape
    p = min(m, n)
    u = np.empty((m, p), order="F")
    s = np.empty(p)
    v = np.empty((n, p), order="F")
    _check(lib().orc_full_svd(m, n, _ptr(a), _ptr(u), _ptr(s), _ptr(v)))
    return u, s, v


# ----------------------------------------------------------- operators
class LinearOperator:
    _h = None
    _owned = True

    def __del__(self):
        if self._h and self._owned:
            lib().orc_op_free(self._h)
            self._h = None

    def rows(self) -> int:
        return int(lib().orc_op_rows(self._h))

    def cols(self) -> int:
        return int(lib().orc_op_cols(self._h))

    def application_count(self) -> int:
        return int(lib().orc_op_count(self._h))

    def apply_block(self, x):
        x = F(x)
        y = np.empty((self.rows(), x.shape[1]), order="F")
        _check(lib().orc_op_apply_block(self._h, x.shape[1], _ptr(x), _ptr(y)))
        return y

    def apply_pair_block(self, left, right):
        left, right = F(left), F(right)
        b = right.shape[1]
        top = np.empty((self.rows(), b), order="F")
        bot = np.empty((self.cols(), b), order="F")
        _check(lib().orc_op_apply_pair_block(self._h, b, _ptr(left), _ptr(right), _ptr(top), _ptr(bot)))
        return top, bot


class DenseOperator(LinearOperator):
    def __init__(self, w):
        w = F(w)
        self.m, self.n = w.shape
        h = lib().orc_dense_op_new(self.m, self.n, _ptr(w))
        if not h:
            raise ValueError(lib().orc_last_error().decode())
        self._h = h

    def assign(self, w):
        w = F(w)
        _check(lib().orc_dense_op_assign(self._h, w.shape[0], w.shape[1], _ptr(w)))


class SparseOperator(LinearOperator):
    """CSC (Eigen default) sparse operator; values in compressed order."""

    def __init__(self, m, n, colptr, rowidx, vals):
        self.colptr = np.ascontiguousarray(colptr, dtype=np.int64)
        self.rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        self.m, self.n, self.nnz = m, n, len(vals)
        h = lib().orc_sparse_op_new(m, n, self.nnz, _ptr(self.colptr), _ptr(self.rowidx), _ptr(vals))
        if not h:
            raise ValueError(lib().orc_last_error().decode())
        self._h = h

    def assign_values(self, vals):
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        _check(lib().orc_sparse_op_assign_values(self._h, len(vals), _ptr(vals)))


class AugmentedOperator(LinearOperator):
    def __init__(self, inner: LinearOperator):
        self._inner = inner
        self._h = lib().orc_aug_op_new(inner._h)


# -------------------------------------------------------- block lanczos
@dataclass
class WarmStart:
    u: np.ndarray
    v: np.ndarray
    sigma: np.ndarray

    def rank(self) -> int:
        return len(self.sigma)


def block_lanczos_procedure(op: LinearOperator, x1, k: int):
    x1 = F(x1)
    b = x1.shape[1]
    q = np.empty((op.rows(), k * b), order="F")
    t = np.zeros((k * b) ** 2)
    built = i64(0)
    term = C.c_int(0)
    _check(lib().orc_block_lanczos(op._h, b, _ptr(x1), k, _ptr(q), _ptr(t), C.byref(built), C.byref(term)))
    nb = built.value * b
    tt = t[: nb * nb].reshape((nb, nb), order="F")
    return q[:, :nb].copy(order="F"), tt.copy(order="F"), built.value, bool(term.value)


def bl_evd(op: LinearOperator, x1, k: int, r: int):
    x1 = F(x1)
    b = x1.shape[1]
    u = np.empty((op.rows(), r), order="F")
    vals = np.empty(r)
    avail = i64(0)
    term = C.c_int(0)
    _check(lib().orc_bl_evd(op._h, b, _ptr(x1), k, r, _ptr(u), _ptr(vals), C.byref(avail), C.byref(term)))
    a = avail.value
    return u[:, :a].copy(order="F"), vals[:a].copy(), a, bool(term.value)


def adapt_subspace(warm, r_new, m, n, rng: Rng) -> WarmStart:
    u = np.empty((m, r_new), order="F")
    v = np.empty((n, r_new), order="F")
    s = np.empty(r_new)
    if warm is None or warm.rank() == 0:
        _check(lib().orc_adapt_subspace(0, None, None, None, r_new, m, n, rng._h, _ptr(u), _ptr(v), _ptr(s)))
    else:
        wu, wv, ws = F(warm.u), F(warm.v), np.ascontiguousarray(warm.sigma, dtype=np.float64)
        _check(lib().orc_adapt_subspace(warm.rank(), _ptr(wu), _ptr(wv), _ptr(ws), r_new, m, n, rng._h,
                                        _ptr(u), _ptr(v), _ptr(s)))
    return WarmStart(u, v, s)


@dataclass
class BlwsResult:
    warm: WarmStart
    padded: bool
    k_raised: bool
    terminated_early: bool


def blws_svd(op: LinearOperator, warm: WarmStart, k: int, r: int, rng: Rng) -> BlwsResult:
    m, n = op.rows(), op.cols()
    b = warm.rank()
    wu, wv = F(warm.u), F(warm.v)
    ws = np.ascontiguousarray(warm.sigma, dtype=np.float64)
    u = np.empty((m, r), order="F")
    v = np.empty((n, r), order="F")
    s = np.empty(r)
    flags = C.c_int(0)
    _check(lib().orc_blws_svd(op._h, b, _ptr(wu), _ptr(wv), _ptr(ws), k, r, rng._h, _ptr(u), _ptr(v), _ptr(s),
                              C.byref(flags)))
    f = flags.value
    return BlwsResult(WarmStart(u, v, s), bool(f & 1), bool(f & 2), bool(f & 4))


# -------------------------------------------------------------- lanczos
def lanczos_partial_svd(op: LinearOperator, r: int, tol=1e-8, max_k=0, seed=0x1A2C705):
    m, n = op.rows(), op.cols()
    u = np.empty((m, r), order="F")
    v = np.empty((n, r), order="F")
    s = np.empty(r)
    keep = i64(0)
    stats = np.zeros(4, dtype=np.int64)
    _check(lib().orc_lanczos_partial_svd(op._h, r, tol, max_k, seed, _ptr(u), _ptr(s), _ptr(v), C.byref(keep),
                                         _ptr(stats)))
    k = keep.value
    return u[:, :k].copy(order="F"), s[:k].copy(), v[:, :k].copy(order="F"), stats


def lanczos_partial_evd(op: LinearOperator, r: int, tol=1e-8, max_k=0, seed=0x1A2C705):
    d = op.rows()
    u = np.empty((d, r), order="F")
    vals = np.empty(r)
    avail = i64(0)
    stats = np.zeros(4, dtype=np.int64)
    _check(lib().orc_lanczos_partial_evd(op._h, r, tol, max_k, seed, _ptr(u), _ptr(vals), C.byref(avail),
                                         _ptr(stats)))
    a = avail.value
    return u[:, :a].copy(order="F"), vals[:a].copy(), stats


def lanczos_procedure(op: LinearOperator, q1, k: int):
    d = op.rows()
    q1 = np.ascontiguousarray(q1, dtype=np.float64)
    q = np.empty((d, k), order="F")
    alpha = np.empty(k)
    beta = np.empty(k)
    cols = i64(0)
    resid = dbl(0)
    term = C.c_int(0)
    _check(lib().orc_lanczos_procedure(op._h, _ptr(q1), k, _ptr(q), _ptr(alpha), _ptr(beta), C.byref(cols),
                                       C.byref(resid), C.byref(term)))
    c = cols.value
    return q[:, :c].copy(order="F"), alpha[:c].copy(), beta[: max(c - 1, 0)].copy(), resid.value, bool(term.value)


def spectral_norm(op: LinearOperator, tol=1e-6, seed=0xB1F) -> float:
    v = lib().orc_spectral_norm(op._h, tol, seed)
    if v < 0:
        raise RuntimeError(lib().orc_last_error().decode())
    return float(v)


# ---------------------------------------------------------- backend/svt
class SvdBackend:
    """blws::SvdBackend (svt.hpp:84-196). kind: 0 ExactFull, 1 Lanczos, 2 Blws."""

    EXACT_FULL, LANCZOS, BLWS = 0, 1, 2

    def __init__(self, kind=2, block_steps=2, ritz_tol=1e-8, max_k=0, seed_margin=5, seed=0xB10C):
        self.kind = kind
        self._h = lib().orc_backend_new(kind, block_steps, ritz_tol, max_k, seed_margin, int(seed) & (2**64 - 1))

    @classmethod
    def exact_full(cls):
        return cls(kind=0)

    @classmethod
    def lanczos(cls, **kw):
        return cls(kind=1, **kw)

    @classmethod
    def blws(cls, **kw):
        return cls(kind=2, **kw)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_backend_free(self._h)
            self._h = None

    def warm_state(self, m, n):
        r = int(lib().orc_backend_warm_rank(self._h))
        if r == 0:
            return None
        u = np.empty((m, r), order="F")
        v = np.empty((n, r), order="F")
        s = np.empty(r)
        lib().orc_backend_warm_get(self._h, _ptr(u), _ptr(v), _ptr(s))
        return WarmStart(u, v, s)


@dataclass
class RankPredictor:
    r: int = 10
    increment: int = 5
    max_rank: int = 1
    history: list = field(default_factory=list)


@dataclass
class SvtResult:
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray
    achieved_rank: int
    all_above_threshold: bool

    def dense(self):
        return (self.u * self.sigma) @ self.v.T


def svt(op: LinearOperator, eps: float, backend: SvdBackend, predictor: RankPredictor) -> SvtResult:
    m, n = op.rows(), op.cols()
    p = min(m, n)
    pred = np.array([predictor.r, predictor.increment, predictor.max_rank], dtype=np.int64)
    cap = len(predictor.history) + 1
    hist = np.zeros(cap, dtype=np.int64)
    hist[: len(predictor.history)] = predictor.history
    hl = i64(len(predictor.history))
    u = np.empty((m, p), order="F")
    v = np.empty((n, p), order="F")
    s = np.empty(p)
    ach = i64(0)
    above = C.c_int(0)
    _check(lib().orc_svt(op._h, eps, backend._h, _ptr(pred), _ptr(hist), cap, C.byref(hl), _ptr(u), _ptr(s), _ptr(v),
                         C.byref(ach), C.byref(above)))
    predictor.r = int(pred[0])
    predictor.history = [int(x) for x in hist[: hl.value]]
    a = ach.value
    return SvtResult(u[:, :a].copy(order="F"), s[:a].copy(), v[:, :a].copy(order="F"), a, bool(above.value))


# -------------------------------------------------------------- solvers
@dataclass
class SolverStats:
    iterations: int = 0
    wall_time_s: float = 0.0
    matvec_count: int = 0
    matvec_init: int = 0
    rel_err: float = -1.0
    rank_hat: int = 0
    e_l0: int = -1
    converged: bool = False
    predicted_ranks: list = field(default_factory=list)
    matvec_history: list = field(default_factory=list)
    residual_history: list = field(default_factory=list)


def _stats(ist, dst, ph, mh, rh):
    it = int(ist[0])
    return SolverStats(iterations=it, wall_time_s=float(dst[0]), matvec_count=int(ist[1]), matvec_init=int(ist[2]),
                       rel_err=float(dst[1]), rank_hat=int(ist[3]), e_l0=int(ist[4]), converged=bool(ist[5]),
                       predicted_ranks=[int(x) for x in ph[:it]], matvec_history=[int(x) for x in mh[:it]],
                       residual_history=[float(x) for x in rh[:it]])


def rpca_adm(d, backend: SvdBackend, lam=0.0, tol_outer=1e-7, max_iter=1000, rho=1.5, mu_max_factor=1e7,
             initial_rank=10, rank_increment=5, truth=None, want_outputs=True):
    d = F(d)
    m = d.shape[0]
    if d.shape[0] != d.shape[1]:
        raise ValueError("rpca_adm: D must be square")
    a = np.empty((m, m), order="F") if want_outputs else None
    e = np.empty((m, m), order="F") if want_outputs else None
    ist = np.zeros(8, dtype=np.int64)
    dst = np.zeros(2)
    ph = np.zeros(max_iter + 1, dtype=np.int64)
    mh = np.zeros(max_iter + 1, dtype=np.int64)
    rh = np.zeros(max_iter + 1)
    tr = F(truth) if truth is not None else None
    _check(lib().orc_rpca_adm(m, _ptr(d), lam, backend._h, tol_outer, max_iter, rho, mu_max_factor, initial_rank,
                              rank_increment, _ptr(tr), _ptr(a), _ptr(e), _ptr(ist), _ptr(dst), _ptr(ph), _ptr(mh),
                              _ptr(rh)))
    st = _stats(ist, dst, ph, mh, rh)
    return a, e, st, int(ist[6])


def mc_svt(m, n, colptr, rowidx, vals, backend: SvdBackend, tau=0.0, delta=0.0, tol_outer=1e-4, max_iter=500,
           initial_rank=10, rank_increment=5, truth_ml=None, truth_mr=None, cap=None):
    colptr = np.ascontiguousarray(colptr, dtype=np.int64)
    rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    cap = cap or min(m, n)
    u = np.empty((m, cap), order="F")
    s = np.empty(cap)
    v = np.empty((n, cap), order="F")
    ist = np.zeros(8, dtype=np.int64)
    dst = np.zeros(2)
    ph = np.zeros(max_iter + 1, dtype=np.int64)
    mh = np.zeros(max_iter + 1, dtype=np.int64)
    rh = np.zeros(max_iter + 1)
    r_true = 0
    ml = mr = None
    if truth_ml is not None:
        ml, mr = F(truth_ml), F(truth_mr)
        r_true = ml.shape[1]
    _check(lib().orc_mc_svt(m, n, len(vals), _ptr(colptr), _ptr(rowidx), _ptr(vals), tau, delta, backend._h,
                            tol_outer, max_iter, initial_rank, rank_increment, r_true, _ptr(ml), _ptr(mr), _ptr(u),
                            _ptr(s), _ptr(v), cap, _ptr(ist), _ptr(dst), _ptr(ph), _ptr(mh), _ptr(rh)))
    k = int(ist[4])
    st = _stats(ist, dst, ph, mh, rh)
    return u[:, :k].copy(order="F"), s[:k].copy(), v[:, :k].copy(order="F"), st


# ---------------------------------------------------------------- trace
def trace_enable(on=True):
    lib().orc_trace_enable(1 if on else 0)


def trace_clear():
    lib().orc_trace_clear()


def trace_records():
    out = []
    n = int(lib().orc_trace_size())
    ints = np.zeros(10, dtype=np.int64)
    for i in range(n):
        sig = np.zeros(8192)
        lib().orc_trace_get(i, _ptr(ints), _ptr(sig), len(sig))
        ns = int(ints[9])
        out.append(dict(kind=int(ints[0]), b=int(ints[1]), r=int(ints[2]), k_eff=int(ints[3]), keep=int(ints[4]),
                        steps=int(ints[5]), restarts=int(ints[6]), converged=int(ints[7]), flags=int(ints[8]),
                        sigma=sig[:ns].copy()))
    return out
