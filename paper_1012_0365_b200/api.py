"""ctypes binding of libblws_cuda.so (include/blws_cuda.h).

Mirrors the reference's C++ API (proj/include/blws): Rng, DenseOperator,
SparseOperator, WarmStart, blws_svd, adapt_subspace, lanczos_partial_svd,
spectral_norm, SvdBackend, RankPredictor, svt, rpca_adm, mc_svt. Every call
runs on the GPU through the C ABI; there is no CPU fallback — if the
extension or a GPU is missing, loading raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BLWS_LIB_PATH") or os.path.join(_HERE, "_lib", "libblws_cuda.so")

i64, u64, dbl, vp, ci = C.c_int64, C.c_uint64, C.c_double, C.c_void_p, C.c_int
P = C.POINTER

HOST, DEVICE = 0, 1


class SolverStatsC(C.Structure):
    _fields_ = [("iterations", i64), ("wall_time_s", dbl), ("matvec_count", i64), ("matvec_init", i64),
                ("rel_err", dbl), ("rank_hat", i64), ("e_l0", i64), ("e_nnz", i64), ("converged", C.c_int32),
                ("pad_", C.c_int32)]


class RpcaOptionsC(C.Structure):
    _fields_ = [("tol_outer", dbl), ("max_iter", i64), ("rho", dbl), ("mu_max_factor", dbl),
                ("initial_rank", i64), ("rank_increment", i64)]


class McOptionsC(C.Structure):
    _fields_ = [("tol_outer", dbl), ("max_iter", i64), ("initial_rank", i64), ("rank_increment", i64)]


class PredictorC(C.Structure):
    _fields_ = [("r", i64), ("increment", i64), ("max_rank", i64)]


# name -> (restype, argtypes); the exported-symbol test checks this against include/blws_cuda.h
SIGNATURES = {
    "blws_last_error": (C.c_char_p, []),
    "blws_abi_version": (ci, []),
    "blws_context_create": (ci, [ci, P(vp)]),
    "blws_context_destroy": (ci, [vp]),
    "blws_context_synchronize": (ci, [vp]),
    "blws_context_stream": (vp, [vp]),
    "blws_context_launches": (i64, [vp]),
    "blws_context_set_profiling": (ci, [vp, ci]),
    "blws_context_region_stats": (ci, [vp, ci, P(dbl), P(i64), P(dbl), P(dbl)]),
    "blws_context_region_reset": (ci, [vp]),
    "blws_fp64_peak": (ci, [vp, ci, P(dbl)]),
    "blws_microbench": (ci, [vp, ci, i64, i64, ci, vp]),
    "blws_rng_create": (ci, [u64, P(vp)]),
    "blws_rng_destroy": (ci, [vp]),
    "blws_rng_split": (ci, [vp, u64, P(vp)]),
    "blws_rng_next_u64": (u64, [vp]),
    "blws_rng_uniform": (dbl, [vp, dbl, dbl]),
    "blws_rng_uniform_fill": (ci, [vp, i64, dbl, dbl, vp]),
    "blws_rng_uniform_index": (u64, [vp, u64]),
    "blws_rng_normal": (dbl, [vp]),
    "blws_rng_gaussian_matrix": (ci, [vp, i64, i64, vp]),
    "blws_sample_distinct": (i64, [i64, i64, vp, vp]),
    "blws_dense_operator_create": (ci, [vp, i64, i64, vp, i64, ci, ci, P(vp)]),
    "blws_dense_operator_assign": (ci, [vp, vp, i64, ci]),
    "blws_dense_operator_assign_async": (ci, [vp, vp, i64]),
    "blws_nccl_unique_id": (ci, [vp]),
    "blws_context_init_comm": (ci, [vp, ci, ci, vp]),
    "blws_context_init_host_comm": (ci, [vp, ci, ci, vp, vp]),
    "blws_l2_probe": (ci, [vp, ci, ci, vp]),
    "blws_context_comm_info": (ci, [vp, P(ci), P(ci)]),
    "blws_dense_operator_set_row_shard": (ci, [vp, i64, i64]),
    "blws_sparse_operator_create": (ci, [vp, i64, i64, i64, vp, vp, vp, P(vp)]),
    "blws_sparse_operator_assign_values": (ci, [vp, vp, i64, ci]),
    "blws_operator_destroy": (ci, [vp]),
    "blws_operator_rows": (i64, [vp]),
    "blws_operator_cols": (i64, [vp]),
    "blws_operator_application_count": (i64, [vp]),
    "blws_operator_apply_pair_block": (ci, [vp, i64, vp, vp, vp, vp]),
    "blws_operator_apply_pair": (ci, [vp, vp, vp, vp, vp]),
    "blws_warm_start_create": (ci, [vp, i64, i64, i64, vp, i64, vp, i64, vp, ci, P(vp)]),
    "blws_warm_start_copy": (ci, [vp, P(vp)]),
    "blws_warm_start_rank": (i64, [vp]),
    "blws_warm_start_get": (ci, [vp, vp, i64, vp, i64, vp, ci]),
    "blws_warm_start_destroy": (ci, [vp]),
    "blws_svd_deferred_fallbacks": (i64, []),
    "blws_svd_graph_launches": (i64, []),
    "blws_svd": (ci, [vp, vp, i64, i64, vp, P(vp), P(ci)]),
    "blws_adapt_subspace": (ci, [vp, vp, i64, i64, i64, vp, P(vp)]),
    "blws_block_lanczos_procedure": (ci, [vp, i64, vp, i64, vp, vp, P(i64), P(ci)]),
    "blws_lanczos_partial_svd": (ci, [vp, i64, dbl, i64, u64, P(vp), vp]),
    "blws_spectral_norm": (ci, [vp, dbl, u64, P(dbl)]),
    "blws_thin_qr": (ci, [vp, i64, i64, vp, vp, vp, P(i64)]),
    "blws_mm_write_dense": (ci, [C.c_char_p, i64, i64, vp, i64]),
    "blws_mm_write_sparse": (ci, [C.c_char_p, i64, i64, i64, vp, vp, vp]),
    "blws_mm_read_dense": (ci, [C.c_char_p, P(i64), P(i64), vp, i64]),
    "blws_mm_read_sparse": (ci, [C.c_char_p, P(i64), P(i64), P(i64), vp, vp, vp]),
    "blws_full_svd_small": (ci, [vp, i64, i64, vp, vp, vp, vp]),
    "blws_sym_evd": (ci, [vp, i64, vp, vp, vp]),
    "blws_sym_evd_tridiagonal_top": (ci, [vp, i64, vp, vp, i64, vp, vp]),
    "blws_dgemm": (ci, [vp, ci, ci, i64, i64, i64, dbl, vp, i64, vp, i64, dbl, vp, i64]),
    "blws_svd_backend_create": (ci, [vp, ci, i64, dbl, i64, i64, u64, P(vp)]),
    "blws_svd_backend_destroy": (ci, [vp]),
    "blws_svd_backend_warm_state": (ci, [vp, P(vp)]),
    "blws_svd_backend_set_warm_state": (ci, [vp, vp]),
    "blws_svt": (ci, [vp, dbl, vp, P(PredictorC), vp, i64, P(i64), P(vp), P(i64), P(ci)]),
    "blws_rpca_adm": (ci, [vp, i64, vp, i64, ci, dbl, vp, P(RpcaOptionsC), vp, vp, vp, P(SolverStatsC), vp, vp, vp,
                           i64]),
    "blws_mc_svt": (ci, [vp, i64, i64, i64, vp, vp, vp, dbl, dbl, vp, P(McOptionsC), vp, vp, i64, vp, vp, vp, i64,
                         P(i64), P(SolverStatsC), vp, vp, vp, i64]),
    "blws_rpca_adm_sharded": (ci, [vp, i64, i64, i64, vp, i64, ci, dbl, vp, P(RpcaOptionsC), vp, vp, vp,
                                   P(SolverStatsC), vp, vp, vp, i64]),
    "blws_mc_svt_sharded": (ci, [vp, i64, i64, i64, i64, i64, vp, vp, vp, dbl, dbl, vp, P(McOptionsC), vp, vp, i64,
                                 vp, vp, vp, i64, P(i64), P(SolverStatsC), vp, vp, vp, i64]),
}

_lib = None


def lib():
    """Load the CUDA extension; fails loudly when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_1012_0365_b200/build.py (no CPU fallback exists)")
        if "BLWS_NCCL_LIB" not in os.environ:
            # the NCCL torch bundles (nvidia-nccl wheel), found without importing
            # torch: comm.cu dlopens it in preference to the system libnccl
            import importlib.util

            spec = importlib.util.find_spec("nvidia")
            for root in list(spec.submodule_search_locations or []) if spec else []:
                cand = os.path.join(root, "nccl", "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ["BLWS_NCCL_LIB"] = cand
                    break
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class BlwsError(RuntimeError):
    pass


def _check(rc):
    if rc == 0:
        return
    msg = lib().blws_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise RuntimeError(msg)
    if rc == 5:
        raise OSError(msg)
    raise BlwsError(f"status {rc}: {msg}")


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):  # torch tensor
        return a.data_ptr()
    return a.ctypes.data_as(vp)


def F(a):
    return np.asfortranarray(a, dtype=np.float64)


# ------------------------------------------------------------------ context
class Context:
    def __init__(self, device: int = 0):
        h = vp()
        _check(lib().blws_context_create(device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().blws_context_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def synchronize(self):
        _check(lib().blws_context_synchronize(self._h))

    @property
    def stream(self) -> int:
        return int(lib().blws_context_stream(self._h) or 0)

    @property
    def launches(self) -> int:
        return int(lib().blws_context_launches(self._h))

    def init_comm(self, nranks: int, rank: int, unique_id: bytes):
        """Attach an NCCL communicator (collective over all ranks; see dist.init_comm)."""
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(unique_id))
        _check(lib().blws_context_init_comm(self._h, int(nranks), int(rank), C.cast(buf, vp)))

    # int (*)(double* buf, size_t count, int op, void* user)
    HOST_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_size_t, C.c_int, C.c_void_p)

    def init_host_comm(self, nranks: int, rank: int, allreduce):
        """Host-staged collectives (tests: several ranks on one GPU). `allreduce(arr, op)`
        reduces the float64 numpy array in place over the ranks (op 0 sum, 1 max)."""
        import numpy as _np

        def _cb(buf, count, op, user):
            try:
                allreduce(_np.ctypeslib.as_array(buf, shape=(int(count),)), int(op))
                return 0
            except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
                import traceback
                traceback.print_exc()
                return 1

        self._host_cb = self.HOST_ALLREDUCE(_cb)  # kept alive with the context
        _check(lib().blws_context_init_host_comm(self._h, int(nranks), int(rank), C.cast(self._host_cb, vp), None))

    def comm_info(self):
        nr, rk = ci(0), ci(0)
        _check(lib().blws_context_comm_info(self._h, C.byref(nr), C.byref(rk)))
        return nr.value, rk.value

    def set_profiling(self, on: bool):
        _check(lib().blws_context_set_profiling(self._h, 1 if on else 0))

    def region_stats(self, region: int = 0):
        ms, cnt, fl, by = dbl(0), i64(0), dbl(0), dbl(0)
        _check(lib().blws_context_region_stats(self._h, region, C.byref(ms), C.byref(cnt), C.byref(fl), C.byref(by)))
        return dict(ms=ms.value, count=cnt.value, flops=fl.value, bytes=by.value)

    def region_reset(self):
        _check(lib().blws_context_region_reset(self._h))

    def microbench(self, which: int, n: int, b: int = 0, reps: int = 10, detail: bool = False):
        out = np.zeros(8)
        _check(lib().blws_microbench(self._h, which, n, b, reps, _ptr(out)))
        return out if detail else float(out[0])

    def l2_probe(self, mode: int = 0, row: int = 50) -> float:
        """L2 throughput in GB/s: mode 0 streaming, mode 1 random `row`-double row gathers."""
        out = dbl(0)
        _check(lib().blws_l2_probe(self._h, int(mode), int(row), C.byref(out)))
        return out.value

    def fp64_peak(self, mode: int = 0) -> float:
        out = dbl(0)
        _check(lib().blws_fp64_peak(self._h, mode, C.byref(out)))
        return out.value


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ---------------------------------------------------------------------- rng
class Rng:
    """blws::Rng (core/rng.hpp:17-90)."""

    def __init__(self, seed: int = 0, _handle=None):
        if _handle is None:
            h = vp()
            _check(lib().blws_rng_create(int(seed) & (2**64 - 1), C.byref(h)))
            _handle = h
        self._h = _handle

    def __del__(self):
        if getattr(self, "_h", None):
            lib().blws_rng_destroy(self._h)
            self._h = None

    def split(self, tag: int) -> "Rng":
        h = vp()
        _check(lib().blws_rng_split(self._h, int(tag), C.byref(h)))
        return Rng(_handle=h)

    def next_u64(self) -> int:
        return int(lib().blws_rng_next_u64(self._h))

    def uniform(self, lo=0.0, hi=1.0) -> float:
        return float(lib().blws_rng_uniform(self._h, lo, hi))

    def uniform_index(self, n: int) -> int:
        return int(lib().blws_rng_uniform_index(self._h, int(n)))

    def normal(self) -> float:
        return float(lib().blws_rng_normal(self._h))

    def gaussian_matrix(self, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), order="F")
        _check(lib().blws_rng_gaussian_matrix(self._h, rows, cols, _ptr(out)))
        return out

    def uniform_fill(self, n, lo, hi) -> np.ndarray:
        out = np.empty(int(n))
        _check(lib().blws_rng_uniform_fill(self._h, int(n), float(lo), float(hi), _ptr(out)))
        return out


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (blws_nccl_unique_id)."""
    buf = (C.c_uint8 * 128)()
    _check(lib().blws_nccl_unique_id(C.cast(buf, vp)))
    return bytes(buf)


def sample_distinct(n: int, s: int, rng: Rng) -> np.ndarray:
    out = np.empty(s, dtype=np.int64)
    got = lib().blws_sample_distinct(n, s, rng._h, _ptr(out))
    return out[:got]


# --------------------------------------------------------------- operators
class LinearOperator:
    _h = None

    def __del__(self):
        if self._h:
            lib().blws_operator_destroy(self._h)
            self._h = None

    def rows(self) -> int:
        return int(lib().blws_operator_rows(self._h))

    def cols(self) -> int:
        return int(lib().blws_operator_cols(self._h))

    def application_count(self) -> int:
        return int(lib().blws_operator_application_count(self._h))

    def apply_pair_vec(self, left, right):
        """apply_pair (linear_operator.hpp:51-54): (W right, W^T left), counts 1."""
        left = np.ascontiguousarray(left, dtype=np.float64)
        right = np.ascontiguousarray(right, dtype=np.float64)
        top, bot = np.empty(self.rows()), np.empty(self.cols())
        _check(lib().blws_operator_apply_pair(self._h, _ptr(left), _ptr(right), _ptr(top), _ptr(bot)))
        return top, bot

    def apply_pair_block(self, left, right):
        left, right = F(left), F(right)
        b = right.shape[1]
        top = np.empty((self.rows(), b), order="F")
        bot = np.empty((self.cols(), b), order="F")
        _check(lib().blws_operator_apply_pair_block(self._h, b, _ptr(left), _ptr(right), _ptr(top), _ptr(bot)))
        return top, bot


class DenseOperator(LinearOperator):
    """DenseOperator (core/linear_operator.hpp:102-131). `w` is a host array or,
    with device=True, a device pointer / torch tensor (column-major, ld)."""

    def __init__(self, w, ctx: Context | None = None, device: bool = False, shape=None, ld=None, borrow=True):
        self.ctx = ctx or default_context()
        h = vp()
        if device:
            m, n = shape
            ld = ld or m
            _check(lib().blws_dense_operator_create(self.ctx._h, m, n, _ptr(w), ld, DEVICE, 1 if borrow else 0,
                                                    C.byref(h)))
            self._keep = w
        else:
            w = F(w)
            m, n = w.shape
            _check(lib().blws_dense_operator_create(self.ctx._h, m, n, _ptr(w), m, HOST, 0, C.byref(h)))
        self._h = h
        self.m, self.n = m, n

    def assign_ptr(self, ptr: int, ld: int, where: int):
        _check(lib().blws_dense_operator_assign(self._h, ptr, ld, where))

    def set_row_shard(self, m_total: int, row0: int):
        """This operator's rows are rows [row0, row0 + rows()) of an m_total x n
        matrix distributed over the context's ranks (blws_dense_operator_set_row_shard)."""
        _check(lib().blws_dense_operator_set_row_shard(self._h, int(m_total), int(row0)))

    def assign_async(self, ptr: int, ld: int):
        """Queue a pinned-host upload on the copy stream; the next use waits
        for it (blws_dense_operator_assign_async). The caller keeps the host
        buffer alive and unchanged until then."""
        _check(lib().blws_dense_operator_assign_async(self._h, ptr, ld))

    def assign(self, w, device=False, ld=None):
        if device:
            _check(lib().blws_dense_operator_assign(self._h, _ptr(w), ld or self.m, DEVICE))
        else:
            w = F(w)
            _check(lib().blws_dense_operator_assign(self._h, _ptr(w), w.shape[0], HOST))


class SparseOperator(LinearOperator):
    """SparseOperator (core/linear_operator.hpp:136-169) from CSC."""

    def __init__(self, m, n, colptr, rowidx, vals, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        colptr = np.ascontiguousarray(colptr, dtype=np.int64)
        rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        h = vp()
        _check(lib().blws_sparse_operator_create(self.ctx._h, m, n, len(vals), _ptr(colptr), _ptr(rowidx),
                                                 _ptr(vals), C.byref(h)))
        self._h = h
        self.m, self.n, self.nnz = m, n, len(vals)

    def assign_values(self, vals):
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        _check(lib().blws_sparse_operator_assign_values(self._h, _ptr(vals), len(vals), HOST))


# --------------------------------------------------------------- warm start
class DeviceWarmStart:
    """Device-resident WarmStart (block_lanczos.hpp:45-52)."""

    def __init__(self, handle, ctx: Context):
        self._h = handle
        self.ctx = ctx

    @classmethod
    def from_host(cls, u, v, sigma, ctx: Context | None = None):
        ctx = ctx or default_context()
        u, v = F(u), F(v)
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        h = vp()
        _check(lib().blws_warm_start_create(ctx._h, u.shape[0], v.shape[0], len(sigma), _ptr(u), u.shape[0],
                                            _ptr(v), v.shape[0], _ptr(sigma), HOST, C.byref(h)))
        return cls(h, ctx)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().blws_warm_start_destroy(self._h)
            self._h = None

    def rank(self) -> int:
        return int(lib().blws_warm_start_rank(self._h))

    def sigma(self) -> np.ndarray:
        s = np.empty(self.rank())
        _check(lib().blws_warm_start_get(self._h, None, 1, None, 1, _ptr(s), HOST))
        return s

    def copy(self) -> "DeviceWarmStart":
        h = vp()
        _check(lib().blws_warm_start_copy(self._h, C.byref(h)))
        return DeviceWarmStart(h, self.ctx)

    def to_host(self, m, n, out: "WarmStart | None" = None):
        """Download U, V, sigma; `out` (F-ordered arrays, e.g. views of pinned
        memory, with at least rank() columns) is filled in place and trimmed."""
        r = self.rank()
        if out is not None:
            u, v, s = out.u, out.v, out.sigma
            if not (u.flags.f_contiguous and v.flags.f_contiguous and u.shape[0] == m and v.shape[0] == n
                    and u.shape[1] >= r and v.shape[1] >= r and s.shape[0] >= r):
                raise ValueError("to_host: out arrays must be F-ordered (m, >=r), (n, >=r), (>=r,)")
            _check(lib().blws_warm_start_get(self._h, _ptr(u), m, _ptr(v), n, _ptr(s), HOST))
            return WarmStart(u[:, :r], v[:, :r], s[:r])
        u = np.empty((m, r), order="F")
        v = np.empty((n, r), order="F")
        s = np.empty(r)
        _check(lib().blws_warm_start_get(self._h, _ptr(u), m, _ptr(v), n, _ptr(s), HOST))
        return WarmStart(u, v, s)


@dataclass
class WarmStart:
    u: np.ndarray
    v: np.ndarray
    sigma: np.ndarray

    def rank(self) -> int:
        return len(self.sigma)


@dataclass
class BlwsResult:
    warm: WarmStart
    padded: bool
    k_raised: bool
    terminated_early: bool


def blws_svd(op: LinearOperator, warm, k: int, r: int, rng: Rng, keep_device=False):
    """blws_svd (block_lanczos.hpp:204-261) on the GPU."""
    dw = warm if isinstance(warm, DeviceWarmStart) else DeviceWarmStart.from_host(warm.u, warm.v, warm.sigma, op.ctx)
    h = vp()
    flags = ci(0)
    _check(lib().blws_svd(op._h, dw._h, k, r, rng._h, C.byref(h), C.byref(flags)))
    out = DeviceWarmStart(h, op.ctx)
    f = flags.value
    w = out if keep_device else out.to_host(op.rows(), op.cols())
    return BlwsResult(w, bool(f & 1), bool(f & 2), bool(f & 4))


def deferred_fallbacks() -> int:
    """blws_svd calls redone on the exact path (blws_svd_deferred_fallbacks)."""
    return int(lib().blws_svd_deferred_fallbacks())


def graph_launches() -> int:
    """blws_svd calls served by a captured CUDA graph (blws_svd_graph_launches)."""
    return int(lib().blws_svd_graph_launches())


def adapt_subspace(warm, r_new, m, n, rng: Rng, ctx: Context | None = None) -> WarmStart:
    ctx = ctx or default_context()
    dw = None
    if warm is not None and warm.rank() > 0:
        dw = DeviceWarmStart.from_host(warm.u, warm.v, warm.sigma, ctx)
    h = vp()
    _check(lib().blws_adapt_subspace(ctx._h, dw._h if dw else None, r_new, m, n, rng._h, C.byref(h)))
    return DeviceWarmStart(h, ctx).to_host(m, n)


def block_lanczos_procedure(op: LinearOperator, x1, k: int):
    """block_lanczos_procedure (block_lanczos.hpp:70-126) on the augmented view of op."""
    x1 = F(x1)
    b = x1.shape[1]
    dim = op.rows() + op.cols()
    q = np.zeros((dim, k * b), order="F")
    t = np.zeros((k * b) ** 2)
    built = i64(0)
    term = ci(0)
    _check(lib().blws_block_lanczos_procedure(op._h, b, _ptr(x1), k, _ptr(q), _ptr(t), C.byref(built),
                                              C.byref(term)))
    nb = built.value * b
    tt = t[: nb * nb].reshape((nb, nb), order="F")
    return q[:, :nb].copy(order="F"), tt.copy(order="F"), built.value, bool(term.value)


def lanczos_partial_svd(op: LinearOperator, r: int, tol=1e-8, max_k=0, seed=0x1A2C705):
    h = vp()
    stats = np.zeros(4, dtype=np.int64)
    _check(lib().blws_lanczos_partial_svd(op._h, r, tol, max_k, seed, C.byref(h), _ptr(stats)))
    w = DeviceWarmStart(h, op.ctx).to_host(op.rows(), op.cols())
    return w.u, w.sigma, w.v, stats


def spectral_norm(op: LinearOperator, tol=1e-6, seed=0xB1F) -> float:
    out = dbl(0)
    _check(lib().blws_spectral_norm(op._h, tol, seed, C.byref(out)))
    return out.value


def thin_qr(m, ctx: Context | None = None):
    ctx = ctx or default_context()
    m = F(m)
    if m.ndim != 2:
        raise ValueError("thin_qr: 2-D input required")
    rows, cols = m.shape
    q = np.empty((rows, cols), order="F")
    r = np.empty((cols, cols), order="F")
    rank = i64(0)
    _check(lib().blws_thin_qr(ctx._h, rows, cols, _ptr(m), _ptr(q), _ptr(r), C.byref(rank)))
    return q, r, rank.value


# ------------------------------------------------ Matrix Market (core/matrix_market.hpp)
def mm_write_dense(path, a):
    a = F(a)
    _check(lib().blws_mm_write_dense(os.fsencode(path), a.shape[0], a.shape[1], _ptr(a), a.shape[0]))


def mm_write_sparse(path, m, n, colptr, rowidx, vals):
    colptr = np.ascontiguousarray(colptr, dtype=np.int64)
    rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    _check(lib().blws_mm_write_sparse(os.fsencode(path), m, n, len(vals), _ptr(colptr), _ptr(rowidx), _ptr(vals)))


def mm_read_dense(path) -> np.ndarray:
    r, c = i64(0), i64(0)
    _check(lib().blws_mm_read_dense(os.fsencode(path), C.byref(r), C.byref(c), None, 0))
    out = np.empty((r.value, c.value), order="F")
    _check(lib().blws_mm_read_dense(os.fsencode(path), C.byref(r), C.byref(c), _ptr(out), r.value))
    return out


def mm_read_sparse(path):
    """-> (rows, cols, colptr int64, rowidx int32, values): CSC, rows ascending."""
    r, c, nz = i64(0), i64(0), i64(0)
    _check(lib().blws_mm_read_sparse(os.fsencode(path), C.byref(r), C.byref(c), C.byref(nz), None, None, None))
    colptr = np.empty(c.value + 1, dtype=np.int64)
    rowidx = np.empty(nz.value, dtype=np.int32)
    vals = np.empty(nz.value)
    _check(lib().blws_mm_read_sparse(os.fsencode(path), C.byref(r), C.byref(c), C.byref(nz), _ptr(colptr),
                                     _ptr(rowidx), _ptr(vals)))
    return r.value, c.value, colptr, rowidx, vals


def full_svd_small(w, ctx: Context | None = None):
    """full_svd_small (small_dense.hpp:72-87) on the GPU: (u, sigma, v), descending."""
    ctx = ctx or default_context()
    w = F(w)
    m, n = w.shape
    p = min(m, n)
    s = np.empty(p)
    u = np.empty((m, p), order="F")
    v = np.empty((n, p), order="F")
    _check(lib().blws_full_svd_small(ctx._h, m, n, _ptr(w), _ptr(s), _ptr(u), _ptr(v)))
    return u, s, v


def sym_evd_small(t, ctx: Context | None = None):
    ctx = ctx or default_context()
    t = F(t)
    if t.ndim != 2 or t.shape[0] != t.shape[1]:
        raise ValueError("sym_evd_small: not square")
    n = t.shape[0]
    vals = np.empty(n)
    vecs = np.empty((n, n), order="F")
    _check(lib().blws_sym_evd(ctx._h, n, _ptr(t), _ptr(vals), _ptr(vecs)))
    return vals, vecs


def sym_evd_tridiagonal_top(d, e, want, ctx: Context | None = None):
    ctx = ctx or default_context()
    d = np.ascontiguousarray(d, dtype=np.float64)
    e = np.ascontiguousarray(e, dtype=np.float64)
    n = len(d)
    vals = np.empty(want)
    vecs = np.empty((n, want), order="F")
    _check(lib().blws_sym_evd_tridiagonal_top(ctx._h, n, _ptr(d), _ptr(e), want, _ptr(vals), _ptr(vecs)))
    return vals, vecs


def dgemm(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, ctx: Context | None = None):
    """Device-pointer GEMM (a, b, c: torch tensors or raw pointers)."""
    ctx = ctx or default_context()
    _check(lib().blws_dgemm(ctx._h, 1 if ta else 0, 1 if tb else 0, m, n, k, alpha, _ptr(a), lda, _ptr(b), ldb, beta,
                            _ptr(c), ldc))


# ------------------------------------------------------------ backend / svt
class SvdBackend:
    """SvdBackend<double> (svt.hpp:84-196); kinds EXACT_FULL=0, LANCZOS=1, BLWS=2."""

    EXACT_FULL, LANCZOS, BLWS = 0, 1, 2

    def __init__(self, kind=2, block_steps=2, ritz_tol=1e-8, max_k=0, seed_margin=5, seed=0xB10C,
                 ctx: Context | None = None):
        self.ctx = ctx or default_context()
        h = vp()
        _check(lib().blws_svd_backend_create(self.ctx._h, kind, block_steps, ritz_tol, max_k, seed_margin,
                                             int(seed) & (2**64 - 1), C.byref(h)))
        self._h = h
        self.kind = kind

    @classmethod
    def exact_full(cls, **kw):
        """svt.hpp:108-116: full SVD of the dense W on the device (m + n <= 4096)."""
        return cls(kind=0, **kw)

    @classmethod
    def lanczos(cls, **kw):
        return cls(kind=1, **kw)

    @classmethod
    def blws(cls, **kw):
        return cls(kind=2, **kw)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().blws_svd_backend_destroy(self._h)
            self._h = None

    def warm_state(self, m, n):
        h = vp()
        _check(lib().blws_svd_backend_warm_state(self._h, C.byref(h)))
        if not h.value:
            return None
        return DeviceWarmStart(h, self.ctx).to_host(m, n)

    def set_warm_state(self, w: DeviceWarmStart):
        _check(lib().blws_svd_backend_set_warm_state(self._h, w._h))


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


def svt(op: LinearOperator, eps: float, backend: SvdBackend, predictor: RankPredictor, keep_device=False):
    pred = PredictorC(predictor.r, predictor.increment, predictor.max_rank)
    hist = np.zeros(1, dtype=np.int64)
    hl = i64(0)
    h = vp()
    ach = i64(0)
    above = ci(0)
    _check(lib().blws_svt(op._h, eps, backend._h, C.byref(pred), _ptr(hist), 1, C.byref(hl), C.byref(h),
                          C.byref(ach), C.byref(above)))
    predictor.r = int(pred.r)
    predictor.history.append(int(hist[0]))
    dw = DeviceWarmStart(h, op.ctx)
    if keep_device:
        return dw, ach.value, bool(above.value)
    w = dw.to_host(op.rows(), op.cols())
    return SvtResult(w.u, w.sigma, w.v, ach.value, bool(above.value))


# ----------------------------------------------------------------- solvers
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


def _stats(s: SolverStatsC, ph, mh, rh):
    it = int(s.iterations)
    return SolverStats(iterations=it, wall_time_s=s.wall_time_s, matvec_count=int(s.matvec_count),
                       matvec_init=int(s.matvec_init), rel_err=s.rel_err, rank_hat=int(s.rank_hat), e_l0=int(s.e_l0),
                       converged=bool(s.converged), predicted_ranks=[int(x) for x in ph[:it]],
                       matvec_history=[int(x) for x in mh[:it]], residual_history=[float(x) for x in rh[:it]])


def rpca_adm(d, backend: SvdBackend, lam=0.0, tol_outer=1e-7, max_iter=1000, rho=1.5, mu_max_factor=1e7,
             initial_rank=10, rank_increment=5, truth=None, want_outputs=True, device=False, m=None, ld=None,
             a_out=None, e_out=None):
    """rpca_adm (solvers.hpp:72-157) on the GPU. Host numpy input by default;
    device=True takes device pointers / torch tensors (then a_out/e_out are
    caller device buffers)."""
    ctx = backend.ctx
    opts = RpcaOptionsC(tol_outer, max_iter, rho, mu_max_factor, initial_rank, rank_increment)
    st = SolverStatsC()
    ph = np.zeros(max_iter + 1, dtype=np.int64)
    mh = np.zeros(max_iter + 1, dtype=np.int64)
    rh = np.zeros(max_iter + 1)
    if device:
        ld = ld or m
        _check(lib().blws_rpca_adm(ctx._h, m, _ptr(d), ld, DEVICE, lam, backend._h, C.byref(opts), _ptr(truth),
                                   _ptr(a_out), _ptr(e_out), C.byref(st), _ptr(ph), _ptr(mh), _ptr(rh), max_iter + 1))
        return a_out, e_out, _stats(st, ph, mh, rh), int(st.e_nnz)
    d = F(d)
    m = d.shape[0]
    if d.shape[0] != d.shape[1]:
        raise ValueError("rpca_adm: D must be square")
    a = np.empty((m, m), order="F") if want_outputs else None
    e = np.empty((m, m), order="F") if want_outputs else None
    tr = F(truth) if truth is not None else None
    _check(lib().blws_rpca_adm(ctx._h, m, _ptr(d), m, HOST, lam, backend._h, C.byref(opts), _ptr(tr), _ptr(a),
                               _ptr(e), C.byref(st), _ptr(ph), _ptr(mh), _ptr(rh), max_iter + 1))
    return a, e, _stats(st, ph, mh, rh), int(st.e_nnz)


def mc_svt(m, n, colptr, rowidx, vals, backend: SvdBackend, tau=0.0, delta=0.0, tol_outer=1e-4, max_iter=500,
           initial_rank=10, rank_increment=5, truth_ml=None, truth_mr=None, cap=None):
    """mc_svt (solvers.hpp:202-270) on the GPU; observation as host CSC."""
    ctx = backend.ctx
    colptr = np.ascontiguousarray(colptr, dtype=np.int64)
    rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    cap = cap or min(m, n)
    u = np.empty((m, cap), order="F")
    s = np.empty(cap)
    v = np.empty((n, cap), order="F")
    rank = i64(0)
    opts = McOptionsC(tol_outer, max_iter, initial_rank, rank_increment)
    st = SolverStatsC()
    ph = np.zeros(max_iter + 1, dtype=np.int64)
    mh = np.zeros(max_iter + 1, dtype=np.int64)
    rh = np.zeros(max_iter + 1)
    r_true = 0
    ml = mr = None
    if truth_ml is not None:
        ml, mr = F(truth_ml), F(truth_mr)
        r_true = ml.shape[1]
    _check(lib().blws_mc_svt(ctx._h, m, n, len(vals), _ptr(colptr), _ptr(rowidx), _ptr(vals), tau, delta, backend._h,
                             C.byref(opts), _ptr(ml), _ptr(mr), r_true, _ptr(u), _ptr(s), _ptr(v), cap, C.byref(rank),
                             C.byref(st), _ptr(ph), _ptr(mh), _ptr(rh), max_iter + 1))
    k = rank.value
    return u[:, :k].copy(order="F"), s[:k].copy(), v[:, :k].copy(order="F"), _stats(st, ph, mh, rh)


def rpca_adm_sharded(d_rows, m, row0, backend: SvdBackend, lam=0.0, tol_outer=1e-7, max_iter=1000, rho=1.5,
                     mu_max_factor=1e7, initial_rank=10, rank_increment=5, truth_rows=None, want_outputs=True):
    """Row-sharded rpca_adm: this rank holds rows [row0, row0 + rows)
    of the m x m D (host numpy, rows x m); the backend's context carries the
    communicator (Context.init_comm; without one it runs as a single rank).
    Returns this rank's rows of A and E and the (rank-identical) stats."""
    ctx = backend.ctx
    d = F(d_rows)
    rows = d.shape[0]
    if d.shape[1] != m:
        raise ValueError("rpca_adm_sharded: D rows must have m columns")
    opts = RpcaOptionsC(tol_outer, max_iter, rho, mu_max_factor, initial_rank, rank_increment)
    st = SolverStatsC()
    ph = np.zeros(max_iter + 1, dtype=np.int64)
    mh = np.zeros(max_iter + 1, dtype=np.int64)
    rh = np.zeros(max_iter + 1)
    a = np.empty((rows, m), order="F") if want_outputs else None
    e = np.empty((rows, m), order="F") if want_outputs else None
    tr = F(truth_rows) if truth_rows is not None else None
    _check(lib().blws_rpca_adm_sharded(ctx._h, m, rows, row0, _ptr(d), rows, HOST, lam, backend._h, C.byref(opts),
                                       _ptr(tr), _ptr(a), _ptr(e), C.byref(st), _ptr(ph), _ptr(mh), _ptr(rh),
                                       max_iter + 1))
    return a, e, _stats(st, ph, mh, rh), int(st.e_nnz)


def mc_svt_sharded(m, row0, rows, n, colptr, rowidx, vals, backend: SvdBackend, tau=0.0, delta=0.0, tol_outer=1e-4,
                   max_iter=500, initial_rank=10, rank_increment=5, truth_ml_rows=None, truth_mr=None, cap=None):
    """Row-sharded mc_svt: this rank's observed rows [row0, row0 + rows) as a
    local CSC over the n columns (row indices local). Returns this rank's rows
    of U, sigma, V and the stats (dist.shard_csc builds the local CSC)."""
    ctx = backend.ctx
    colptr = np.ascontiguousarray(colptr, dtype=np.int64)
    rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    cap = cap or min(m, n)
    u = np.empty((rows, cap), order="F")
    s = np.empty(cap)
    v = np.empty((n, cap), order="F")
    rank = i64(0)
    opts = McOptionsC(tol_outer, max_iter, initial_rank, rank_increment)
    st = SolverStatsC()
    ph = np.zeros(max_iter + 1, dtype=np.int64)
    mh = np.zeros(max_iter + 1, dtype=np.int64)
    rh = np.zeros(max_iter + 1)
    r_true = 0
    ml = mr = None
    if truth_ml_rows is not None:
        ml, mr = F(truth_ml_rows), F(truth_mr)
        r_true = ml.shape[1]
    _check(lib().blws_mc_svt_sharded(ctx._h, m, rows, row0, n, len(vals), _ptr(colptr), _ptr(rowidx), _ptr(vals),
                                     tau, delta, backend._h, C.byref(opts), _ptr(ml), _ptr(mr), r_true, _ptr(u),
                                     _ptr(s), _ptr(v), cap, C.byref(rank), C.byref(st), _ptr(ph), _ptr(mh), _ptr(rh),
                                     max_iter + 1))
    k = rank.value
    return u[:, :k].copy(order="F"), s[:k].copy(), v[:, :k].copy(order="F"), _stats(st, ph, mh, rh)
