"""B200-native (sm_100a) BLWS partial singular value thresholding.

The hot path of arXiv 1012.0365's block Lanczos with warm start — the
per-iteration partial SVT inside the RPCA (inexact ALM) and MC (SVT) solvers —
as hand-written CUDA behind a C ABI (include/blws_cuda.h). This package is the
Python mirror of the reference's C++ API (proj/include/blws); see api.py.
"""
from . import api  # noqa: F401
from .api import (  # noqa: F401
    Context,
    DenseOperator,
    DeviceWarmStart,
    RankPredictor,
    Rng,
    SparseOperator,
    SvdBackend,
    WarmStart,
    adapt_subspace,
    blws_svd,
    deferred_fallbacks,
    full_svd_small,
    graph_launches,
    block_lanczos_procedure,
    lanczos_partial_svd,
    mc_svt,
    mc_svt_sharded,
    rpca_adm,
    rpca_adm_sharded,
    sample_distinct,
    spectral_norm,
    svt,
    sym_evd_small,
    sym_evd_tridiagonal_top,
    thin_qr,
)
from .api import LIB_PATH  # noqa: F401
