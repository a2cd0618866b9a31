"""GPU parity of the dense building blocks against the CPU oracle / numpy.

Each test restates a reference test (proj/tests/test_dense_core.cpp,
test_lanczos.cpp) with the device path under test; tolerances are the
reference's unless stated.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu(G):
    import torch

    assert torch.cuda.is_available(), "GPU tests need a B200"
    return G


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("m,n,k", [(64, 64, 16), (257, 33, 1001), (1000, 100, 4000), (7, 5, 3), (100, 100, 20000)])
def test_dgemm_matches_numpy(gpu, ta, tb, m, n, k):
    import torch

    rs = np.random.default_rng(m * 7 + n * 3 + k)
    A = rs.standard_normal((k, m) if ta else (m, k))
    B = rs.standard_normal((n, k) if tb else (k, n))
    C0 = rs.standard_normal((m, n))
    ref = 1.5 * ((A.T if ta else A) @ (B.T if tb else B)) - 0.5 * C0
    dev = torch.device("cuda:0")
    # column-major = transpose of a contiguous row-major tensor
    At = torch.tensor(A.T.copy(), device=dev)
    Bt = torch.tensor(B.T.copy(), device=dev)
    Ct = torch.tensor(C0.T.copy(), device=dev)
    gpu.api.dgemm(ta, tb, m, n, k, 1.5, At, A.shape[0], Bt, B.shape[0], -0.5, Ct, m)
    torch.cuda.synchronize()
    got = Ct.cpu().numpy().T
    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()) * np.sqrt(k)


def test_thin_qr_known_answers(gpu, O):
    q, r, rank = gpu.thin_qr(np.array([[3.0], [4.0]]))
    assert abs(q[0, 0] - 0.6) <= 1e-14 and abs(q[1, 0] - 0.8) <= 1e-14 and abs(r[0, 0] - 5.0) <= 1e-14
    assert rank == 1
    g = O.Rng(11).gaussian_matrix(12, 4)
    qq = O.thin_qr(g).q
    q2, r2, rk = gpu.thin_qr(qq)
    assert np.linalg.norm(q2 - qq) <= 1e-12 and np.linalg.norm(r2 - np.eye(4)) <= 1e-12 and rk == 4


@pytest.mark.parametrize("m,b", [(5, 1), (20, 4), (50, 10), (200, 30), (8000, 100), (4000, 205)])
def test_thin_qr_recomposition_and_oracle(gpu, O, m, b):
    a = O.Rng(17 + m).gaussian_matrix(m, b)
    q, r, rank = gpu.thin_qr(a)
    assert np.linalg.norm(a - q @ r) <= 1e-12 * np.linalg.norm(a)
    assert np.linalg.norm(q.T @ q - np.eye(b)) <= 1e-12
    assert np.all(np.diag(r) >= 0) and rank == b
    assert np.allclose(np.tril(r, -1), 0.0)
    ref = O.thin_qr(a)
    assert np.abs(q - ref.q).max() <= 1e-10
    assert np.abs(r - ref.r).max() <= 1e-10 * np.abs(ref.r).max()


def test_thin_qr_rank_deficiency(gpu, O):
    col = O.Rng(3).gaussian_vector(10)
    m = np.stack([col, 2.0 * col], axis=1)
    assert gpu.thin_qr(m)[2] == 1
    assert O.thin_qr(m).rank == 1
    with pytest.raises(ValueError):
        gpu.thin_qr(np.zeros((2, 5)))
    with pytest.raises(ValueError):
        gpu.thin_qr(np.array([[1.0], [np.nan]]))


def test_thin_qr_ill_conditioned_uses_shifted_cholqr(gpu, O):
    rs = np.random.default_rng(5)
    u, _ = np.linalg.qr(rs.standard_normal((3000, 40)))
    v, _ = np.linalg.qr(rs.standard_normal((40, 40)))
    a = (u * np.logspace(0, -11, 40)) @ v.T
    q, r, rank = gpu.thin_qr(a)
    assert np.linalg.norm(q.T @ q - np.eye(40)) <= 1e-12
    assert np.linalg.norm(a - q @ r) <= 1e-12 * np.linalg.norm(a)
    assert rank == O.thin_qr(a).rank


def test_sym_evd_known_answers(gpu):
    vals, vecs = gpu.sym_evd_small(np.diag([3.0, 1.0, 2.0]))
    assert np.allclose(vals, [3, 2, 1])
    assert np.allclose(np.abs(vecs).max(axis=0), 1.0, atol=1e-12)
    vals, vecs = gpu.sym_evd_small(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert abs(vals[0] - 1) <= 1e-14 and abs(vals[1] + 1) <= 1e-14
    assert abs(abs(vecs[0, 0] * vecs[1, 0]) - 0.5) <= 1e-12
    assert abs(vecs[0, 1] * vecs[1, 1] + 0.5) <= 1e-12
    with pytest.raises(ValueError):
        gpu.sym_evd_small(np.array([[0.0, 1.0], [5.0, 0.0]]))


@pytest.mark.parametrize("n", [12, 61, 110, 200, 216, 222, 224, 230, 260, 810, 1056, 1900])  # 1900: global-memory back-transformation
def test_sym_evd_matches_oracle(gpu, O, n):
    g = O.Rng(23 + n).gaussian_matrix(n, n)
    t = 0.5 * (g + g.T)
    vals, vecs = gpu.sym_evd_small(t)
    ref_vals, _ = O.sym_evd_small(t)
    tn = np.linalg.norm(t)
    assert np.abs(vals - ref_vals).max() <= 1e-12 * tn
    assert np.linalg.norm(t @ vecs - vecs * vals) <= 1e-10 * tn
    assert np.linalg.norm(vecs.T @ vecs - np.eye(n)) <= 1e-10


@pytest.mark.parametrize("n", [16, 17, 40, 63, 96, 127, 150, 199, 200])
def test_sym_evd_two_stage(gpu, O, n, monkeypatch):
    # dense -> band 8 -> tridiagonal (sytrd2.cu), forced on for every order here
    monkeypatch.setenv("BLWS_EVD2", "1")
    g = O.Rng(57 + n).gaussian_matrix(n, n)
    tn_cases = [0.5 * (g + g.T)]
    # repeated eigenvalues and a zero block: Q diag(3,3,3,1,...,0,0) Q^T
    q, _ = np.linalg.qr(O.Rng(5 + n).gaussian_matrix(n, n))
    lam = np.concatenate([[3.0, 3.0, 3.0], np.linspace(1, 0, n - 3)])
    lam[-min(4, n - 3):] = 0.0
    tn_cases.append((q * lam) @ q.T)
    for t in tn_cases:
        t = 0.5 * (t + t.T)
        vals, vecs = gpu.sym_evd_small(t)
        ref_vals, _ = O.sym_evd_small(t)
        tn = np.linalg.norm(t)
        assert np.abs(vals - ref_vals).max() <= 1e-12 * tn
        assert np.linalg.norm(t @ vecs - vecs * vals) <= 1e-10 * tn
        assert np.linalg.norm(vecs.T @ vecs - np.eye(n)) <= 1e-10


@pytest.mark.parametrize("n", [64, 110, 208, 260])
def test_sym_evd_cluster_tridiagonalisation(gpu, O, n, monkeypatch):
    # opt-in cluster-distributed Householder stage (sytrd_cluster.cu)
    monkeypatch.setenv("BLWS_SYTRD", "cluster")
    g = O.Rng(41 + n).gaussian_matrix(n, n)
    t = 0.5 * (g + g.T)
    vals, vecs = gpu.sym_evd_small(t)
    ref_vals, _ = O.sym_evd_small(t)
    tn = np.linalg.norm(t)
    assert np.abs(vals - ref_vals).max() <= 1e-12 * tn
    assert np.linalg.norm(t @ vecs - vecs * vals) <= 1e-10 * tn


def test_tridiagonal_top_matches_oracle(gpu, O):
    rs = np.random.default_rng(9)
    for n, want in [(10, 3), (60, 20), (500, 40), (2600, 12)]:  # > 2048: global-memory path
        d = rs.standard_normal(n)
        e = np.abs(rs.standard_normal(n - 1))
        vals, vecs = gpu.sym_evd_tridiagonal_top(d, e, want)
        rv, rvec = O.sym_evd_tridiagonal(d, e)
        assert np.abs(vals - rv[:want]).max() <= 1e-13 * np.abs(rv).max()
        t = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
        assert np.linalg.norm(t @ vecs - vecs * vals) <= 1e-11 * np.abs(rv).max()
        assert np.linalg.norm(vecs.T @ vecs - np.eye(want)) <= 1e-10


def test_tridiagonal_degenerate_clusters(gpu):
    # identity blocks decoupled by zero couplings (Lanczos restarts on I)
    d = np.ones(9)
    e = np.zeros(8)
    vals, vecs = gpu.sym_evd_tridiagonal_top(d, e, 3)
    assert np.allclose(vals, 1.0, atol=1e-14)
    assert np.linalg.norm(vecs.T @ vecs - np.eye(3)) <= 1e-10


@pytest.mark.parametrize("m,n", [(1, 1), (37, 1029), (2500, 700), (5000, 3001)])
def test_pair_gemv_matches_numpy(gpu, m, n):
    # K10: W x and W^T y from one pass over W (Lanczos step), via the single-vector pair apply
    rs = np.random.default_rng(m + n)
    w = rs.standard_normal((m, n))
    x, y = rs.standard_normal(n), rs.standard_normal(m)
    op = gpu.DenseOperator(w)
    top, bot = op.apply_pair_block(y[:, None], x[:, None])  # block path (reference)
    t1, b1 = op.apply_pair_vec(y, x)
    assert np.abs(t1 - w @ x).max() <= 1e-12 * np.sqrt(n) * np.abs(w @ x).max()
    assert np.abs(b1 - w.T @ y).max() <= 1e-12 * np.sqrt(m) * np.abs(w.T @ y).max()


@pytest.mark.parametrize("b", [1, 3, 4, 7, 8, 9, 32, 33, 64, 100, 128, 130])
def test_sparse_pair_block_matches_numpy(gpu, b):
    # K8 (csr_spmm_k, one template per 32-column slot count + the wide path):
    # ragged columns and rows, including empty ones and one dense row
    rs = np.random.default_rng(b)
    m, n = 700, 450
    dense = np.where(rs.random((m, n)) < 0.05, rs.standard_normal((m, n)), 0.0)
    dense[13, :] = 0.0
    dense[:, 17] = 0.0
    dense[200, :] = rs.standard_normal(n)
    colptr = np.zeros(n + 1, dtype=np.int64)
    rows, vals = [], []
    for j in range(n):
        nz = np.nonzero(dense[:, j])[0]
        rows.append(nz)
        vals.append(dense[nz, j])
        colptr[j + 1] = colptr[j] + len(nz)
    op = gpu.api.SparseOperator(m, n, colptr, np.concatenate(rows).astype(np.int32), np.concatenate(vals))
    left, right = rs.standard_normal((m, b)), rs.standard_normal((n, b))
    top, bot = op.apply_pair_block(left, right)
    ref_top, ref_bot = dense @ right, dense.T @ left
    assert np.abs(top - ref_top).max() <= 1e-12 * np.abs(ref_top).max()
    assert np.abs(bot - ref_bot).max() <= 1e-12 * np.abs(ref_bot).max()


@pytest.mark.parametrize("b", [9, 55, 100])
def test_sparse_spmm_large_ragged(gpu, b):
    # K8 at a larger size: 21000 x 1500 at 1% density, odd b, a dense row and
    # an empty column (more rows than the grid has warps: grid-stride rows)
    import scipy.sparse as sp

    rs = np.random.default_rng(100 + b)
    m, n = 21000, 1500
    a = sp.random(m, n, density=0.01, format="csc", random_state=rs, data_rvs=rs.standard_normal)
    a = a.tolil()
    a[5, :] = rs.standard_normal(n)
    a[:, 7] = 0.0
    a = a.tocsc()
    a.sort_indices()
    op = gpu.api.SparseOperator(m, n, a.indptr.astype(np.int64), a.indices.astype(np.int32), a.data.copy())
    left, right = rs.standard_normal((m, b)), rs.standard_normal((n, b))
    top, bot = op.apply_pair_block(left, right)
    ref_top, ref_bot = a @ right, a.T @ left
    assert np.abs(top - ref_top).max() <= 1e-12 * np.abs(ref_top).max()
    assert np.abs(bot - ref_bot).max() <= 1e-12 * np.abs(ref_bot).max()


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("m,n,k", [(1001, 37, 999), (5000, 104, 130), (300, 128, 17), (4000, 100, 4000),
                                   (2047, 64, 61), (640, 8, 1)])
def test_tall_skinny_gemm_edges(gpu, ta, m, n, k):
    # the tall-skinny path (TMA-staged, dgemm_tma.cuh): ragged M / K / N and
    # padded leading dimensions (even, as the 16-byte TMA strides require);
    # out-of-range rows and k are zero-filled by the tensor loads
    import torch

    rs = np.random.default_rng(m + 3 * n + 7 * k + int(ta))
    A = rs.standard_normal((k, m) if ta else (m, k))
    B = rs.standard_normal((k, n))
    C0 = rs.standard_normal((m, n))
    ref = 1.25 * ((A.T if ta else A) @ B) + 0.5 * C0
    dev = torch.device("cuda:0")

    def padded(x):
        rows, cols = x.shape
        ld = rows + (2 if rows % 2 == 0 else 1)
        t = torch.zeros((cols, ld), dtype=torch.float64, device=dev)  # column-major with ld
        t[:, :rows] = torch.tensor(x.T.copy(), device=dev)
        return t, ld

    At, lda = padded(A)
    Bt, ldb = padded(B)
    Ct, ldc = padded(C0)
    gpu.api.dgemm(ta, False, m, n, k, 1.25, At, lda, Bt, ldb, 0.5, Ct, ldc)
    torch.cuda.synchronize()
    got = Ct[:, :m].cpu().numpy().T
    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()) * np.sqrt(k)
    assert torch.all(Ct[:, m:] == 0)  # the padding rows are left alone


@pytest.mark.parametrize("m,b", [(600, 16), (3000, 100), (2000, 111), (900, 37), (400, 112), (300, 113)])
@pytest.mark.parametrize("kind", ["orthonormal", "near", "general", "graded"])
def test_thin_qr_factor_modes(gpu, O, m, b, kind):
    # cholqr.cu picks the factorisation on the device: a scaled-identity Gram
    # (skip), a near-identity Gram (closed form I + F, ||E|| <= 1e-9), or the
    # blocked Cholesky; b = 113 takes the chol_inv_upper path. Every mode must
    # reproduce the oracle's Householder Q / R.
    rng = O.Rng(1000 + m + b)
    a = rng.gaussian_matrix(m, b)
    if kind in ("orthonormal", "near"):
        a = O.thin_qr(a).q * 3.0
        if kind == "near":
            a = a + 1e-12 * rng.gaussian_matrix(m, b)
    elif kind == "graded":
        a = a * np.logspace(0, -4, b)
    q, r, rank = gpu.thin_qr(a)
    ref = O.thin_qr(a)
    assert rank == ref.rank == b
    assert np.linalg.norm(q.T @ q - np.eye(b)) <= 1e-13
    assert np.linalg.norm(a - q @ r) <= 1e-13 * np.linalg.norm(a)
    assert np.allclose(np.tril(r, -1), 0.0) and np.all(np.diag(r) > 0)
    assert np.abs(q - ref.q).max() <= 1e-9
    assert np.abs(r - ref.r).max() <= 1e-12 * np.abs(ref.r).max()


@pytest.mark.parametrize("m,n,k,sym", [(100, 100, 8000, True), (100, 100, 8000, False), (7, 13, 300, False),
                                       (128, 128, 5000, True), (111, 111, 2001, True), (64, 32, 777, False)])
def test_dgemm_tn_small_output(gpu, m, n, k, sym):
    # the K2 Grams / projections: A^T B with M, N <= 128 over many rows (split-K
    # with a deterministic reduction); beta != 0, ragged K, a Gram (A == B), and
    # the result bitwise reproducible run to run (fixed reduction order)
    import torch

    rs = np.random.default_rng(m + 5 * n + k)
    A = rs.standard_normal((k, m))
    B = A if sym else rs.standard_normal((k, n))
    C0 = rs.standard_normal((m, n))
    ref = 0.75 * (A.T @ B) + 0.25 * C0
    dev = torch.device("cuda:0")
    At = torch.tensor(A.T.copy(), device=dev)
    Bt = At if sym else torch.tensor(B.T.copy(), device=dev)
    outs = []
    for _ in range(2):
        Ct = torch.tensor(C0.T.copy(), device=dev)
        gpu.api.dgemm(True, False, m, n, k, 0.75, At, k, Bt, k, 0.25, Ct, m)
        torch.cuda.synchronize()
        outs.append(Ct.cpu().numpy().T)
    assert np.abs(outs[0] - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()) * np.sqrt(k)
    assert np.array_equal(outs[0], outs[1])
    if sym:
        assert np.array_equal(outs[0] - 0.25 * C0, (outs[0] - 0.25 * C0).T) or np.abs(
            (outs[0] - 0.25 * C0) - (outs[0] - 0.25 * C0).T).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("rows,b", [(4000, 100), (4003, 97), (37, 7), (5, 112), (20001, 64), (1, 1), (9000, 16)])
def test_gram16_matches_split_k(gpu, rows, b):
    # gram16.cu (the CholQR Grams, b <= 112): one cluster launch per Gram, every
    # 16 x 16 tile of the upper triangle reduced over an 8-CTA cluster through
    # DSMEM and mirrored. Compared with the split-K GEMM on the same panel
    # (microbench mode 10 returns max |G16 - G| / max |G|), ragged rows / widths
    # included, and run repeatedly (the DSMEM hand-off must not race).
    ctx = gpu.Context(0)
    for _ in range(3):
        d = ctx.microbench(10, rows, b, 2, detail=True)
        assert d[1] <= 1e-14 * max(1.0, np.sqrt(rows)), (rows, b, d[1])
