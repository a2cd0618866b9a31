// Host-callable launchers for every device kernel of the BLWS hot path.
// Each launcher enqueues on ctx.stream() and counts its launches.
#pragma once
#include "common.cuh"

namespace blws {

// ------------------------------------------------------------------ GEMM (K1, K2, K5)
/// C = alpha * op(A) * op(B) + beta * C, column-major fp64, DMMA tensor cores.
/// op(A) is M x K, op(B) is K x N. Split-K with a deterministic reduction
/// when the output tile grid alone cannot fill the SMs.
void gemm(Context& ctx, bool ta, bool tb, Index M, Index N, Index K, double alpha, const double* A, Index lda,
          const double* B, Index ldb, double beta, double* C, Index ldc);

// ------------------------------------------------------------------ level-1 / small
void fill(Context& ctx, View x, double v);
/// full_svd_small (small_dense.hpp:72-87) via the symmetric embedding: sigma (p),
/// u (m x p), v (n x p), p = min(m, n), descending.
void full_svd_small(Context& ctx, View w, double* sigma, View u, View v);
/// Lanczos steps l0..l1-1 on the augmented view of a dense W (m <= 4096) in one
/// cooperative launch (lanczos_coop.cu); false if not applicable. q holds the
/// basis (column l0 already set); column l+1 receives each next direction.
bool lanczos_coop_steps(Context& ctx, const double* w, Index ldw, Index m, Index n, Index mp, double* q, Index ldq,
                        double* r,
                        double* alpha, double* lastbeta, double* coup, double* state, double* coef, Index cap,
                        Index dim, Index l0, Index l1);
// row-owned variant with the basis resident in shared memory (lanczos_rows.cu)
bool lanczos_rows_steps(Context& ctx, const double* w, Index ldw, Index m, Index n, Index mp, double* q, Index ldq,
                        double* r,
                        double* alpha, double* lastbeta, double* coup, double* state, double* coef, Index cap,
                        Index dim, Index l0, Index l1);
/// top = W x (m), bot = W^T y (n) in one pass over column-major W (K10).
void pair_gemv(Context& ctx, Index m, Index n, const double* w, Index ld, const double* x, const double* y,
               double* top, double* bot);
/// Zeroes `bytes` (multiple of 4) with a kernel: a cudaMemsetAsync may be
/// queued on a copy engine behind a pending host upload.
void zero(Context& ctx, void* p, size_t bytes);
/// dst (x.rows x x.cols, row-major) = x; and back (column-major view dst).
void pack_rows(Context& ctx, View x, double* dst);
void unpack_rows(Context& ctx, const double* src, View dst);
void copy(Context& ctx, View dst, View src, double alpha = 1.0);  // dst = alpha * src
void axpy(Context& ctx, View y, View x, double alpha);            // y += alpha * x
/// out[0] = sum of squares of x (deterministic two-pass reduction).
void sumsq(Context& ctx, View x, double* out);
/// *flag = 1 if x has a non-finite entry, else 0 (device; stream-ordered)
void nonfinite_count(Context& ctx, View x, int* flag);
/// out[0] = sum of squares of (X - I) for a square X.
void sumsq_minus_identity(Context& ctx, View x, double* out);
/// dst = 0.5 * (src + src^T), square.
void symmetrize(Context& ctx, View dst, View src);
/// Scatter a b x b block (or its transpose) into a larger matrix.
void place_block(Context& ctx, View dst, View src, bool transpose);
/// dst(:, j) = src(:, j) * s[j]   (s on device)
void scale_columns(Context& ctx, View dst, View src, const double* s);
/// Gather selected columns: dst(:, j) = src(:, idx[j]) (idx on device).
void gather_columns(Context& ctx, View dst, View src, const int* idx);

// ------------------------------------------------------------------ small dense (K3, K4)
/// In-place upper Cholesky of the leading n x n of G (G = R^T R, R upper).
/// status[0] = 0 on success, j+1 if pivot j was not positive or not finite.
/// min_diag/max_diag of R written to status-adjacent doubles diag[0..1].
void potrf_upper(Context& ctx, View g, int* status, double* diag);
/// Fused blocked Cholesky + inverse: G <- R (upper, zero lower), rinv <- R^{-1};
/// status / diag as potrf_upper. With skip_rel > 0 a Gram with ||G - cI||_F <=
/// skip_rel c (c = tr(G) / n) yields R = sqrt(c) I, Rinv = I / sqrt(c) without
/// factorising (device-predicated CholQR pass skip); tr(G) -> *trace_out if set.
void chol_inv_upper(Context& ctx, View g, View rinv, int* status, double* diag, double skip_rel = 0.0,
                    double* trace_out = nullptr);
/// The same for 112 < n <= 1024 by 112-column blocks (cholblk.cu): diagonal
/// blocks on cholqr_factor_k, panels / trailing updates / R^{-1} on the GEMM;
/// no whole-matrix skip mode. chol_inv_upper routes there (BLWS_CHOL_BLOCKED=0: not).
bool chol_blocked_fits(Index n);
void chol_inv_blocked(Context& ctx, View g, View rinv, int* status, double* diag, double* trace_out);
/// One CholQR pass factor for n <= 112 (cholqr.cu): G <- R (upper), rinv <-
/// R^{-1}; with r_prev, r_out <- R * r_prev (upper) when r_out is set and
/// rank_out <- #diag(R * r_prev) > 1e-12 sqrt(trace_ref[0]) (trace_ref = null:
/// this G's trace). The factorisation (scaled identity / near identity / blocked
/// Cholesky) is picked on the device; status, diag, trace_out as chol_inv_upper.
/// G = X^T X (full, exactly symmetric) for b = x.cols <= 112 (gram16.cu): one
/// cluster launch, no split-K workspace, fixed summation order.
bool gram16_fits(Index rows, Index b);
void gram16(Context& ctx, View x, double* g, Index ldg);
bool cholqr_factor_fits(Index n);
void cholqr_factor(Context& ctx, View g, View rinv, const double* r_prev, Index ldp, View* r_out, int* status,
                   double* diag, double* trace_out, const double* trace_ref, std::int64_t* rank_out);
/// R^{-1} of an upper-triangular n x n R (out may not alias r).
void trtri_upper(Context& ctx, View out, View r);
/// C = A * B for upper-triangular n x n A, B (C upper triangular).
void trmm_upper(Context& ctx, View c, View a, View b);
/// G += s * I
void add_diagonal(Context& ctx, View g, const double* s_dev);
/// count of diag(R) > tau (tau = scale * sqrt(sumsq[0])) -> out[0]
void count_diag_above(Context& ctx, View r, const double* sumsq_dev, double scale, std::int64_t* out);

/// Top `want` eigenpairs (descending) of a dense symmetric n x n T:
/// Householder tridiagonalisation + bisection / inverse iteration + back-transform.
void sym_evd_top(Context& ctx, View t, Index want, double* values, View vectors);
/// The same by two-stage tridiagonalisation (sytrd2.cu: dense -> band 8 on
/// DMMA, bulge chasing as a warp wavefront, back-transformation bt2_k);
/// sym_evd_top routes there when sytrd2_fits(n): opt-in, BLWS_EVD2=1 (n >= 16,
/// on-chip sizes); slower than the one-stage kernel at order 200 (2.0 vs 0.74 ms).
bool sytrd2_fits(Index n);
void sym_evd_top_two_stage(Context& ctx, View t, Index want, double* values, View vectors);
/// Top `want` eigenpairs of the symmetric tridiagonal (d, e): values
/// descending, vectors n x want. Bisection + inverse iteration with cluster
/// reorthogonalisation.
void tridiag_eig_top(Context& ctx, Index n, const double* d, const double* e, Index want, double* values,
                     View vectors);

// ------------------------------------------------------------------ GEMV (K10)
/// y = alpha * op(A) x + beta * y for column-major A (rows x cols).
void gemv(Context& ctx, bool trans, Index rows, Index cols, double alpha, const double* A, Index lda,
          const double* x, double beta, double* y);
/// out = dot(x, y) (device scalar).
void dot(Context& ctx, Index n, const double* x, const double* y, double* out);

// ------------------------------------------------------------------ sparse (K8, K9)
/// Y (rows x b) = S * X where S is CSR (rowptr, colidx, val); X col-major.
/// xt is scratch of cols(S) * b doubles (row-major copy of X). nnz >= 0 with
/// ascending column indices in every row allows the shared-memory tiled kernel
/// (csr_spmm_tiled_k) when it pays; nnz < 0 keeps the L2 gather kernel.
void csr_spmm(Context& ctx, Index rows, const std::int64_t* rowptr, const std::int32_t* colidx,
              const double* val, Index ncols, Index b, const double* X, Index ldx, double* Y, Index ldy,
              double* xt, Index nnz = -1);
/// CSR view of a CSC pattern on the device (csr_build.cu): rowptr (m + 1),
/// colidx and perm (CSR slot -> CSC position) in column order within a row,
/// colof (column of each CSC position); throws on bad row indices / non-finite values.
/// Returns whether the row indices ascend within every column (the CSR columns
/// within a row always do): what the tiled SpMM needs of the CSC arrays.
bool build_csr_device(Context& ctx, Index m, Index n, Index nnz, const std::int64_t* colptr,
                      const std::int32_t* rowidx, const double* val, std::int64_t* rowptr, std::int32_t* colidx,
                      std::int64_t* perm, std::int32_t* colof);
void gather_values(Context& ctx, Index nnz, double* dst, const double* src, const std::int64_t* perm);

// ------------------------------------------------------------------ misc
/// FP64 peak microbenchmark in TFLOP/s (mode 0 DMMA tensor pipe, 1 DFMA).
double fp64_peak_tflops(Context& ctx, int mode);
/// L2 throughput probe (GB/s): mode 0 stream, mode 1 random row gathers of `row` doubles.
double l2_probe_gbps(Context& ctx, int mode, int row);
void reduce_partials(Context& ctx, const double* partials, Index count, double* out);

}  // namespace blws
