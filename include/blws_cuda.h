/*
 * blws_cuda.h — C ABI of the B200-native BLWS partial-SVT library
 * (libblws_cuda.so, built from paper_1012_0365_b200/csrc).
 *
 * The reference (arXiv 1012.0365 BLWS, /root/reference/proj) is a header-only
 * C++20 template library with no FFI; its seam is the C++ API in
 * proj/include/blws. Each entry point below replaces one reference function
 * (cited as file:line) behind plain pointers and sizes. A C++ shim with the
 * reference's own names (blws::blws_svd, blws::SvdBackend, blws::svt,
 * blws::rpca_adm, blws::mc_svt, ...) lives in include/blws/blws.hpp and maps
 * the status codes back to the reference's exceptions.
 *
 * Conventions
 *  - fp64, column-major, leading dimension arguments in elements.
 *  - `where` = BLWS_HOST (pointer is host memory) or BLWS_DEVICE (device
 *    memory on the context's GPU).
 *  - Status codes: 0 ok; 1 invalid argument (std::invalid_argument in the
 *    reference); 2 numerical failure (std::runtime_error); 3 CUDA error;
 *    4 NCCL error. blws_last_error() returns the message of the last failure
 *    on the calling thread.
 *  - One context per solve, single-threaded use (as the reference).
 */
#ifndef BLWS_CUDA_H
#define BLWS_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BLWS_OK 0
#define BLWS_INVALID_ARGUMENT 1
#define BLWS_NUMERICAL_FAILURE 2
#define BLWS_CUDA_ERROR 3
#define BLWS_NCCL_ERROR 4
#define BLWS_IO_ERROR 5

#define BLWS_HOST 0
#define BLWS_DEVICE 1

typedef struct blws_context blws_context;
typedef struct blws_operator blws_operator;
typedef struct blws_warm_start blws_warm_start;
typedef struct blws_rng blws_rng;
typedef struct blws_svd_backend blws_svd_backend;

const char* blws_last_error(void);
int blws_abi_version(void);

/* ---------------------------------------------------------------- context */
int blws_context_create(int device, blws_context** out);
int blws_context_destroy(blws_context* ctx);
int blws_context_synchronize(blws_context* ctx);
/* cudaStream_t the library enqueues on (for CUDA-event timing by callers). */
void* blws_context_stream(blws_context* ctx);
/* kernels launched through this context so far */
int64_t blws_context_launches(const blws_context* ctx);
/* CUDA-event timing of the K1 paired W products (region 0) for roofline
 * evidence; stats = {total_ms, count, flops, algorithmic bytes}. */
int blws_context_set_profiling(blws_context* ctx, int on);
int blws_context_region_stats(blws_context* ctx, int region, double* total_ms, int64_t* count, double* flops,
                              double* bytes);
int blws_context_region_reset(blws_context* ctx);
/* FP64 peak microbenchmark on this GPU, TFLOP/s (mode 0 DMMA, 1 DFMA). */
int blws_fp64_peak(blws_context* ctx, int mode, double* tflops);
/* L2 throughput probe, GB/s of requested bytes (roofline of the gather-form
 * sparse kernels): mode 0 streams an L2-resident buffer; mode 1 gathers random
 * rows of `row` doubles from a 4 MB matrix (K8 / K9's access pattern). */
int blws_l2_probe(blws_context* ctx, int mode, int row, double* gbps);

/* -------------------------------------------------------------------- rng
 * blws::Rng (core/rng.hpp:17-90), bit-exact: std::mt19937_64 + 53-bit
 * uniform + rejection index + Box-Muller with spare. */
int blws_rng_create(uint64_t seed, blws_rng** out);
int blws_rng_destroy(blws_rng* rng);
int blws_rng_split(const blws_rng* rng, uint64_t tag, blws_rng** out);       /* rng.hpp:22-24 */
uint64_t blws_rng_next_u64(blws_rng* rng);                                 /* rng.hpp:26 */
double blws_rng_uniform(blws_rng* rng, double lo, double hi);              /* rng.hpp:29-32 */
/* n successive rng.uniform(lo, hi) draws (instance generation, synth.hpp:88-89). */
int blws_rng_uniform_fill(blws_rng* rng, int64_t n, double lo, double hi, double* out);
uint64_t blws_rng_uniform_index(blws_rng* rng, uint64_t n);                /* rng.hpp:35-42 */
double blws_rng_normal(blws_rng* rng);                                     /* rng.hpp:45-60 */
int blws_rng_gaussian_matrix(blws_rng* rng, int64_t rows, int64_t cols, double* out); /* rng.hpp:63-68 */
/* synth.hpp:23-33 (sample_distinct, Floyd), sorted ascending; returns count */
int64_t blws_sample_distinct(int64_t n, int64_t s, blws_rng* rng, int64_t* out);

/* -------------------------------------------------------------- operators
 * DenseOperator (core/linear_operator.hpp:102-131). BLWS_HOST copies W to
 * the device; BLWS_DEVICE with borrow=1 aliases caller memory (ldw even,
 * 16-byte aligned), borrow=0 copies. */
int blws_dense_operator_create(blws_context* ctx, int64_t m, int64_t n, const double* w, int64_t ldw, int where,
                               int borrow, blws_operator** out);
/* ---- row-sharded multi-GPU path (no reference counterpart: the
   reference is single-process). One process per GPU; each holds a row panel
   of W (rows [row0, row0 + m_local) of m_total) and the matching rows of U,
   with V replicated. blws_svd then allreduces every reduction over panel rows
   (Grams, norms, M = Q^T Z, W^T U) over NCCL; T, its EVD and every host
   decision are computed from identical allreduced values on all ranks. */
/* A fresh NCCL unique id (128 bytes): made on one rank, broadcast to the others. */
int blws_nccl_unique_id(uint8_t* out128);
/* Collective over all ranks: attach an NCCL communicator to the context. */
int blws_context_init_comm(blws_context* ctx, int nranks, int rank, const uint8_t* id128);
/* Host-staged collectives instead of NCCL (several ranks sharing one GPU in
 * tests): every reduction synchronises the context's stream and calls
 * fn(buf, count, op, user) on a host copy (op 0 sum, 1 max); fn returns 0 after
 * leaving the reduced values in buf on every rank. No CUDA-graph capture while
 * set. Not a product path: NCCL (blws_context_init_comm) is. */
typedef int (*blws_host_allreduce_fn)(double* buf, size_t count, int op, void* user);
int blws_context_init_host_comm(blws_context* ctx, int nranks, int rank, blws_host_allreduce_fn fn, void* user);
int blws_context_comm_info(const blws_context* ctx, int* nranks, int* rank);
/* Mark a dense operator holding m_local = rows() rows as rows [row0, row0 +
   m_local) of an m_total x n matrix distributed over the context's ranks. */
int blws_dense_operator_set_row_shard(blws_operator* op, int64_t m_total, int64_t row0);
/* DenseOperator::assign (linear_operator.hpp:113-116): replace W, non-finite check. */
int blws_dense_operator_assign(blws_operator* op, const double* w, int64_t ldw, int where);
/* Asynchronous host assign (B200 extension of DenseOperator::assign): queues the
   upload on the context's copy stream behind the kernels already queued and
   returns at once, so the next W uploads while the current solve runs on another
   operator. The next call using `op` waits for the copy and performs the
   reference's non-finite check then (BLWS_EINVAL from that call). `w` (pinned
   host memory for real overlap) must stay valid and unchanged until then. */
int blws_dense_operator_assign_async(blws_operator* op, const double* w, int64_t ldw);
/* SparseOperator (linear_operator.hpp:136-169) from host CSC (Eigen's default order). */
int blws_sparse_operator_create(blws_context* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* colptr,
                                const int32_t* rowidx, const double* values, blws_operator** out);
/* SparseOperator::assign_values (:149-153), compressed (CSC) order. */
int blws_sparse_operator_assign_values(blws_operator* op, const double* values, int64_t nnz, int where);
int blws_operator_destroy(blws_operator* op);
int64_t blws_operator_rows(const blws_operator* op);
int64_t blws_operator_cols(const blws_operator* op);
/* LinearOperator::application_count (linear_operator.hpp:76) */
int64_t blws_operator_application_count(const blws_operator* op);
/* LinearOperator::apply_pair_block (:57-61): top = W*right (m x b), bot = W^T*left (n x b); host buffers. */
int blws_operator_apply_pair_block(blws_operator* op, int64_t b, const double* left, const double* right,
                                   double* top, double* bot);
/* LinearOperator::apply_pair (:51-54): top = W*right (m), bot = W^T*left (n); one
   pass over a dense W (K10); counts 1. Host buffers. */
int blws_operator_apply_pair(blws_operator* op, const double* left, const double* right, double* top,
                             double* bot);

/* ------------------------------------------------------------- warm start
 * WarmStart (block_lanczos.hpp:45-52): U m x r, V n x r, sigma r. */
int blws_warm_start_create(blws_context* ctx, int64_t m, int64_t n, int64_t r, const double* u, int64_t ldu,
                           const double* v, int64_t ldv, const double* sigma, int where, blws_warm_start** out);
int blws_warm_start_copy(const blws_warm_start* src, blws_warm_start** out);
int64_t blws_warm_start_rank(const blws_warm_start* w);
/* copy out (any pointer may be NULL); sigma always host */
int blws_warm_start_get(const blws_warm_start* w, double* u, int64_t ldu, double* v, int64_t ldv, double* sigma,
                        int where);
int blws_warm_start_destroy(blws_warm_start* w);

/* --------------------------------------------------------- block lanczos */
/* Number of blws_svd calls (process-wide) whose deferred single-round-trip
   path was redone on the exact path because a host test would have branched
   away from the common case (breakdown, rank loss, ill-conditioned Gram,
   keep < min(r, d)). BLWS_EXACT=1 in the environment forces the exact path. */
int64_t blws_svd_deferred_fallbacks(void);
/* Number of blws_svd calls (process-wide) served by replaying a captured CUDA
   graph of the deferred launch sequence (cached per operator data and
   (rank, k, r); captured on the second call with the same key, replayed after).
   BLWS_GRAPHS=0 disables the graphs; they are also skipped while region
   profiling is on. */
int64_t blws_svd_graph_launches(void);
/* blws_svd (block_lanczos.hpp:204-261). flags: bit0 padded, bit1 k_raised,
 * bit2 terminated_early. *out receives a new warm start of rank r. */
int blws_svd(blws_operator* w, const blws_warm_start* warm, int64_t k, int64_t r, blws_rng* rng,
             blws_warm_start** out, int* flags);
/* adapt_subspace (block_lanczos.hpp:157-187); warm may be NULL. */
int blws_adapt_subspace(blws_context* ctx, const blws_warm_start* warm, int64_t r_new, int64_t m, int64_t n,
                        blws_rng* rng, blws_warm_start** out);
/* block_lanczos_procedure (block_lanczos.hpp:70-126) on the augmented view of
 * W from x1 ((m+n) x b host); q ((m+n) x k*b host), t (k*b x k*b host). */
int blws_block_lanczos_procedure(blws_operator* w, int64_t b, const double* x1, int64_t k, double* q, double* t,
                                 int64_t* built, int* terminated_early);

/* ---------------------------------------------------------------- lanczos */
/* lanczos_partial_svd (lanczos.hpp:289-329). stats: steps, restarts, converged, all_converged. */
int blws_lanczos_partial_svd(blws_operator* w, int64_t r, double tol, int64_t max_k, uint64_t seed,
                             blws_warm_start** out, int64_t stats[4]);
/* spectral_norm (lanczos.hpp:332-340) */
int blws_spectral_norm(blws_operator* w, double tol, uint64_t seed, double* out);

/* ------------------------------------------------- dense kernels (device) */
/* thin_qr (core/qr.hpp:24-47) on the device; host buffers. */
int blws_thin_qr(blws_context* ctx, int64_t rows, int64_t cols, const double* m, double* q, double* r,
                 int64_t* rank);
/* full_svd_small (small_dense.hpp:72-87): SVD of a host m x n W (m + n <= 4096)
   via the top min(m, n) eigenpairs of the symmetric embedding; sigma
   descending, u (m x p), v (n x p) column-major, p = min(m, n). */
int blws_full_svd_small(blws_context* ctx, int64_t m, int64_t n, const double* w, double* sigma, double* u,
                        double* v);
/* sym_evd_small (core/small_dense.hpp:24-43): values descending. host buffers */
int blws_sym_evd(blws_context* ctx, int64_t n, const double* t, double* values, double* vectors);
/* top `want` pairs of sym_evd_tridiagonal (small_dense.hpp:46-62); vectors n x want. host buffers */
int blws_sym_evd_tridiagonal_top(blws_context* ctx, int64_t n, const double* d, const double* e, int64_t want,
                                 double* values, double* vectors);
/* C = alpha op(A) op(B) + beta C on device pointers (the K1/K2/K5 GEMM) */
int blws_dgemm(blws_context* ctx, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* a,
               int64_t lda, const double* b, int64_t ldb, double beta, double* c, int64_t ldc);

/* development: average device microseconds of one hot-path piece on a seeded
 * input (0 chol_inv n, 1 sym_evd_top n, 2 thin_qr n x b, 3 gemm NN, 4 gemm TN) */
int blws_microbench(blws_context* ctx, int which, int64_t n, int64_t b, int reps, double* us);

/* ------------------------------------------------------------ backend/svt */
#define BLWS_BACKEND_EXACT_FULL 0 /* svt.hpp:108-116: dense full SVD (m + n <= 4096) */
#define BLWS_BACKEND_LANCZOS 1
#define BLWS_BACKEND_BLWS 2
/* SvdBackend<double>::lanczos / ::blws (svt.hpp:84-98) with Options (:88-94). */
int blws_svd_backend_create(blws_context* ctx, int kind, int64_t block_steps, double ritz_tol, int64_t max_k,
                            int64_t seed_margin, uint64_t seed, blws_svd_backend** out);
int blws_svd_backend_destroy(blws_svd_backend* b);
/* warm_state() (svt.hpp:102): copy of the held warm start or *out = NULL */
int blws_svd_backend_warm_state(const blws_svd_backend* b, blws_warm_start** out);
/* replace the held warm start (harness: reset to a fixed warm start) */
int blws_svd_backend_set_warm_state(blws_svd_backend* b, const blws_warm_start* w);

/* RankPredictor (svt.hpp:48-53); history is appended to `history`
 * (capacity history_cap, current length *history_len). */
typedef struct {
    int64_t r;
    int64_t increment;
    int64_t max_rank;
} blws_rank_predictor;

/* svt (svt.hpp:216-254): *out gets the retained triplets with shrunk sigma. */
int blws_svt(blws_operator* w, double eps, blws_svd_backend* backend, blws_rank_predictor* pred,
             int64_t* history, int64_t history_cap, int64_t* history_len, blws_warm_start** out,
             int64_t* achieved_rank, int* all_above_threshold);

/* ---------------------------------------------------------------- solvers */
typedef struct {
    double tol_outer;      /* 1e-7 */
    int64_t max_iter;      /* 1000 */
    double rho;            /* 1.5 (solvers.hpp:60) */
    double mu_max_factor;  /* 1e7 */
    int64_t initial_rank;  /* 10 */
    int64_t rank_increment;/* 5 */
} blws_rpca_options;

typedef struct {
    double tol_outer;      /* 1e-4 */
    int64_t max_iter;      /* 500 */
    int64_t initial_rank;  /* 10 */
    int64_t rank_increment;/* 5 */
} blws_mc_options;

typedef struct {
    int64_t iterations;
    double wall_time_s;
    int64_t matvec_count;
    int64_t matvec_init;
    double rel_err;
    int64_t rank_hat;
    int64_t e_l0;
    int64_t e_nnz;
    int32_t converged;
    int32_t pad_;
} blws_solver_stats;

/* rpca_adm (solvers.hpp:72-157). d / truth / a_out / e_out share `where` and
 * ldd; truth, a_out, e_out may be NULL. Histories (predicted ranks,
 * per-iteration counter deltas, residuals) are written up to hist_cap. */
int blws_rpca_adm(blws_context* ctx, int64_t m, const double* d, int64_t ldd, int where, double lambda,
                  blws_svd_backend* backend, const blws_rpca_options* opts, const double* truth, double* a_out,
                  double* e_out, blws_solver_stats* stats, int64_t* predicted_ranks, int64_t* matvec_history,
                  double* residual_history, int64_t hist_cap);

/* mc_svt (solvers.hpp:202-270), observation as host CSC. Outputs (host):
 * u m x cap, sigma cap, v n x cap; *rank receives the retained count. */
int blws_mc_svt(blws_context* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* colptr, const int32_t* rowidx,
                const double* values, double tau, double delta, blws_svd_backend* backend, const blws_mc_options* opts,
                const double* truth_ml, const double* truth_mr, int64_t r_true, double* u, double* sigma, double* v,
                int64_t cap, int64_t* rank, blws_solver_stats* stats, int64_t* predicted_ranks,
                int64_t* matvec_history, double* residual_history, int64_t hist_cap);

/* Row-sharded solvers (one process per GPU, the context's NCCL
 * communicator from blws_context_init_comm; a context without one runs the same
 * code path on one rank). This rank holds rows [row0, row0 + rows) of the
 * m x m RPCA problem (d / truth / a_out / e_out are rows x m panels, ldd >=
 * rows) or of the m x n MC observation (local CSC over n columns, row indices
 * in [0, rows), nnz local; truth_ml its rows x r_true rows of ML; u comes back
 * as this rank's rows x cap). Stats and histories are identical on every rank.
 * Replaces solvers.hpp:72-74 / :202-204 for a row-distributed problem. */
int blws_rpca_adm_sharded(blws_context* ctx, int64_t m, int64_t rows, int64_t row0, const double* d, int64_t ldd,
                          int where, double lambda, blws_svd_backend* backend, const blws_rpca_options* opts,
                          const double* truth, double* a_out, double* e_out, blws_solver_stats* stats,
                          int64_t* predicted_ranks, int64_t* matvec_history, double* residual_history,
                          int64_t hist_cap);
int blws_mc_svt_sharded(blws_context* ctx, int64_t m, int64_t rows, int64_t row0, int64_t n, int64_t nnz,
                        const int64_t* colptr, const int32_t* rowidx, const double* values, double tau, double delta,
                        blws_svd_backend* backend, const blws_mc_options* opts, const double* truth_ml,
                        const double* truth_mr, int64_t r_true, double* u, double* sigma, double* v, int64_t cap,
                        int64_t* rank, blws_solver_stats* stats, int64_t* predicted_ranks, int64_t* matvec_history,
                        double* residual_history, int64_t hist_cap);

/* ---- Matrix Market I/O (core/matrix_market.hpp:63-168): host files; the
   reference's std::runtime_error becomes BLWS_IO_ERROR. Dense = "array"
   column-major (lda), sparse = "coordinate" read into / written from CSC. */
int blws_mm_write_dense(const char* path, int64_t rows, int64_t cols, const double* a, int64_t lda);
int blws_mm_write_sparse(const char* path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* colptr,
                         const int32_t* rowidx, const double* values);
/* out == NULL: only rows / cols are returned. */
int blws_mm_read_dense(const char* path, int64_t* rows, int64_t* cols, double* out, int64_t ldo);
/* colptr == NULL: only rows / cols / nnz are returned (then call again with
   colptr (cols + 1), rowidx (nnz), values (nnz)). */
int blws_mm_read_sparse(const char* path, int64_t* rows, int64_t* cols, int64_t* nnz, int64_t* colptr,
                        int32_t* rowidx, double* values);

#ifdef __cplusplus
}
#endif

#endif /* BLWS_CUDA_H */
