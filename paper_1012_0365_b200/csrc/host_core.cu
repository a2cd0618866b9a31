// Operators, CholQR thin_qr, block Lanczos / BLWS and the cold Lanczos reseed.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <stdexcept>

#include "host.hpp"
#include "ops.cuh"

namespace blws {

// kSmallDenseLimit (small_dense.hpp:13): the reference throws
// std::invalid_argument for a symmetric / tridiagonal EVD above order 4096. The
// device path has no such limit (the C5 reseeds exceed it); BLWS_STRICT_SMALL_DENSE=1
// restores the reference's error.
static void small_dense_guard(Index n, const char* what) {
    static const bool strict = [] {
        const char* e = std::getenv("BLWS_STRICT_SMALL_DENSE");
        return e && e[0] == '1';
    }();
    if (strict && n > 4096) throw std::invalid_argument(what);
}

// =================================================================== Rng
std::uint64_t Rng::uniform_index(std::uint64_t n) {
    const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    std::uint64_t x;
    do {
        x = engine_();
    } while (x >= limit);
    return x % n;
}

double Rng::normal() {
    if (have_spare_) {
        have_spare_ = false;
        return spare_;
    }
    double u1, u2;
    do {
        u1 = uniform();
    } while (u1 <= 0.0);
    u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 6.283185307179586476925287 * u2;
    spare_ = r * std::sin(theta);
    have_spare_ = true;
    return r * std::cos(theta);
}

void Rng::gaussian_matrix(Index rows, Index cols, double* out, Index ld) {
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i < rows; ++i) out[i + j * ld] = normal();
}

std::vector<double> Rng::gaussian_vector(Index n) {
    std::vector<double> v(static_cast<size_t>(n));
    for (auto& x : v) x = normal();
    return v;
}

std::vector<double> Rng::unit_vector(Index n) {
    auto v = gaussian_vector(n);
    double s = 0;
    for (double x : v) s += x * x;
    const double nv = std::sqrt(s);
    for (auto& x : v) x /= nv;
    return v;
}

// ============================================================ small kernels
namespace {

constexpr int kT = 256;
inline unsigned gridn(long total, long cap = 4096) {
    return static_cast<unsigned>(std::max<long>(1, std::min<long>(cap, (total + kT - 1) / kT)));
}

__global__ void nonfinite_count_k(const double* x, long rows, long cols, long ld, int* flag) {
    const long total = rows * cols;
    int bad = 0;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x)
        if (!isfinite(x[idx % rows + (idx / rows) * ld])) bad = 1;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// Paired SpMV of the sparse Lanczos apply (one launch for W x over the CSR
// rows and W^T y over the CSC columns; warps [0, rows_a) take the first,
// the rest the second): warp per row, y[i] = sum_p val[p] x[col[p]]. Each
// lane keeps 4 nonzeros in flight (index loads, then the gathers, then the
// FMAs) so a row's ~1000 nonzeros are not one dependent load chain.
__device__ __forceinline__ double spmv_row(long b, long e, const std::int32_t* __restrict__ idx,
                                           const double* __restrict__ val, const double* __restrict__ x, int lane) {
    double s0 = 0.0, s1 = 0.0;
    long p = b + lane;
    // 8 gathers in flight per lane; the accumulation order is the 4-wide loop's
    // (two of its iterations per pass), so the sums are bitwise unchanged
    for (; p + 224 < e; p += 256) {
        int c[8];
        double v[8], xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            c[u] = idx[p + 32 * u];
            v[u] = val[p + 32 * u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = x[c[u]];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (u & 1)
                s1 = fma(v[u], xv[u], s1);
            else
                s0 = fma(v[u], xv[u], s0);
        }
    }
    for (; p + 96 < e; p += 128) {
        const int c0 = idx[p], c1 = idx[p + 32], c2 = idx[p + 64], c3 = idx[p + 96];
        const double v0 = val[p], v1 = val[p + 32], v2 = val[p + 64], v3 = val[p + 96];
        const double x0 = x[c0], x1 = x[c1], x2 = x[c2], x3 = x[c3];
        s0 = fma(v0, x0, s0);
        s1 = fma(v1, x1, s1);
        s0 = fma(v2, x2, s0);
        s1 = fma(v3, x3, s1);
    }
    for (; p < e; p += 32) s0 = fma(val[p], x[idx[p]], s0);
    double s = s0 + s1;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

__global__ void csr_spmv_pair_k(long rows_a, const std::int64_t* __restrict__ ptr_a,
                                const std::int32_t* __restrict__ idx_a, const double* __restrict__ val_a,
                                const double* __restrict__ x_a, double* y_a, long rows_b,
                                const std::int64_t* __restrict__ ptr_b, const std::int32_t* __restrict__ idx_b,
                                const double* __restrict__ val_b, const double* __restrict__ x_b, double* y_b) {
    const long warps = (static_cast<long>(gridDim.x) * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (long w = (blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x) >> 5; w < rows_a + rows_b;
         w += warps) {
        if (w < rows_a) {
            const double s = spmv_row(ptr_a[w], ptr_a[w + 1], idx_a, val_a, x_a, lane);
            if (lane == 0) y_a[w] = s;
        } else {
            const long i = w - rows_a;
            const double s = spmv_row(ptr_b[i], ptr_b[i + 1], idx_b, val_b, x_b, lane);
            if (lane == 0) y_b[i] = s;
        }
    }
}

// r -= alpha[l] q_l + coup[l] q_{l-1}
__global__ void lanczos_three_term_k(double* r, const double* q, long ld, long l, const double* alpha,
                                     const double* coup, long n) {
    const double a = alpha[l];
    const double b = l > 0 ? coup[l] : 0.0;
    const double* ql = q + l * ld;
    const double* qp = l > 0 ? q + (l - 1) * ld : q;
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long>(gridDim.x) * blockDim.x) {
        double v = r[i] - a * ql[i];
        if (l > 0) v -= b * qp[i];
        r[i] = v;
    }
}

// beta = ||r|| (from sumsq), breakdown test, next_dir = r / beta; state[0] =
// first broken step (or -1), state[1] = tau (set at step 0).
__global__ void lanczos_finalize_k(const double* r, double* next, long n, long l, long dim, const double* rsq,
                                   const double* alpha, double* lastbeta, double* coup, long cap, double* state) {
    const double beta = sqrt(rsq[0]);
    __shared__ int broken;
    if (threadIdx.x == 0) {
        if (l == 0) state[1] = 1e-12 * fabs(alpha[0]);
        const bool already = state[0] >= 0.0;
        const bool now = beta <= state[1] || (l + 1) >= dim;
        if (!already && now) state[0] = static_cast<double>(l);
        broken = already || now;
        lastbeta[l] = beta;
        if (!broken && l + 1 < cap) coup[l + 1] = beta;
    }
    __syncthreads();
    const double inv = broken ? 0.0 : 1.0 / beta;
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long>(gridDim.x) * blockDim.x)
        next[i] = broken ? 0.0 : r[i] * inv;
}

__global__ void scale_by_inv_sqrt_k(double* x, long n, const double* ss) {
    const double inv = 1.0 / sqrt(ss[0]);
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long>(gridDim.x) * blockDim.x)
        x[i] *= inv;
}

__global__ void shift_for_cholqr3_k(const double* ss, double factor, double* out) { out[0] = factor * ss[0]; }

}  // namespace

// ======================================================== upload / download
void upload(Context& ctx, View dst, const double* host, Index ldh) {
    if (dst.rows * dst.cols == 0) return;
    BLWS_CUDA(cudaMemcpy2DAsync(dst.p, sizeof(double) * dst.ld, host, sizeof(double) * ldh,
                                sizeof(double) * dst.rows, dst.cols, cudaMemcpyHostToDevice, ctx.stream()));
    ctx.sync();
}

void download(Context& ctx, View src, double* host, Index ldh) {
    if (src.rows * src.cols == 0) return;
    BLWS_CUDA(cudaMemcpy2DAsync(host, sizeof(double) * ldh, src.p, sizeof(double) * src.ld,
                                sizeof(double) * src.rows, src.cols, cudaMemcpyDeviceToHost, ctx.stream()));
    ctx.sync();
}

static void launch_nonfinite(Context& ctx, View v, int* flag) {
    if (v.rows * v.cols == 0) return;
    nonfinite_count_k<<<gridn(v.rows * v.cols), kT, 0, ctx.stream()>>>(v.p, v.rows, v.cols, v.ld, flag);
    ctx.note_launch();
    ctx.check_launch("nonfinite");
}

void nonfinite_count(Context& ctx, View v, int* flag) {
    zero(ctx, flag, sizeof(int));
    launch_nonfinite(ctx, v, flag);
}

static void check_finite_view(Context& ctx, View v, const char* what) {
    DBuf<int> flag(ctx, 1);
    zero(ctx, flag.get(), sizeof(int));
    if (v.rows * v.cols > 0) {
        nonfinite_count_k<<<gridn(v.rows * v.cols), kT, 0, ctx.stream()>>>(v.p, v.rows, v.cols, v.ld, flag.get());
        ctx.note_launch();
        ctx.check_launch("nonfinite");
    }
    int h = 0;
    BLWS_CUDA(cudaMemcpyAsync(&h, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx.stream()));
    ctx.sync();
    if (h) throw std::invalid_argument(what);
}

__global__ void flag_to_double_k(const int* f, double* d) { *d = *f != 0 ? 1.0 : 0.0; }

// the async-upload non-finite verdict of this rank -> slot `dst` as 0/1, summed
// over the ranks, so every rank takes the same branch
void share_flag(Context& ctx, const int* flag, double* dst) {
    if (!ctx.has_comm()) return;
    flag_to_double_k<<<1, 1, 0, ctx.stream()>>>(flag, dst);
    ctx.note_launch();
    ctx.allreduce_sum(dst, 1);
}

// region timing for whole calls (regions 3: Lanczos reseed, 4: Ritz checkpoint,
// 5: blws_svd) -- host-side event records, also around graph launches


// ======================================================== row sharding
void LinearOperator::set_row_shard(Index m_total, Index row0) {
    if (m_total < rows() || row0 < 0 || row0 + rows() > m_total)
        throw std::invalid_argument("set_row_shard: local rows outside [0, m_total)");
    shard_ = RowShard{m_total, row0};
}

RowSplit LinearOperator::panel_split() const {
    // the top of a stacked panel (rows [0, mp), padding row included: it is zero);
    // with column sharding the whole panel
    if (col_sharded()) return RowSplit{Stack{rows(), panel_n()}.ld()};
    return RowSplit{row_sharded() && ctx_.has_comm() ? round_up(rows(), 2) : 0};
}

bool LinearOperator::col_sharded() const {
    // BLWS_NSHARD=0: bottom rows replicated; =force: split even on a one-rank
    // communicator (tests of the NCCL all-gather / reduce-scatter, graph capture)
    static const int mode = [] {
        const char* e = std::getenv("BLWS_NSHARD");
        if (!e) return 1;
        const std::string v(e);
        return v == "0" ? 0 : (v == "force" ? 2 : 1);
    }();
    if (mode == 0 || !row_sharded() || !ctx_.has_comm()) return false;
    return ctx_.nranks() > 1 || mode == 2;
}

Index LinearOperator::col_chunk() const { return ceil_div(cols(), std::max(1, ctx_.nranks())); }

// ---- column-sharded panels: gather / scatter of the bottom rows
// dst (npad x b, col-major, ld npad) = the bottom rows of every rank, in rank
// order (chunk x b each, `src` with its own ld)
void gather_cols(LinearOperator& w, View src, double* dst) {
    Context& ctx = w.ctx();
    const Index chunk = w.col_chunk(), b = src.cols, N = ctx.nranks();
    DBuf<double> send(ctx, static_cast<size_t>(chunk * b)), recv(ctx, static_cast<size_t>(chunk * b * N));
    pack_rows(ctx, src, send.get());  // row-major chunk x b: one contiguous block per rank
    ctx.allgather(send.get(), recv.get(), static_cast<size_t>(chunk * b));
    unpack_rows(ctx, recv.get(), View{dst, chunk * N, b, chunk * N});
}

// dst (chunk x b, this rank's bottom rows) = sum over the ranks of the rows
// [col0, col0 + chunk) of `part` (npad x b, col-major, ld npad; rows past n zero)
void scatter_cols(LinearOperator& w, View part, View dst) {
    Context& ctx = w.ctx();
    const Index chunk = w.col_chunk(), b = part.cols, N = ctx.nranks();
    DBuf<double> send(ctx, static_cast<size_t>(chunk * b * N)), recv(ctx, static_cast<size_t>(chunk * b));
    pack_rows(ctx, part, send.get());
    ctx.reduce_scatter_sum(send.get(), recv.get(), static_cast<size_t>(chunk * b));
    unpack_rows(ctx, recv.get(), dst);
}

// ======================================================== DenseOperator
DenseOperator::DenseOperator(Context& ctx, Index m, Index n)
    : LinearOperator(ctx), m_(m), n_(n), ld_(std::max<Index>(2, round_up(m, 2))) {
    own_ = DBuf<double>(ctx, static_cast<size_t>(ld_ * std::max<Index>(n, 1)));
    zero(ctx, own_.get(), sizeof(double) * own_.size());
    p_ = own_.get();
}

DenseOperator::DenseOperator(Context& ctx, Index m, Index n, double* dev, Index ld)
    : LinearOperator(ctx), m_(m), n_(n), ld_(ld), p_(dev) {}

DenseOperator::~DenseOperator() {
    // the owned buffer is freed on the compute stream: order it after a pending upload
    if (pending_) cudaStreamWaitEvent(ctx_.stream(), ready_, 0);
    if (consumed_) cudaEventDestroy(consumed_);
    if (ready_) cudaEventDestroy(ready_);
}

void DenseOperator::check_finite() {
    check_finite_view(ctx_, View{p_, m_, n_, ld_}, "DenseOperator: non-finite entries");
}

void DenseOperator::ensure_ready() const {
    if (poisoned_) throw std::invalid_argument("DenseOperator: non-finite entries");
    if (!pending_) return;
    pending_ = false;
    BLWS_CUDA(cudaStreamWaitEvent(ctx_.stream(), ready_, 0));
    poisoned_ = true;  // until the check passes
    check_finite_view(ctx_, View{p_, m_, n_, ld_}, "DenseOperator: non-finite entries");
    poisoned_ = false;
}

void DenseOperator::assign_host(const double* w_host, Index ldw) {
    poisoned_ = false;
    upload(ctx_, w(), w_host, ldw);
    poisoned_ = true;  // until the check passes
    check_finite();
    poisoned_ = false;
}

void DenseOperator::defer_pending_check(int* flag) {
    if (poisoned_) throw std::invalid_argument("DenseOperator: non-finite entries");
    if (!pending_) return;
    pending_ = false;
    BLWS_CUDA(cudaStreamWaitEvent(ctx_.stream(), ready_, 0));
    launch_nonfinite(ctx_, View{p_, m_, n_, ld_}, flag);
}

void DenseOperator::assign_host_async(const double* w_host, Index ldw) {
    if (ldw < m_) throw std::invalid_argument("assign: ldw < rows");
    if (!poisoned_) ensure_ready();  // a previous pending upload is checked and ordered first
    else if (pending_) BLWS_CUDA(cudaStreamWaitEvent(ctx_.stream(), ready_, 0));
    poisoned_ = false;
    if (!consumed_) {
        BLWS_CUDA(cudaEventCreateWithFlags(&consumed_, cudaEventDisableTiming));
        BLWS_CUDA(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming));
    }
    cudaStream_t cs = ctx_.copy_stream();
    // everything queued so far on the compute stream may still read W
    BLWS_CUDA(cudaEventRecord(consumed_, ctx_.stream()));
    BLWS_CUDA(cudaStreamWaitEvent(cs, consumed_, 0));
    BLWS_CUDA(cudaMemcpy2DAsync(p_, sizeof(double) * ld_, w_host, sizeof(double) * ldw, sizeof(double) * m_, n_,
                                cudaMemcpyHostToDevice, cs));
    BLWS_CUDA(cudaEventRecord(ready_, cs));
    pending_ = true;
}

void DenseOperator::assign_device(const double* w_dev, Index ldw) {
    poisoned_ = false;
    if (w_dev != p_) copy(ctx_, w(), View{const_cast<double*>(w_dev), m_, n_, ldw});
    poisoned_ = true;  // until the check passes
    check_finite();
    poisoned_ = false;
}

void DenseOperator::pair_block_impl(View left, View right, View top, View bot) {
    ensure_ready();
    const Index b = right.cols;
    // K1: region 0 times the paired product (both GEMMs incl. split-K reduce)
    ctx_.region_begin(0);
    if (col_sharded()) {
        // X_bot is split over the ranks: all-gather it for W X_bot; W^T X_top
        // over the local rows is reduce-scattered into this rank's bottom rows
        const Index npad = col_chunk() * ctx_.nranks();
        DBuf<double> xfull(ctx_, static_cast<size_t>(npad * b)), part(ctx_, static_cast<size_t>(npad * b));
        if (npad > n_) zero(ctx_, part.get(), sizeof(double) * static_cast<size_t>(npad * b));  // padding rows
        // collectives on the main stream only, outside the fork (same order on
        // every rank; a gather issued while the W^T X_top GEMM ran on the
        // auxiliary stream raced at large panels): gather, then the two GEMMs
        // side by side, then the scatter after the join
        gather_cols(*this, right, xfull.get());
        {
            AuxScope aux(ctx_);
            gemm(ctx_, true, false, n_, b, m_, 1.0, p_, ld_, left.p, left.ld, 0.0, part.get(), npad);
            aux.main();
            gemm(ctx_, false, false, m_, b, n_, 1.0, p_, ld_, xfull.get(), npad, 0.0, top.p, top.ld);
        }
        scatter_cols(*this, View{part.get(), npad, b, npad}, bot);
    } else if (row_sharded() && ctx_.has_comm()) {
        // W^T U over the local rows, summed over the ranks (contiguous n x b
        // buffer for the allreduce), while W V runs on the local rows only
        DBuf<double> part(ctx_, static_cast<size_t>(n_ * b));
        AuxScope aux(ctx_);
        gemm(ctx_, true, false, n_, b, m_, 1.0, p_, ld_, left.p, left.ld, 0.0, part.get(), n_);
        ctx_.allreduce_sum(part.get(), static_cast<size_t>(n_ * b));
        copy(ctx_, bot, View{part.get(), n_, b, n_});
        aux.main();
        gemm(ctx_, false, false, m_, b, n_, 1.0, p_, ld_, right.p, right.ld, 0.0, top.p, top.ld);
    } else {
        AuxScope aux(ctx_);  // W^T U on the auxiliary stream, overlapping W V
        gemm(ctx_, true, false, n_, b, m_, 1.0, p_, ld_, left.p, left.ld, 0.0, bot.p, bot.ld);
        aux.main();
        gemm(ctx_, false, false, m_, b, n_, 1.0, p_, ld_, right.p, right.ld, 0.0, top.p, top.ld);
    }
    ctx_.region_end(0, 4.0 * static_cast<double>(m_) * n_ * b, 16.0 * static_cast<double>(m_) * n_);
}

void DenseOperator::pair_impl(const double* left, const double* right, double* top, double* bot) {
    ensure_ready();
    if (col_sharded()) {
        // right / bot are this rank's chunk of the n-length halves
        const Index chunk = col_chunk(), npad = chunk * ctx_.nranks();
        DBuf<double> xfull(ctx_, static_cast<size_t>(npad)), part(ctx_, static_cast<size_t>(npad));
        if (npad > n_) zero(ctx_, part.get() + n_, sizeof(double) * static_cast<size_t>(npad - n_));
        ctx_.allgather(right, xfull.get(), static_cast<size_t>(chunk));
        pair_gemv(ctx_, m_, n_, p_, ld_, xfull.get(), left, top, part.get());  // one read of W for both products
        ctx_.reduce_scatter_sum(part.get(), bot, static_cast<size_t>(chunk));
        return;
    }
    pair_gemv(ctx_, m_, n_, p_, ld_, right, left, top, bot);  // one read of W for both products
    if (row_sharded() && ctx_.has_comm()) ctx_.allreduce_sum(bot, static_cast<size_t>(n_));  // W^T left over the ranks
}

// ======================================================== SparseOperator
SparseOperator::SparseOperator(Context& ctx, Index m, Index n, Index nnz, const std::int64_t* colptr,
                               const std::int32_t* rowidx, const double* values)
    : LinearOperator(ctx), m_(m), n_(n), nnz_(nnz) {
    // The CSC arrays are uploaded as given; the CSR view and the CSC -> CSR
    // position permutation are built on the device: a stable radix sort of the
    // positions by row (equal rows keep CSC = column order, the order of the
    // reference-order host transpose), a row histogram and its exclusive scan.
    // (Host-side, the random-scatter transpose of 10^7 entries took ~0.2 s of
    // the C4 solve.)
    const size_t nz = static_cast<size_t>(std::max<Index>(nnz, 1));
    colptr_ = DBuf<std::int64_t>(ctx, static_cast<size_t>(n + 1));
    rowidx_ = DBuf<std::int32_t>(ctx, nz);
    val_csc_ = DBuf<double>(ctx, nz);
    val_csr_ = DBuf<double>(ctx, nz);
    rowptr_ = DBuf<std::int64_t>(ctx, static_cast<size_t>(m + 1));
    perm_ = DBuf<std::int64_t>(ctx, nz);
    colidx_ = DBuf<std::int32_t>(ctx, nz);
    colof_ = DBuf<std::int32_t>(ctx, nz);
    BLWS_CUDA(cudaMemcpyAsync(colptr_.get(), colptr, sizeof(std::int64_t) * (n + 1), cudaMemcpyHostToDevice,
                              ctx.stream()));
    if (nnz > 0) {
        BLWS_CUDA(cudaMemcpyAsync(rowidx_.get(), rowidx, sizeof(std::int32_t) * nnz, cudaMemcpyHostToDevice,
                                  ctx.stream()));
        BLWS_CUDA(cudaMemcpyAsync(val_csc_.get(), values, sizeof(double) * nnz, cudaMemcpyHostToDevice,
                                  ctx.stream()));
    }
    csc_rows_ascend_ = build_csr_device(ctx, m, n, nnz, colptr_.get(), rowidx_.get(), val_csc_.get(), rowptr_.get(),
                                        colidx_.get(), perm_.get(), colof_.get());
    gather_values(ctx, nnz_, val_csr_.get(), val_csc_.get(), perm_.get());
    ctx.sync();
}

void SparseOperator::assign_values_host(const double* vals) {
    BLWS_CUDA(cudaMemcpyAsync(val_csc_.get(), vals, sizeof(double) * nnz_, cudaMemcpyHostToDevice, ctx_.stream()));
    gather_values(ctx_, nnz_, val_csr_.get(), val_csc_.get(), perm_.get());
    ctx_.sync();
}

void SparseOperator::assign_values_device(const double* vals) {
    if (vals != val_csc_.get())
        BLWS_CUDA(cudaMemcpyAsync(val_csc_.get(), vals, sizeof(double) * nnz_, cudaMemcpyDeviceToDevice,
                                  ctx_.stream()));
    gather_values(ctx_, nnz_, val_csr_.get(), val_csc_.get(), perm_.get());
}

void SparseOperator::pair_block_impl(View left, View right, View top, View bot) {
    const Index b = right.cols;
    // Row-major staging of X for the two SpMMs, allocated per call from the
    // stream-ordered pool: under CUDA-graph capture they become the graph's own
    // memory nodes, so a replayed graph never writes into a buffer a later call
    // (with another block width) reallocated. Declared before the AuxScope so
    // they are freed on the main stream after the join.
    const size_t need = static_cast<size_t>(std::max(m_, n_) * b);
    DBuf<double> scratch(ctx_, need), scratch2(ctx_, need);
    if (col_sharded()) {
        // as DenseOperator: all-gather X_bot, reduce-scatter the W^T X_top partial
        const Index npad = col_chunk() * ctx_.nranks();
        DBuf<double> xfull(ctx_, static_cast<size_t>(npad * b)), part(ctx_, static_cast<size_t>(npad * b));
        if (npad > n_) zero(ctx_, part.get(), sizeof(double) * static_cast<size_t>(npad * b));
        gather_cols(*this, right, xfull.get());  // collectives outside the fork (see DenseOperator)
        {
            AuxScope aux(ctx_);
            csr_spmm(ctx_, n_, colptr_.get(), rowidx_.get(), val_csc_.get(), m_, b, left.p, left.ld, part.get(), npad,
                     scratch2.get(), csc_rows_ascend_ ? nnz_ : -1);
            aux.main();
            csr_spmm(ctx_, m_, rowptr_.get(), colidx_.get(), val_csr_.get(), n_, b, xfull.get(), npad, top.p, top.ld,
                     scratch.get(), nnz_);
        }
        scatter_cols(*this, View{part.get(), npad, b, npad}, bot);
        return;
    }
    const bool reduce = row_sharded() && ctx_.has_comm();
    DBuf<double> part;  // row shard: W^T x over the local rows, summed over the ranks
    if (reduce && bot.ld != n_) part = DBuf<double>(ctx_, static_cast<size_t>(n_ * b));
    AuxScope aux(ctx_);  // W^T x on the auxiliary stream, overlapping W x
    if (reduce && bot.ld != n_) {
        csr_spmm(ctx_, n_, colptr_.get(), rowidx_.get(), val_csc_.get(), m_, b, left.p, left.ld, part.get(), n_,
                 scratch2.get(), csc_rows_ascend_ ? nnz_ : -1);
        ctx_.allreduce_sum(part.get(), static_cast<size_t>(n_ * b));
        copy(ctx_, bot, View{part.get(), n_, b, n_});
    } else {
        csr_spmm(ctx_, n_, colptr_.get(), rowidx_.get(), val_csc_.get(), m_, b, left.p, left.ld, bot.p, bot.ld,
                 scratch2.get(), csc_rows_ascend_ ? nnz_ : -1);
        if (reduce) ctx_.allreduce_sum(bot.p, static_cast<size_t>(n_ * b));
    }
    aux.main();
    csr_spmm(ctx_, m_, rowptr_.get(), colidx_.get(), val_csr_.get(), n_, b, right.p, right.ld, top.p, top.ld,
             scratch.get(), nnz_);
}

void SparseOperator::pair_impl(const double* left, const double* right, double* top, double* bot) {
    if (col_sharded()) {
        const Index chunk = col_chunk(), npad = chunk * ctx_.nranks();
        DBuf<double> xfull(ctx_, static_cast<size_t>(npad)), part(ctx_, static_cast<size_t>(npad));
        if (npad > n_) zero(ctx_, part.get() + n_, sizeof(double) * static_cast<size_t>(npad - n_));
        ctx_.allgather(right, xfull.get(), static_cast<size_t>(chunk));
        csr_spmv_pair_k<<<gridn((m_ + n_) * 32, 8192), kT, 0, ctx_.stream()>>>(
            m_, rowptr_.get(), colidx_.get(), val_csr_.get(), xfull.get(), top, n_, colptr_.get(), rowidx_.get(),
            val_csc_.get(), left, part.get());
        ctx_.note_launch();
        ctx_.check_launch("csr_spmv_pair");
        ctx_.reduce_scatter_sum(part.get(), bot, static_cast<size_t>(chunk));
        return;
    }
    csr_spmv_pair_k<<<gridn((m_ + n_) * 32, 8192), kT, 0, ctx_.stream()>>>(
        m_, rowptr_.get(), colidx_.get(), val_csr_.get(), right, top, n_, colptr_.get(), rowidx_.get(),
        val_csc_.get(), left, bot);
    ctx_.note_launch();
    ctx_.check_launch("csr_spmv_pair");
    if (row_sharded() && ctx_.has_comm()) ctx_.allreduce_sum(bot, static_cast<size_t>(n_));  // W^T left over the ranks
}

// ======================================================== warm start
DWarm make_warm(Context& ctx, Index m, Index n, Index b) {
    DWarm w;
    w.geo = Stack{m, n};
    w.uv = DMat(ctx, w.geo.ld(), std::max<Index>(b, 1), true);
    w.uv.cols = b;
    w.sigma.assign(static_cast<size_t>(b), 0.0);
    return w;
}

DWarm copy_warm(Context& ctx, const DWarm& src, Index cols) {
    DWarm w = make_warm(ctx, src.geo.m, src.geo.n, cols);
    copy(ctx, w.panel().left(cols), src.panel().left(cols));
    w.sigma.assign(src.sigma.begin(), src.sigma.begin() + cols);
    return w;
}

// ======================================================== thin_qr (CholQR)
namespace {

struct CholStep {
    DMat r, rinv;
    bool ok = false;
    double dmin = 0, dmax = 0;
};

constexpr double kSkipRel = 1e-14;  // CholQR pass skip: ||G - cI||_F <= 1e-14 c (cholinv.cu)

// R = chol(G) in place (or sqrt(c) I for a scaled-identity Gram), Rinv = R^{-1};
// reads back status, diag range and tr(G) (one sync). `trace_dev`, if set,
// receives tr(G) on the device too (the rank threshold reads it there).
// the same through cholqr_factor (b <= 112): with r_prev, also R_total =
// R * R_prev into *r_total and its rank into *rank_dev (the deferred path's
// second pass, so both paths stay bitwise identical)
CholStep chol_step_q(Context& ctx, DMat g, double* trace_dev, double* trace_host, const DMat* r_prev = nullptr,
                     View* r_total = nullptr, const double* trace_ref = nullptr, std::int64_t* rank_dev = nullptr) {
    CholStep s;
    const Index b = g.rows;
    s.r = std::move(g);
    s.rinv = DMat(ctx, b, b, false);
    DBuf<int> status(ctx, 1);
    DBuf<double> diag(ctx, 3);
    cholqr_factor(ctx, s.r.view(), s.rinv.view(), r_prev ? r_prev->data() : nullptr, r_prev ? r_prev->ld : 0,
                  r_total, status.get(), diag.get(), diag.get() + 2, trace_ref, rank_dev);
    if (trace_dev) copy(ctx, View{trace_dev, 1, 1, 2}, View{diag.get() + 2, 1, 1, 2});
    int st = 0;
    double dd[3] = {0, 0, 0};
    BLWS_CUDA(cudaMemcpyAsync(&st, status.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx.stream()));
    ctx.read(diag.get(), dd, 3);
    s.ok = st == 0;
    s.dmin = dd[0];
    s.dmax = dd[1];
    if (trace_host) *trace_host = dd[2];
    return s;
}

CholStep chol_step(Context& ctx, DMat g, double* trace_dev = nullptr, double* trace_host = nullptr) {
    CholStep s;
    const Index b = g.rows;
    s.r = std::move(g);
    s.rinv = DMat(ctx, b, b, false);
    DBuf<int> status(ctx, 1);
    DBuf<double> diag(ctx, 3);
    chol_inv_upper(ctx, s.r.view(), s.rinv.view(), status.get(), diag.get(), kSkipRel, diag.get() + 2);
    if (trace_dev) copy(ctx, View{trace_dev, 1, 1, 2}, View{diag.get() + 2, 1, 1, 2});
    int st = 0;
    double dd[3] = {0, 0, 0};
    BLWS_CUDA(cudaMemcpyAsync(&st, status.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx.stream()));
    ctx.read(diag.get(), dd, 3);
    s.ok = st == 0;
    s.dmin = dd[0];
    s.dmax = dd[1];
    if (trace_host) *trace_host = dd[2];
    return s;
}

}  // namespace

// C (a.cols x b.cols, ldc) = A^T B over the rows of two panels of the same row
// structure; rows [0, split.sharded) are summed over the ranks.
void panel_tn(Context& ctx, View a, View b, RowSplit split, double* c, Index ldc) {
    const Index rows = a.rows, s = split.sharded;
    if (s == 0 || !ctx.has_comm()) {
        gemm(ctx, true, false, a.cols, b.cols, rows, 1.0, a.p, a.ld, b.p, b.ld, 0.0, c, ldc);
        return;
    }
    gemm(ctx, true, false, a.cols, b.cols, s, 1.0, a.p, a.ld, b.p, b.ld, 0.0, c, ldc);
    ctx.allreduce_sum(c, static_cast<size_t>(ldc * b.cols));
    if (rows > s) gemm(ctx, true, false, a.cols, b.cols, rows - s, 1.0, a.p + s, a.ld, b.p + s, b.ld, 1.0, c, ldc);
}

// ||X||_F^2 of a panel -> out (device scalar), sharded rows summed over the ranks
void panel_sumsq(Context& ctx, View x, RowSplit split, double* out) {
    const Index s = split.sharded;
    if (s == 0 || !ctx.has_comm()) {
        sumsq(ctx, x, out);
        return;
    }
    sumsq(ctx, View{x.p, s, x.cols, x.ld}, out);
    ctx.allreduce_sum(out, 1);
    if (x.rows > s) {
        DBuf<double> t(ctx, 1);
        sumsq(ctx, View{x.p + s, x.rows - s, x.cols, x.ld}, t.get());
        axpy(ctx, View{out, 1, 1, 1}, View{t.get(), 1, 1, 1}, 1.0);
    }
}

// x^T y of two panel vectors -> out (device scalar), sharded rows summed over the ranks
void panel_dot(Context& ctx, Index rows, const double* x, const double* y, RowSplit split, double* out) {
    const Index s = split.sharded;
    if (s == 0 || !ctx.has_comm()) {
        dot(ctx, rows, x, y, out);
        return;
    }
    dot(ctx, s, x, y, out);
    ctx.allreduce_sum(out, 1);
    if (rows > s) {
        DBuf<double> t(ctx, 1);
        dot(ctx, rows - s, x + s, y + s, t.get());
        axpy(ctx, View{out, 1, 1, 1}, View{t.get(), 1, 1, 1}, 1.0);
    }
}

// coef (cols) = Q^T r over the panel rows, sharded rows summed over the ranks
void panel_gemv_t(Context& ctx, Index rows, Index cols, const double* q, Index ldq, const double* r, RowSplit split,
                  double* coef) {
    const Index s = split.sharded;
    if (s == 0 || !ctx.has_comm()) {
        gemv(ctx, true, rows, cols, 1.0, q, ldq, r, 0.0, coef);
        return;
    }
    gemv(ctx, true, s, cols, 1.0, q, ldq, r, 0.0, coef);
    ctx.allreduce_sum(coef, static_cast<size_t>(cols));
    if (rows > s) gemv(ctx, true, rows - s, cols, 1.0, q + s, ldq, r + s, 1.0, coef);
}

namespace {

DMat gram(Context& ctx, View x, RowSplit split = {}) {
    DMat g(ctx, x.cols, x.cols, false);
    static const bool g16 = [] {
        const char* e = std::getenv("BLWS_GRAM16");
        return !(e && e[0] == '0');
    }();
    if (g16 && (split.sharded == 0 || !ctx.has_comm()) && gram16_fits(x.rows, x.cols)) {
        gram16(ctx, x, g.data(), g.ld);
        return g;
    }
    panel_tn(ctx, x, x, split, g.data(), g.ld);
    return g;
}

}  // namespace

Index thin_qr_impl(Context& ctx, View x, View* r_out, RowSplit split);

Index thin_qr(Context& ctx, View x, View* r_out, RowSplit split) {
    ctx.region_begin(2);
    const Index rank = thin_qr_impl(ctx, x, r_out, split);
    ctx.region_end(2, 0.0, 0.0);
    return rank;
}

// thin_qr (core/qr.hpp:24-47) as CholQR2 with a shifted-CholQR3 fallback. Q is
// the unique orthonormal factor with diag(R) > 0, i.e. the reference's
// sign-normalised Householder Q. A pass whose Gram is a scaled identity
// (||G - cI||_F <= 1e-14 c) is skipped on the device (R = sqrt(c) I), so the
// launch sequence is fixed -- the same one thin_qr_deferred() issues.
Index thin_qr_impl(Context& ctx, View x, View* r_out, RowSplit split) {
    const Index rows = x.rows, b = x.cols;
    if (rows == 0 || b == 0) throw std::invalid_argument("thin_qr: empty matrix");
    if (rows < b) throw std::invalid_argument("thin_qr: requires rows >= cols");
    DBuf<double> ss(ctx, 2);  // ss[0] = ||X||_F^2 = tr(X^T X)
    std::vector<CholStep> steps;
    double hss = 0;
    const bool q = cholqr_factor_fits(b);
    CholStep s1 = q ? chol_step_q(ctx, gram(ctx, x, split), ss.get(), &hss)
                    : chol_step(ctx, gram(ctx, x, split), ss.get(), &hss);
    if (!std::isfinite(hss)) throw std::invalid_argument("thin_qr: non-finite entries");
    const bool ill = !s1.ok || !(s1.dmin > 0) || s1.dmax / s1.dmin > 1e6;
    DMat y(ctx, rows, b, false);
    if (!ill && q) {
        gemm(ctx, false, false, rows, b, b, 1.0, x.p, x.ld, s1.rinv.data(), s1.rinv.ld, 0.0, y.data(), y.ld);
        DMat rt(ctx, b, b, false);
        View rtv = rt.view();
        DBuf<std::int64_t> rank(ctx, 1);
        CholStep s2 = chol_step_q(ctx, gram(ctx, y.view(), split), nullptr, nullptr, &s1.r, &rtv, ss.get(),
                                  rank.get());
        if (!s2.ok) throw NumericalError("thin_qr: CholQR2 second pass failed");
        gemm(ctx, false, false, rows, b, b, 1.0, y.data(), y.ld, s2.rinv.data(), s2.rinv.ld, 0.0, x.p, x.ld);
        std::int64_t hr = 0;
        ctx.read_i64(rank.get(), &hr, 1);
        if (r_out) copy(ctx, *r_out, rtv);
        return hr;
    }
    if (!ill) {
        gemm(ctx, false, false, rows, b, b, 1.0, x.p, x.ld, s1.rinv.data(), s1.rinv.ld, 0.0, y.data(), y.ld);
        steps.push_back(std::move(s1));
        CholStep s2 = chol_step(ctx, gram(ctx, y.view(), split));
        if (!s2.ok) throw NumericalError("thin_qr: CholQR2 second pass failed");
        gemm(ctx, false, false, rows, b, b, 1.0, y.data(), y.ld, s2.rinv.data(), s2.rinv.ld, 0.0, x.p, x.ld);
        steps.push_back(std::move(s2));
    } else {
        // shifted CholQR3 (Fukaya et al. 2020): s = 11 (rows*b + b(b+1)) u ||X||_F^2
        DMat g = gram(ctx, x, split);
        DBuf<double> shift(ctx, 1);
        const double factor =
            11.0 * (static_cast<double>(rows) * b + static_cast<double>(b) * (b + 1)) * 1.1102230246251565e-16;
        shift_for_cholqr3_k<<<1, 1, 0, ctx.stream()>>>(ss.get(), factor, shift.get());
        ctx.note_launch();
        add_diagonal(ctx, g.view(), shift.get());
        CholStep a = chol_step(ctx, std::move(g));
        if (!a.ok) {
            if (hss == 0.0) {
                if (r_out) fill(ctx, *r_out, 0.0);
                return 0;
            }
            throw NumericalError("thin_qr: shifted CholQR failed");
        }
        gemm(ctx, false, false, rows, b, b, 1.0, x.p, x.ld, a.rinv.data(), a.rinv.ld, 0.0, y.data(), y.ld);
        copy(ctx, x, y.view());
        steps.push_back(std::move(a));
        for (int k = 0; k < 2; ++k) {
            CholStep c = chol_step(ctx, gram(ctx, x, split));
            if (!c.ok) break;  // remaining directions are numerically null
            gemm(ctx, false, false, rows, b, b, 1.0, x.p, x.ld, c.rinv.data(), c.rinv.ld, 0.0, y.data(), y.ld);
            copy(ctx, x, y.view());
            steps.push_back(std::move(c));
        }
    }
    // R = R_last * ... * R_1
    DMat r = std::move(steps.back().r);
    for (int k = static_cast<int>(steps.size()) - 2; k >= 0; --k) {
        DMat t(ctx, b, b, false);
        gemm(ctx, false, false, b, b, b, 1.0, r.data(), r.ld, steps[k].r.data(), steps[k].r.ld, 0.0, t.data(), t.ld);
        r = std::move(t);
    }
    DBuf<std::int64_t> rank(ctx, 1);
    count_diag_above(ctx, r.view(), ss.get(), 1e-12, rank.get());
    std::int64_t hr = 0;
    ctx.read_i64(rank.get(), &hr, 1);
    if (r_out) copy(ctx, *r_out, r.view());
    return hr;
}

// ======================================================== adapt_subspace
DWarm adapt_subspace(Context& ctx, const DWarm* warm, Index r_new, Index m, Index n, Rng& rng,
                     const RowShard* shard, Index col0, Index chunk) {
    // with a row shard, U's Gaussian columns are drawn for all m_total rows in the
    // reference's (column-major) order and this rank keeps rows [row0, row0 + m);
    // with a column slice (chunk >= 0) V's are drawn for all n rows and this rank
    // keeps rows [col0, col0 + chunk) (rows past n stay zero padding)
    const bool sh = shard && shard->m_total > 0;
    const bool cs = chunk >= 0;
    const Index mt = sh ? shard->m_total : m, r0 = sh ? shard->row0 : 0, pn = cs ? chunk : n;
    const RowSplit usplit{sh && ctx.has_comm() ? m : 0};
    const RowSplit vsplit{cs && ctx.has_comm() ? pn : 0};
    if (r_new < 1 || r_new > std::min(mt, n)) throw std::invalid_argument("adapt_subspace: r_new out of range");
    auto put_v = [&](View dst, const double* h) {  // the drawn n x cols block, this rank's rows
        if (!cs) return upload(ctx, dst, h, n);
        const Index take = std::max<Index>(0, std::min(n, col0 + chunk) - col0);
        if (take > 0) upload(ctx, View{dst.p, take, dst.cols, dst.ld}, h + col0, n);
    };
    if (!warm || warm->rank() == 0) {
        DWarm out = make_warm(ctx, m, pn, r_new);
        std::vector<double> h(static_cast<size_t>(std::max(mt, n) * r_new));
        rng.gaussian_matrix(mt, r_new, h.data(), mt);
        upload(ctx, out.u(), h.data() + r0, mt);
        rng.gaussian_matrix(n, r_new, h.data(), n);
        put_v(out.v(), h.data());
        View u = out.u(), v = out.v();
        thin_qr(ctx, u, nullptr, usplit);
        thin_qr(ctx, v, nullptr, vsplit);
        return out;
    }
    const Index r_old = warm->rank();
    if (r_new == r_old) return copy_warm(ctx, *warm, r_old);
    if (r_new < r_old) return copy_warm(ctx, *warm, r_new);
    const Index add = r_new - r_old;
    DWarm out = make_warm(ctx, m, pn, r_new);
    copy(ctx, out.panel().left(r_old), warm->panel().left(r_old));
    std::vector<double> h(static_cast<size_t>(std::max(mt, n) * add));
    rng.gaussian_matrix(mt, add, h.data(), mt);
    upload(ctx, out.u().cols_range(r_old, add), h.data() + r0, mt);
    rng.gaussian_matrix(n, add, h.data(), n);
    put_v(out.v().cols_range(r_old, add), h.data());
    View u = out.u(), v = out.v();
    thin_qr(ctx, u, nullptr, usplit);
    thin_qr(ctx, v, nullptr, vsplit);
    std::copy(warm->sigma.begin(), warm->sigma.end(), out.sigma.begin());
    return out;
}

// ======================================================== block lanczos
namespace {

/// Augmented block apply (augmented_operator.hpp:50-57): Z = [[0,W],[W^T,0]] X.
void aug_apply(LinearOperator& w, const Stack& geo, View x, View z) {
    View xt{x.p, geo.m, x.cols, x.ld}, xb{x.p + geo.mp(), geo.n, x.cols, x.ld};
    View zt{z.p, geo.m, z.cols, z.ld}, zb{z.p + geo.mp(), geo.n, z.cols, z.ld};
    w.apply_pair_block(xt, xb, zt, zb);
}

double read_scalar(Context& ctx, const double* d) {
    double h = 0;
    ctx.read(d, &h, 1);
    return h;
}

}  // namespace

// block_lanczos.hpp:70-126 on the augmented view; x1 is a stacked panel.
BlockLanczos block_lanczos_procedure(LinearOperator& w, View x1, Index k) {
    Context& ctx = w.ctx();
    const Stack geo{w.rows(), w.panel_n()};  // bottom rows: this rank's columns when column-sharded
    const Index dim = global_rows(w) + w.cols(), bs = x1.cols, ld = geo.ld();
    if (k < 1) throw std::invalid_argument("block_lanczos_procedure: k must be >= 1");
    if (bs < 1 || x1.rows != ld) throw std::invalid_argument("block_lanczos_procedure: bad initial block");
    if (k * bs > dim) throw std::invalid_argument("block_lanczos_procedure: k*b exceeds dimension");
    const RowSplit split = w.panel_split();  // row-sharded operator: the top rows are this rank's
    DBuf<double> sc(ctx, 4);
    {
        DMat g = gram(ctx, x1, split);
        sumsq_minus_identity(ctx, g.view(), sc.get());
        if (std::sqrt(read_scalar(ctx, sc.get())) > 1e-8)
            throw std::invalid_argument("block_lanczos_procedure: X1 not orthonormal");
    }
    BlockLanczos out;
    out.q = DMat(ctx, ld, k * bs, true);
    View Q = out.q.view();
    copy(ctx, Q.cols_range(0, bs), x1);
    DMat z(ctx, ld, bs, true);
    DMat mtmp(ctx, bs, bs, false);
    auto block = [&](Index l) { return View{Q.p + l * bs * Q.ld, ld, bs, Q.ld}; };

    aug_apply(w, geo, block(0), z.view());
    panel_sumsq(ctx, z.view(), split, sc.get());
    double scale = std::sqrt(read_scalar(ctx, sc.get()));
    panel_tn(ctx, block(0), z.view(), split, mtmp.data(), mtmp.ld);
    out.m.emplace_back(ctx, bs, bs, false);
    symmetrize(ctx, out.m.back().view(), mtmp.view());
    out.built = 1;
    for (Index l = 1; l < k; ++l) {
        View xc = block(l - 1);
        // R = Z - X_l M_l - X_{l-1} B_{l-1}^T, in place in z
        gemm(ctx, false, false, ld, bs, bs, -1.0, xc.p, xc.ld, out.m.back().data(), out.m.back().ld, 1.0, z.data(),
             z.ld);
        if (l > 1) {
            View xp = block(l - 2);
            gemm(ctx, false, true, ld, bs, bs, -1.0, xp.p, xp.ld, out.b.back().data(), out.b.back().ld, 1.0,
                 z.data(), z.ld);
        }
        panel_sumsq(ctx, z.view(), split, sc.get());
        const double rn = std::sqrt(read_scalar(ctx, sc.get()));
        if (rn <= 1e-10 * scale) {  // kBlockBreakdownTol (block_lanczos.hpp:64, :103)
            out.terminated_early = true;
            break;
        }
        View xn = block(l);
        copy(ctx, xn, z.view());
        DMat rb(ctx, bs, bs, true);
        View rv = rb.view();
        const Index rank = thin_qr(ctx, xn, &rv, split);
        if (rank < bs) {
            fill(ctx, xn, 0.0);
            out.terminated_early = true;
            break;
        }
        out.b.push_back(std::move(rb));
        ++out.built;
        aug_apply(w, geo, xn, z.view());
        panel_sumsq(ctx, z.view(), split, sc.get());
        scale = std::max(scale, std::sqrt(read_scalar(ctx, sc.get())));
        panel_tn(ctx, xn, z.view(), split, mtmp.data(), mtmp.ld);
        out.m.emplace_back(ctx, bs, bs, false);
        symmetrize(ctx, out.m.back().view(), mtmp.view());
    }
    out.q.cols = out.built * bs;
    return out;
}

// block_lanczos.hpp:204-261, every host decision taken when it arises (the
// exact path; blws_svd() below tries the deferred path first).
static BlwsResult blws_svd_exact(LinearOperator& w, const DWarm& warm, Index k, Index r, Rng& rng) {
    Context& ctx = w.ctx();
    const Index m = w.rows(), n = w.cols(), pn = w.panel_n();  // pn: the panels' bottom rows
    const Index bs = warm.rank();
    if (bs < 1) throw std::invalid_argument("blws_svd: empty warm start (seed via adapt_subspace)");
    const Index m_all = w.row_sharded() ? w.shard().m_total : m;
    if (r < 1 || r > std::min(m_all, n)) throw std::invalid_argument("blws_svd: bad r");
    if (warm.geo.m != m || warm.geo.n != pn) throw std::invalid_argument("blws_svd: warm start does not match operator");
    BlwsResult out;
    Index k_eff = k;
    if (r > k_eff * bs) {
        k_eff = (r + bs - 1) / bs;
        out.k_raised = true;
    }
    k_eff = std::min(k_eff, (m_all + n) / bs);
    k_eff = std::max<Index>(k_eff, 1);
    const Stack geo{m, pn};

    // X1 = qr([U; V] / sqrt(2)).q -- Q is invariant under the positive scale,
    // so the 1/sqrt(2) is folded away.
    DMat x1(ctx, geo.ld(), bs, false);
    copy(ctx, x1.view(), warm.panel());
    const RowSplit split = w.panel_split();
    const RowSplit usplit{split.sharded ? m : 0};
    const RowSplit vsplit{w.col_sharded() ? pn : 0};
    {
        View xv = x1.view();
        thin_qr(ctx, xv, nullptr, split);
    }
    BlockLanczos fac = block_lanczos_procedure(w, x1.view(), k_eff);
    out.terminated_early = fac.terminated_early;
    const Index d = fac.built * bs;

    // T = embed() (block_lanczos.hpp:28-40), EVD descending (small_dense.hpp:24-43)
    DMat t(ctx, d, d, true);
    for (Index l = 0; l < fac.built; ++l) {
        place_block(ctx, t.view().sub(l * bs, l * bs, bs, bs), fac.m[l].view(), false);
        if (l + 1 < fac.built) {
            place_block(ctx, t.view().sub(l * bs + bs, l * bs, bs, bs), fac.b[l].view(), false);
            place_block(ctx, t.view().sub(l * bs, l * bs + bs, bs, bs), fac.b[l].view(), true);
        }
    }
    // only the leading min(r, d) pairs can be kept (block_lanczos.hpp:235-238)
    const Index want = std::min(r, d);
    DBuf<double> vals(ctx, static_cast<size_t>(want));
    DMat vecs(ctx, d, want, false);
    ctx.region_begin(1);
    small_dense_guard(t.rows, "sym_evd_small: too large");
    sym_evd_top(ctx, t.view(), want, vals.get(), vecs.view());
    ctx.region_end(1, 0.0, 0.0);
    std::vector<double> hv(static_cast<size_t>(want));
    ctx.read(vals.get(), hv.data(), want);
    for (double v : hv)
        if (!std::isfinite(v)) throw NumericalError("sym_evd_small: failed to converge");

    // keep the strictly positive part (block_lanczos.hpp:233-238); avail = d >= r
    const Index avail = std::min(k_eff * bs, want);
    const double floor = d > 0 ? 1e-12 * std::fabs(hv[0]) : 0.0;
    Index keep = 0;
    while (keep < avail && keep < r && hv[static_cast<size_t>(keep)] > floor) ++keep;

    DWarm next = make_warm(ctx, m, pn, keep);
    if (keep > 0) {
        // Ritz lift of the kept columns only, sqrt(2) unpack fused (:240-248)
        gemm(ctx, false, false, geo.ld(), keep, d, std::sqrt(2.0), fac.q.data(), fac.q.ld, vecs.data(), vecs.ld, 0.0,
             next.uv.data(), next.uv.ld);
        std::copy(hv.begin(), hv.begin() + keep, next.sigma.begin());
        View u = next.u(), v = next.v();
        thin_qr(ctx, u, nullptr, usplit);
        thin_qr(ctx, v, nullptr, vsplit);
    }
    if (keep < r) {
        next = adapt_subspace(ctx, keep > 0 ? &next : nullptr, r, m, n, rng, w.row_sharded() ? &w.shard() : nullptr,
                              w.col0(), w.col_sharded() ? pn : -1);
        out.padded = true;
    }
    out.warm = std::move(next);
    return out;
}

// ======================================================== deferred (optimistic) path
// The exact path reads ~26 scalars back per call (norms for the rank and
// breakdown tests, Cholesky status and conditioning, the Ritz values for
// `keep`); every read drains the launch queue (and, while an async upload
// shares the PCIe link, costs several times more). The deferred path launches
// the common-case sequence with each of those scalars written to a slot of one
// device buffer, reads the buffer ONCE, and replays the exact path's host tests
// on the values. If any test would have branched away from the common case
// (breakdown, rank loss, ill-conditioned Gram, keep < min(r, d), non-finite),
// the call is redone on the exact path -- which the deferred path never
// perturbs: it does not draw from the Rng and writes only fresh buffers.
// Where both run, results are bitwise identical (tests/test_gpu_blws.py):
// the device-predicated pass skip yields R = Rinv = I and X I == X exactly.
namespace {

struct Slots {
    DBuf<double> buf;
    int used = 0, cap = 0;
    std::vector<double> h;
    Slots(Context& ctx, int capacity) : buf(ctx, static_cast<size_t>(capacity)), cap(capacity) {
        zero(ctx, buf.get(), sizeof(double) * static_cast<size_t>(capacity));
    }
    int take(int k = 1) {
        if (used + k > cap) throw std::logic_error("deferred slots exhausted");
        const int s0 = used;
        used += k;
        return s0;
    }
    double* at(int s0) { return buf.get() + s0; }
    void fetch(Context& ctx) {
        h.assign(static_cast<size_t>(used), 0.0);
        if (used) ctx.read(buf.get(), h.data(), static_cast<size_t>(used));
    }
    double val(int s0) const { return h[static_cast<size_t>(s0)]; }
    int as_int(int s0) const {
        int v = 0;
        std::memcpy(&v, &h[static_cast<size_t>(s0)], sizeof(int));
        return v;
    }
    std::int64_t as_i64(int s0) const {
        std::int64_t v = 0;
        std::memcpy(&v, &h[static_cast<size_t>(s0)], sizeof(v));
        return v;
    }
};

struct QrRec {
    int hss, st1, dg1, st2, dg2, rank;
};

// thin_qr_impl's common case as a fixed launch sequence (both CholQR passes,
// each skipped on the device for a scaled-identity Gram).
QrRec thin_qr_deferred(Context& ctx, View x, View* r_out, Slots& sl, RowSplit split) {
    const Index rows = x.rows, b = x.cols;
    QrRec q{sl.take(), sl.take(), sl.take(3), sl.take(), sl.take(3), sl.take()};
    ctx.region_begin(2);
    DMat r1 = gram(ctx, x, split);
    DMat ri1(ctx, b, b, false);
    DMat y(ctx, rows, b, false);
    if (cholqr_factor_fits(b)) {
        // one launch per pass (cholqr.cu): factor + inverse, and in the second
        // pass R = R2 R1 and the rank count as well
        cholqr_factor(ctx, r1.view(), ri1.view(), nullptr, 0, nullptr, reinterpret_cast<int*>(sl.at(q.st1)),
                      sl.at(q.dg1), sl.at(q.hss), nullptr, nullptr);
        gemm(ctx, false, false, rows, b, b, 1.0, x.p, x.ld, ri1.data(), ri1.ld, 0.0, y.data(), y.ld);
        DMat r2 = gram(ctx, y.view(), split);
        DMat ri2(ctx, b, b, false);
        cholqr_factor(ctx, r2.view(), ri2.view(), r1.data(), r1.ld, r_out, reinterpret_cast<int*>(sl.at(q.st2)),
                      sl.at(q.dg2), sl.at(q.dg2 + 2), sl.at(q.hss), reinterpret_cast<std::int64_t*>(sl.at(q.rank)));
        gemm(ctx, false, false, rows, b, b, 1.0, y.data(), y.ld, ri2.data(), ri2.ld, 0.0, x.p, x.ld);
        ctx.region_end(2, 0.0, 0.0);
        return q;
    }
    chol_inv_upper(ctx, r1.view(), ri1.view(), reinterpret_cast<int*>(sl.at(q.st1)), sl.at(q.dg1), kSkipRel,
                   sl.at(q.hss));
    gemm(ctx, false, false, rows, b, b, 1.0, x.p, x.ld, ri1.data(), ri1.ld, 0.0, y.data(), y.ld);
    DMat r2 = gram(ctx, y.view(), split);
    DMat ri2(ctx, b, b, false);
    chol_inv_upper(ctx, r2.view(), ri2.view(), reinterpret_cast<int*>(sl.at(q.st2)), sl.at(q.dg2), kSkipRel,
                   sl.at(q.dg2 + 2));
    gemm(ctx, false, false, rows, b, b, 1.0, y.data(), y.ld, ri2.data(), ri2.ld, 0.0, x.p, x.ld);
    DMat r(ctx, b, b, false);
    gemm(ctx, false, false, b, b, b, 1.0, r2.data(), r2.ld, r1.data(), r1.ld, 0.0, r.data(), r.ld);
    count_diag_above(ctx, r.view(), sl.at(q.hss), 1e-12, reinterpret_cast<std::int64_t*>(sl.at(q.rank)));
    if (r_out) copy(ctx, *r_out, r.view());
    ctx.region_end(2, 0.0, 0.0);
    return q;
}

// thin_qr_impl's host tests on the deferred values; false = it would have
// taken another branch (shifted CholQR3, a failed pass, non-finite input).
bool qr_check(const QrRec& q, const Slots& sl, Index b, Index* rank) {
    (void)b;
    if (!std::isfinite(sl.val(q.hss))) return false;
    const double dmin = sl.val(q.dg1), dmax = sl.val(q.dg1 + 1);
    if (sl.as_int(q.st1) != 0 || !(dmin > 0) || dmax / dmin > 1e6) return false;
    if (sl.as_int(q.st2) != 0) return false;
    *rank = sl.as_i64(q.rank);
    return true;
}

struct LanczosRec {
    int scale0 = -1;
    std::vector<int> rn, scale;
    std::vector<QrRec> qr;
};

// block_lanczos_procedure without reads: every block is built (the breakdown
// and rank tests are replayed by lanczos_check). X1 comes from thin_qr here,
// so the caller-input orthonormality check of the exact path is not repeated.
BlockLanczos block_lanczos_deferred(LinearOperator& w, View x1, Index k, Slots& sl, LanczosRec& rec) {
    Context& ctx = w.ctx();
    const Stack geo{w.rows(), w.panel_n()};
    const Index bs = x1.cols, ld = geo.ld();
    const RowSplit split = w.panel_split();
    BlockLanczos out;
    // no zero fills unless a padding row exists: every block of Q is written
    // over all ld rows (copies of full panels), and Z's rows are all written by
    // the paired apply when m and n are even
    const bool pad = (geo.m % 2) != 0 || (geo.n % 2) != 0;
    out.q = DMat(ctx, ld, k * bs, false);
    View Q = out.q.view();
    copy(ctx, Q.cols_range(0, bs), x1);
    DMat z(ctx, ld, bs, pad);
    DMat mtmp(ctx, bs, bs, false);
    auto block = [&](Index l) { return View{Q.p + l * bs * Q.ld, ld, bs, Q.ld}; };
    aug_apply(w, geo, block(0), z.view());
    rec.scale0 = sl.take();
    panel_sumsq(ctx, z.view(), split, sl.at(rec.scale0));
    panel_tn(ctx, block(0), z.view(), split, mtmp.data(), mtmp.ld);
    out.m.emplace_back(ctx, bs, bs, false);
    symmetrize(ctx, out.m.back().view(), mtmp.view());
    out.built = 1;
    for (Index l = 1; l < k; ++l) {
        View xc = block(l - 1);
        gemm(ctx, false, false, ld, bs, bs, -1.0, xc.p, xc.ld, out.m.back().data(), out.m.back().ld, 1.0, z.data(),
             z.ld);
        if (l > 1) {
            View xp = block(l - 2);
            gemm(ctx, false, true, ld, bs, bs, -1.0, xp.p, xp.ld, out.b.back().data(), out.b.back().ld, 1.0,
                 z.data(), z.ld);
        }
        rec.rn.push_back(sl.take());
        panel_sumsq(ctx, z.view(), split, sl.at(rec.rn.back()));
        View xn = block(l);
        copy(ctx, xn, z.view());
        DMat rb(ctx, bs, bs, false);  // thin_qr writes all of R (zeros below the diagonal)
        View rv = rb.view();
        rec.qr.push_back(thin_qr_deferred(ctx, xn, &rv, sl, split));
        out.b.push_back(std::move(rb));
        ++out.built;
        aug_apply(w, geo, xn, z.view());
        rec.scale.push_back(sl.take());
        panel_sumsq(ctx, z.view(), split, sl.at(rec.scale.back()));
        panel_tn(ctx, xn, z.view(), split, mtmp.data(), mtmp.ld);
        out.m.emplace_back(ctx, bs, bs, false);
        symmetrize(ctx, out.m.back().view(), mtmp.view());
    }
    out.q.cols = out.built * bs;
    return out;
}

// block_lanczos_procedure's breakdown (block_lanczos.hpp:103) and rank tests
bool lanczos_check(const LanczosRec& rec, const Slots& sl, Index bs) {
    double scale = std::sqrt(sl.val(rec.scale0));
    for (size_t l = 0; l < rec.rn.size(); ++l) {
        const double rn = std::sqrt(sl.val(rec.rn[l]));
        if (rn <= 1e-10 * scale) return false;
        Index rank = 0;
        if (!qr_check(rec.qr[l], sl, bs, &rank) || rank < bs) return false;
        scale = std::max(scale, std::sqrt(sl.val(rec.scale[l])));
    }
    return true;
}

bool force_exact() {
    const char* e = std::getenv("BLWS_EXACT");
    return e && *e && std::string(e) != "0";
}

// BLWS_EXACT_PAD=1: a deferred call that needs padding is redone on the exact
// path (the r01 behaviour) instead of padding its own kept columns
bool force_exact_pad() {
    static const bool on = [] {
        const char* e = std::getenv("BLWS_EXACT_PAD");
        return e && *e && std::string(e) != "0";
    }();
    return on;
}

}  // namespace

namespace {

struct DeferredShape {
    Index m, n, bs, k, r, k_eff, d, want;
    bool k_raised;
};

struct DeferredRecs {
    QrRec q1{}, qu{}, qv{};
    LanczosRec lrec;
    int vslot = -1;
};

// blws_svd's common case as one launch sequence with no host reads (capturable
// as a CUDA graph): input the warm panel `src` (ld x bs), output the next warm
// panel in `next_uv` (ld x want) and the slots.
DeferredRecs enqueue_deferred(LinearOperator& w, View src, const DeferredShape& sh, Slots& sl, View next_uv) {
    Context& ctx = w.ctx();
    const Stack geo{sh.m, sh.n};
    DeferredRecs rec;
    const RowSplit split = w.panel_split();
    const RowSplit usplit{split.sharded ? sh.m : 0};
    DMat x1(ctx, geo.ld(), sh.bs, false);
    copy(ctx, x1.view(), src);
    {
        View xv = x1.view();
        rec.q1 = thin_qr_deferred(ctx, xv, nullptr, sl, split);
    }
    BlockLanczos fac = block_lanczos_deferred(w, x1.view(), sh.k_eff, sl, rec.lrec);
    const Index bs = sh.bs, d = sh.d, want = sh.want;
    DMat t(ctx, d, d, fac.built > 2);  // built <= 2 blocks cover all of T
    for (Index l = 0; l < fac.built; ++l) {
        place_block(ctx, t.view().sub(l * bs, l * bs, bs, bs), fac.m[l].view(), false);
        if (l + 1 < fac.built) {
            place_block(ctx, t.view().sub(l * bs + bs, l * bs, bs, bs), fac.b[l].view(), false);
            place_block(ctx, t.view().sub(l * bs, l * bs + bs, bs, bs), fac.b[l].view(), true);
        }
    }
    rec.vslot = sl.take(static_cast<int>(want));
    DMat vecs(ctx, d, want, false);
    ctx.region_begin(1);
    small_dense_guard(t.rows, "sym_evd_small: too large");
    sym_evd_top(ctx, t.view(), want, sl.at(rec.vslot), vecs.view());
    ctx.region_end(1, 0.0, 0.0);
    // keep = want is assumed (verified by finish_deferred); lift + sqrt(2) unpack
    gemm(ctx, false, false, geo.ld(), want, d, std::sqrt(2.0), fac.q.data(), fac.q.ld, vecs.data(), vecs.ld, 0.0,
         next_uv.p, next_uv.ld);
    View u{next_uv.p, sh.m, want, next_uv.ld}, v{next_uv.p + geo.mp(), sh.n, want, next_uv.ld};
    {
        AuxScope aux(ctx);  // the two QRs are independent
        rec.qv = thin_qr_deferred(ctx, v, nullptr, sl, RowSplit{w.col_sharded() ? sh.n : 0});
        aux.main();
        rec.qu = thin_qr_deferred(ctx, u, nullptr, sl, usplit);
    }
    return rec;
}

// the exact path's host tests on the fetched slots (BLWS_DEBUG=1: the failing one on stderr)
// *kept_short: set to the kept count when keep < want is the ONLY failed test
// (the call then needs just the exact path's Rng padding), else -1.
bool finish_deferred(const DeferredRecs& rec, const Slots& sl, const DeferredShape& sh, Index* kept_short) {
    const bool dbg = std::getenv("BLWS_DEBUG") != nullptr;
    *kept_short = -1;
    auto fail = [&](const char* why) {
        if (dbg) std::fprintf(stderr, "blws_svd deferred -> exact: %s\n", why);
        return false;
    };
    auto qr_dbg = [&](const char* nm, const QrRec& q) {
        if (dbg)
            std::fprintf(stderr, "  %s: hss %.3e st %d/%d diag [%.3e, %.3e] rank %lld\n", nm, sl.val(q.hss),
                         sl.as_int(q.st1), sl.as_int(q.st2), sl.val(q.dg1), sl.val(q.dg1 + 1),
                         static_cast<long long>(sl.as_i64(q.rank)));
    };
    Index rank = 0;
    if (!qr_check(rec.q1, sl, sh.bs, &rank)) {
        qr_dbg("x1", rec.q1);
        return fail("X1 QR");
    }
    if (!lanczos_check(rec.lrec, sl, sh.bs)) {
        for (const auto& q : rec.lrec.qr) qr_dbg("lanczos", q);
        return fail("block Lanczos breakdown / rank");
    }
    if (!qr_check(rec.qu, sl, sh.want, &rank)) {
        qr_dbg("u", rec.qu);
        return fail("U QR");
    }
    if (!qr_check(rec.qv, sl, sh.want, &rank)) {
        qr_dbg("v", rec.qv);
        return fail("V QR");
    }
    const double* hv = sl.h.data() + rec.vslot;
    for (Index i = 0; i < sh.want; ++i)
        if (!std::isfinite(hv[i])) return fail("non-finite Ritz value");
    const double floor = 1e-12 * std::fabs(hv[0]);
    Index kept = 0;
    while (kept < sh.want && hv[kept] > floor) ++kept;
    if (kept != sh.want) {
        *kept_short = kept;
        return fail("keep < min(r, d)");
    }
    return true;
}

bool graphs_enabled() {
    const char* e = std::getenv("BLWS_GRAPHS");
    return !(e && std::string(e) == "0");
}

}  // namespace

/// A captured deferred blws_svd for one (operator data, bs, k, r): stable input
/// and output panels around a CUDA graph of the whole launch sequence. The
/// kernel nodes live in device memory, so there is no per-kernel command fetch
/// over PCIe (which an async upload saturates) and no per-launch host cost.
struct SvdGraph {
    const void* key_data = nullptr;
    Index bs = 0, k = 0, r = 0;
    std::uint64_t last_use = 0;  // LRU stamp (the cache holds kMaxSvdGraphs plans per operator)
    bool comm = false;  // captured with the allreduces of a row-sharded operator
    int seen = 0;
    bool failed = false;
    cudaGraphExec_t exec = nullptr;
    std::unique_ptr<Slots> sl;
    DMat src, next;
    DeferredRecs rec;
    int finite_slot = 0;
    std::int64_t launches = 0, applications = 0;
    std::vector<Context::CapturedRegion> regions;  // K1 / EVD / thin_qr, timed by stamp nodes
    DBuf<std::uint64_t> stamps;
    ~SvdGraph() {
        if (exec) cudaGraphExecDestroy(exec);
    }
};

// diagnostics (tests) and the graph-cache LRU clock; atomic because
// independent solves may run on several threads (one context each)
std::atomic<std::int64_t> g_blws_deferred_fallbacks{0};
constexpr size_t kMaxSvdGraphs = 4;
static std::atomic<std::uint64_t> g_svd_graph_clock{0};
std::atomic<std::int64_t> g_blws_graph_launches{0};

// blws_svd on warm starts in the operator's panel layout (V = this rank's
// columns when column-sharded); blws_svd() converts at the boundary.
static BlwsResult blws_svd_panel(LinearOperator& w, const DWarm& warm, Index k, Index r, Rng& rng) {
    Context& ctx = w.ctx();
    RegionGuard region(ctx, 5);
    const Index m = w.rows(), n = w.cols(), pn = w.panel_n();
    const Index bs = warm.rank();
    const Index m_all = w.row_sharded() ? w.shard().m_total : m;  // global rows of a row shard
    if (bs < 1 || r < 1 || r > std::min(m_all, n) || warm.geo.m != m || warm.geo.n != pn)
        return blws_svd_exact(w, warm, k, r, rng);  // throws the reference's errors
    DeferredShape sh{m, pn, bs, k, r, k, 0, 0, false};
    if (r > sh.k_eff * bs) {
        sh.k_eff = (r + bs - 1) / bs;
        sh.k_raised = true;
    }
    sh.k_eff = std::max<Index>(std::min(sh.k_eff, (m_all + n) / bs), 1);
    sh.d = sh.k_eff * bs;
    sh.want = std::min(r, sh.d);
    // keep < r needs the Rng padding: the exact path owns that case
    if (force_exact() || sh.want < r || k < 1 || k * bs > m_all + n) return blws_svd_exact(w, warm, k, r, rng);
    const Stack geo{m, pn};
    const int cap = 16 * static_cast<int>(sh.k_eff + 3) + static_cast<int>(sh.want) + 9;

    // ---- graph plan for this (operator data, shape); eager on first sight
    SvdGraph* plan = nullptr;
    if (graphs_enabled() && !ctx.host_comm()) {  // host-staged collectives cannot be captured
        for (auto& g : w.svd_graphs())
            if (g->key_data == w.data_key() && g->bs == bs && g->k == k && g->r == r && g->comm == ctx.has_comm())
                plan = g.get();
        if (!plan) {
            // bounded cache: a solve whose rank keeps changing must not pin one
            // graph (panels + graph memory pool) per rank it ever visited
            auto& gs = w.svd_graphs();
            if (gs.size() >= kMaxSvdGraphs) {
                auto lru = std::min_element(gs.begin(), gs.end(), [](const std::shared_ptr<SvdGraph>& a,
                                                                     const std::shared_ptr<SvdGraph>& b) {
                    return a->last_use < b->last_use;
                });
                ctx.sync();  // nothing in flight may still use the evicted graph
                gs.erase(lru);
            }
            auto g = std::make_shared<SvdGraph>();
            g->key_data = w.data_key();
            g->bs = bs;
            g->k = k;
            g->r = r;
            g->comm = ctx.has_comm();
            w.svd_graphs().push_back(g);
            plan = g.get();
        }
        plan->last_use = ++g_svd_graph_clock;
        // captured on the third call with this key (one-off shapes stay eager:
        // capture + instantiate costs tens of ms)
        if (plan->failed || (!plan->exec && plan->seen++ < 2)) plan = nullptr;
    }

    std::unique_ptr<Slots> local;
    Slots* sl = nullptr;
    DeferredRecs rec;
    DWarm next;
    int finite_slot = 0;
    if (plan) {
        if (!plan->exec) {
            // capture once: stable buffers outside the graph, temporaries inside
            plan->sl = std::make_unique<Slots>(ctx, cap);
            plan->finite_slot = plan->sl->take(2);
            plan->src = DMat(ctx, geo.ld(), bs, false);
            plan->next = DMat(ctx, geo.ld(), sh.want, true);
            plan->stamps = DBuf<std::uint64_t>(ctx, 64);
        }
        sl = plan->sl.get();
        finite_slot = plan->finite_slot;
        // a pending async upload is waited for and checked outside the graph
        zero(ctx, sl->at(finite_slot), 2 * sizeof(double));
        w.defer_pending_check(reinterpret_cast<int*>(sl->at(finite_slot)));
        share_flag(ctx, reinterpret_cast<int*>(sl->at(finite_slot)), sl->at(finite_slot + 1));
        if (!plan->exec) {
            const std::int64_t l0 = ctx.launches(), a0 = w.application_count();
            BLWS_CUDA(cudaStreamBeginCapture(ctx.stream(), cudaStreamCaptureModeRelaxed));
            ctx.begin_region_capture(plan->stamps.get(), 64);
            cudaGraph_t graph = nullptr;
            bool captured = true;
            try {
                plan->rec = enqueue_deferred(w, plan->src.view(), sh, *plan->sl, plan->next.view());
            } catch (...) {
                captured = false;
            }
            plan->regions = ctx.end_region_capture();
            const cudaError_t ce = cudaStreamEndCapture(ctx.stream(), &graph);
            cudaError_t ie = cudaErrorUnknown;
            if (captured && ce == cudaSuccess) ie = cudaGraphInstantiate(&plan->exec, graph, 0);
            if (graph) cudaGraphDestroy(graph);
            // the capture's host-side counts are re-added per replay
            plan->launches = ctx.launches() - l0;
            plan->applications = w.application_count() - a0;
            ctx.note_launch(-plan->launches);
            w.add_applications(-plan->applications);
            if (ie != cudaSuccess) {
                cudaGetLastError();  // clear a capture error; run eagerly from now on
                plan->exec = nullptr;
                plan->failed = true;
            }
        }
    }
    const bool graphed = plan && plan->exec;
    if (graphed) {
        copy(ctx, plan->src.view(), warm.panel());
        BLWS_CUDA(cudaGraphLaunch(plan->exec, ctx.stream()));
        ctx.note_launch(plan->launches);
        w.add_applications(plan->applications);
        ++g_blws_graph_launches;
        rec = plan->rec;
    } else {
        local = std::make_unique<Slots>(ctx, cap);
        sl = local.get();
        finite_slot = sl->take(2);
        w.defer_pending_check(reinterpret_cast<int*>(sl->at(finite_slot)));  // async-assigned W
        share_flag(ctx, reinterpret_cast<int*>(sl->at(finite_slot)), sl->at(finite_slot + 1));
        next = make_warm(ctx, m, pn, sh.want);
        rec = enqueue_deferred(w, warm.panel(), sh, *sl, next.panel());
    }
    sl->fetch(ctx);  // the one host round trip
    if (graphed) ctx.add_replayed_regions(plan->regions, plan->stamps.get());
    if (ctx.has_comm() ? sl->val(finite_slot + 1) != 0.0 : sl->as_int(finite_slot) != 0) {
        w.mark_poisoned();
        throw std::invalid_argument("DenseOperator: non-finite entries");
    }
    Index kept_short = -1;
    if (!finish_deferred(rec, *sl, sh, &kept_short)) {
        ++g_blws_deferred_fallbacks;
        if (kept_short < 0 || force_exact_pad()) return blws_svd_exact(w, warm, k, r, rng);
        // Only keep < r failed: every other test of the exact path passed on the
        // same values, so its result would be this call's kept leading columns
        // (the leading columns of a QR depend only on the leading input columns)
        // padded by adapt_subspace with the same Rng draws (block_lanczos.hpp:249-255).
        // Reusing them saves recomputing the whole call.
        DWarm part = make_warm(ctx, m, pn, kept_short);
        if (kept_short > 0) {
            copy(ctx, part.panel(), (graphed ? plan->next.view() : next.panel()).left(kept_short));
            const double* hv = sl->h.data() + rec.vslot;
            part.sigma.assign(hv, hv + kept_short);
        }
        BlwsResult out;
        out.k_raised = sh.k_raised;
        out.padded = true;
        out.warm = adapt_subspace(ctx, kept_short > 0 ? &part : nullptr, r, m, n, rng,
                                  w.row_sharded() ? &w.shard() : nullptr, w.col0(), w.col_sharded() ? pn : -1);
        return out;
    }
    if (graphed) {
        next = make_warm(ctx, m, pn, sh.want);
        copy(ctx, next.panel(), plan->next.view().left(sh.want));
    }
    BlwsResult out;
    out.k_raised = sh.k_raised;
    const double* hv = sl->h.data() + rec.vslot;
    next.sigma.assign(hv, hv + sh.want);
    out.warm = std::move(next);
    return out;
}

// ---- column-sharded warm starts: the public form holds V whole (n rows), the
// panel form this rank's rows [col0, col0 + chunk) (zero past n)
DWarm to_panel_warm(LinearOperator& w, const DWarm& a) {
    Context& ctx = w.ctx();
    const Index n = w.cols(), chunk = w.col_chunk(), c0 = w.col0();
    DWarm p = make_warm(ctx, a.geo.m, chunk, a.rank());
    if (a.rank() > 0) {
        copy(ctx, p.u(), a.u());
        const Index take = std::max<Index>(0, std::min(n, c0 + chunk) - c0);
        if (take > 0) copy(ctx, View{p.v().p, take, a.rank(), p.uv.ld}, View{a.v().p + c0, take, a.rank(), a.uv.ld});
    }
    p.sigma = a.sigma;
    return p;
}

DWarm to_api_warm(LinearOperator& w, const DWarm& p) {
    Context& ctx = w.ctx();
    const Index n = w.cols(), npad = w.col_chunk() * ctx.nranks();
    DWarm a = make_warm(ctx, p.geo.m, n, p.rank());
    if (p.rank() > 0) {
        copy(ctx, a.u(), p.u());
        DBuf<double> full(ctx, static_cast<size_t>(npad * p.rank()));
        gather_cols(w, p.v(), full.get());
        copy(ctx, a.v(), View{full.get(), n, p.rank(), npad});
    }
    a.sigma = p.sigma;
    return a;
}

BlwsResult blws_svd(LinearOperator& w, const DWarm& warm, Index k, Index r, Rng& rng) {
    if (!w.col_sharded()) return blws_svd_panel(w, warm, k, r, rng);
    if (warm.geo.m != w.rows() || warm.geo.n != w.cols())
        throw std::invalid_argument("blws_svd: warm start does not match operator");
    BlwsResult res = blws_svd_panel(w, to_panel_warm(w, warm), k, r, rng);
    res.warm = to_api_warm(w, res.warm);
    return res;
}

// ======================================================== Lanczos (reseed)
namespace {

/// LanczosRun (lanczos.hpp:85-183) on the augmented view. Steps run on the
/// device without host round trips; breakdown is latched on the device and
/// read back at the Ritz checkpoints.
class DeviceLanczos {
public:
    DeviceLanczos(LinearOperator& w, const std::vector<double>& q1_logical, Index cap)
        : w_(w), ctx_(w.ctx()), geo_{w.rows(), w.panel_n()},
          m_all_(w.row_sharded() ? w.shard().m_total : geo_.m), row0_(w.row_sharded() ? w.shard().row0 : 0),
          n_all_(w.cols()), col0_(w.col0()), dim_(m_all_ + n_all_), ld_(geo_.ld()), cap_(cap),
          split_(w.panel_split()) {
        q_ = DMat(ctx_, ld_, cap_, true);
        next_ = DMat(ctx_, ld_, 1, true);
        r_ = DMat(ctx_, ld_, 1, true);
        alpha_ = DBuf<double>(ctx_, static_cast<size_t>(cap_));
        lastbeta_ = DBuf<double>(ctx_, static_cast<size_t>(cap_));
        coup_ = DBuf<double>(ctx_, static_cast<size_t>(cap_ + 1));
        state_ = DBuf<double>(ctx_, 2);
        coef_ = DBuf<double>(ctx_, static_cast<size_t>(cap_));
        ss_ = DBuf<double>(ctx_, 1);
        zero(ctx_, coup_.get(), sizeof(double) * coup_.size());
        const double st[2] = {-1.0, 0.0};
        ctx_.write(state_.get(), st, 2);
        set_logical(next_.data(), q1_logical);
    }

    Index cols() const { return cols_; }
    bool breakdown() const { return breakdown_; }
    double residual_norm() const { return last_beta_; }
    View basis() const { return View{q_.data(), ld_, cols_, q_.ld}; }

    /// Launch steps until `target` columns; returns after syncing the state.
    void step_to(Index target) {
        if (cols_ < target && coop_steps(target)) {
            cols_ = target;
        } else {
            while (cols_ < target) {
                launch_step(cols_);
                ++cols_;
            }
        }
        sync_state();
    }

    /// restart (lanczos.hpp:144-160)
    bool restart(Rng& rng) {
        if (cols_ >= dim_) return false;
        for (int attempt = 0; attempt < 3; ++attempt) {
            std::vector<double> v = rng.gaussian_vector(dim_);
            double s = 0;
            for (double x : v) s += x * x;
            const double n0 = std::sqrt(s);
            for (auto& x : v) x /= n0;
            set_logical(r_.data(), v);
            reorth(r_.data());
            reorth(r_.data());
            panel_sumsq(ctx_, r_.view(), split_, ss_.get());
            double nv2 = 0;
            ctx_.read(ss_.get(), &nv2, 1);
            const double nv = std::sqrt(nv2);
            if (nv > 1e-8) {
                copy(ctx_, next_.view(), r_.view(), 1.0 / nv);
                const double zero = 0.0;
                ctx_.write(coup_.get() + cols_, &zero, 1);  // recorded coupling is zero
                const double st[1] = {-1.0};
                ctx_.write(state_.get(), st, 1);
                breakdown_ = false;
                return true;
            }
        }
        return false;
    }

    void read_tridiagonal(std::vector<double>& alpha, std::vector<double>& coup) {
        alpha.resize(static_cast<size_t>(cols_));
        coup.resize(static_cast<size_t>(std::max<Index>(cols_ - 1, 0)));
        ctx_.read(alpha_.get(), alpha.data(), cols_);
        if (cols_ > 1) ctx_.read(coup_.get() + 1, coup.data(), cols_ - 1);
    }
    const double* alpha_dev() const { return alpha_.get(); }
    const double* coup_dev() const { return coup_.get(); }

private:
    // a logical (m_all + n) vector into this rank's panel layout (its top rows,
    // its bottom rows: all of them, or [col0, col0 + chunk) when column-sharded)
    void set_logical(double* dst, const std::vector<double>& v) {
        std::vector<double> h(static_cast<size_t>(ld_), 0.0);
        std::copy(v.begin() + row0_, v.begin() + row0_ + geo_.m, h.begin());
        const Index b0 = std::min(n_all_, col0_), b1 = std::min(n_all_, col0_ + geo_.n);
        std::copy(v.begin() + m_all_ + b0, v.begin() + m_all_ + b1, h.begin() + geo_.mp());
        BLWS_CUDA(cudaMemcpyAsync(dst, h.data(), sizeof(double) * ld_, cudaMemcpyHostToDevice, ctx_.stream()));
        ctx_.sync();
    }

    // r -= Q (Q^T r) over the current basis
    void reorth(double* r) {
        if (cols_ == 0) return;
        panel_gemv_t(ctx_, ld_, cols_, q_.data(), q_.ld, r, split_, coef_.get());
        gemv(ctx_, false, ld_, cols_, -1.0, q_.data(), q_.ld, coef_.get(), 1.0, r);
    }

    // the whole step range in one cooperative launch (dense, unsharded, m <= 4096)
    bool coop_steps(Index target) {
        auto* dense = dynamic_cast<DenseOperator*>(&w_);
        if (!dense || split_.sharded || ctx_.has_comm() || std::getenv("BLWS_NO_COOP")) return false;
        const View wv = dense->w();
        double* ql = q_.data() + cols_ * q_.ld;
        BLWS_CUDA(cudaMemcpyAsync(ql, next_.data(), sizeof(double) * ld_, cudaMemcpyDeviceToDevice, ctx_.stream()));
        if (geo_.m > 4096) return false;  // large operators: the HBM-bound paired GEMV path
        static const bool cols_variant = [] {
            const char* e = std::getenv("BLWS_COOP");
            return e && std::string(e) == "cols";
        }();
        const bool ok =
            (!cols_variant && lanczos_rows_steps(ctx_, wv.p, wv.ld, geo_.m, geo_.n, geo_.mp(), q_.data(), q_.ld,
                                                 r_.data(), alpha_.get(), lastbeta_.get(), coup_.get(), state_.get(),
                                                 coef_.get(), cap_, dim_, cols_, target)) ||
            lanczos_coop_steps(ctx_, wv.p, wv.ld, geo_.m, geo_.n, geo_.mp(), q_.data(), q_.ld, r_.data(),
                               alpha_.get(), lastbeta_.get(), coup_.get(), state_.get(), coef_.get(), cap_, dim_,
                               cols_, target);
        if (!ok) return false;
        w_.add_applications(target - cols_);  // one paired apply per step (linear_operator.hpp:51-54)
        if (target < cap_)  // the last direction, for a later step_to / the restart logic
            BLWS_CUDA(cudaMemcpyAsync(next_.data(), q_.data() + target * q_.ld, sizeof(double) * ld_,
                                      cudaMemcpyDeviceToDevice, ctx_.stream()));
        return true;
    }

    void launch_step(Index l) {
        double* ql = q_.data() + l * q_.ld;
        BLWS_CUDA(cudaMemcpyAsync(ql, next_.data(), sizeof(double) * ld_, cudaMemcpyDeviceToDevice, ctx_.stream()));
        // r = A q_l: (W q_bot ; W^T q_top)
        w_.apply_pair(ql, ql + geo_.mp(), r_.data(), r_.data() + geo_.mp());
        panel_dot(ctx_, ld_, ql, r_.data(), split_, alpha_.get() + l);
        lanczos_three_term_k<<<gridn(ld_), kT, 0, ctx_.stream()>>>(r_.data(), q_.data(), q_.ld, l, alpha_.get(),
                                                                   coup_.get(), ld_);
        ctx_.note_launch();
        // full reorthogonalisation, twice (lanczos.hpp:123-126); basis includes column l
        const Index c = l + 1;
        for (int pass = 0; pass < 2; ++pass) {
            panel_gemv_t(ctx_, ld_, c, q_.data(), q_.ld, r_.data(), split_, coef_.get());
            gemv(ctx_, false, ld_, c, -1.0, q_.data(), q_.ld, coef_.get(), 1.0, r_.data());
        }
        panel_sumsq(ctx_, r_.view(), split_, ss_.get());
        lanczos_finalize_k<<<gridn(ld_), kT, 0, ctx_.stream()>>>(r_.data(), next_.data(), ld_, l, dim_, ss_.get(),
                                                                 alpha_.get(), lastbeta_.get(), coup_.get(), cap_,
                                                                 state_.get());
        ctx_.note_launch();
        ctx_.check_launch("lanczos step");
    }

    void sync_state() {
        double st[2];
        ctx_.read(state_.get(), st, 2);
        const Index first_broken = st[0] >= 0 ? static_cast<Index>(st[0]) : -1;
        if (first_broken >= 0 && first_broken + 1 < cols_) cols_ = first_broken + 1;
        breakdown_ = first_broken >= 0;
        if (cols_ > 0) ctx_.read(lastbeta_.get() + cols_ - 1, &last_beta_, 1);
    }

    LinearOperator& w_;
    Context& ctx_;
    Stack geo_;
    Index m_all_, row0_, n_all_, col0_, dim_, ld_, cap_;
    RowSplit split_;
    DMat q_, next_, r_;
    DBuf<double> alpha_, lastbeta_, coup_, state_, coef_, ss_;
    Index cols_ = 0;
    bool breakdown_ = false;
    double last_beta_ = 0;
};

struct Checkpoint {
    std::vector<double> values;  // top `want`, descending
    DMat vecs;                   // cols x want
    Index converged = 0;
};

// ritz_checkpoint (lanczos.hpp:191-207), top min(r, cols) pairs
Checkpoint ritz_checkpoint(Context& ctx, DeviceLanczos& run, Index r, double tol) {
    RegionGuard region(ctx, 4);
    Checkpoint cp;
    const Index k = run.cols();
    const Index want = std::min(r, k);
    DBuf<double> vals(ctx, static_cast<size_t>(want));
    cp.vecs = DMat(ctx, k, want, false);
    small_dense_guard(k, "sym_evd_tridiagonal: too large");
    tridiag_eig_top(ctx, k, run.alpha_dev(), run.coup_dev() + 1, want, vals.get(), cp.vecs.view());
    cp.values.resize(static_cast<size_t>(want));
    ctx.read(vals.get(), cp.values.data(), want);
    std::vector<double> last(static_cast<size_t>(want));
    BLWS_CUDA(cudaMemcpy2DAsync(last.data(), sizeof(double), cp.vecs.data() + (k - 1), sizeof(double) * cp.vecs.ld,
                                sizeof(double), want, cudaMemcpyDeviceToHost, ctx.stream()));
    ctx.sync();
    const double scale = std::fabs(cp.values[0]);
    const double limit = tol * scale;
    for (Index j = 0; j < want; ++j) {
        const double res = run.residual_norm() * std::fabs(last[static_cast<size_t>(j)]);
        if (res <= limit)
            ++cp.converged;
        else
            break;
    }
    return cp;
}

}  // namespace

// lanczos.hpp:209-252 (partial_evd_impl) + :289-329 (lanczos_partial_svd)
PartialSvd lanczos_partial_svd(LinearOperator& w, Index r, const LanczosOptions& opts) {
    Context& ctx = w.ctx();
    RegionGuard region(ctx, 3);
    const Index m = w.rows(), n = w.cols();
    const Index m_all = w.row_sharded() ? w.shard().m_total : m;  // a row shard: the global rows
    if (r < 1 || r > std::min(m_all, n)) throw std::invalid_argument("lanczos_partial_svd: bad r");
    const Index dim = m_all + n;
    Rng seed_rng = Rng(opts.seed).split(13);
    std::vector<double> top = seed_rng.unit_vector(m_all);
    std::vector<double> q1(static_cast<size_t>(dim), 0.0);
    std::copy(top.begin(), top.end(), q1.begin());

    Index max_k = opts.max_k > 0 ? std::min(opts.max_k, dim) : std::min(dim, 10 * r + 20);
    max_k = std::max(max_k, std::min(dim, r));
    DeviceLanczos run(w, q1, max_k);
    Rng rng = Rng(opts.seed).split(11);
    LanczosStats stats;
    Index k_target = std::min(max_k, std::max<Index>(2 * r, 10));
    static const bool lzdbg = std::getenv("BLWS_DEBUG_LZ") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t_begin = now();
    double t_steps = 0.0, t_cp = 0.0;
    Index n_cp = 0;
    while (true) {
        if (!run.breakdown() && run.cols() < k_target) {
            const auto t0 = now();
            const Index c0 = run.cols();
            run.step_to(k_target);
            const double dt = std::chrono::duration<double>(now() - t0).count();
            t_steps += dt;
            if (lzdbg)
                std::fprintf(stderr, "  lanczos r %lld: steps %lld -> %lld in %.2f ms (%.1f us/step)\n",
                             static_cast<long long>(r), static_cast<long long>(c0), static_cast<long long>(run.cols()),
                             1e3 * dt, 1e6 * dt / std::max<Index>(1, run.cols() - c0));
            continue;
        }
        const auto tc0 = now();
        Checkpoint cp = ritz_checkpoint(ctx, run, r, opts.tol);
        t_cp += std::chrono::duration<double>(now() - tc0).count();
        ++n_cp;
        bool done = cp.converged >= r || run.cols() >= max_k;
        if (!done) {
            if (run.breakdown()) {
                if (run.restart(rng))
                    ++stats.restarts;
                else
                    done = true;
            } else {
                k_target = std::min(max_k, 2 * k_target);
            }
        }
        if (done) {
            const Index avail = std::min(r, run.cols());
            Index keep = 0;
            while (keep < avail && cp.values[static_cast<size_t>(keep)] > 0.0) ++keep;
            PartialSvd out;
            const auto td0 = now();
            out.uv = make_warm(ctx, m, w.panel_n(), keep);
            if (lzdbg) {
                ctx.sync();
                std::fprintf(stderr, "  done: make_warm %.2f ms\n", 1e3 * std::chrono::duration<double>(now() - td0).count());
            }
            if (keep > 0) {
                View B = run.basis();
                const auto tg0 = now();
                gemm(ctx, false, false, B.rows, keep, B.cols, std::sqrt(2.0), B.p, B.ld, cp.vecs.data(), cp.vecs.ld,
                     0.0, out.uv.uv.data(), out.uv.uv.ld);
                if (lzdbg) {
                    ctx.sync();
                    std::fprintf(stderr, "  done: lift gemm %lld x %lld x %lld: %.2f ms\n", static_cast<long long>(B.rows),
                                 static_cast<long long>(keep), static_cast<long long>(B.cols),
                                 1e3 * std::chrono::duration<double>(now() - tg0).count());
                }
                std::copy(cp.values.begin(), cp.values.begin() + keep, out.uv.sigma.begin());
            }
            if (w.col_sharded()) out.uv = to_api_warm(w, out.uv);  // V whole for the caller
            if (lzdbg) {
                ctx.sync();
                std::fprintf(stderr, "lanczos r %lld: %lld steps, total %.2f ms: steps %.2f, %lld checkpoints %.2f ms\n",
                             static_cast<long long>(r), static_cast<long long>(run.cols()),
                             1e3 * std::chrono::duration<double>(now() - t_begin).count(), 1e3 * t_steps,
                             static_cast<long long>(n_cp), 1e3 * t_cp);
            }
            stats.steps = run.cols();
            stats.converged = std::min(cp.converged, avail);
            stats.all_converged = avail == r && cp.converged >= r;
            out.stats = stats;
            out.stats.converged = std::min(out.stats.converged, keep);
            out.stats.all_converged = stats.all_converged && keep == r;
            return out;
        }
    }
}

double spectral_norm(LinearOperator& w, double tol, std::uint64_t seed) {
    LanczosOptions o;
    o.tol = tol;
    o.seed = seed;
    auto svd = lanczos_partial_svd(w, 1, o);
    return svd.uv.rank() > 0 ? svd.uv.sigma[0] : 0.0;
}

}  // namespace blws
