// blws/blws.hpp — header-only C++ shim with the reference's API names over the
// C ABI of libblws_cuda.so (include/blws_cuda.h).
//
// Drop-in for the hot-path entry points of /root/reference/proj/include/blws:
//   blws::Rng                    core/rng.hpp:17-90
//   blws::DenseOperator          core/linear_operator.hpp:102-131
//   blws::SparseOperator         core/linear_operator.hpp:136-169
//   blws::WarmStart, blws_svd    block_lanczos.hpp:45-52, :204-261
//   blws::adapt_subspace         block_lanczos.hpp:157-187
//   blws::lanczos_partial_svd    lanczos.hpp:289-329
//   blws::spectral_norm          lanczos.hpp:332-340
//   blws::SvdBackend, RankPredictor, svt   svt.hpp:48-254
//   blws::rpca_adm, mc_svt       solvers.hpp:72-157, :202-270
// Matrices are plain column-major std::vector<double> (the reference uses
// Eigen, which this build does not depend on). Status codes map back to the
// reference's exceptions: 1 -> std::invalid_argument, 2 -> std::runtime_error,
// 3/4 (CUDA/NCCL) -> std::runtime_error with the library message.
#ifndef BLWS_BLWS_HPP
#define BLWS_BLWS_HPP

#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../blws_cuda.h"

namespace blws {

using Index = std::int64_t;

inline void check(int rc) {
    if (rc == BLWS_OK) return;
    const std::string msg = blws_last_error();
    if (rc == BLWS_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

/// Column-major dense matrix (the reference's DenseMatrix<double>).
struct Matrix {
    Index rows = 0, cols = 0;
    std::vector<double> data;
    Matrix() = default;
    Matrix(Index r, Index c) : rows(r), cols(c), data(static_cast<size_t>(r * c), 0.0) {}
    double& operator()(Index i, Index j) { return data[static_cast<size_t>(i + j * rows)]; }
    double operator()(Index i, Index j) const { return data[static_cast<size_t>(i + j * rows)]; }
};

/// Compressed sparse column matrix (the reference's SparseMatrix<double>,
/// Eigen's default column-major storage): colptr (cols + 1), row indices
/// sorted within a column, values in the same order.
struct SparseMatrix {
    Index rows = 0, cols = 0;
    std::vector<std::int64_t> colptr;
    std::vector<std::int32_t> rowidx;
    std::vector<double> values;
    Index nonZeros() const { return static_cast<Index>(values.size()); }
};

/// One device context per solve.
class Context {
public:
    explicit Context(int device = 0) {
        blws_context* c = nullptr;
        check(blws_context_create(device, &c));
        h_.reset(c);
    }
    blws_context* get() const { return h_.get(); }
    void synchronize() { check(blws_context_synchronize(h_.get())); }

private:
    struct Del {
        void operator()(blws_context* c) const { blws_context_destroy(c); }
    };
    std::unique_ptr<blws_context, Del> h_;
};

/// The process-wide context on device 0 that the reference-shaped overloads
/// (no Context argument) use; created on first use and never destroyed (its
/// teardown would race the CUDA runtime's own at process exit).
inline Context& default_context() {
    static Context* ctx = new Context(0);
    return *ctx;
}

class Rng {
public:
    explicit Rng(std::uint64_t seed) {
        blws_rng* r = nullptr;
        check(blws_rng_create(seed, &r));
        h_.reset(r);
    }
    Rng split(std::uint64_t tag) const {
        blws_rng* r = nullptr;
        check(blws_rng_split(h_.get(), tag, &r));
        return Rng(r);
    }
    std::uint64_t next_u64() { return blws_rng_next_u64(h_.get()); }
    double uniform(double lo = 0.0, double hi = 1.0) { return blws_rng_uniform(h_.get(), lo, hi); }
    std::uint64_t uniform_index(std::uint64_t n) { return blws_rng_uniform_index(h_.get(), n); }
    double normal() { return blws_rng_normal(h_.get()); }
    Matrix gaussian_matrix(Index rows, Index cols) {
        Matrix m(rows, cols);
        check(blws_rng_gaussian_matrix(h_.get(), rows, cols, m.data.data()));
        return m;
    }
    blws_rng* get() const { return h_.get(); }

private:
    explicit Rng(blws_rng* r) { h_.reset(r); }
    struct Del {
        void operator()(blws_rng* r) const { blws_rng_destroy(r); }
    };
    std::unique_ptr<blws_rng, Del> h_;
};

class LinearOperator {
public:
    Index rows() const { return blws_operator_rows(h_.get()); }
    Index cols() const { return blws_operator_cols(h_.get()); }
    std::int64_t application_count() const { return blws_operator_application_count(h_.get()); }
    blws_operator* get() const { return h_.get(); }
    Context& context() const { return *ctx_; }

protected:
    explicit LinearOperator(Context& ctx) : ctx_(&ctx) {}
    struct Del {
        void operator()(blws_operator* o) const { blws_operator_destroy(o); }
    };
    std::unique_ptr<blws_operator, Del> h_;
    Context* ctx_;
};

class DenseOperator : public LinearOperator {
public:
    /// DenseOperator(W) (linear_operator.hpp:109) on the default context
    explicit DenseOperator(const Matrix& w) : DenseOperator(default_context(), w) {}
    DenseOperator(Context& ctx, const Matrix& w) : LinearOperator(ctx) {
        blws_operator* o = nullptr;
        check(blws_dense_operator_create(ctx.get(), w.rows, w.cols, w.data.data(), w.rows, BLWS_HOST, 0, &o));
        h_.reset(o);
    }
    /// Borrow a device-resident column-major W (ld even, 16-byte aligned).
    DenseOperator(Context& ctx, Index m, Index n, const double* dev_w, Index ld) : LinearOperator(ctx) {
        blws_operator* o = nullptr;
        check(blws_dense_operator_create(ctx.get(), m, n, dev_w, ld, BLWS_DEVICE, 1, &o));
        h_.reset(o);
    }
    void assign(const Matrix& w) { check(blws_dense_operator_assign(h_.get(), w.data.data(), w.rows, BLWS_HOST)); }
};

class SparseOperator : public LinearOperator {
public:
    /// SparseOperator(S) (linear_operator.hpp:141) on the default context
    explicit SparseOperator(const SparseMatrix& s) : SparseOperator(default_context(), s) {}
    SparseOperator(Context& ctx, const SparseMatrix& s)
        : SparseOperator(ctx, s.rows, s.cols, s.colptr, s.rowidx, s.values) {}
    SparseOperator(Context& ctx, Index m, Index n, const std::vector<std::int64_t>& colptr,
                   const std::vector<std::int32_t>& rowidx, const std::vector<double>& values)
        : LinearOperator(ctx), nnz_(static_cast<Index>(values.size())) {
        blws_operator* o = nullptr;
        check(blws_sparse_operator_create(ctx.get(), m, n, nnz_, colptr.data(), rowidx.data(), values.data(), &o));
        h_.reset(o);
    }
    void assign_values(const std::vector<double>& v) {
        check(blws_sparse_operator_assign_values(h_.get(), v.data(), static_cast<Index>(v.size()), BLWS_HOST));
    }
    Index nnz() const { return nnz_; }

private:
    Index nnz_;
};

/// Host copy of a warm start (U m x r, V n x r, sigma r).
struct WarmStart {
    Matrix u, v;
    std::vector<double> sigma;
    Index rank() const { return static_cast<Index>(sigma.size()); }
};

namespace detail {
struct WarmDel {
    void operator()(blws_warm_start* w) const { blws_warm_start_destroy(w); }
};
using WarmPtr = std::unique_ptr<blws_warm_start, WarmDel>;

inline WarmPtr upload(Context& ctx, const WarmStart& w) {
    blws_warm_start* h = nullptr;
    check(blws_warm_start_create(ctx.get(), w.u.rows, w.v.rows, w.rank(), w.u.data.data(), w.u.rows,
                                 w.v.data.data(), w.v.rows, w.sigma.data(), BLWS_HOST, &h));
    return WarmPtr(h);
}
inline WarmStart download(blws_warm_start* h, Index m, Index n) {
    WarmStart w;
    const Index r = blws_warm_start_rank(h);
    w.u = Matrix(m, r);
    w.v = Matrix(n, r);
    w.sigma.assign(static_cast<size_t>(r), 0.0);
    check(blws_warm_start_get(h, w.u.data.data(), m, w.v.data.data(), n, w.sigma.data(), BLWS_HOST));
    return w;
}
}  // namespace detail

struct BlwsResult {
    WarmStart warm;
    bool padded = false, k_raised = false, terminated_early = false;
};

/// blws_svd (block_lanczos.hpp:204-261)
inline BlwsResult blws_svd(const LinearOperator& w, const WarmStart& warm, Index k, Index r, Rng& rng) {
    auto in = detail::upload(w.context(), warm);
    blws_warm_start* out = nullptr;
    int flags = 0;
    check(::blws_svd(w.get(), in.get(), k, r, rng.get(), &out, &flags));
    detail::WarmPtr keep(out);
    BlwsResult res;
    res.warm = detail::download(out, w.rows(), w.cols());
    res.padded = flags & 1;
    res.k_raised = flags & 2;
    res.terminated_early = flags & 4;
    return res;
}

/// adapt_subspace (block_lanczos.hpp:157-187)
inline WarmStart adapt_subspace(Context& ctx, const std::optional<WarmStart>& warm, Index r_new, Index m, Index n,
                                Rng& rng) {
    detail::WarmPtr in;
    if (warm && warm->rank() > 0) in = detail::upload(ctx, *warm);
    blws_warm_start* out = nullptr;
    check(blws_adapt_subspace(ctx.get(), in.get(), r_new, m, n, rng.get(), &out));
    detail::WarmPtr keep(out);
    return detail::download(out, m, n);
}

/// spectral_norm (lanczos.hpp:332-340)
inline double spectral_norm(const LinearOperator& w, double tol = 1e-6, std::uint64_t seed = 0xb1f) {
    double s = 0;
    check(blws_spectral_norm(w.get(), tol, seed, &s));
    return s;
}

struct RankPredictor {
    Index r = 10, increment = 5, max_rank = 1;
    std::vector<Index> history;
};

class SvdBackend {
public:
    enum class Kind { ExactFull = BLWS_BACKEND_EXACT_FULL, Lanczos = BLWS_BACKEND_LANCZOS, Blws = BLWS_BACKEND_BLWS };
    struct Options {
        Index block_steps = 2;
        double ritz_tol = 1e-8;
        Index max_k = 0;
        Index seed_margin = 5;
        std::uint64_t seed = 0xb10c;
    };
    // svt.hpp:96-98: the reference's factories, on the default context
    static SvdBackend exact_full() { return SvdBackend(default_context(), Kind::ExactFull, Options()); }
    static SvdBackend lanczos(Options o) { return SvdBackend(default_context(), Kind::Lanczos, o); }
    static SvdBackend lanczos() { return SvdBackend(default_context(), Kind::Lanczos, Options()); }
    static SvdBackend blws(Options o) { return SvdBackend(default_context(), Kind::Blws, o); }
    static SvdBackend blws() { return SvdBackend(default_context(), Kind::Blws, Options()); }
    // the same on an explicit context (one context per solve)
    static SvdBackend exact_full(Context& ctx) { return SvdBackend(ctx, Kind::ExactFull, Options()); }
    static SvdBackend blws(Context& ctx, Options o) { return SvdBackend(ctx, Kind::Blws, o); }
    static SvdBackend blws(Context& ctx) { return SvdBackend(ctx, Kind::Blws, Options()); }
    static SvdBackend lanczos(Context& ctx, Options o) { return SvdBackend(ctx, Kind::Lanczos, o); }
    static SvdBackend lanczos(Context& ctx) { return SvdBackend(ctx, Kind::Lanczos, Options()); }
    blws_svd_backend* get() const { return h_.get(); }
    Context& context() const { return *ctx_; }

private:
    SvdBackend(Context& ctx, Kind k, Options o) : ctx_(&ctx) {
        blws_svd_backend* b = nullptr;
        check(blws_svd_backend_create(ctx.get(), static_cast<int>(k), o.block_steps, o.ritz_tol, o.max_k,
                                      o.seed_margin, o.seed, &b));
        h_.reset(b);
    }
    struct Del {
        void operator()(blws_svd_backend* b) const { blws_svd_backend_destroy(b); }
    };
    std::unique_ptr<blws_svd_backend, Del> h_;
    Context* ctx_;
};

struct SvtResult {
    Matrix u, v;
    std::vector<double> sigma;  // shrunk values of the retained triplets
    Index achieved_rank = 0;
    bool all_above_threshold = false;
};

/// svt (svt.hpp:216-254)
inline SvtResult svt(const LinearOperator& w, double eps, SvdBackend& backend, RankPredictor& predictor) {
    blws_rank_predictor p{predictor.r, predictor.increment, predictor.max_rank};
    std::int64_t hist = 0, hl = 0, ach = 0;
    int above = 0;
    blws_warm_start* out = nullptr;
    check(blws_svt(w.get(), eps, backend.get(), &p, &hist, 1, &hl, &out, &ach, &above));
    detail::WarmPtr keep(out);
    predictor.r = p.r;
    if (hl) predictor.history.push_back(hist);
    SvtResult res;
    WarmStart t = detail::download(out, w.rows(), w.cols());
    res.u = std::move(t.u);
    res.v = std::move(t.v);
    res.sigma = std::move(t.sigma);
    res.achieved_rank = ach;
    res.all_above_threshold = above != 0;
    return res;
}

struct SolverStats {
    Index iterations = 0;
    double wall_time_s = 0;
    std::int64_t matvec_count = 0, matvec_init = 0;
    double rel_err = -1;
    Index rank_hat = 0;
    std::int64_t e_l0 = -1;
    bool converged = false;
    std::vector<Index> predicted_ranks;
    std::vector<std::int64_t> matvec_history;
    std::vector<double> residual_history;
};

struct RpcaOptions {
    double tol_outer = 1e-7;
    Index max_iter = 1000;
    double rho = 1.5;
    double mu_max_factor = 1e7;
    Index initial_rank = 10, rank_increment = 5;
    const Matrix* truth = nullptr;
};

/// RpcaProblem (solvers.hpp:17-26)
struct RpcaProblem {
    Matrix d;           ///< square observation, low rank + sparse
    double lambda = 0;  ///< sparsity weight; <= 0 selects 1/sqrt(m)
    double effective_lambda() const { return lambda > 0 ? lambda : 1.0 / std::sqrt(static_cast<double>(d.rows)); }
};

/// RpcaSolution (solvers.hpp:49-54): A dense, E sparse (the nonzeros of the
/// final shrink, column-major order, as solvers.hpp:133-146)
struct RpcaSolution {
    Matrix a;
    SparseMatrix e;
    SolverStats stats;
};

namespace detail {
inline SolverStats stats(const blws_solver_stats& s, const std::vector<std::int64_t>& pr,
                         const std::vector<std::int64_t>& mh, const std::vector<double>& rh) {
    SolverStats o;
    o.iterations = s.iterations;
    o.wall_time_s = s.wall_time_s;
    o.matvec_count = s.matvec_count;
    o.matvec_init = s.matvec_init;
    o.rel_err = s.rel_err;
    o.rank_hat = s.rank_hat;
    o.e_l0 = s.e_l0;
    o.converged = s.converged != 0;
    o.predicted_ranks.assign(pr.begin(), pr.begin() + s.iterations);
    o.matvec_history.assign(mh.begin(), mh.begin() + s.iterations);
    o.residual_history.assign(rh.begin(), rh.begin() + s.iterations);
    return o;
}

/// the nonzeros of a dense column-major m x n matrix as CSC (solvers.hpp:133-146)
inline SparseMatrix sparse_from_dense(const std::vector<double>& e, Index m, Index n) {
    SparseMatrix s;
    s.rows = m;
    s.cols = n;
    s.colptr.assign(static_cast<size_t>(n + 1), 0);
    for (Index j = 0; j < n; ++j) {
        for (Index i = 0; i < m; ++i) {
            const double v = e[static_cast<size_t>(i + j * m)];
            if (v != 0.0) {
                s.rowidx.push_back(static_cast<std::int32_t>(i));
                s.values.push_back(v);
            }
        }
        s.colptr[static_cast<size_t>(j + 1)] = static_cast<std::int64_t>(s.values.size());
    }
    return s;
}
}  // namespace detail

/// rpca_adm (solvers.hpp:72-157) as the reference declares it; the solve runs
/// on the backend's context
inline RpcaSolution rpca_adm(const RpcaProblem& problem, SvdBackend& backend, const RpcaOptions& opts = {}) {
    const Matrix& d = problem.d;
    const Index m = d.rows;
    if (d.rows != d.cols) throw std::invalid_argument("rpca_adm: D must be square");
    blws_rpca_options o{opts.tol_outer, opts.max_iter, opts.rho, opts.mu_max_factor, opts.initial_rank,
                        opts.rank_increment};
    RpcaSolution sol;
    sol.a = Matrix(m, m);
    std::vector<double> e(static_cast<size_t>(m * m));
    blws_solver_stats st{};
    std::vector<std::int64_t> pr(static_cast<size_t>(opts.max_iter + 1)), mh(pr.size());
    std::vector<double> rh(pr.size());
    check(blws_rpca_adm(backend.context().get(), m, d.data.data(), m, BLWS_HOST, problem.lambda, backend.get(), &o,
                        opts.truth ? opts.truth->data.data() : nullptr, sol.a.data.data(), e.data(), &st, pr.data(),
                        mh.data(), rh.data(), static_cast<std::int64_t>(pr.size())));
    sol.e = detail::sparse_from_dense(e, m, m);
    sol.stats = detail::stats(st, pr, mh, rh);
    return sol;
}

/// the same with D and lambda given directly
inline RpcaSolution rpca_adm(const Matrix& d, double lambda, SvdBackend& backend, const RpcaOptions& opts = {}) {
    return rpca_adm(RpcaProblem{d, lambda}, backend, opts);
}

struct McOptions {
    double tol_outer = 1e-4;
    Index max_iter = 500;
    Index initial_rank = 10, rank_increment = 5;
    const Matrix* truth_ml = nullptr;
    const Matrix* truth_mr = nullptr;
};

struct McSolution {
    Matrix u, v;
    std::vector<double> sigma;
    SolverStats stats;
};

/// McProblem (solvers.hpp:28-33)
struct McProblem {
    SparseMatrix observed;  ///< observed entries of A on the support
    double tau = 0;         ///< threshold; <= 0 selects 5 m
    double delta = 0;       ///< step size; <= 0 selects 1.2 m^2 / s
};

/// mc_svt (solvers.hpp:202-270); observation as CSC; tau/delta <= 0 select the defaults
inline McSolution mc_svt(Context& ctx, Index m, Index n, const std::vector<std::int64_t>& colptr,
                         const std::vector<std::int32_t>& rowidx, const std::vector<double>& values, double tau,
                         double delta, SvdBackend& backend, const McOptions& opts = {}) {
    blws_mc_options o{opts.tol_outer, opts.max_iter, opts.initial_rank, opts.rank_increment};
    const Index cap = std::min(m, n);
    McSolution sol;
    sol.u = Matrix(m, cap);
    sol.v = Matrix(n, cap);
    sol.sigma.assign(static_cast<size_t>(cap), 0.0);
    blws_solver_stats st{};
    std::vector<std::int64_t> pr(static_cast<size_t>(opts.max_iter + 1)), mh(pr.size());
    std::vector<double> rh(pr.size());
    std::int64_t rank = 0;
    const Index rt = opts.truth_ml ? opts.truth_ml->cols : 0;
    check(blws_mc_svt(ctx.get(), m, n, static_cast<Index>(values.size()), colptr.data(), rowidx.data(),
                      values.data(), tau, delta, backend.get(), &o, opts.truth_ml ? opts.truth_ml->data.data() : nullptr,
                      opts.truth_mr ? opts.truth_mr->data.data() : nullptr, rt, sol.u.data.data(), sol.sigma.data(),
                      sol.v.data.data(), cap, &rank, &st, pr.data(), mh.data(), rh.data(),
                      static_cast<std::int64_t>(pr.size())));
    sol.u.cols = rank;
    sol.u.data.resize(static_cast<size_t>(m * rank));
    sol.v.cols = rank;
    sol.v.data.resize(static_cast<size_t>(n * rank));
    sol.sigma.resize(static_cast<size_t>(rank));
    sol.stats = detail::stats(st, pr, mh, rh);
    return sol;
}

/// mc_svt (solvers.hpp:202-270) as the reference declares it
inline McSolution mc_svt(const McProblem& problem, SvdBackend& backend, const McOptions& opts = {}) {
    const SparseMatrix& s = problem.observed;
    return mc_svt(backend.context(), s.rows, s.cols, s.colptr, s.rowidx, s.values, problem.tau, problem.delta,
                  backend, opts);
}

}  // namespace blws

#endif  // BLWS_BLWS_HPP
