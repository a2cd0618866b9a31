// TEST INFRASTRUCTURE ONLY — CPU oracle for the BLWS partial-SVT hot path.
//
// A line-by-line restatement of the reference algorithm in
// /root/reference/proj/include/blws (header-only C++20 over Eigen 3.4), written
// against oracle/la.hpp (OpenBLAS/LAPACK from numpy) because Eigen is absent
// from this image, so the reference itself cannot be compiled.
// Every function cites the reference file:line it restates. Control flow,
// constants and RNG consumption order follow the reference exactly; the dense
// kernels (Householder QR, symmetric EVD, GEMM) are the LAPACK/BLAS members of
// the same algorithm classes Eigen uses, so results agree with the reference
// to rounding, not bitwise.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
// --impl reference legs may load this code.
#pragma once
#include <algorithm>
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <random>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

#include "la.hpp"

namespace orc {

// ---------------------------------------------------------------- rng.hpp
/// Restates blws::Rng (core/rng.hpp:17-90): std::mt19937_64 plus the
/// hand-written 53-bit uniform, rejection index and Box–Muller with spare.
class Rng {
public:
    explicit Rng(std::uint64_t seed) : engine_(seed), seed_(seed) {}
    Rng split(std::uint64_t tag) const { return Rng(seed_ ^ (0x9e3779b97f4a7c15ull * (tag + 1))); }
    std::uint64_t next_u64() { return engine_(); }
    double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    std::uint64_t uniform_index(std::uint64_t n) {
        const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        std::uint64_t x;
        do {
            x = engine_();
        } while (x >= limit);
        return x % n;
    }
    double normal() {
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
    Mat gaussian_matrix(Index rows, Index cols) {
        Mat m(rows, cols);
        for (Index j = 0; j < cols; ++j)
            for (Index i = 0; i < rows; ++i) m(i, j) = normal();
        return m;
    }
    Vec gaussian_vector(Index n) {
        Vec v(static_cast<size_t>(n));
        for (Index i = 0; i < n; ++i) v[static_cast<size_t>(i)] = normal();
        return v;
    }
    Vec unit_vector(Index n) {
        Vec v = gaussian_vector(n);
        const double nv = vnorm(v);
        for (auto& x : v) x /= nv;
        return v;
    }

private:
    std::mt19937_64 engine_;
    std::uint64_t seed_ = 0;
    double spare_ = 0.0;
    bool have_spare_ = false;
};

// ------------------------------------------------------ linear_operator.hpp
/// Restates LinearOperator (core/linear_operator.hpp:20-98) with its
/// single-vector application counter (bump :94).
class LinearOperator {
public:
    virtual ~LinearOperator() = default;
    virtual Index rows() const = 0;
    virtual Index cols() const = 0;

    Vec apply(const Vec& x) const {
        bump(1);
        return apply_impl(x);
    }
    Vec apply_adjoint(const Vec& y) const {
        bump(1);
        return apply_adjoint_impl(y);
    }
    Mat apply_block(const Mat& x) const {
        bump(x.c);
        return apply_block_impl(x);
    }
    Mat apply_adjoint_block(const Mat& y) const {
        bump(y.c);
        return apply_adjoint_block_impl(y);
    }
    std::pair<Vec, Vec> apply_pair(const Vec& left, const Vec& right) const {
        bump(1);
        return {apply_impl(right), apply_adjoint_impl(left)};
    }
    std::pair<Mat, Mat> apply_pair_block(const Mat& left, const Mat& right) const {
        bump(right.c);
        return {apply_block_impl(right), apply_adjoint_block_impl(left)};
    }
    virtual Mat dense() const {
        Mat m(rows(), cols());
        Vec e(static_cast<size_t>(cols()), 0.0);
        for (Index j = 0; j < cols(); ++j) {
            e[static_cast<size_t>(j)] = 1.0;
            Vec c = apply(e);
            std::copy(c.begin(), c.end(), m.col(j));
            e[static_cast<size_t>(j)] = 0.0;
        }
        return m;
    }
    std::int64_t application_count() const { return count_; }

protected:
    virtual Vec apply_impl(const Vec& x) const = 0;
    virtual Vec apply_adjoint_impl(const Vec& y) const = 0;
    virtual Mat apply_block_impl(const Mat& x) const {
        Mat y(rows(), x.c);
        for (Index j = 0; j < x.c; ++j) {
            Vec c = apply_impl(Vec(x.col(j), x.col(j) + x.r));
            std::copy(c.begin(), c.end(), y.col(j));
        }
        return y;
    }
    virtual Mat apply_adjoint_block_impl(const Mat& y) const {
        Mat x(cols(), y.c);
        for (Index j = 0; j < y.c; ++j) {
            Vec c = apply_adjoint_impl(Vec(y.col(j), y.col(j) + y.r));
            std::copy(c.begin(), c.end(), x.col(j));
        }
        return x;
    }
    void bump(Index n) const { count_ += n; }

private:
    mutable std::int64_t count_ = 0;
};

/// DenseOperator (core/linear_operator.hpp:102-131): owned W, non-finite scan
/// on assign (:113-116), GEMM products (:124-127).
class DenseOperator final : public LinearOperator {
public:
    DenseOperator() = default;
    explicit DenseOperator(Mat m) : mat_(std::move(m)) {
        if (!all_finite(mat_)) throw std::invalid_argument("DenseOperator: non-finite entries");
    }
    void assign(Mat m) {
        if (!all_finite(m)) throw std::invalid_argument("DenseOperator: non-finite entries");
        mat_ = std::move(m);
    }
    Index rows() const override { return mat_.r; }
    Index cols() const override { return mat_.c; }
    const Mat& matrix() const { return mat_; }
    Mat dense() const override { return mat_; }

protected:
    Vec apply_impl(const Vec& x) const override {
        Vec y(static_cast<size_t>(mat_.r));
        gemm('N', 'N', mat_.r, 1, mat_.c, 1.0, mat_.data(), mat_.r, x.data(), mat_.c, 0.0, y.data(),
             mat_.r);
        return y;
    }
    Vec apply_adjoint_impl(const Vec& y) const override {
        Vec x(static_cast<size_t>(mat_.c));
        gemm('T', 'N', mat_.c, 1, mat_.r, 1.0, mat_.data(), mat_.r, y.data(), mat_.r, 0.0, x.data(),
             mat_.c);
        return x;
    }
    Mat apply_block_impl(const Mat& x) const override { return mul(mat_, x); }
    Mat apply_adjoint_block_impl(const Mat& y) const override { return mul(mat_, y, 'T', 'N'); }

private:
    Mat mat_;
};

/// Compressed sparse column matrix (Eigen::SparseMatrix default, types.hpp:18-20).
struct Csc {
    Index rows = 0, cols = 0;
    std::vector<std::int64_t> colptr;  // cols + 1
    std::vector<std::int32_t> rowidx;  // nnz, sorted within a column
    std::vector<double> val;
    Index nnz() const { return static_cast<Index>(val.size()); }
};

/// SparseOperator (core/linear_operator.hpp:136-169): assign_values in
/// compressed order (:149-153), SpMM products (:162-165).
class SparseOperator final : public LinearOperator {
public:
    explicit SparseOperator(Csc m) : mat_(std::move(m)) {
        if (!all_finite(mat_.val.data(), mat_.nnz()))
            throw std::invalid_argument("SparseOperator: non-finite entries");
    }
    void assign_values(const Vec& values) {
        if (static_cast<Index>(values.size()) != mat_.nnz())
            throw std::invalid_argument("SparseOperator: value count does not match pattern");
        mat_.val = values;
    }
    Index rows() const override { return mat_.rows; }
    Index cols() const override { return mat_.cols; }
    Index nnz() const { return mat_.nnz(); }
    const Csc& matrix() const { return mat_; }
    Mat dense() const override {
        Mat d(mat_.rows, mat_.cols);
        for (Index j = 0; j < mat_.cols; ++j)
            for (auto p = mat_.colptr[j]; p < mat_.colptr[j + 1]; ++p) d(mat_.rowidx[p], j) = mat_.val[p];
        return d;
    }

protected:
    Vec apply_impl(const Vec& x) const override {
        Mat X(mat_.cols, 1);
        std::copy(x.begin(), x.end(), X.col(0));
        Mat Y = apply_block_impl(X);
        return Vec(Y.col(0), Y.col(0) + Y.r);
    }
    Vec apply_adjoint_impl(const Vec& y) const override {
        Mat Y(mat_.rows, 1);
        std::copy(y.begin(), y.end(), Y.col(0));
        Mat X = apply_adjoint_block_impl(Y);
        return Vec(X.col(0), X.col(0) + X.r);
    }
    // Threaded over (column of x, row slab): each y(i, c) is accumulated by one
    // thread over j ascending, the serial order, so the result is bitwise the
    // same for any thread count.
    Mat apply_block_impl(const Mat& x) const override {
        Mat y(mat_.rows, x.c);
        const Index slabs = std::max<Index>(1, (4 * loop_threads() + x.c - 1) / std::max<Index>(x.c, 1));
        const Index rs = (mat_.rows + slabs - 1) / slabs;
        parallel_tasks(x.c * slabs, [&](Index t) {
            const Index c = t / slabs, r0 = (t % slabs) * rs, r1 = std::min(mat_.rows, r0 + rs);
            if (r0 >= r1) return;
            double* yc = y.col(c);
            for (Index j = 0; j < mat_.cols; ++j) {
                const double xj = x(j, c);
                const std::int32_t* b = mat_.rowidx.data() + mat_.colptr[j];
                const std::int32_t* e = mat_.rowidx.data() + mat_.colptr[j + 1];
                const std::int32_t* p0 = slabs == 1 ? b : std::lower_bound(b, e, static_cast<std::int32_t>(r0));
                for (const std::int32_t* p = p0; p < e && *p < r1; ++p)
                    yc[*p] += mat_.val[static_cast<size_t>(p - mat_.rowidx.data())] * xj;
            }
        });
        return y;
    }
    Mat apply_adjoint_block_impl(const Mat& y) const override {
        Mat x(mat_.cols, y.c);
        const Index chunks = 4 * loop_threads();
        const Index cs = (mat_.cols + chunks - 1) / chunks;
        parallel_tasks(y.c * chunks, [&](Index t) {
            const Index c = t / chunks, j0 = (t % chunks) * cs, j1 = std::min(mat_.cols, j0 + cs);
            for (Index j = j0; j < j1; ++j) {
                double s = 0;
                for (auto p = mat_.colptr[j]; p < mat_.colptr[j + 1]; ++p) s += mat_.val[p] * y(mat_.rowidx[p], c);
                x(j, c) = s;
            }
        });
        return x;
    }

private:
    Csc mat_;
};

/// AugmentedOperator (core/augmented_operator.hpp:18-63): [[0,W],[W^T,0]],
/// non-owning, one paired W application per augmented apply.
class AugmentedOperator final : public LinearOperator {
public:
    explicit AugmentedOperator(const LinearOperator& inner) : inner_(inner) {}
    Index rows() const override { return inner_.rows() + inner_.cols(); }
    Index cols() const override { return rows(); }
    Mat dense() const override {
        const Index m = inner_.rows(), n = inner_.cols();
        Mat w = inner_.dense();
        Mat out(m + n, m + n);
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < m; ++i) {
                out(i, m + j) = w(i, j);
                out(m + j, i) = w(i, j);
            }
        return out;
    }

protected:
    Vec apply_impl(const Vec& x) const override {
        const Index m = inner_.rows(), n = inner_.cols();
        Vec top(x.begin(), x.begin() + m), bot(x.begin() + m, x.end());
        auto [t, b] = inner_.apply_pair(top, bot);
        Vec out(static_cast<size_t>(m + n));
        std::copy(t.begin(), t.end(), out.begin());
        std::copy(b.begin(), b.end(), out.begin() + m);
        return out;
    }
    Vec apply_adjoint_impl(const Vec& x) const override { return apply_impl(x); }
    Mat apply_block_impl(const Mat& x) const override {
        const Index m = inner_.rows(), n = inner_.cols();
        auto [t, b] = inner_.apply_pair_block(x.top_rows(m), x.bottom_rows(n));
        Mat out(m + n, x.c);
        for (Index j = 0; j < x.c; ++j) {
            std::copy(t.col(j), t.col(j) + m, out.col(j));
            std::copy(b.col(j), b.col(j) + n, out.col(j) + m);
        }
        return out;
    }
    Mat apply_adjoint_block_impl(const Mat& x) const override { return apply_block_impl(x); }

private:
    const LinearOperator& inner_;
};

// ------------------------------------------------------------------ qr.hpp
struct ThinQr {
    Mat q, r;
    Index rank = 0;
};
ThinQr thin_qr(const Mat& m);  // core/qr.hpp:24-47

// ---------------------------------------------------------- small_dense.hpp
constexpr Index kSmallDenseLimit = 4096;  // small_dense.hpp:13
/// largest symmetric / tridiagonal EVD order met so far (see blws_oracle.cpp)
Index small_dense_max_order();
struct SymEvd {
    Mat vectors;
    Vec values;  // descending
};
SymEvd sym_evd_small(const Mat& t);                               // small_dense.hpp:24-43
SymEvd sym_evd_tridiagonal(const Vec& diag, const Vec& subdiag);  // small_dense.hpp:46-62
struct FullSvd {
    Mat u;
    Vec sigma;
    Mat v;
};
FullSvd full_svd_small(const Mat& m);  // small_dense.hpp:72-87 (ExactFull backend / tests)

// ---------------------------------------------------------------- trace
/// Parity trace (not in the reference): one record per partial-SVD call so
/// tests can compare block widths, keeps, flags and singular values call by
/// call against the device path.
struct TraceRecord {
    int kind = 0;  // 1 = blws_svd, 2 = lanczos reseed, 3 = spectral_norm
    Index b = 0, r = 0, k_eff = 0, keep = 0, steps = 0, restarts = 0, converged = 0;
    int flags = 0;  // bit0 padded, bit1 k_raised, bit2 terminated_early
    Vec sigma;
};
std::vector<TraceRecord>& trace();
bool& trace_enabled();

// ------------------------------------------------------------- lanczos.hpp
struct LanczosStats {
    Index steps = 0, restarts = 0, converged = 0;
    bool all_converged = false;
};
struct PartialEvd {
    Mat u;
    Vec values;
    LanczosStats stats;
};
struct PartialSvd {
    Mat u;
    Vec sigma;
    Mat v;
    LanczosStats stats;
};
struct LanczosOptions {
    double tol = 1e-8;
    Index max_k = 0;
    bool full_reorth = true;
    std::uint64_t seed = 0x1a2c705u;
};
PartialEvd lanczos_partial_evd(const LinearOperator& w, Index r, const LanczosOptions& o = {});
PartialSvd lanczos_partial_svd(const LinearOperator& w, Index r, const LanczosOptions& o = {},
                               const Vec* u1 = nullptr);
double spectral_norm(const LinearOperator& w, double tol = 1e-6, std::uint64_t seed = 0xb1f);
struct LanczosFactorization {
    Mat q;
    Vec alpha, beta;
    double residual_norm = 0;
    bool terminated_early = false;
};
LanczosFactorization lanczos_procedure(const LinearOperator& w, const Vec& q1, Index k,
                                       bool full_reorth = true);

// ------------------------------------------------------- block_lanczos.hpp
struct WarmStart {
    Mat u, v;
    Vec sigma;
    Index rank() const { return static_cast<Index>(sigma.size()); }
};
struct BlockLanczosFactorization {
    Mat q;
    std::vector<Mat> m, b;
    bool terminated_early = false;
    Mat embed() const;
};
BlockLanczosFactorization block_lanczos_procedure(const LinearOperator& w, const Mat& x1, Index k);
struct BlockEvd {
    Mat u;
    Vec values;
    Index available = 0;
    bool terminated_early = false;
};
BlockEvd bl_evd(const LinearOperator& w, const Mat& x1, Index k, Index r);
WarmStart adapt_subspace(const std::optional<WarmStart>& warm, Index r_new, Index m, Index n, Rng& rng);
struct BlwsResult {
    WarmStart warm;
    bool padded = false, k_raised = false, terminated_early = false;
};
BlwsResult blws_svd(const LinearOperator& w, const WarmStart& warm, Index k, Index r, Rng& rng);

// ------------------------------------------------------------------ svt.hpp
double shrink(double x, double eps);
struct RankPredictor {
    Index r = 10, increment = 5, max_rank = 1;
    std::vector<Index> history;
};
RankPredictor predict_rank(RankPredictor p, Index achieved, bool all_above);
struct SvdTriplets {
    Mat u;
    Vec sigma;
    Mat v;
    Index converged = 0;
    bool hit_cap = false;
};
class SvdBackend {
public:
    enum class Kind { ExactFull = 0, Lanczos = 1, Blws = 2 };
    struct Options {
        Index block_steps = 2;
        double ritz_tol = 1e-8;
        Index max_k = 0;
        Index seed_margin = 5;
        std::uint64_t seed = 0xb10c;
    };
    SvdBackend(Kind k, Options o) : kind_(k), opt_(o), rng_(o.seed) {}
    SvdTriplets compute(const LinearOperator& w, Index r);
    Kind kind() const { return kind_; }
    const std::optional<WarmStart>& warm_state() const { return warm_; }

private:
    Kind kind_;
    Options opt_;
    std::optional<WarmStart> warm_;
    Rng rng_;
    Index growth_streak_ = 0;
};
struct SvtResult {
    Mat u;
    Vec sigma;
    Mat v;
    Index achieved_rank = 0;
    bool all_above_threshold = false;
    Mat dense() const;
};
SvtResult svt(const LinearOperator& w, double eps, SvdBackend& backend, RankPredictor& predictor);

// -------------------------------------------------------------- solvers.hpp
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
    const Mat* truth = nullptr;
};
struct RpcaSolution {
    Mat a, e;  // e returned dense (reference: sparse from the nonzeros)
    std::int64_t e_nnz = 0;
    SolverStats stats;
};
RpcaSolution rpca_adm(const Mat& d, double lambda, SvdBackend& backend, const RpcaOptions& o = {});
struct McOptions {
    double tol_outer = 1e-4;
    Index max_iter = 500;
    Index initial_rank = 10, rank_increment = 5;
    const Mat* truth_ml = nullptr;
    const Mat* truth_mr = nullptr;
};
struct McSolution {
    Mat u;
    Vec sigma;
    Mat v;
    SolverStats stats;
};
McSolution mc_svt(const Csc& observed, double tau, double delta, SvdBackend& backend,
                  const McOptions& o = {});

// --------------------------------------------------------------- synth.hpp
std::vector<std::int64_t> sample_distinct(std::int64_t n, std::int64_t s, Rng& rng);

}  // namespace orc
