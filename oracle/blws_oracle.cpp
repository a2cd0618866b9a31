// TEST INFRASTRUCTURE ONLY — CPU oracle implementation (see blws_oracle.hpp).
#include <cstdlib>
#include "blws_oracle.hpp"

#include <chrono>
#include <sstream>

namespace orc {

std::vector<TraceRecord>& trace() {
    static std::vector<TraceRecord> t;
    return t;
}
bool& trace_enabled() {
    static bool on = false;
    return on;
}
static void push_trace(TraceRecord rec) {
    if (trace_enabled()) trace().push_back(std::move(rec));
}

// ------------------------------------------------------------------ qr.hpp
// core/qr.hpp:24-47. Householder (LAPACK dgeqrf + dorgqr, the algorithm class
// of Eigen::HouseholderQR), diag(R) >= 0 normalisation (:39-43), rank counted
// against tau = 1e-12 ||M||_F (:33, :44).
ThinQr thin_qr(const Mat& m_in) {
    const Index rows = m_in.r, cols = m_in.c;
    if (rows == 0 || cols == 0) throw std::invalid_argument("thin_qr: empty matrix");
    if (rows < cols) throw std::invalid_argument("thin_qr: requires rows >= cols");
    if (!all_finite(m_in)) throw std::invalid_argument("thin_qr: non-finite entries");
    const double tau = 1e-12 * fro(m_in);

    Mat a = m_in;
    Vec tauv(static_cast<size_t>(cols));
    Index info = 0, lwork = -1;
    double wq = 0;
    scipy_dgeqrf_64_(&rows, &cols, a.data(), &rows, tauv.data(), &wq, &lwork, &info);
    lwork = std::max<Index>(1, static_cast<Index>(wq));
    Vec work(static_cast<size_t>(lwork));
    scipy_dgeqrf_64_(&rows, &cols, a.data(), &rows, tauv.data(), work.data(), &lwork, &info);
    if (info != 0) throw std::runtime_error("thin_qr: dgeqrf failed");
    ThinQr out;
    out.r = Mat(cols, cols);
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i <= j; ++i) out.r(i, j) = a(i, j);
    lwork = -1;
    scipy_dorgqr_64_(&rows, &cols, &cols, a.data(), &rows, tauv.data(), &wq, &lwork, &info);
    lwork = std::max<Index>(1, static_cast<Index>(wq));
    work.assign(static_cast<size_t>(lwork), 0.0);
    scipy_dorgqr_64_(&rows, &cols, &cols, a.data(), &rows, tauv.data(), work.data(), &lwork, &info);
    if (info != 0) throw std::runtime_error("thin_qr: dorgqr failed");
    out.q = std::move(a);
    for (Index j = 0; j < cols; ++j) {
        if (out.r(j, j) < 0.0) {
            for (Index c = 0; c < cols; ++c) out.r(j, c) = -out.r(j, c);
            for (Index i = 0; i < rows; ++i) out.q(i, j) = -out.q(i, j);
        }
        if (out.r(j, j) > tau) ++out.rank;
    }
    return out;
}

// ---------------------------------------------------------- small_dense.hpp
// kSmallDenseLimit (small_dense.hpp:13) is the reference's guard; with
// ORC_LIFT_SMALL_DENSE_LIMIT=1 the oracle runs past it (the device path has no
// such limit: DESIGN.md §3) and records the largest order it met.
static Index g_small_dense_max = 0;
static bool small_dense_limit_lifted() {
    static const bool lifted = [] {
        const char* e = std::getenv("ORC_LIFT_SMALL_DENSE_LIMIT");
        return e && e[0] == '1';
    }();
    return lifted;
}
static void small_dense_guard(Index n, const char* what) {
    g_small_dense_max = std::max(g_small_dense_max, n);
    if (n > kSmallDenseLimit && !small_dense_limit_lifted()) throw std::invalid_argument(what);
}
Index small_dense_max_order() { return g_small_dense_max; }

// small_dense.hpp:24-43: checks, symmetrise, EVD, descending order.
SymEvd sym_evd_small(const Mat& t_in) {
    if (t_in.r != t_in.c) throw std::invalid_argument("sym_evd_small: not square");
    small_dense_guard(t_in.r, "sym_evd_small: too large");
    if (!all_finite(t_in)) throw std::invalid_argument("sym_evd_small: non-finite entries");
    const Index n = t_in.r;
    const double nrm = fro(t_in);
    double asym = 0;
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
            const double d = t_in(i, j) - t_in(j, i);
            asym += d * d;
        }
    if (std::sqrt(asym) > 1e-10 * nrm && nrm > 0.0)
        throw std::invalid_argument("sym_evd_small: input is not symmetric");
    Mat t(n, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) t(i, j) = 0.5 * (t_in(i, j) + t_in(j, i));
    Vec w(static_cast<size_t>(n));
    Index info = 0, lwork = -1, liwork = -1, iwq = 0;
    double wq = 0;
    const char jobz = 'V', uplo = 'L';
    scipy_dsyevd_64_(&jobz, &uplo, &n, t.data(), &n, w.data(), &wq, &lwork, &iwq, &liwork, &info, 1, 1);
    lwork = std::max<Index>(1, static_cast<Index>(wq));
    liwork = std::max<Index>(1, iwq);
    Vec work(static_cast<size_t>(lwork));
    std::vector<Index> iwork(static_cast<size_t>(liwork));
    scipy_dsyevd_64_(&jobz, &uplo, &n, t.data(), &n, w.data(), work.data(), &lwork, iwork.data(),
                     &liwork, &info, 1, 1);
    if (info != 0) throw std::runtime_error("sym_evd_small: failed to converge");
    SymEvd out;
    out.values.resize(static_cast<size_t>(n));
    out.vectors = Mat(n, n);
    for (Index j = 0; j < n; ++j) {
        out.values[static_cast<size_t>(j)] = w[static_cast<size_t>(n - 1 - j)];
        std::copy(t.col(n - 1 - j), t.col(n - 1 - j) + n, out.vectors.col(j));
    }
    return out;
}

// small_dense.hpp:46-62 (computeFromTridiagonal -> LAPACK dsteqr 'I').
SymEvd sym_evd_tridiagonal(const Vec& diag, const Vec& subdiag) {
    if (diag.empty()) throw std::invalid_argument("sym_evd_tridiagonal: empty");
    if (subdiag.size() + 1 != diag.size()) throw std::invalid_argument("sym_evd_tridiagonal: size mismatch");
    const Index n = static_cast<Index>(diag.size());
    small_dense_guard(n, "sym_evd_tridiagonal: too large");
    Vec d = diag, e = subdiag;
    e.push_back(0.0);
    Mat z(n, n);
    Vec work(static_cast<size_t>(std::max<Index>(1, 2 * n - 2)));
    Index info = 0;
    const char compz = 'I';
    scipy_dsteqr_64_(&compz, &n, d.data(), e.data(), z.data(), &n, work.data(), &info, 1);
    if (info != 0) throw std::runtime_error("sym_evd_tridiagonal: failed to converge");
    SymEvd out;
    out.values.resize(static_cast<size_t>(n));
    out.vectors = Mat(n, n);
    for (Index j = 0; j < n; ++j) {
        out.values[static_cast<size_t>(j)] = d[static_cast<size_t>(n - 1 - j)];
        std::copy(z.col(n - 1 - j), z.col(n - 1 - j) + n, out.vectors.col(j));
    }
    return out;
}

// small_dense.hpp:72-87 (BDCSVD -> LAPACK dgesdd). ExactFull backend only.
FullSvd full_svd_small(const Mat& m_in) {
    if (m_in.r == 0 || m_in.c == 0) throw std::invalid_argument("full_svd_small: empty");
    if (std::min(m_in.r, m_in.c) > kSmallDenseLimit) throw std::invalid_argument("full_svd_small: too large");
    if (!all_finite(m_in)) throw std::invalid_argument("full_svd_small: non-finite entries");
    const Index m = m_in.r, n = m_in.c, p = std::min(m, n);
    Mat a = m_in;
    FullSvd out;
    out.sigma.resize(static_cast<size_t>(p));
    out.u = Mat(m, p);
    Mat vt(p, n);
    Index info = 0, lwork = -1;
    double wq = 0;
    std::vector<Index> iwork(static_cast<size_t>(8 * p));
    const char jobz = 'S';
    scipy_dgesdd_64_(&jobz, &m, &n, a.data(), &m, out.sigma.data(), out.u.data(), &m, vt.data(), &p,
                     &wq, &lwork, iwork.data(), &info, 1);
    lwork = std::max<Index>(1, static_cast<Index>(wq));
    Vec work(static_cast<size_t>(lwork));
    scipy_dgesdd_64_(&jobz, &m, &n, a.data(), &m, out.sigma.data(), out.u.data(), &m, vt.data(), &p,
                     work.data(), &lwork, iwork.data(), &info, 1);
    if (info != 0) throw std::runtime_error("full_svd_small: dgesdd failed");
    out.v = vt.transpose();
    return out;
}

// ------------------------------------------------------------- lanczos.hpp
namespace {

/// lanczos.hpp:85-183 LanczosRun: incremental three-term recurrence with
/// full double classical Gram-Schmidt and deflation restarts.
class LanczosRun {
public:
    LanczosRun(const LinearOperator& w, const Vec& q1, bool full)
        : w_(w), full_(full), dim_(w.rows()) {
        if (w.rows() != w.cols()) throw std::invalid_argument("lanczos: operator not square");
        if (static_cast<Index>(q1.size()) != dim_) throw std::invalid_argument("lanczos: bad start vector size");
        if (std::abs(vnorm(q1) - 1.0) > 1e-12) throw std::invalid_argument("lanczos: start vector is not unit");
        next_dir_ = q1;
    }
    Index cols() const { return cols_; }
    bool breakdown() const { return breakdown_; }
    double residual_norm() const { return last_beta_; }
    const std::vector<double>& alpha() const { return alpha_; }
    const std::vector<double>& beta() const { return beta_; }
    Mat basis() const {
        Mat b(dim_, cols_);
        std::copy(q_.begin(), q_.begin() + dim_ * cols_, b.data());
        return b;
    }

    // lanczos.hpp:112-138
    void step() {
        const Index l = cols_;
        q_.insert(q_.end(), next_dir_.begin(), next_dir_.end());
        if (l > 0) beta_.push_back(next_coupling_);
        cols_ = l + 1;
        const double* ql = q_.data() + l * dim_;
        Vec ql_v(ql, ql + dim_);
        Vec r = w_.apply(ql_v);
        const double alpha = dot(ql, r.data(), dim_);
        for (Index i = 0; i < dim_; ++i) r[i] -= alpha * ql[i];
        if (l > 0) {
            const double* qp = q_.data() + (l - 1) * dim_;
            const double bl = beta_.back();
            for (Index i = 0; i < dim_; ++i) r[i] -= bl * qp[i];
        }
        if (full_) {
            reorth(r);
            reorth(r);
        }
        alpha_.push_back(alpha);
        if (alpha_.size() == 1) tau_ = 1e-12 * std::abs(alpha);
        last_beta_ = vnorm(r);
        if (last_beta_ <= tau_ || cols_ >= dim_) {
            breakdown_ = true;
        } else {
            breakdown_ = false;
            next_dir_.resize(static_cast<size_t>(dim_));
            for (Index i = 0; i < dim_; ++i) next_dir_[i] = r[i] / last_beta_;
            next_coupling_ = last_beta_;
        }
    }

    // lanczos.hpp:144-160
    bool restart(Rng& rng) {
        if (cols_ >= dim_) return false;
        for (int attempt = 0; attempt < 3; ++attempt) {
            Vec v = rng.gaussian_vector(dim_);
            const double n0 = vnorm(v);
            for (auto& x : v) x /= n0;
            reorth(v);
            reorth(v);
            const double nv = vnorm(v);
            if (nv > 1e-8) {
                for (auto& x : v) x /= nv;
                next_dir_ = v;
                next_coupling_ = 0.0;
                breakdown_ = false;
                return true;
            }
        }
        return false;
    }

private:
    // r -= B (B^T r) over the current basis (lanczos.hpp:124-125, :149-150)
    void reorth(Vec& r) const {
        Vec c(static_cast<size_t>(cols_));
        gemm('T', 'N', cols_, 1, dim_, 1.0, q_.data(), dim_, r.data(), dim_, 0.0, c.data(), cols_);
        gemm('N', 'N', dim_, 1, cols_, -1.0, q_.data(), dim_, c.data(), cols_, 1.0, r.data(), dim_);
    }

    const LinearOperator& w_;
    bool full_;
    Index dim_;
    std::vector<double> q_;
    Index cols_ = 0;
    std::vector<double> alpha_, beta_;
    Vec next_dir_;
    double next_coupling_ = 0, last_beta_ = 0, tau_ = 0;
    bool breakdown_ = false;
};

struct RitzCheckpoint {
    SymEvd evd;
    Index converged = 0;
};

// lanczos.hpp:191-207
RitzCheckpoint ritz_checkpoint(const LanczosRun& run, double tol) {
    RitzCheckpoint cp;
    cp.evd = sym_evd_tridiagonal(run.alpha(), run.beta());
    const Index k = run.cols();
    const double scale = std::abs(cp.evd.values[0]);
    const double limit = tol * scale;
    for (Index j = 0; j < k; ++j) {
        const double res = run.residual_norm() * std::abs(cp.evd.vectors(k - 1, j));
        if (res <= limit)
            ++cp.converged;
        else
            break;
    }
    return cp;
}

// lanczos.hpp:209-252
PartialEvd partial_evd_impl(const LinearOperator& w, Index r, const LanczosOptions& opts, const Vec& q1) {
    const Index m = w.rows();
    if (r < 1 || r > m) throw std::invalid_argument("lanczos_partial_evd: bad r");
    Index max_k = opts.max_k > 0 ? std::min(opts.max_k, m) : std::min(m, 10 * r + 20);
    max_k = std::max(max_k, std::min(m, r));
    LanczosRun run(w, q1, opts.full_reorth);
    Rng rng = Rng(opts.seed).split(11);
    LanczosStats stats;
    Index k_target = std::min(max_k, std::max<Index>(2 * r, 10));
    while (true) {
        if (!run.breakdown() && run.cols() < k_target) {
            run.step();
            continue;
        }
        auto cp = ritz_checkpoint(run, opts.tol);
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
            PartialEvd out;
            out.values.assign(cp.evd.values.begin(), cp.evd.values.begin() + avail);
            out.u = mul(run.basis(), cp.evd.vectors.left_cols(avail));
            stats.steps = run.cols();
            stats.converged = std::min(cp.converged, avail);
            stats.all_converged = avail == r && cp.converged >= r;
            out.stats = stats;
            return out;
        }
    }
}

}  // namespace

// lanczos.hpp:259-272
LanczosFactorization lanczos_procedure(const LinearOperator& w, const Vec& q1, Index k, bool full) {
    if (k < 1) throw std::invalid_argument("lanczos_procedure: k must be >= 1");
    LanczosRun run(w, q1, full);
    while (run.cols() < k && !run.breakdown()) run.step();
    LanczosFactorization out;
    out.q = run.basis();
    out.alpha = run.alpha();
    out.beta = run.beta();
    out.residual_norm = run.residual_norm();
    out.terminated_early = run.cols() < k;
    return out;
}

// lanczos.hpp:277-283
PartialEvd lanczos_partial_evd(const LinearOperator& w, Index r, const LanczosOptions& opts) {
    Rng rng = Rng(opts.seed).split(7);
    Vec q1 = rng.unit_vector(w.rows());
    return partial_evd_impl(w, r, opts, q1);
}

// lanczos.hpp:289-329
PartialSvd lanczos_partial_svd(const LinearOperator& w, Index r, const LanczosOptions& opts, const Vec* u1) {
    const Index m = w.rows(), n = w.cols();
    if (r < 1 || r > std::min(m, n)) throw std::invalid_argument("lanczos_partial_svd: bad r");
    Vec top;
    if (u1) {
        if (static_cast<Index>(u1->size()) != m) throw std::invalid_argument("lanczos_partial_svd: bad seed size");
        const double nu = vnorm(*u1);
        if (!(nu > 0.0)) throw std::invalid_argument("lanczos_partial_svd: zero seed");
        top = *u1;
        for (auto& x : top) x /= nu;
    } else {
        Rng rng = Rng(opts.seed).split(13);
        top = rng.unit_vector(m);
    }
    Vec q1(static_cast<size_t>(m + n), 0.0);
    std::copy(top.begin(), top.end(), q1.begin());
    AugmentedOperator aug(w);
    PartialEvd evd = partial_evd_impl(aug, r, opts, q1);
    Index keep = 0;
    while (keep < static_cast<Index>(evd.values.size()) && evd.values[keep] > 0.0) ++keep;
    PartialSvd out;
    out.sigma.assign(evd.values.begin(), evd.values.begin() + keep);
    out.u = Mat(m, keep);
    out.v = Mat(n, keep);
    const double root2 = std::sqrt(2.0);
    for (Index j = 0; j < keep; ++j) {
        for (Index i = 0; i < m; ++i) out.u(i, j) = root2 * evd.u(i, j);
        for (Index i = 0; i < n; ++i) out.v(i, j) = root2 * evd.u(m + i, j);
    }
    out.stats = evd.stats;
    out.stats.converged = std::min(out.stats.converged, keep);
    out.stats.all_converged = evd.stats.all_converged && keep == r;
    return out;
}

// lanczos.hpp:332-340
double spectral_norm(const LinearOperator& w, double tol, std::uint64_t seed) {
    LanczosOptions opts;
    opts.tol = tol;
    opts.seed = seed;
    auto svd = lanczos_partial_svd(w, 1, opts);
    TraceRecord rec;
    rec.kind = 3;
    rec.r = 1;
    rec.steps = svd.stats.steps;
    rec.converged = svd.stats.converged;
    rec.sigma = svd.sigma;
    push_trace(rec);
    return svd.sigma.empty() ? 0.0 : svd.sigma[0];
}

// ------------------------------------------------------- block_lanczos.hpp
// block_lanczos.hpp:28-40
Mat BlockLanczosFactorization::embed() const {
    const Index bs = m.empty() ? 0 : m.front().r;
    const Index d = static_cast<Index>(m.size()) * bs;
    Mat t(d, d);
    for (size_t l = 0; l < m.size(); ++l) {
        const Index off = static_cast<Index>(l) * bs;
        for (Index j = 0; j < bs; ++j)
            for (Index i = 0; i < bs; ++i) t(off + i, off + j) = m[l](i, j);
        if (l + 1 < m.size()) {
            for (Index j = 0; j < bs; ++j)
                for (Index i = 0; i < bs; ++i) {
                    t(off + bs + i, off + j) = b[l](i, j);
                    t(off + j, off + bs + i) = b[l](i, j);
                }
        }
    }
    return t;
}

static Mat sym_half(const Mat& a) {
    Mat s(a.r, a.c);
    for (Index j = 0; j < a.c; ++j)
        for (Index i = 0; i < a.r; ++i) s(i, j) = 0.5 * (a(i, j) + a(j, i));
    return s;
}

constexpr double kBlockBreakdownTol = 1e-10;  // block_lanczos.hpp:64

// block_lanczos.hpp:70-126
BlockLanczosFactorization block_lanczos_procedure(const LinearOperator& w, const Mat& x1, Index k) {
    const Index m = w.rows(), bs = x1.c;
    if (w.rows() != w.cols()) throw std::invalid_argument("block_lanczos_procedure: operator not square");
    if (k < 1) throw std::invalid_argument("block_lanczos_procedure: k must be >= 1");
    if (bs < 1 || x1.r != m) throw std::invalid_argument("block_lanczos_procedure: bad initial block");
    if (k * bs > m) throw std::invalid_argument("block_lanczos_procedure: k*b exceeds dimension");
    {
        Mat g = mul(x1, x1, 'T', 'N');
        for (Index i = 0; i < bs; ++i) g(i, i) -= 1.0;
        if (fro(g) > 1e-8) throw std::invalid_argument("block_lanczos_procedure: X1 not orthonormal");
    }
    BlockLanczosFactorization out;
    out.q = Mat(m, k * bs);
    std::copy(x1.a.begin(), x1.a.end(), out.q.a.begin());
    Mat x_cur = x1, x_prev;
    Mat z = w.apply_block(x_cur);
    double scale = fro(z);
    out.m.push_back(sym_half(mul(x_cur, z, 'T', 'N')));
    Index built = 1;
    for (Index l = 1; l < k; ++l) {
        Mat r = z;
        gemm('N', 'N', m, bs, bs, -1.0, x_cur.data(), m, out.m.back().data(), bs, 1.0, r.data(), m);
        if (l > 1) gemm('N', 'T', m, bs, bs, -1.0, x_prev.data(), m, out.b.back().data(), bs, 1.0, r.data(), m);
        if (fro(r) <= kBlockBreakdownTol * scale) {
            out.terminated_early = true;
            break;
        }
        auto qr = thin_qr(r);
        if (qr.rank < bs) {
            out.terminated_early = true;
            break;
        }
        x_prev = x_cur;
        x_cur = qr.q;
        out.b.push_back(qr.r);
        std::copy(x_cur.a.begin(), x_cur.a.end(), out.q.a.begin() + l * bs * m);
        ++built;
        z = w.apply_block(x_cur);
        scale = std::max(scale, fro(z));
        out.m.push_back(sym_half(mul(x_cur, z, 'T', 'N')));
    }
    out.q = out.q.left_cols(built * bs);
    return out;
}

// block_lanczos.hpp:139-152
BlockEvd bl_evd(const LinearOperator& w, const Mat& x1, Index k, Index r) {
    if (r < 1 || r > k * x1.c) throw std::invalid_argument("bl_evd: bad r");
    auto fac = block_lanczos_procedure(w, x1, k);
    auto evd = sym_evd_small(fac.embed());
    const Index dim = static_cast<Index>(fac.m.size()) * x1.c;
    const Index avail = std::min(r, dim);
    BlockEvd out;
    out.values.assign(evd.values.begin(), evd.values.begin() + avail);
    out.u = mul(fac.q, evd.vectors.left_cols(avail));
    out.available = avail;
    out.terminated_early = fac.terminated_early;
    return out;
}

// block_lanczos.hpp:157-187
WarmStart adapt_subspace(const std::optional<WarmStart>& warm, Index r_new, Index m, Index n, Rng& rng) {
    if (r_new < 1 || r_new > std::min(m, n)) throw std::invalid_argument("adapt_subspace: r_new out of range");
    WarmStart out;
    if (!warm || warm->rank() == 0) {
        out.u = thin_qr(rng.gaussian_matrix(m, r_new)).q;
        out.v = thin_qr(rng.gaussian_matrix(n, r_new)).q;
        out.sigma.assign(static_cast<size_t>(r_new), 0.0);
        return out;
    }
    const Index r_old = warm->rank();
    if (r_new == r_old) return *warm;
    if (r_new < r_old) {
        out.u = warm->u.left_cols(r_new);
        out.v = warm->v.left_cols(r_new);
        out.sigma.assign(warm->sigma.begin(), warm->sigma.begin() + r_new);
        return out;
    }
    const Index add = r_new - r_old;
    Mat ue(m, r_new), ve(n, r_new);
    std::copy(warm->u.a.begin(), warm->u.a.end(), ue.a.begin());
    Mat gu = rng.gaussian_matrix(m, add);
    std::copy(gu.a.begin(), gu.a.end(), ue.a.begin() + m * r_old);
    std::copy(warm->v.a.begin(), warm->v.a.end(), ve.a.begin());
    Mat gv = rng.gaussian_matrix(n, add);
    std::copy(gv.a.begin(), gv.a.end(), ve.a.begin() + n * r_old);
    out.u = thin_qr(ue).q;
    out.v = thin_qr(ve).q;
    out.sigma.assign(static_cast<size_t>(r_new), 0.0);
    std::copy(warm->sigma.begin(), warm->sigma.end(), out.sigma.begin());
    return out;
}

// block_lanczos.hpp:204-261
BlwsResult blws_svd(const LinearOperator& w, const WarmStart& warm, Index k, Index r, Rng& rng) {
    const Index m = w.rows(), n = w.cols();
    const Index bs = warm.rank();
    if (bs < 1) throw std::invalid_argument("blws_svd: empty warm start (seed via adapt_subspace)");
    if (r < 1 || r > std::min(m, n)) throw std::invalid_argument("blws_svd: bad r");
    if (warm.u.r != m || warm.v.r != n || warm.u.c != bs || warm.v.c != bs)
        throw std::invalid_argument("blws_svd: warm start does not match operator");
    BlwsResult out;
    Index k_eff = k;
    if (r > k_eff * bs) {
        k_eff = (r + bs - 1) / bs;
        out.k_raised = true;
    }
    k_eff = std::min(k_eff, (m + n) / bs);
    k_eff = std::max<Index>(k_eff, 1);

    const double inv_root2 = 1.0 / std::sqrt(2.0);
    Mat stacked(m + n, bs);
    for (Index j = 0; j < bs; ++j) {
        for (Index i = 0; i < m; ++i) stacked(i, j) = inv_root2 * warm.u(i, j);
        for (Index i = 0; i < n; ++i) stacked(m + i, j) = inv_root2 * warm.v(i, j);
    }
    Mat x1 = thin_qr(stacked).q;
    AugmentedOperator aug(w);
    auto evd = bl_evd(aug, x1, k_eff, k_eff * bs);
    out.terminated_early = evd.terminated_early;

    const double positive_floor = !evd.values.empty() ? 1e-12 * std::abs(evd.values[0]) : 0.0;
    Index keep = 0;
    while (keep < static_cast<Index>(evd.values.size()) && keep < r && evd.values[keep] > positive_floor) ++keep;

    const double root2 = std::sqrt(2.0);
    WarmStart next;
    next.sigma.assign(evd.values.begin(), evd.values.begin() + keep);
    next.u = Mat(m, keep);
    next.v = Mat(n, keep);
    for (Index j = 0; j < keep; ++j) {
        for (Index i = 0; i < m; ++i) next.u(i, j) = root2 * evd.u(i, j);
        for (Index i = 0; i < n; ++i) next.v(i, j) = root2 * evd.u(m + i, j);
    }
    if (keep > 0) {
        next.u = thin_qr(next.u).q;
        next.v = thin_qr(next.v).q;
    }
    if (keep < r) {
        std::optional<WarmStart> partial;
        if (keep > 0) partial = next;
        next = adapt_subspace(partial, r, m, n, rng);
        out.padded = true;
    }
    out.warm = std::move(next);
    TraceRecord rec;
    rec.kind = 1;
    rec.b = bs;
    rec.r = r;
    rec.k_eff = k_eff;
    rec.keep = keep;
    rec.flags = (out.padded ? 1 : 0) | (out.k_raised ? 2 : 0) | (out.terminated_early ? 4 : 0);
    rec.sigma = out.warm.sigma;
    push_trace(rec);
    return out;
}

// ------------------------------------------------------------------ svt.hpp
// svt.hpp:20-26
double shrink(double x, double eps) {
    if (eps < 0.0) throw std::invalid_argument("shrink: negative threshold");
    if (x > eps) return x - eps;
    if (x < -eps) return x + eps;
    return 0.0;
}

// svt.hpp:58-64
RankPredictor predict_rank(RankPredictor p, Index achieved, bool all_above) {
    Index next = achieved + (all_above ? p.increment : 1);
    p.r = std::clamp<Index>(next, 1, p.max_rank);
    p.history.push_back(p.r);
    return p;
}

// svt.hpp:104-186
SvdTriplets SvdBackend::compute(const LinearOperator& w, Index r) {
    const Index p = std::min(w.rows(), w.cols());
    if (r < 1 || r > p) throw std::invalid_argument("SvdBackend: bad r");
    switch (kind_) {
        case Kind::ExactFull: {
            auto svd = full_svd_small(w.dense());
            SvdTriplets t;
            t.u = svd.u.left_cols(r);
            t.sigma.assign(svd.sigma.begin(), svd.sigma.begin() + r);
            t.v = svd.v.left_cols(r);
            t.converged = r;
            return t;
        }
        case Kind::Lanczos: {
            LanczosOptions lo;
            lo.tol = opt_.ritz_tol;
            lo.max_k = opt_.max_k;
            lo.seed = rng_.next_u64();
            auto svd = lanczos_partial_svd(w, r, lo);
            TraceRecord rec;
            rec.kind = 2;
            rec.r = r;
            rec.steps = svd.stats.steps;
            rec.restarts = svd.stats.restarts;
            rec.converged = svd.stats.converged;
            rec.sigma = svd.sigma;
            push_trace(rec);
            SvdTriplets t;
            t.u = std::move(svd.u);
            t.sigma = std::move(svd.sigma);
            t.v = std::move(svd.v);
            t.converged = svd.stats.converged;
            t.hit_cap = !svd.stats.all_converged;
            return t;
        }
        case Kind::Blws: {
            const Index held = warm_ ? warm_->rank() : 0;
            if (held < r) {
                const Index margin = opt_.seed_margin * (Index(1) << std::min<Index>(growth_streak_, 5));
                ++growth_streak_;
                const Index r_seed = std::min(p, r + margin);
                LanczosOptions lo;
                lo.tol = opt_.ritz_tol;
                lo.max_k = opt_.max_k;
                lo.seed = rng_.next_u64();
                auto svd = lanczos_partial_svd(w, r_seed, lo);
                TraceRecord rec;
                rec.kind = 2;
                rec.r = r_seed;
                rec.steps = svd.stats.steps;
                rec.restarts = svd.stats.restarts;
                rec.converged = svd.stats.converged;
                rec.sigma = svd.sigma;
                push_trace(rec);
                WarmStart ws;
                ws.u = std::move(svd.u);
                ws.sigma = std::move(svd.sigma);
                ws.v = std::move(svd.v);
                if (ws.rank() < r_seed) {
                    std::optional<WarmStart> partial;
                    if (ws.rank() > 0) partial = ws;
                    ws = adapt_subspace(partial, r_seed, w.rows(), w.cols(), rng_);
                }
                warm_ = std::move(ws);
                SvdTriplets t;
                t.u = warm_->u;
                t.sigma = warm_->sigma;
                t.v = warm_->v;
                t.converged = svd.stats.converged;
                t.hit_cap = !svd.stats.all_converged;
                return t;
            }
            if (r < held) growth_streak_ = 0;
            if (held > r + 2 * opt_.seed_margin)
                warm_ = adapt_subspace(warm_, r + opt_.seed_margin, w.rows(), w.cols(), rng_);
            auto res = blws_svd(w, *warm_, opt_.block_steps, warm_->rank(), rng_);
            warm_ = res.warm;
            SvdTriplets t;
            t.u = warm_->u;
            t.sigma = warm_->sigma;
            t.v = warm_->v;
            t.converged = res.padded ? std::min(r, res.warm.rank()) : warm_->rank();
            return t;
        }
    }
    throw std::logic_error("SvdBackend: unreachable");
}

Mat SvtResult::dense() const {
    Mat us = u;
    for (Index j = 0; j < us.c; ++j)
        for (Index i = 0; i < us.r; ++i) us(i, j) *= sigma[j];
    return mul(us, v, 'N', 'T');
}

// svt.hpp:216-254
SvtResult svt(const LinearOperator& w, double eps, SvdBackend& backend, RankPredictor& predictor) {
    if (eps < 0.0) throw std::invalid_argument("svt: negative threshold");
    const Index p = std::min(w.rows(), w.cols());
    Index r = std::clamp<Index>(predictor.r, 1, p);
    SvdTriplets t;
    bool all_above = false;
    while (true) {
        t = backend.compute(w, r);
        const Index have = static_cast<Index>(t.sigma.size());
        const bool smallest_above = have > 0 && t.sigma[have - 1] > eps;
        if (!smallest_above || std::max(r, have) >= p) {
            all_above = smallest_above;
            break;
        }
        r = std::min<Index>(std::max(r, have) + predictor.increment, p);
    }
    if (t.hit_cap && t.converged == 0 && !t.sigma.empty() && t.sigma[0] > eps) {
        std::ostringstream msg;
        msg << "svt: partial SVD backend hit its step cap with no converged triplet (requested " << r
            << " of " << p << ")";
        throw std::runtime_error(msg.str());
    }
    Index achieved = 0;
    while (achieved < static_cast<Index>(t.sigma.size()) && t.sigma[achieved] > eps) ++achieved;
    SvtResult out;
    out.u = t.u.left_cols(achieved);
    out.v = t.v.left_cols(achieved);
    out.sigma.resize(static_cast<size_t>(achieved));
    for (Index j = 0; j < achieved; ++j) out.sigma[j] = t.sigma[j] - eps;
    out.achieved_rank = achieved;
    out.all_above_threshold = all_above;
    predictor = predict_rank(predictor, achieved, all_above);
    return out;
}

// -------------------------------------------------------------- solvers.hpp
// solvers.hpp:72-157
RpcaSolution rpca_adm(const Mat& d, double lambda_in, SvdBackend& backend, const RpcaOptions& opts) {
    const auto t0 = std::chrono::steady_clock::now();
    const Index m = d.r;
    if (d.r != d.c) throw std::invalid_argument("rpca_adm: D must be square");
    if (!all_finite(d)) throw std::invalid_argument("rpca_adm: D has non-finite entries");
    const double lambda = lambda_in > 0.0 ? lambda_in : 1.0 / std::sqrt(static_cast<double>(m));
    const double norm_d_fro = fro(d);
    RpcaSolution sol;
    if (norm_d_fro == 0.0) {
        sol.a = Mat(m, m);
        sol.e = Mat(m, m);
        sol.stats.converged = true;
        sol.stats.e_l0 = 0;
        return sol;
    }
    DenseOperator op(d);
    const double norm2_d = spectral_norm(op);
    double mu = 1.25 / norm2_d;
    const double mu_max = mu * opts.mu_max_factor;
    double dmax = 0;
    for (double x : d.a) dmax = std::max(dmax, std::abs(x));
    const double dual_scale = std::max(norm2_d, dmax / lambda);
    const Index mm = m * m;
    Mat y(m, m), e(m, m), a(m, m);
    for (Index i = 0; i < mm; ++i) y.a[i] = d.a[i] / dual_scale;

    RankPredictor predictor;
    predictor.r = opts.initial_rank;
    predictor.increment = opts.rank_increment;
    predictor.max_rank = m;
    SolverStats& stats = sol.stats;
    stats.matvec_init = op.application_count();
    std::int64_t mark = stats.matvec_init;
    Index last_rank = 0;
    Mat w(m, m), resid(m, m);
    for (Index it = 1; it <= opts.max_iter; ++it) {
        for (Index i = 0; i < mm; ++i) w.a[i] = d.a[i] - e.a[i] + y.a[i] / mu;
        op.assign(w);
        auto prox = svt(op, 1.0 / mu, backend, predictor);
        a = prox.dense();
        last_rank = prox.achieved_rank;
        const double thr = lambda / mu;
        for (Index i = 0; i < mm; ++i) e.a[i] = shrink(d.a[i] - a.a[i] + y.a[i] / mu, thr);
        for (Index i = 0; i < mm; ++i) resid.a[i] = d.a[i] - a.a[i] - e.a[i];
        for (Index i = 0; i < mm; ++i) y.a[i] += mu * resid.a[i];
        mu = std::min(opts.rho * mu, mu_max);
        stats.matvec_history.push_back(op.application_count() - mark);
        mark = op.application_count();
        const double feas = fro(resid) / norm_d_fro;
        stats.residual_history.push_back(feas);
        stats.iterations = it;
        if (feas <= opts.tol_outer) {
            stats.converged = true;
            break;
        }
    }
    sol.a = a;
    const double e_tol = 1e-8 * dmax;
    std::int64_t e_l0 = 0, nnz = 0;
    for (Index i = 0; i < mm; ++i) {
        if (e.a[i] != 0.0) ++nnz;
        if (std::abs(e.a[i]) > e_tol) ++e_l0;
    }
    sol.e = std::move(e);
    sol.e_nnz = nnz;
    stats.rank_hat = last_rank;
    stats.e_l0 = e_l0;
    stats.matvec_count = op.application_count();
    stats.predicted_ranks = predictor.history;
    if (opts.truth) {
        Mat diff = a;
        for (Index i = 0; i < mm; ++i) diff.a[i] -= opts.truth->a[i];
        stats.rel_err = fro(diff) / fro(*opts.truth);
    }
    stats.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return sol;
}

// solvers.hpp:181-196
static Vec project_low_rank(const Csc& pattern, const Mat& u, const Vec& s, const Mat& v) {
    Vec out(static_cast<size_t>(pattern.nnz()), 0.0);
    if (u.c == 0) return out;
    Mat us = u;
    for (Index j = 0; j < us.c; ++j)
        for (Index i = 0; i < us.r; ++i) us(i, j) *= s[j];
    const Index chunks = 4 * loop_threads();
    const Index cs = (pattern.cols + chunks - 1) / chunks;
    parallel_tasks(chunks, [&](Index t) {
        for (Index k = t * cs; k < std::min(pattern.cols, (t + 1) * cs); ++k)
            for (auto p = pattern.colptr[k]; p < pattern.colptr[k + 1]; ++p) {
                const Index row = pattern.rowidx[p];
                double acc = 0;
                for (Index c = 0; c < us.c; ++c) acc += us(row, c) * v(k, c);
                out[static_cast<size_t>(p)] = acc;
            }
    });
    return out;
}

// solvers.hpp:202-270
McSolution mc_svt(const Csc& pd, double tau_in, double delta_in, SvdBackend& backend, const McOptions& opts) {
    const auto t0 = std::chrono::steady_clock::now();
    const Index m = pd.rows, n = pd.cols;
    const std::int64_t s = pd.nnz();
    if (s == 0) throw std::invalid_argument("mc_svt: empty observation set");
    if (!all_finite(pd.val.data(), s)) throw std::invalid_argument("mc_svt: non-finite observations");
    const double tau = tau_in > 0.0 ? tau_in : 5.0 * static_cast<double>(m);
    const double delta = delta_in > 0.0 ? delta_in
                                        : 1.2 * static_cast<double>(m) * static_cast<double>(n) / static_cast<double>(s);
    SparseOperator op(pd);
    const double norm2_pd = spectral_norm(op);
    const double k0 = std::ceil(tau / (delta * norm2_pd));
    const Vec& obs = pd.val;
    const double obs_norm = vnorm(obs);
    Vec y(static_cast<size_t>(s));
    for (std::int64_t i = 0; i < s; ++i) y[i] = (k0 * delta) * obs[i];

    RankPredictor predictor;
    predictor.r = opts.initial_rank;
    predictor.increment = opts.rank_increment;
    predictor.max_rank = std::min(m, n);
    McSolution sol;
    SolverStats& stats = sol.stats;
    stats.matvec_init = op.application_count();
    std::int64_t mark = stats.matvec_init;
    Vec resid(static_cast<size_t>(s));
    for (Index it = 1; it <= opts.max_iter; ++it) {
        op.assign_values(y);
        auto prox = svt(op, tau, backend, predictor);
        sol.u = std::move(prox.u);
        sol.sigma = std::move(prox.sigma);
        sol.v = std::move(prox.v);
        stats.rank_hat = prox.achieved_rank;
        Vec a_vals = project_low_rank(pd, sol.u, sol.sigma, sol.v);
        for (std::int64_t i = 0; i < s; ++i) resid[i] = obs[i] - a_vals[i];
        stats.matvec_history.push_back(op.application_count() - mark);
        mark = op.application_count();
        const double rel = vnorm(resid) / obs_norm;
        stats.residual_history.push_back(rel);
        stats.iterations = it;
        if (rel <= opts.tol_outer) {
            stats.converged = true;
            break;
        }
        for (std::int64_t i = 0; i < s; ++i) y[i] += delta * resid[i];
    }
    stats.matvec_count = op.application_count();
    stats.predicted_ranks = predictor.history;
    if (opts.truth_ml && opts.truth_mr) {
        Mat a_true = mul(*opts.truth_ml, *opts.truth_mr, 'N', 'T');
        Mat us = sol.u;
        for (Index j = 0; j < us.c; ++j)
            for (Index i = 0; i < us.r; ++i) us(i, j) *= sol.sigma[j];
        Mat a_hat = us.c > 0 ? mul(us, sol.v, 'N', 'T') : Mat(m, n);
        for (size_t i = 0; i < a_hat.a.size(); ++i) a_hat.a[i] -= a_true.a[i];
        stats.rel_err = fro(a_hat) / fro(a_true);
    }
    stats.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return sol;
}

// --------------------------------------------------------------- synth.hpp
// synth.hpp:23-33 Floyd's algorithm, sorted output. For large draws a bitmap
// replaces the hash set; the accepted set (and so the RNG consumption) is the
// same, because membership, not container, decides each insertion.
std::vector<std::int64_t> sample_distinct(std::int64_t n, std::int64_t s, Rng& rng) {
    std::vector<std::int64_t> out;
    out.reserve(static_cast<size_t>(s));
    if (s > 2000000) {
        std::vector<std::uint64_t> bits(static_cast<size_t>((n + 63) / 64), 0);
        auto test_set = [&](std::int64_t t) {
            std::uint64_t& w = bits[static_cast<size_t>(t >> 6)];
            const std::uint64_t mask = 1ull << (t & 63);
            const bool had = (w & mask) != 0;
            w |= mask;
            return had;
        };
        for (std::int64_t j = n - s; j < n; ++j) {
            auto t = static_cast<std::int64_t>(rng.uniform_index(static_cast<std::uint64_t>(j + 1)));
            if (test_set(t)) test_set(j);
        }
        for (std::int64_t w = 0; w < static_cast<std::int64_t>(bits.size()); ++w) {
            std::uint64_t x = bits[static_cast<size_t>(w)];
            while (x) {
                const int b = __builtin_ctzll(x);
                out.push_back(w * 64 + b);
                x &= x - 1;
            }
        }
        return out;
    }
    std::unordered_set<std::int64_t> chosen;
    chosen.reserve(static_cast<size_t>(s));
    for (std::int64_t j = n - s; j < n; ++j) {
        auto t = static_cast<std::int64_t>(rng.uniform_index(static_cast<std::uint64_t>(j + 1)));
        if (!chosen.insert(t).second) chosen.insert(j);
    }
    out.assign(chosen.begin(), chosen.end());
    std::sort(out.begin(), out.end());
    return out;
}

}  // namespace orc
