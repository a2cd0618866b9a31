// TEST INFRASTRUCTURE ONLY — extern "C" surface of the CPU oracle, bound by
// oracle/oracle.py through ctypes. All matrices are column-major doubles.
// Return codes: 0 ok, 1 invalid argument, 2 numerical failure.
#include <cstring>
#include <string>

#include "blws_oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

Mat to_mat(Index r, Index c, const double* p) {
    Mat m(r, c);
    if (r * c > 0) std::memcpy(m.data(), p, sizeof(double) * static_cast<size_t>(r * c));
    return m;
}
void put(const Mat& m, double* out) {
    if (!m.a.empty()) std::memcpy(out, m.data(), sizeof(double) * m.a.size());
}
void put(const Vec& v, double* out) {
    if (!v.empty()) std::memcpy(out, v.data(), sizeof(double) * v.size());
}
Csc to_csc(Index m, Index n, Index nnz, const std::int64_t* colptr, const std::int32_t* rowidx, const double* v) {
    Csc c;
    c.rows = m;
    c.cols = n;
    c.colptr.assign(colptr, colptr + n + 1);
    c.rowidx.assign(rowidx, rowidx + nnz);
    c.val.assign(v, v + nnz);
    return c;
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
void orc_set_threads(int n) { set_threads(n); }
int64_t orc_small_dense_max_order() { return small_dense_max_order(); }

// ---------------------------------------------------------------- rng
void* orc_rng_new(std::uint64_t seed) { return new Rng(seed); }
void orc_rng_free(void* r) { delete static_cast<Rng*>(r); }
void* orc_rng_split(void* r, std::uint64_t tag) { return new Rng(static_cast<Rng*>(r)->split(tag)); }
std::uint64_t orc_rng_next_u64(void* r) { return static_cast<Rng*>(r)->next_u64(); }
double orc_rng_uniform(void* r) { return static_cast<Rng*>(r)->uniform(); }
double orc_rng_uniform_range(void* r, double lo, double hi) { return static_cast<Rng*>(r)->uniform(lo, hi); }
double orc_rng_normal(void* r) { return static_cast<Rng*>(r)->normal(); }
std::uint64_t orc_rng_uniform_index(void* r, std::uint64_t n) { return static_cast<Rng*>(r)->uniform_index(n); }
void orc_rng_gaussian_matrix(void* r, Index rows, Index cols, double* out) {
    put(static_cast<Rng*>(r)->gaussian_matrix(rows, cols), out);
}
void orc_rng_unit_vector(void* r, Index n, double* out) { put(static_cast<Rng*>(r)->unit_vector(n), out); }
void orc_rng_uniform_fill(void* r, Index n, double lo, double hi, double* out) {
    for (Index i = 0; i < n; ++i) out[i] = static_cast<Rng*>(r)->uniform(lo, hi);
}
Index orc_sample_distinct(std::int64_t n, std::int64_t s, void* r, std::int64_t* out) {
    auto v = sample_distinct(n, s, *static_cast<Rng*>(r));
    std::memcpy(out, v.data(), sizeof(std::int64_t) * v.size());
    return static_cast<Index>(v.size());
}

// ------------------------------------------------------ dense kernels
int orc_thin_qr(Index rows, Index cols, const double* m, double* q, double* r, Index* rank) {
    return guard([&] {
        auto qr = thin_qr(to_mat(rows, cols, m));
        put(qr.q, q);
        put(qr.r, r);
        *rank = qr.rank;
    });
}
int orc_sym_evd(Index n, const double* t, double* values, double* vectors) {
    return guard([&] {
        auto e = sym_evd_small(to_mat(n, n, t));
        put(e.values, values);
        put(e.vectors, vectors);
    });
}
int orc_sym_evd_tridiagonal(Index n, const double* d, const double* e, double* values, double* vectors) {
    return guard([&] {
        auto r = sym_evd_tridiagonal(Vec(d, d + n), Vec(e, e + (n > 0 ? n - 1 : 0)));
        put(r.values, values);
        put(r.vectors, vectors);
    });
}
int orc_full_svd(Index m, Index n, const double* a, double* u, double* s, double* v) {
    return guard([&] {
        auto r = full_svd_small(to_mat(m, n, a));
        put(r.u, u);
        put(r.sigma, s);
        put(r.v, v);
    });
}

// ---------------------------------------------------------- operators
void* orc_dense_op_new(Index m, Index n, const double* w) {
    try {
        return new DenseOperator(to_mat(m, n, w));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
int orc_dense_op_assign(void* op, Index m, Index n, const double* w) {
    return guard([&] { static_cast<DenseOperator*>(op)->assign(to_mat(m, n, w)); });
}
void* orc_sparse_op_new(Index m, Index n, Index nnz, const std::int64_t* colptr, const std::int32_t* rowidx,
                        const double* vals) {
    try {
        return new SparseOperator(to_csc(m, n, nnz, colptr, rowidx, vals));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
int orc_sparse_op_assign_values(void* op, Index nnz, const double* vals) {
    return guard([&] { static_cast<SparseOperator*>(op)->assign_values(Vec(vals, vals + nnz)); });
}
void* orc_aug_op_new(void* inner) { return new AugmentedOperator(*static_cast<LinearOperator*>(inner)); }
std::int64_t orc_op_count(void* op) { return static_cast<LinearOperator*>(op)->application_count(); }
Index orc_op_rows(void* op) { return static_cast<LinearOperator*>(op)->rows(); }
Index orc_op_cols(void* op) { return static_cast<LinearOperator*>(op)->cols(); }
void orc_op_free(void* op) { delete static_cast<LinearOperator*>(op); }
int orc_op_apply_block(void* op, Index b, const double* x, double* y) {
    return guard([&] {
        auto* o = static_cast<LinearOperator*>(op);
        put(o->apply_block(to_mat(o->cols(), b, x)), y);
    });
}
int orc_op_apply_pair_block(void* op, Index b, const double* left, const double* right, double* top, double* bot) {
    return guard([&] {
        auto* o = static_cast<LinearOperator*>(op);
        auto [t, bt] = o->apply_pair_block(to_mat(o->rows(), b, left), to_mat(o->cols(), b, right));
        put(t, top);
        put(bt, bot);
    });
}

// ------------------------------------------------------- block lanczos
int orc_block_lanczos(void* op, Index b, const double* x1, Index k, double* q, double* t, Index* built, int* term) {
    return guard([&] {
        auto* o = static_cast<LinearOperator*>(op);
        auto f = block_lanczos_procedure(*o, to_mat(o->rows(), b, x1), k);
        put(f.q, q);
        put(f.embed(), t);
        *built = static_cast<Index>(f.m.size());
        *term = f.terminated_early ? 1 : 0;
    });
}
int orc_bl_evd(void* op, Index b, const double* x1, Index k, Index r, double* u, double* values, Index* avail,
               int* term) {
    return guard([&] {
        auto* o = static_cast<LinearOperator*>(op);
        auto e = bl_evd(*o, to_mat(o->rows(), b, x1), k, r);
        put(e.u, u);
        put(e.values, values);
        *avail = e.available;
        *term = e.terminated_early ? 1 : 0;
    });
}
int orc_adapt_subspace(Index r_old, const double* u, const double* v, const double* s, Index r_new, Index m,
                       Index n, void* rng, double* u_out, double* v_out, double* s_out) {
    return guard([&] {
        std::optional<WarmStart> w;
        if (r_old > 0) {
            WarmStart ws;
            ws.u = to_mat(m, r_old, u);
            ws.v = to_mat(n, r_old, v);
            ws.sigma.assign(s, s + r_old);
            w = ws;
        }
        auto o = adapt_subspace(w, r_new, m, n, *static_cast<Rng*>(rng));
        put(o.u, u_out);
        put(o.v, v_out);
        put(o.sigma, s_out);
    });
}
int orc_blws_svd(void* op, Index b, const double* u, const double* v, const double* s, Index k, Index r, void* rng,
                 double* u_out, double* v_out, double* s_out, int* flags) {
    return guard([&] {
        auto* o = static_cast<LinearOperator*>(op);
        WarmStart ws;
        ws.u = to_mat(o->rows(), b, u);
        ws.v = to_mat(o->cols(), b, v);
        ws.sigma.assign(s, s + b);
        auto res = blws_svd(*o, ws, k, r, *static_cast<Rng*>(rng));
        put(res.warm.u, u_out);
        put(res.warm.v, v_out);
        put(res.warm.sigma, s_out);
        *flags = (res.padded ? 1 : 0) | (res.k_raised ? 2 : 0) | (res.terminated_early ? 4 : 0);
    });
}

// ------------------------------------------------------------ lanczos
int orc_lanczos_partial_svd(void* op, Index r, double tol, Index max_k, std::uint64_t seed, double* u, double* s,
                            double* v, Index* keep, Index* stats) {
    return guard([&] {
        LanczosOptions lo;
        lo.tol = tol;
        lo.max_k = max_k;
        lo.seed = seed;
        auto res = lanczos_partial_svd(*static_cast<LinearOperator*>(op), r, lo);
        put(res.u, u);
        put(res.sigma, s);
        put(res.v, v);
        *keep = static_cast<Index>(res.sigma.size());
        stats[0] = res.stats.steps;
        stats[1] = res.stats.restarts;
        stats[2] = res.stats.converged;
        stats[3] = res.stats.all_converged ? 1 : 0;
    });
}
int orc_lanczos_partial_evd(void* op, Index r, double tol, Index max_k, std::uint64_t seed, double* u,
                            double* values, Index* avail, Index* stats) {
    return guard([&] {
        LanczosOptions lo;
        lo.tol = tol;
        lo.max_k = max_k;
        lo.seed = seed;
        auto res = lanczos_partial_evd(*static_cast<LinearOperator*>(op), r, lo);
        put(res.u, u);
        put(res.values, values);
        *avail = static_cast<Index>(res.values.size());
        stats[0] = res.stats.steps;
        stats[1] = res.stats.restarts;
        stats[2] = res.stats.converged;
        stats[3] = res.stats.all_converged ? 1 : 0;
    });
}
int orc_lanczos_procedure(void* op, const double* q1, Index k, double* q, double* alpha, double* beta,
                          Index* cols, double* resid, int* term) {
    return guard([&] {
        auto* o = static_cast<LinearOperator*>(op);
        auto f = lanczos_procedure(*o, Vec(q1, q1 + o->rows()), k, true);
        put(f.q, q);
        put(f.alpha, alpha);
        put(f.beta, beta);
        *cols = f.q.c;
        *resid = f.residual_norm;
        *term = f.terminated_early ? 1 : 0;
    });
}
double orc_spectral_norm(void* op, double tol, std::uint64_t seed) {
    try {
        return spectral_norm(*static_cast<LinearOperator*>(op), tol, seed);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

// --------------------------------------------------------- backend/svt
void* orc_backend_new(int kind, Index block_steps, double ritz_tol, Index max_k, Index seed_margin,
                      std::uint64_t seed) {
    SvdBackend::Options o;
    o.block_steps = block_steps;
    o.ritz_tol = ritz_tol;
    o.max_k = max_k;
    o.seed_margin = seed_margin;
    o.seed = seed;
    return new SvdBackend(static_cast<SvdBackend::Kind>(kind), o);
}
void orc_backend_free(void* b) { delete static_cast<SvdBackend*>(b); }
Index orc_backend_warm_rank(void* b) {
    auto& w = static_cast<SvdBackend*>(b)->warm_state();
    return w ? w->rank() : 0;
}
void orc_backend_warm_get(void* b, double* u, double* v, double* s) {
    auto& w = static_cast<SvdBackend*>(b)->warm_state();
    if (!w) return;
    put(w->u, u);
    put(w->v, v);
    put(w->sigma, s);
}
int orc_svt(void* op, double eps, void* backend, Index* pred, Index* hist, Index hist_cap, Index* hist_len,
            double* u, double* s, double* v, Index* achieved, int* all_above) {
    return guard([&] {
        RankPredictor p;
        p.r = pred[0];
        p.increment = pred[1];
        p.max_rank = pred[2];
        for (Index i = 0; i < *hist_len; ++i) p.history.push_back(hist[i]);
        auto res = svt(*static_cast<LinearOperator*>(op), eps, *static_cast<SvdBackend*>(backend), p);
        pred[0] = p.r;
        *hist_len = std::min<Index>(hist_cap, static_cast<Index>(p.history.size()));
        for (Index i = 0; i < *hist_len; ++i) hist[i] = p.history[i];
        put(res.u, u);
        put(res.sigma, s);
        put(res.v, v);
        *achieved = res.achieved_rank;
        *all_above = res.all_above_threshold ? 1 : 0;
    });
}

// ------------------------------------------------------------ solvers
// istats: iterations, matvec_count, matvec_init, rank_hat, e_l0, converged, e_nnz
// dstats: wall_time_s, rel_err
int orc_rpca_adm(Index m, const double* d, double lambda, void* backend, double tol, Index max_iter, double rho,
                 double mu_max_factor, Index initial_rank, Index rank_increment, const double* truth, double* a_out,
                 double* e_out, Index* istats, double* dstats, Index* pred_hist, Index* mv_hist, double* res_hist) {
    return guard([&] {
        RpcaOptions o;
        o.tol_outer = tol;
        o.max_iter = max_iter;
        o.rho = rho;
        o.mu_max_factor = mu_max_factor;
        o.initial_rank = initial_rank;
        o.rank_increment = rank_increment;
        Mat tr;
        if (truth) {
            tr = to_mat(m, m, truth);
            o.truth = &tr;
        }
        auto sol = rpca_adm(to_mat(m, m, d), lambda, *static_cast<SvdBackend*>(backend), o);
        if (a_out) put(sol.a, a_out);
        if (e_out) put(sol.e, e_out);
        const auto& st = sol.stats;
        istats[0] = st.iterations;
        istats[1] = st.matvec_count;
        istats[2] = st.matvec_init;
        istats[3] = st.rank_hat;
        istats[4] = st.e_l0;
        istats[5] = st.converged ? 1 : 0;
        istats[6] = sol.e_nnz;
        dstats[0] = st.wall_time_s;
        dstats[1] = st.rel_err;
        for (size_t i = 0; i < st.predicted_ranks.size(); ++i) pred_hist[i] = st.predicted_ranks[i];
        for (size_t i = 0; i < st.matvec_history.size(); ++i) mv_hist[i] = st.matvec_history[i];
        for (size_t i = 0; i < st.residual_history.size(); ++i) res_hist[i] = st.residual_history[i];
    });
}
int orc_mc_svt(Index m, Index n, Index nnz, const std::int64_t* colptr, const std::int32_t* rowidx,
               const double* vals, double tau, double delta, void* backend, double tol, Index max_iter,
               Index initial_rank, Index rank_increment, Index r_true, const double* ml, const double* mr,
               double* u_out, double* s_out, double* v_out, Index cap, Index* istats, double* dstats,
               Index* pred_hist, Index* mv_hist, double* res_hist) {
    return guard([&] {
        McOptions o;
        o.tol_outer = tol;
        o.max_iter = max_iter;
        o.initial_rank = initial_rank;
        o.rank_increment = rank_increment;
        Mat tl, tr;
        if (ml && mr) {
            tl = to_mat(m, r_true, ml);
            tr = to_mat(n, r_true, mr);
            o.truth_ml = &tl;
            o.truth_mr = &tr;
        }
        auto sol = mc_svt(to_csc(m, n, nnz, colptr, rowidx, vals), tau, delta, *static_cast<SvdBackend*>(backend), o);
        const Index rank = static_cast<Index>(sol.sigma.size());
        if (rank > cap) throw std::runtime_error("orc_mc_svt: output capacity too small");
        put(sol.u, u_out);
        put(sol.sigma, s_out);
        put(sol.v, v_out);
        const auto& st = sol.stats;
        istats[0] = st.iterations;
        istats[1] = st.matvec_count;
        istats[2] = st.matvec_init;
        istats[3] = st.rank_hat;
        istats[4] = rank;
        istats[5] = st.converged ? 1 : 0;
        dstats[0] = st.wall_time_s;
        dstats[1] = st.rel_err;
        for (size_t i = 0; i < st.predicted_ranks.size(); ++i) pred_hist[i] = st.predicted_ranks[i];
        for (size_t i = 0; i < st.matvec_history.size(); ++i) mv_hist[i] = st.matvec_history[i];
        for (size_t i = 0; i < st.residual_history.size(); ++i) res_hist[i] = st.residual_history[i];
    });
}

// -------------------------------------------------------------- trace
void orc_trace_enable(int on) { trace_enabled() = on != 0; }
void orc_trace_clear() { trace().clear(); }
Index orc_trace_size() { return static_cast<Index>(trace().size()); }
// ints: kind, b, r, k_eff, keep, steps, restarts, converged, flags, nsigma
int orc_trace_get(Index i, Index* ints, double* sigma, Index cap) {
    if (i < 0 || i >= static_cast<Index>(trace().size())) return 1;
    const auto& t = trace()[static_cast<size_t>(i)];
    ints[0] = t.kind;
    ints[1] = t.b;
    ints[2] = t.r;
    ints[3] = t.k_eff;
    ints[4] = t.keep;
    ints[5] = t.steps;
    ints[6] = t.restarts;
    ints[7] = t.converged;
    ints[8] = t.flags;
    ints[9] = static_cast<Index>(t.sigma.size());
    for (Index j = 0; j < std::min<Index>(cap, static_cast<Index>(t.sigma.size())); ++j) sigma[j] = t.sigma[j];
    return 0;
}

}  // extern "C"
