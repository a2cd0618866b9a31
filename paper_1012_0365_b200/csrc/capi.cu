// extern "C" boundary (include/blws_cuda.h): handles, status codes, copies.
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_set>

#include "../../include/blws_cuda.h"
#include "host.hpp"
#include "matrix_market.hpp"
#include "ops.cuh"

using namespace blws;
namespace blws {
void chol_probe_read(double* out);
}

// Every handle keeps its Context alive (shared ownership): callers may destroy
// the context handle first (e.g. interpreter shutdown order) without the
// dependent handles' device buffers freeing through a dangling context.
struct blws_context {
    std::shared_ptr<Context> ctx;
};
struct blws_rng {
    Rng rng;
};
struct blws_operator {
    std::shared_ptr<Context> keep;  // declared first: destroyed last
    blws_context* owner;
    std::unique_ptr<LinearOperator> op;
    bool dense = true;
};
struct blws_warm_start {
    std::shared_ptr<Context> keep;
    DWarm w;
};
struct blws_svd_backend {
    std::shared_ptr<Context> keep;
    blws_context* owner;
    std::unique_ptr<SvdBackend> b;
};

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return BLWS_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return BLWS_INVALID_ARGUMENT;
    } catch (const CudaError& e) {
        g_err = e.what();
        return BLWS_CUDA_ERROR;
    } catch (const CommError& e) {
        g_err = e.what();
        return BLWS_NCCL_ERROR;
    } catch (const IoError& e) {
        g_err = e.what();
        return BLWS_IO_ERROR;
    } catch (const std::bad_alloc& e) {
        g_err = std::string("allocation failed: ") + e.what();
        return BLWS_CUDA_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return BLWS_NUMERICAL_FAILURE;
    }
}

void need(bool c, const char* msg) {
    if (!c) throw std::invalid_argument(msg);
}

blws_warm_start* wrap(const std::shared_ptr<Context>& keep, DWarm w) { return new blws_warm_start{keep, std::move(w)}; }

void copy_in(Context& ctx, View dst, const double* src, Index ld, int where) {
    if (where == BLWS_HOST)
        upload(ctx, dst, src, ld);
    else
        copy(ctx, dst, View{const_cast<double*>(src), dst.rows, dst.cols, ld});
}

void copy_out(Context& ctx, View src, double* dst, Index ld, int where) {
    if (!dst) return;
    if (where == BLWS_HOST)
        download(ctx, src, dst, ld);
    else
        copy(ctx, View{dst, src.rows, src.cols, ld}, src);
}

void put_stats(const SolverStats& s, blws_solver_stats* o, int64_t* pr, int64_t* mh, double* rh, int64_t cap) {
    if (o) {
        o->iterations = s.iterations;
        o->wall_time_s = s.wall_time_s;
        o->matvec_count = s.matvec_count;
        o->matvec_init = s.matvec_init;
        o->rel_err = s.rel_err;
        o->rank_hat = s.rank_hat;
        o->e_l0 = s.e_l0;
        o->e_nnz = s.e_nnz;
        o->converged = s.converged ? 1 : 0;
    }
    for (int64_t i = 0; i < std::min<int64_t>(cap, static_cast<int64_t>(s.predicted_ranks.size())); ++i)
        if (pr) pr[i] = s.predicted_ranks[i];
    for (int64_t i = 0; i < std::min<int64_t>(cap, static_cast<int64_t>(s.matvec_history.size())); ++i)
        if (mh) mh[i] = s.matvec_history[i];
    for (int64_t i = 0; i < std::min<int64_t>(cap, static_cast<int64_t>(s.residual_history.size())); ++i)
        if (rh) rh[i] = s.residual_history[i];
}
}  // namespace

extern "C" {

const char* blws_last_error(void) { return g_err.c_str(); }
int blws_abi_version(void) { return 1; }

// ---------------------------------------------------------------- context
int blws_context_create(int device, blws_context** out) {
    return guard([&] {
        need(out != nullptr, "blws_context_create: null out");
        auto c = std::make_unique<blws_context>();
        c->ctx = std::make_shared<Context>(device);
        *out = c.release();
    });
}
int blws_context_destroy(blws_context* ctx) {
    return guard([&] { delete ctx; });
}
int blws_context_synchronize(blws_context* ctx) {
    return guard([&] { ctx->ctx->sync(); });
}
void* blws_context_stream(blws_context* ctx) { return ctx ? ctx->ctx->stream() : nullptr; }
int64_t blws_context_launches(const blws_context* ctx) { return ctx ? ctx->ctx->launches() : 0; }
int blws_context_set_profiling(blws_context* ctx, int on) {
    return guard([&] { ctx->ctx->set_profiling(on != 0); });
}
int blws_context_region_stats(blws_context* ctx, int region, double* total_ms, int64_t* count, double* flops,
                              double* bytes) {
    return guard([&] {
        need(region >= 0 && region < Context::kRegions, "region out of range");
        ctx->ctx->region_stats(region, total_ms, count, flops, bytes);
    });
}
int blws_context_region_reset(blws_context* ctx) {
    return guard([&] { ctx->ctx->region_reset(); });
}
int blws_fp64_peak(blws_context* ctx, int mode, double* tflops) {
    return guard([&] { *tflops = fp64_peak_tflops(*ctx->ctx, mode); });
}

int blws_l2_probe(blws_context* ctx, int mode, int row, double* gbps) {
    return guard([&] {
        need(mode == 0 || (mode == 1 && row >= 1 && row <= 128), "l2_probe: bad mode / row");
        *gbps = l2_probe_gbps(*ctx->ctx, mode, row);
    });
}

// -------------------------------------------------------------------- rng
int blws_rng_create(uint64_t seed, blws_rng** out) {
    return guard([&] { *out = new blws_rng{Rng(seed)}; });
}
int blws_rng_destroy(blws_rng* r) {
    delete r;
    return BLWS_OK;
}
int blws_rng_split(const blws_rng* r, uint64_t tag, blws_rng** out) {
    return guard([&] { *out = new blws_rng{r->rng.split(tag)}; });
}
uint64_t blws_rng_next_u64(blws_rng* r) { return r->rng.next_u64(); }
double blws_rng_uniform(blws_rng* r, double lo, double hi) { return r->rng.uniform(lo, hi); }
int blws_rng_uniform_fill(blws_rng* r, int64_t n, double lo, double hi, double* out) {
    return guard([&] {
        need(r && (n == 0 || out), "uniform_fill: null argument");
        for (int64_t i = 0; i < n; ++i) out[i] = r->rng.uniform(lo, hi);
    });
}
uint64_t blws_rng_uniform_index(blws_rng* r, uint64_t n) { return r->rng.uniform_index(n); }
double blws_rng_normal(blws_rng* r) { return r->rng.normal(); }
int blws_rng_gaussian_matrix(blws_rng* r, int64_t rows, int64_t cols, double* out) {
    return guard([&] { r->rng.gaussian_matrix(rows, cols, out, rows); });
}
int64_t blws_sample_distinct(int64_t n, int64_t s, blws_rng* r, int64_t* out) {
    // Floyd's algorithm (synth.hpp:23-33); the accepted set decides each step,
    // so a bitmap gives the same draws as the reference's hash set.
    std::vector<std::uint64_t> bits(static_cast<size_t>((n + 63) / 64), 0);
    auto test_set = [&](int64_t t) {
        std::uint64_t& w = bits[static_cast<size_t>(t >> 6)];
        const std::uint64_t mask = 1ull << (t & 63);
        const bool had = (w & mask) != 0;
        w |= mask;
        return had;
    };
    for (int64_t j = n - s; j < n; ++j) {
        const auto t = static_cast<int64_t>(r->rng.uniform_index(static_cast<uint64_t>(j + 1)));
        if (test_set(t)) test_set(j);
    }
    int64_t c = 0;
    for (int64_t w = 0; w < static_cast<int64_t>(bits.size()); ++w) {
        std::uint64_t x = bits[static_cast<size_t>(w)];
        while (x) {
            out[c++] = w * 64 + __builtin_ctzll(x);
            x &= x - 1;
        }
    }
    return c;
}

// -------------------------------------------------------------- operators
int blws_dense_operator_create(blws_context* ctx, int64_t m, int64_t n, const double* w, int64_t ldw, int where,
                               int borrow, blws_operator** out) {
    return guard([&] {
        need(m > 0 && n > 0 && w && ldw >= m, "DenseOperator: bad shape");
        Context& c = *ctx->ctx;
        auto h = std::make_unique<blws_operator>();
        h->keep = ctx->ctx;
        h->owner = ctx;
        if (where == BLWS_DEVICE && borrow) {
            need(ldw % 2 == 0 && reinterpret_cast<uintptr_t>(w) % 16 == 0,
                 "DenseOperator: borrowed W needs an even leading dimension and 16-byte alignment");
            auto op = std::make_unique<DenseOperator>(c, m, n, const_cast<double*>(w), ldw);
            op->check_finite();
            h->op = std::move(op);
        } else {
            auto op = std::make_unique<DenseOperator>(c, m, n);
            if (where == BLWS_HOST)
                op->assign_host(w, ldw);
            else
                op->assign_device(w, ldw);
            h->op = std::move(op);
        }
        *out = h.release();
    });
}
int blws_dense_operator_assign(blws_operator* op, const double* w, int64_t ldw, int where) {
    return guard([&] {
        need(op->dense, "assign: not a dense operator");
        auto* d = static_cast<DenseOperator*>(op->op.get());
        if (where == BLWS_HOST)
            d->assign_host(w, ldw);
        else
            d->assign_device(w, ldw);
    });
}
int blws_nccl_unique_id(uint8_t* out128) {
    return guard([&] {
        need(out128 != nullptr, "nccl_unique_id: null output");
        comm_unique_id(out128);
    });
}
int blws_context_init_host_comm(blws_context* ctx, int nranks, int rank, blws_host_allreduce_fn fn, void* user) {
    return guard([&] {
        need(ctx && fn, "init_host_comm: null argument");
        ctx->ctx->init_host_comm(nranks, rank, fn, user);
    });
}

int blws_context_init_comm(blws_context* ctx, int nranks, int rank, const uint8_t* id128) {
    return guard([&] {
        need(ctx && id128, "init_comm: null argument");
        ctx->ctx->init_comm(nranks, rank, id128);
    });
}
int blws_context_comm_info(const blws_context* ctx, int* nranks, int* rank) {
    return guard([&] {
        need(ctx != nullptr, "comm_info: null context");
        if (nranks) *nranks = ctx->ctx->nranks();
        if (rank) *rank = ctx->ctx->rank();
    });
}
int blws_dense_operator_set_row_shard(blws_operator* op, int64_t m_total, int64_t row0) {
    return guard([&] {
        need(op && op->dense, "set_row_shard: not a dense operator");
        op->op->set_row_shard(m_total, row0);
    });
}
int blws_dense_operator_assign_async(blws_operator* op, const double* w, int64_t ldw) {
    return guard([&] {
        need(op->dense, "assign_async: not a dense operator");
        need(w != nullptr, "assign_async: null source");
        static_cast<DenseOperator*>(op->op.get())->assign_host_async(w, ldw);
    });
}
int blws_sparse_operator_create(blws_context* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* colptr,
                                const int32_t* rowidx, const double* values, blws_operator** out) {
    return guard([&] {
        need(m > 0 && n > 0 && nnz >= 0, "SparseOperator: bad shape");
        auto h = std::make_unique<blws_operator>();
        h->keep = ctx->ctx;
        h->owner = ctx;
        h->dense = false;
        h->op = std::make_unique<SparseOperator>(*ctx->ctx, m, n, nnz, colptr, rowidx, values);
        *out = h.release();
    });
}
int blws_sparse_operator_assign_values(blws_operator* op, const double* values, int64_t nnz, int where) {
    return guard([&] {
        need(!op->dense, "assign_values: not a sparse operator");
        auto* s = static_cast<SparseOperator*>(op->op.get());
        need(nnz == s->nnz(), "SparseOperator: value count does not match pattern");
        if (where == BLWS_HOST) {
            for (int64_t i = 0; i < nnz; ++i)
                if (!std::isfinite(values[i])) throw std::invalid_argument("SparseOperator: non-finite entries");
            s->assign_values_host(values);
        } else {
            s->assign_values_device(values);
        }
    });
}
int blws_operator_destroy(blws_operator* op) {
    return guard([&] { delete op; });
}
int64_t blws_operator_rows(const blws_operator* op) { return op->op->rows(); }
int64_t blws_operator_cols(const blws_operator* op) { return op->op->cols(); }
int64_t blws_operator_application_count(const blws_operator* op) { return op->op->application_count(); }
int blws_operator_apply_pair_block(blws_operator* op, int64_t b, const double* left, const double* right,
                                   double* top, double* bot) {
    return guard([&] {
        Context& c = op->op->ctx();
        const Index m = op->op->rows(), n = op->op->cols();
        DMat l(c, m, b), r(c, n, b), t(c, m, b), bt(c, n, b);
        upload(c, l.view(), left, m);
        upload(c, r.view(), right, n);
        op->op->apply_pair_block(l.view(), r.view(), t.view(), bt.view());
        download(c, t.view(), top, m);
        download(c, bt.view(), bot, n);
    });
}

int blws_operator_apply_pair(blws_operator* op, const double* left, const double* right, double* top,
                             double* bot) {
    return guard([&] {
        need(op && left && right && top && bot, "apply_pair: null argument");
        Context& c = op->op->ctx();
        const Index m = op->op->rows(), n = op->op->cols();
        DBuf<double> l(c, static_cast<size_t>(m)), r(c, static_cast<size_t>(n)), t(c, static_cast<size_t>(m)),
            bt(c, static_cast<size_t>(n));
        upload(c, View{l.get(), m, 1, m}, left, m);
        upload(c, View{r.get(), n, 1, n}, right, n);
        op->op->apply_pair(l.get(), r.get(), t.get(), bt.get());
        download(c, View{t.get(), m, 1, m}, top, m);
        download(c, View{bt.get(), n, 1, n}, bot, n);
    });
}

// ------------------------------------------------------------- warm start
int blws_warm_start_create(blws_context* ctx, int64_t m, int64_t n, int64_t r, const double* u, int64_t ldu,
                           const double* v, int64_t ldv, const double* sigma, int where, blws_warm_start** out) {
    return guard([&] {
        need(m > 0 && n > 0 && r >= 0, "WarmStart: bad shape");
        Context& c = *ctx->ctx;
        DWarm w = make_warm(c, m, n, r);
        if (r > 0) {
            copy_in(c, w.u(), u, ldu, where);
            copy_in(c, w.v(), v, ldv, where);
            std::copy(sigma, sigma + r, w.sigma.begin());
        }
        *out = wrap(ctx->ctx, std::move(w));
    });
}
int blws_warm_start_copy(const blws_warm_start* src, blws_warm_start** out) {
    return guard([&] { *out = wrap(src->keep, copy_warm(*src->keep, src->w, src->w.rank())); });
}
int64_t blws_warm_start_rank(const blws_warm_start* w) { return w->w.rank(); }
int blws_warm_start_get(const blws_warm_start* w, double* u, int64_t ldu, double* v, int64_t ldv, double* sigma,
                        int where) {
    return guard([&] {
        Context& c = *w->keep;
        copy_out(c, w->w.u(), u, ldu, where);
        copy_out(c, w->w.v(), v, ldv, where);
        if (sigma) std::copy(w->w.sigma.begin(), w->w.sigma.end(), sigma);
        c.sync();
    });
}
int blws_warm_start_destroy(blws_warm_start* w) {
    return guard([&] { delete w; });
}

// ---------------------------------------------------------- block lanczos
int64_t blws_svd_deferred_fallbacks(void) { return blws::g_blws_deferred_fallbacks; }
int64_t blws_svd_graph_launches(void) { return blws::g_blws_graph_launches; }
int blws_svd(blws_operator* w, const blws_warm_start* warm, int64_t k, int64_t r, blws_rng* rng,
             blws_warm_start** out, int* flags) {
    return guard([&] {
        need(w && warm && rng && out, "blws_svd: null argument");
        auto res = blws::blws_svd(*w->op, warm->w, k, r, rng->rng);
        if (flags) *flags = (res.padded ? 1 : 0) | (res.k_raised ? 2 : 0) | (res.terminated_early ? 4 : 0);
        *out = wrap(w->keep, std::move(res.warm));
    });
}
int blws_adapt_subspace(blws_context* ctx, const blws_warm_start* warm, int64_t r_new, int64_t m, int64_t n,
                        blws_rng* rng, blws_warm_start** out) {
    return guard([&] {
        DWarm o = blws::adapt_subspace(*ctx->ctx, warm ? &warm->w : nullptr, r_new, m, n, rng->rng);
        *out = wrap(ctx->ctx, std::move(o));
    });
}
int blws_block_lanczos_procedure(blws_operator* w, int64_t b, const double* x1, int64_t k, double* q, double* t,
                                 int64_t* built, int* terminated_early) {
    return guard([&] {
        Context& c = w->op->ctx();
        need(!w->op->col_sharded(), "block_lanczos_procedure: a column-sharded operator's panels are split");
        const Stack geo{w->op->rows(), w->op->cols()};
        const Index dim = geo.m + geo.n;
        DMat x(c, geo.ld(), b, true);
        upload(c, View{x.data(), geo.m, b, x.ld}, x1, dim);
        upload(c, View{x.data() + geo.mp(), geo.n, b, x.ld}, x1 + geo.m, dim);
        auto f = blws::block_lanczos_procedure(*w->op, x.view(), k);
        const Index cols = f.built * b;
        download(c, View{f.q.data(), geo.m, cols, f.q.ld}, q, dim);
        download(c, View{f.q.data() + geo.mp(), geo.n, cols, f.q.ld}, q + geo.m, dim);
        std::vector<double> tt(static_cast<size_t>(cols * cols), 0.0);
        std::vector<double> blk(static_cast<size_t>(b * b));
        for (Index l = 0; l < f.built; ++l) {
            download(c, f.m[l].view(), blk.data(), b);
            for (Index j = 0; j < b; ++j)
                for (Index i = 0; i < b; ++i) tt[(l * b + i) + (l * b + j) * cols] = blk[i + j * b];
            if (l + 1 < f.built) {
                download(c, f.b[l].view(), blk.data(), b);
                for (Index j = 0; j < b; ++j)
                    for (Index i = 0; i < b; ++i) {
                        tt[(l * b + b + i) + (l * b + j) * cols] = blk[i + j * b];
                        tt[(l * b + j) + (l * b + b + i) * cols] = blk[i + j * b];
                    }
            }
        }
        std::copy(tt.begin(), tt.end(), t);
        *built = f.built;
        *terminated_early = f.terminated_early ? 1 : 0;
    });
}

// ---------------------------------------------------------------- lanczos
int blws_lanczos_partial_svd(blws_operator* w, int64_t r, double tol, int64_t max_k, uint64_t seed,
                             blws_warm_start** out, int64_t stats[4]) {
    return guard([&] {
        LanczosOptions o;
        o.tol = tol;
        o.max_k = max_k;
        o.seed = seed;
        auto res = blws::lanczos_partial_svd(*w->op, r, o);
        if (stats) {
            stats[0] = res.stats.steps;
            stats[1] = res.stats.restarts;
            stats[2] = res.stats.converged;
            stats[3] = res.stats.all_converged ? 1 : 0;
        }
        *out = wrap(w->keep, std::move(res.uv));
    });
}
int blws_spectral_norm(blws_operator* w, double tol, uint64_t seed, double* out) {
    return guard([&] { *out = blws::spectral_norm(*w->op, tol, seed); });
}

// ------------------------------------------------- dense kernels (device)
int blws_thin_qr(blws_context* ctx, int64_t rows, int64_t cols, const double* m, double* q, double* r,
                 int64_t* rank) {
    return guard([&] {
        need(rows > 0 && cols > 0, "thin_qr: empty matrix");
        need(rows >= cols, "thin_qr: requires rows >= cols");
        for (int64_t i = 0; i < rows * cols; ++i)
            if (!std::isfinite(m[i])) throw std::invalid_argument("thin_qr: non-finite entries");
        Context& c = *ctx->ctx;
        DMat x(c, rows, cols), rr(c, cols, cols);
        upload(c, x.view(), m, rows);
        View rv = rr.view();
        *rank = blws::thin_qr(c, x.view(), &rv);
        download(c, x.view(), q, rows);
        if (r) download(c, rr.view(), r, cols);
    });
}
int blws_full_svd_small(blws_context* ctx, int64_t m, int64_t n, const double* w, double* sigma, double* u,
                        double* v) {
    return guard([&] {
        need(ctx && w && sigma && u && v && m > 0 && n > 0, "full_svd_small: bad argument");
        for (int64_t i = 0; i < m * n; ++i)
            if (!std::isfinite(w[i])) throw std::invalid_argument("full_svd_small: non-finite entries");
        Context& c = *ctx->ctx;
        const Index p = std::min(m, n);
        DMat wd(c, m, n), ud(c, m, p), vd(c, n, p);
        upload(c, wd.view(), w, m);
        DBuf<double> s(c, static_cast<size_t>(p));
        full_svd_small(c, wd.view(), s.get(), ud.view(), vd.view());
        c.read(s.get(), sigma, static_cast<size_t>(p));
        download(c, ud.view(), u, m);
        download(c, vd.view(), v, n);
        c.sync();
    });
}
int blws_sym_evd(blws_context* ctx, int64_t n, const double* t, double* values, double* vectors) {
    return guard([&] {
        need(n > 0, "sym_evd_small: not square");
        need(n <= 4096, "sym_evd_small: too large");
        double nrm = 0, asym = 0;
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) {
                const double a = t[i + j * n];
                if (!std::isfinite(a)) throw std::invalid_argument("sym_evd_small: non-finite entries");
                nrm += a * a;
                const double d = a - t[j + i * n];
                asym += d * d;
            }
        if (std::sqrt(asym) > 1e-10 * std::sqrt(nrm) && nrm > 0)
            throw std::invalid_argument("sym_evd_small: input is not symmetric");
        Context& c = *ctx->ctx;
        DMat a(c, n, n), s(c, n, n), vec(c, n, n);
        upload(c, a.view(), t, n);
        blws::symmetrize(c, s.view(), a.view());
        DBuf<double> vals(c, static_cast<size_t>(n));
        sym_evd_top(c, s.view(), n, vals.get(), vec.view());
        c.read(vals.get(), values, n);
        download(c, vec.view(), vectors, n);
    });
}
int blws_sym_evd_tridiagonal_top(blws_context* ctx, int64_t n, const double* d, const double* e, int64_t want,
                                 double* values, double* vectors) {
    return guard([&] {
        need(n > 0, "sym_evd_tridiagonal: empty");
        need(n <= 4096, "sym_evd_tridiagonal: too large");
        need(want >= 1 && want <= n, "sym_evd_tridiagonal: bad want");
        Context& c = *ctx->ctx;
        DBuf<double> dd(c, static_cast<size_t>(n)), ee(c, static_cast<size_t>(std::max<int64_t>(n - 1, 1))),
            vals(c, static_cast<size_t>(want));
        c.write(dd.get(), d, n);
        if (n > 1) c.write(ee.get(), e, n - 1);
        DMat vec(c, n, want);
        tridiag_eig_top(c, n, dd.get(), ee.get(), want, vals.get(), vec.view());
        c.read(vals.get(), values, want);
        download(c, vec.view(), vectors, n);
    });
}
int blws_dgemm(blws_context* ctx, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* a,
               int64_t lda, const double* b, int64_t ldb, double beta, double* c, int64_t ldc) {
    return guard([&] { gemm(*ctx->ctx, ta != 0, tb != 0, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc); });
}

// ------------------------------------------------------------ backend/svt
int blws_svd_backend_create(blws_context* ctx, int kind, int64_t block_steps, double ritz_tol, int64_t max_k,
                            int64_t seed_margin, uint64_t seed, blws_svd_backend** out) {
    return guard([&] {
        need(kind == BLWS_BACKEND_EXACT_FULL || kind == BLWS_BACKEND_LANCZOS || kind == BLWS_BACKEND_BLWS,
             "SvdBackend: kind must be exact-full (0), lanczos (1) or blws (2)");
        SvdBackend::Options o;
        o.block_steps = block_steps;
        o.ritz_tol = ritz_tol;
        o.max_k = max_k;
        o.seed_margin = seed_margin;
        o.seed = seed;
        *out = new blws_svd_backend{ctx->ctx, ctx, std::make_unique<SvdBackend>(*ctx->ctx, static_cast<SvdBackend::Kind>(kind), o)};
    });
}
int blws_svd_backend_destroy(blws_svd_backend* b) {
    return guard([&] { delete b; });
}
int blws_svd_backend_warm_state(const blws_svd_backend* b, blws_warm_start** out) {
    return guard([&] {
        const auto& w = b->b->warm_state();
        *out = w ? wrap(b->keep, copy_warm(*b->keep, *w, w->rank())) : nullptr;
    });
}
int blws_svd_backend_set_warm_state(blws_svd_backend* b, const blws_warm_start* w) {
    return guard([&] { b->b->set_warm(copy_warm(*b->keep, w->w, w->w.rank())); });
}
int blws_svt(blws_operator* w, double eps, blws_svd_backend* backend, blws_rank_predictor* pred, int64_t* history,
             int64_t history_cap, int64_t* history_len, blws_warm_start** out, int64_t* achieved_rank,
             int* all_above_threshold) {
    return guard([&] {
        RankPredictor p;
        p.r = pred->r;
        p.increment = pred->increment;
        p.max_rank = pred->max_rank;
        auto res = blws::svt(*w->op, eps, *backend->b, p);
        pred->r = p.r;
        if (history && history_len && *history_len < history_cap) history[(*history_len)++] = p.history.back();
        if (achieved_rank) *achieved_rank = res.achieved_rank;
        if (all_above_threshold) *all_above_threshold = res.all_above_threshold ? 1 : 0;
        if (out) *out = wrap(w->keep, std::move(res.trip));
    });
}

// ---------------------------------------------------------------- solvers
}  // extern "C"

namespace {
// rpca_adm through the C ABI: the unsharded call has rows = m, shard = null
void rpca_entry(blws_context* ctx, int64_t m, int64_t rows, const RowShard* shard, const double* d, int64_t ldd,
                int where, double lambda, blws_svd_backend* backend, const blws_rpca_options* opts,
                const double* truth, double* a_out, double* e_out, blws_solver_stats* stats,
                int64_t* predicted_ranks, int64_t* matvec_history, double* residual_history, int64_t hist_cap) {
    need(m > 0 && rows > 0 && rows <= m && d && ldd >= rows, "rpca_adm: bad D");
    need(backend != nullptr, "rpca_adm: null backend");
    Context& c = *ctx->ctx;
    RpcaOptions o;
    if (opts) {
        o.tol_outer = opts->tol_outer;
        o.max_iter = opts->max_iter;
        o.rho = opts->rho;
        o.mu_max_factor = opts->mu_max_factor;
        o.initial_rank = opts->initial_rank;
        o.rank_increment = opts->rank_increment;
    }
    const Index ld = std::max<Index>(2, round_up(rows, 2));
    if (where == BLWS_DEVICE && ldd % 2 == 0) {
        auto s = blws::rpca_adm(c, m, d, ldd, lambda, *backend->b, o, truth, a_out, e_out, shard, rows);
        put_stats(s, stats, predicted_ranks, matvec_history, residual_history, hist_cap);
        return;
    }
    DMat dd(c, rows, m, false);
    copy_in(c, dd.view(), d, ldd, where);
    DMat tr, a, e;
    if (truth) {
        tr = DMat(c, rows, m, false);
        copy_in(c, tr.view(), truth, ldd, where);
    }
    if (a_out) a = DMat(c, rows, m, false);
    if (e_out) e = DMat(c, rows, m, false);
    auto s = blws::rpca_adm(c, m, dd.data(), ld, lambda, *backend->b, o, truth ? tr.data() : nullptr,
                            a_out ? a.data() : nullptr, e_out ? e.data() : nullptr, shard, rows);
    if (a_out) copy_out(c, a.view(), a_out, ldd, where);
    if (e_out) copy_out(c, e.view(), e_out, ldd, where);
    c.sync();
    put_stats(s, stats, predicted_ranks, matvec_history, residual_history, hist_cap);
}

void mc_entry(blws_context* ctx, int64_t m, int64_t rows, const RowShard* shard, int64_t n, int64_t nnz,
              const int64_t* colptr, const int32_t* rowidx, const double* values, double tau, double delta,
              blws_svd_backend* backend, const blws_mc_options* opts, const double* truth_ml, const double* truth_mr,
              int64_t r_true, double* u, double* sigma, double* v, int64_t cap, int64_t* rank,
              blws_solver_stats* stats, int64_t* predicted_ranks, int64_t* matvec_history, double* residual_history,
              int64_t hist_cap) {
    need(m > 0 && n > 0 && rows > 0 && rows <= m && nnz >= 0 && colptr && (nnz == 0 || (rowidx && values)),
         "mc_svt: bad observation");
    need(backend != nullptr, "mc_svt: null backend");
    for (int64_t p = 0; p < nnz; ++p) need(rowidx[p] >= 0 && rowidx[p] < rows, "mc_svt: row index out of range");
    Context& c = *ctx->ctx;
    McOptions o;
    if (opts) {
        o.tol_outer = opts->tol_outer;
        o.max_iter = opts->max_iter;
        o.initial_rank = opts->initial_rank;
        o.rank_increment = opts->rank_increment;
    }
    auto sol = blws::mc_svt(c, m, n, nnz, colptr, rowidx, values, tau, delta, *backend->b, o, truth_ml, truth_mr,
                            r_true, shard, rows);
    const Index k = sol.uv.rank();
    if (rank) *rank = k;
    if (k > cap) throw std::invalid_argument("mc_svt: output capacity too small");
    if (u) download(c, sol.uv.u(), u, rows);
    if (v) download(c, sol.uv.v(), v, n);
    if (sigma) std::copy(sol.uv.sigma.begin(), sol.uv.sigma.end(), sigma);
    put_stats(sol.stats, stats, predicted_ranks, matvec_history, residual_history, hist_cap);
}
}  // namespace

extern "C" {

int blws_rpca_adm(blws_context* ctx, int64_t m, const double* d, int64_t ldd, int where, double lambda,
                  blws_svd_backend* backend, const blws_rpca_options* opts, const double* truth, double* a_out,
                  double* e_out, blws_solver_stats* stats, int64_t* predicted_ranks, int64_t* matvec_history,
                  double* residual_history, int64_t hist_cap) {
    return guard([&] {
        rpca_entry(ctx, m, m, nullptr, d, ldd, where, lambda, backend, opts, truth, a_out, e_out, stats,
                   predicted_ranks, matvec_history, residual_history, hist_cap);
    });
}

int blws_rpca_adm_sharded(blws_context* ctx, int64_t m, int64_t rows, int64_t row0, const double* d, int64_t ldd,
                          int where, double lambda, blws_svd_backend* backend, const blws_rpca_options* opts,
                          const double* truth, double* a_out, double* e_out, blws_solver_stats* stats,
                          int64_t* predicted_ranks, int64_t* matvec_history, double* residual_history,
                          int64_t hist_cap) {
    return guard([&] {
        need(row0 >= 0 && row0 + rows <= m, "rpca_adm_sharded: rows outside [0, m)");
        const RowShard sh{m, row0};
        rpca_entry(ctx, m, rows, &sh, d, ldd, where, lambda, backend, opts, truth, a_out, e_out, stats,
                   predicted_ranks, matvec_history, residual_history, hist_cap);
    });
}

int blws_mc_svt(blws_context* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* colptr, const int32_t* rowidx,
                const double* values, double tau, double delta, blws_svd_backend* backend, const blws_mc_options* opts,
                const double* truth_ml, const double* truth_mr, int64_t r_true, double* u, double* sigma, double* v,
                int64_t cap, int64_t* rank, blws_solver_stats* stats, int64_t* predicted_ranks,
                int64_t* matvec_history, double* residual_history, int64_t hist_cap) {
    return guard([&] {
        mc_entry(ctx, m, m, nullptr, n, nnz, colptr, rowidx, values, tau, delta, backend, opts, truth_ml, truth_mr,
                 r_true, u, sigma, v, cap, rank, stats, predicted_ranks, matvec_history, residual_history, hist_cap);
    });
}

int blws_mc_svt_sharded(blws_context* ctx, int64_t m, int64_t rows, int64_t row0, int64_t n, int64_t nnz,
                        const int64_t* colptr, const int32_t* rowidx, const double* values, double tau, double delta,
                        blws_svd_backend* backend, const blws_mc_options* opts, const double* truth_ml,
                        const double* truth_mr, int64_t r_true, double* u, double* sigma, double* v, int64_t cap,
                        int64_t* rank, blws_solver_stats* stats, int64_t* predicted_ranks, int64_t* matvec_history,
                        double* residual_history, int64_t hist_cap) {
    return guard([&] {
        need(row0 >= 0 && row0 + rows <= m, "mc_svt_sharded: rows outside [0, m)");
        const RowShard sh{m, row0};
        mc_entry(ctx, m, rows, &sh, n, nnz, colptr, rowidx, values, tau, delta, backend, opts, truth_ml, truth_mr,
                 r_true, u, sigma, v, cap, rank, stats, predicted_ranks, matvec_history, residual_history, hist_cap);
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Kernel microbenchmarks (development / profiling only): average device time
// in microseconds of one call of a hot-path piece on a seeded input of order n
// (and width b where relevant). which: 0 chol_inv (SPD n x n), 1 sym_evd_top
// (n x n symmetric, want = n/2), 2 thin_qr (rows n, cols b), 3 gemm NN
// (n x b = n x n * n x b), 4 gemm TN (b x b = (n x b)^T (n x b)).
extern "C" int blws_microbench(blws_context* ctx, int which, int64_t n, int64_t b, int reps, double* us) {
    return guard([&] {
        Context& c = *ctx->ctx;
        std::vector<double> h(static_cast<size_t>(std::max<int64_t>(n * n, n * b)));
        Rng rng(12345);
        auto fill_host = [&](Index cnt) {
            for (Index i = 0; i < cnt; ++i) h[static_cast<size_t>(i)] = rng.normal();
        };
        cudaEvent_t e0, e1;
        BLWS_CUDA(cudaEventCreate(&e0));
        BLWS_CUDA(cudaEventCreate(&e1));
        float total = 0;
        if (which >= 5 && which <= 7) {
            // cholqr_factor on G = A^T A + n I (5), I + 1e-12 E (6), 4 I (7)
            fill_host(n * n);
            DMat a(c, n, n), g0(c, n, n), work(c, n, n), rinv(c, n, n);
            upload(c, a.view(), h.data(), n);
            if (which == 5) {
                gemm(c, true, false, n, n, n, 1.0, a.data(), a.ld, a.data(), a.ld, 0.0, g0.data(), g0.ld);
            } else {
                symmetrize(c, g0.view(), a.view());
                DMat id(c, n, n);
                std::vector<double> eye(static_cast<size_t>(n * n), 0.0);
                for (Index i = 0; i < n; ++i) eye[static_cast<size_t>(i + i * n)] = which == 6 ? 1.0 : 4.0;
                upload(c, id.view(), eye.data(), n);
                copy(c, g0.view(), g0.view(), which == 6 ? 1e-12 : 0.0);
                axpy(c, g0.view(), id.view(), 1.0);
            }
            DBuf<int> st(c, 1);
            DBuf<double> dg(c, 8);
            for (int r = -1; r < reps; ++r) {
                copy(c, work.view(), g0.view());
                BLWS_CUDA(cudaEventRecord(e0, c.stream()));
                cholqr_factor(c, work.view(), rinv.view(), nullptr, 0, nullptr, st.get(), dg.get(), dg.get() + 2,
                              nullptr, nullptr);
                BLWS_CUDA(cudaEventRecord(e1, c.stream()));
                BLWS_CUDA(cudaEventSynchronize(e1));
                float ms = 0;
                BLWS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                if (r >= 0) total += ms;
            }
            int hst = 0;
            BLWS_CUDA(cudaMemcpy(&hst, st.get(), sizeof(int), cudaMemcpyDeviceToHost));
            us[1] = hst;  // factor status (0 ok)
        } else if (which == 8 || which == 9) {
            // 8: Gram X^T X of an n x b panel; 9: X * R (n x b times b x b)
            fill_host(n * b);
            DMat x(c, n, b), y(c, n, b), gg(c, b, b);
            upload(c, x.view(), h.data(), n);
            for (int r = -1; r < reps; ++r) {
                BLWS_CUDA(cudaEventRecord(e0, c.stream()));
                if (which == 8)
                    gemm(c, true, false, b, b, n, 1.0, x.data(), x.ld, x.data(), x.ld, 0.0, gg.data(), gg.ld);
                else
                    gemm(c, false, false, n, b, b, 1.0, x.data(), x.ld, gg.data(), gg.ld, 0.0, y.data(), y.ld);
                BLWS_CUDA(cudaEventRecord(e1, c.stream()));
                BLWS_CUDA(cudaEventSynchronize(e1));
                float ms = 0;
                BLWS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                if (r >= 0) total += ms;
            }
        } else if (which == 11 || which == 12) {
            // 11: K7 (fused ALM update) on an n x n problem of rank b; 12: its E-only pass.
            // us[1] = checksum (sum of the residual partials / ||E||_F)
            total = static_cast<float>(alm_microbench(c, n, b, reps, which == 12, &us[1]) * reps / 1e3);
        } else if (which == 10) {
            // 10: gram16 (cluster Gram) of an n x b panel; us[1] = max |G16 - G_gemm| / max |G_gemm|
            fill_host(n * b);
            DMat x(c, n, b), g1(c, b, b), g2(c, b, b);
            upload(c, x.view(), h.data(), n);
            for (int r = -1; r < reps; ++r) {
                BLWS_CUDA(cudaEventRecord(e0, c.stream()));
                gram16(c, x.view(), g1.data(), g1.ld);
                BLWS_CUDA(cudaEventRecord(e1, c.stream()));
                BLWS_CUDA(cudaEventSynchronize(e1));
                float ms = 0;
                BLWS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                if (r >= 0) total += ms;
            }
            gemm(c, true, false, b, b, n, 1.0, x.data(), x.ld, x.data(), x.ld, 0.0, g2.data(), g2.ld);
            std::vector<double> h1(static_cast<size_t>(g1.ld * b)), h2(static_cast<size_t>(g2.ld * b));
            BLWS_CUDA(cudaMemcpy(h1.data(), g1.data(), h1.size() * 8, cudaMemcpyDeviceToHost));
            BLWS_CUDA(cudaMemcpy(h2.data(), g2.data(), h2.size() * 8, cudaMemcpyDeviceToHost));
            double md = 0, mx = 0;
            for (int64_t j = 0; j < b; ++j)
                for (int64_t i = 0; i < b; ++i) {
                    md = std::max(md, std::abs(h1[i + j * g1.ld] - h2[i + j * g2.ld]));
                    mx = std::max(mx, std::abs(h2[i + j * g2.ld]));
                }
            us[1] = mx > 0 ? md / mx : md;
        } else if (which == 0 || which == 1) {
            fill_host(n * n);
            DMat a(c, n, n), s(c, n, n), g0(c, n, n), work(c, n, n), rinv(c, n, n), vec(c, n, std::max<int64_t>(1, n / 2));
            upload(c, a.view(), h.data(), n);
            if (which == 0) {
                // G = A^T A + n I (SPD)
                gemm(c, true, false, n, n, n, 1.0, a.data(), a.ld, a.data(), a.ld, 0.0, g0.data(), g0.ld);
            } else {
                symmetrize(c, g0.view(), a.view());
            }
            DBuf<int> st(c, 1);
            DBuf<double> dg(c, 8), vals(c, static_cast<size_t>(n));
            for (int r = -1; r < reps; ++r) {
                copy(c, work.view(), g0.view());
                BLWS_CUDA(cudaEventRecord(e0, c.stream()));
                if (which == 0)
                    chol_inv_upper(c, work.view(), rinv.view(), st.get(), dg.get());
                else
                    sym_evd_top(c, work.view(), std::max<int64_t>(1, n / 2), vals.get(), vec.view());
                BLWS_CUDA(cudaEventRecord(e1, c.stream()));
                BLWS_CUDA(cudaEventSynchronize(e1));
                float ms = 0;
                BLWS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                if (r >= 0) total += ms;
            }
        } else if (which == 2) {
            fill_host(n * b);
            DMat x0(c, n, b), x(c, n, b);
            upload(c, x0.view(), h.data(), n);
            for (int r = -1; r < reps; ++r) {
                copy(c, x.view(), x0.view());
                BLWS_CUDA(cudaEventRecord(e0, c.stream()));
                blws::thin_qr(c, x.view(), nullptr);
                BLWS_CUDA(cudaEventRecord(e1, c.stream()));
                BLWS_CUDA(cudaEventSynchronize(e1));
                float ms = 0;
                BLWS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                if (r >= 0) total += ms;
            }
        } else {
            DMat a(c, n, which == 3 ? n : b), x(c, n, b), y(c, which == 3 ? n : b, b);
            fill(c, a.view(), 1.0 / static_cast<double>(n));
            fill(c, x.view(), 0.5);
            for (int r = -1; r < reps; ++r) {
                BLWS_CUDA(cudaEventRecord(e0, c.stream()));
                if (which == 3)
                    gemm(c, false, false, n, b, n, 1.0, a.data(), a.ld, x.data(), x.ld, 0.0, y.data(), y.ld);
                else
                    gemm(c, true, false, b, b, n, 1.0, x.data(), x.ld, x.data(), x.ld, 0.0, y.data(), y.ld);
                BLWS_CUDA(cudaEventRecord(e1, c.stream()));
                BLWS_CUDA(cudaEventSynchronize(e1));
                float ms = 0;
                BLWS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                if (r >= 0) total += ms;
            }
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *us = 1e3 * total / std::max(1, reps);
        if (which == 0) {
            double ph[4];
            chol_probe_read(ph);
            us[1] = ph[0];
            us[2] = ph[1];
            us[3] = ph[2];
            us[4] = ph[3];
        }
    });
}

int blws_mm_write_dense(const char* path, int64_t rows, int64_t cols, const double* a, int64_t lda) {
    return guard([&] {
        need(path && a && rows > 0 && cols > 0 && lda >= rows, "mm_write_dense: bad argument");
        mm_write_dense(path, rows, cols, a, lda);
    });
}
int blws_mm_write_sparse(const char* path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* colptr,
                         const int32_t* rowidx, const double* values) {
    return guard([&] {
        need(path && colptr && rows > 0 && cols > 0 && nnz >= 0, "mm_write_sparse: bad argument");
        need(nnz == 0 || (rowidx && values), "mm_write_sparse: null entries");
        mm_write_sparse(path, rows, cols, nnz, colptr, rowidx, values);
    });
}
int blws_mm_read_dense(const char* path, int64_t* rows, int64_t* cols, double* out, int64_t ldo) {
    return guard([&] {
        need(path && rows && cols, "mm_read_dense: bad argument");
        Index r = 0, c = 0;
        std::vector<double> data;
        mm_read_dense(path, &r, &c, out ? &data : nullptr);
        *rows = r;
        *cols = c;
        if (!out) return;
        need(ldo >= r, "mm_read_dense: ldo < rows");
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) out[i + j * ldo] = data[static_cast<size_t>(i + j * r)];
    });
}
int blws_mm_read_sparse(const char* path, int64_t* rows, int64_t* cols, int64_t* nnz, int64_t* colptr,
                        int32_t* rowidx, double* values) {
    return guard([&] {
        need(path && rows && cols && nnz, "mm_read_sparse: bad argument");
        Index r = 0, c = 0;
        std::vector<std::int64_t> cp;
        std::vector<std::int32_t> ri;
        std::vector<double> vs;
        mm_read_sparse(path, &r, &c, &cp, &ri, &vs);
        *rows = r;
        *cols = c;
        *nnz = static_cast<int64_t>(vs.size());
        if (!colptr) return;
        need(rowidx && values, "mm_read_sparse: null outputs");
        std::copy(cp.begin(), cp.end(), colptr);
        std::copy(ri.begin(), ri.end(), rowidx);
        std::copy(vs.begin(), vs.end(), values);
    });
}
