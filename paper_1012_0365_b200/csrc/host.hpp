// Host-side control flow of the BLWS hot path on the device.
//
// The algorithm objects mirror the reference's C++ API
// (/root/reference/proj/include/blws): same names, same control flow, same
// constants, same RNG draw order. All matrices live on the device; the host
// reads back only the scalars and small vectors the control flow branches on.
#pragma once
#include <atomic>
#include <cstdint>
#include <memory>
#include <optional>
#include <random>
#include <vector>

#include "common.cuh"

namespace blws {

// ------------------------------------------------------------------ rng
/// Bit-exact restatement of blws::Rng (core/rng.hpp:17-90). Draws happen on the
/// host so the device path consumes exactly the reference's stream.
class Rng {
public:
    explicit Rng(std::uint64_t seed) : engine_(seed), seed_(seed) {}
    Rng split(std::uint64_t tag) const { return Rng(seed_ ^ (0x9e3779b97f4a7c15ull * (tag + 1))); }
    std::uint64_t next_u64() { return engine_(); }
    double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    std::uint64_t uniform_index(std::uint64_t n);
    double normal();
    /// Column-major rows x cols draws (rng.hpp:63-68).
    void gaussian_matrix(Index rows, Index cols, double* out, Index ld);
    std::vector<double> gaussian_vector(Index n);
    std::vector<double> unit_vector(Index n);

private:
    std::mt19937_64 engine_;
    std::uint64_t seed_ = 0;
    double spare_ = 0.0;
    bool have_spare_ = false;
};

// ------------------------------------------------------------- operators
/// Device-resident W with the reference's application counter
/// (core/linear_operator.hpp:20-98). Only the paired products the augmented
/// view needs are exposed (augmented_operator.hpp:39-57).
struct SvdGraph;  // captured blws_svd launch sequence (host_core.cu)

/// Rows [0, sharded) of a panel are this rank's share of a row-sharded
/// operator: a reduction over the panel's rows allreduces their
/// contribution over the context's communicator and adds the replicated rows'
/// locally. sharded = 0: an ordinary (replicated) panel.
struct RowSplit {
    Index sharded = 0;
};

/// Row-shard geometry of a distributed operator: this rank holds rows
/// [row0, row0 + rows()) of an m_total x n matrix.
struct RowShard {
    Index m_total = 0, row0 = 0;
};

class LinearOperator {
public:
    explicit LinearOperator(Context& ctx) : ctx_(ctx) {}
    virtual ~LinearOperator() = default;
    virtual Index rows() const = 0;
    virtual Index cols() const = 0;
    Context& ctx() const { return ctx_; }

    /// (top, bot) = (W * right, W^T * left); counts right.cols (linear_operator.hpp:57-61).
    void apply_pair_block(View left, View right, View top, View bot) {
        count_ += right.cols;
        pair_block_impl(left, right, top, bot);
    }
    /// Single-vector paired apply; counts 1 (linear_operator.hpp:51-54).
    void apply_pair(const double* left, const double* right, double* top, double* bot) {
        count_ += 1;
        pair_impl(left, right, top, bot);
    }
    std::int64_t application_count() const { return count_; }
    /// If a deferred input check is pending (async upload), queue it now with
    /// its verdict (nonzero = non-finite entries) written to the device int
    /// `*flag`, instead of the synchronous check at the next use.
    virtual void defer_pending_check(int* flag) { (void)flag; }
    /// A deferred check found non-finite data: every later use throws until
    /// the operator is reassigned (the reference rejects it at assign time).
    virtual void mark_poisoned() {}
    /// Identity of the data the kernels read (graph cache key).
    virtual const void* data_key() const { return this; }
    void add_applications(std::int64_t n) { count_ += n; }
    /// Row-sharded operator: the local rows [row0, row0 + rows()) of m_total.
    void set_row_shard(Index m_total, Index row0);
    bool row_sharded() const { return shard_.m_total > 0; }
    const RowShard& shard() const { return shard_; }
    /// The split of a stacked panel of this operator: the top rows, and with
    /// column sharding the bottom rows too, are summed over the ranks.
    RowSplit panel_split() const;
    /// Column (n-side) sharding of the stacked panels: a row-sharded
    /// operator with a communicator keeps only the bottom rows [col0, col0 +
    /// chunk) of every panel (chunk = ceil(n / nranks); rows past n are zero
    /// padding), so V, the bottom halves of the Lanczos bases and every
    /// n-length vector are split across the ranks instead of replicated. The
    /// paired apply all-gathers X_bot before W X_bot and reduce-scatters W^T
    /// X_top. BLWS_NSHARD=0 keeps the bottom rows replicated.
    bool col_sharded() const;
    Index col_chunk() const;
    Index col0() const { return col_sharded() ? col_chunk() * ctx_.rank() : 0; }
    /// bottom rows of this operator's stacked panels (chunk, or n unsharded)
    Index panel_n() const { return col_sharded() ? col_chunk() : cols(); }
    std::vector<std::shared_ptr<SvdGraph>>& svd_graphs() { return svd_graphs_; }

protected:
    virtual void pair_block_impl(View left, View right, View top, View bot) = 0;
    virtual void pair_impl(const double* left, const double* right, double* top, double* bot) = 0;
    Context& ctx_;

private:
    std::int64_t count_ = 0;
    RowShard shard_;
    std::vector<std::shared_ptr<SvdGraph>> svd_graphs_;
};

/// Rows of the whole (possibly row-sharded) operator.
inline Index global_rows(const LinearOperator& w) { return w.row_sharded() ? w.shard().m_total : w.rows(); }

/// DenseOperator (linear_operator.hpp:102-131): column-major W on the device,
/// either owned or borrowed (a caller-owned device buffer).
class DenseOperator final : public LinearOperator {
public:
    DenseOperator(Context& ctx, Index m, Index n);
    /// Borrow caller memory (ld must be even, 16-byte aligned).
    DenseOperator(Context& ctx, Index m, Index n, double* dev, Index ld);
    ~DenseOperator() override;
    Index rows() const override { return m_; }
    Index cols() const override { return n_; }
    /// The held matrix; first waits for (and checks) a pending async upload.
    View w() const {
        ensure_ready();
        return View{p_, m_, n_, ld_};
    }
    /// Host upload with the reference's non-finite check (:113-116).
    void assign_host(const double* w, Index ldw);
    /// Asynchronous host upload (B200 extension of assign): the copy is queued
    /// on the context's copy stream behind every kernel already queued on the
    /// compute stream and returns at once, so it overlaps work in flight on
    /// another operator; the next use of this operator waits for it and runs
    /// the non-finite check then. `w` must stay valid (and pinned, for real
    /// overlap) until that use.
    void assign_host_async(const double* w, Index ldw);
    void defer_pending_check(int* flag) override;
    void mark_poisoned() override { poisoned_ = true; }
    const void* data_key() const override { return p_; }
    /// Device copy with the non-finite check.
    void assign_device(const double* w, Index ldw);
    /// Non-finite scan of the held matrix (throws std::invalid_argument).
    void check_finite();

protected:
    void pair_block_impl(View left, View right, View top, View bot) override;
    void pair_impl(const double* left, const double* right, double* top, double* bot) override;

private:
    void ensure_ready() const;
    Index m_, n_, ld_;
    DBuf<double> own_;
    double* p_ = nullptr;
    mutable bool pending_ = false;
    mutable bool poisoned_ = false;
    cudaEvent_t consumed_ = nullptr, ready_ = nullptr;
};

/// SparseOperator (linear_operator.hpp:136-169): the pattern in CSR (for W*x)
/// and CSC (= CSR of W^T, for W^T*x); values are assigned in compressed (CSC)
/// order like the reference and scattered to CSR order on the device.
class SparseOperator final : public LinearOperator {
public:
    SparseOperator(Context& ctx, Index m, Index n, Index nnz, const std::int64_t* colptr, const std::int32_t* rowidx,
                   const double* values_host);
    Index rows() const override { return m_; }
    Index cols() const override { return n_; }
    Index nnz() const { return nnz_; }
    void assign_values_device(const double* vals_csc);
    void assign_values_host(const double* vals_csc);
    const double* val_csc() const { return val_csc_.get(); }
    const std::int64_t* colptr_csc() const { return colptr_.get(); }
    const std::int32_t* rowidx_csc() const { return rowidx_.get(); }
    const std::int32_t* colof_csc() const { return colof_.get(); }

protected:
    void pair_block_impl(View left, View right, View top, View bot) override;
    void pair_impl(const double* left, const double* right, double* top, double* bot) override;

private:
    Index m_, n_, nnz_;
    DBuf<std::int64_t> rowptr_, colptr_, perm_;  // perm: csr position -> csc position
    DBuf<std::int32_t> colidx_, rowidx_, colof_;
    DBuf<double> val_csr_, val_csc_;
    bool csc_rows_ascend_ = true;  // the tiled SpMM may run on the CSC arrays (W^T x)
};

// ------------------------------------------------------------ warm start
/// WarmStart (block_lanczos.hpp:45-52): U (m x b) and V (n x b) kept as one
/// stacked panel (top / bottom), sigma on the host.
struct DWarm {
    Stack geo;
    DMat uv;  // geo.ld() x b
    std::vector<double> sigma;
    Index rank() const { return static_cast<Index>(sigma.size()); }
    View u() const { return View{uv.data(), geo.m, rank(), uv.ld}; }
    View v() const { return View{uv.data() + geo.mp(), geo.n, rank(), uv.ld}; }
    View panel() const { return View{uv.data(), uv.ld, rank(), uv.ld}; }
};
DWarm make_warm(Context& ctx, Index m, Index n, Index b);
DWarm copy_warm(Context& ctx, const DWarm& w, Index cols);

// ------------------------------------------------------------ dense pieces
/// thin_qr (core/qr.hpp:24-47) as CholQR2 (shifted CholQR3 fallback) in place:
/// X <- Q, R (b x b, optional) upper with positive diagonal; returns the rank,
/// counted as diag(R) > 1e-12 ||X||_F.
Index thin_qr(Context& ctx, View x, View* r_out, RowSplit split = {});

/// Upload / download a host column-major block into a device view.
void upload(Context& ctx, View dst, const double* host, Index ldh);
void download(Context& ctx, View src, double* host, Index ldh);

// ------------------------------------------------------------ block lanczos
struct BlwsResult {
    DWarm warm;
    bool padded = false, k_raised = false, terminated_early = false;
};
/// adapt_subspace (block_lanczos.hpp:157-187).
/// With `shard`, m is the local row count and the Gaussian padding of U is
/// drawn for all m_total rows (the reference's draw order) and sliced.
/// With chunk >= 0, V holds only rows [col0, col0 + chunk) of the n drawn
/// (a column-sharded panel; rows past n zero).
DWarm adapt_subspace(Context& ctx, const DWarm* warm, Index r_new, Index m, Index n, Rng& rng,
                     const RowShard* shard = nullptr, Index col0 = 0, Index chunk = -1);
/// blws_svd (block_lanczos.hpp:204-261).
BlwsResult blws_svd(LinearOperator& w, const DWarm& warm, Index k, Index r, Rng& rng);
extern std::atomic<std::int64_t> g_blws_deferred_fallbacks;
extern std::atomic<std::int64_t> g_blws_graph_launches;

/// Factorisation for tests: block_lanczos_procedure on the augmented view.
struct BlockLanczos {
    DMat q;
    std::vector<DMat> m, b;
    Index built = 0;
    bool terminated_early = false;
};
BlockLanczos block_lanczos_procedure(LinearOperator& w, View x1, Index k);

// ------------------------------------------------------------------ lanczos
struct LanczosStats {
    Index steps = 0, restarts = 0, converged = 0;
    bool all_converged = false;
};
struct LanczosOptions {
    double tol = 1e-8;
    Index max_k = 0;
    std::uint64_t seed = 0x1a2c705u;
};
struct PartialSvd {
    DWarm uv;  // sigma + stacked U/V (not re-orthonormalised, as the reference)
    LanczosStats stats;
};
/// lanczos_partial_svd (lanczos.hpp:289-329) on the augmented view.
PartialSvd lanczos_partial_svd(LinearOperator& w, Index r, const LanczosOptions& opts);
/// spectral_norm (lanczos.hpp:332-340).
double spectral_norm(LinearOperator& w, double tol = 1e-6, std::uint64_t seed = 0xb1f);

// --------------------------------------------------------------------- svt
struct RankPredictor {
    Index r = 10, increment = 5, max_rank = 1;
    std::vector<Index> history;
};
RankPredictor predict_rank(RankPredictor p, Index achieved, bool all_above);  // svt.hpp:58-64

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
    SvdBackend(Context& ctx, Kind k, Options o);
    struct Triplets {
        DWarm own;                    // cold Lanczos result (Lanczos kind)
        const DWarm* held = nullptr;  // the backend's warm start (Blws kind)
        Index converged = 0;
        bool hit_cap = false;
        const DWarm& get() const { return held ? *held : own; }
    };
    /// SvdBackend::compute (svt.hpp:104-186). ExactFull runs the device
    /// full_svd_small (small_dense.hpp:72-87, m + n <= 4096) on a dense copy.
    Triplets compute(LinearOperator& w, Index r);
    Kind kind() const { return kind_; }
    const std::optional<DWarm>& warm_state() const { return warm_; }
    void set_warm(DWarm w) { warm_ = std::move(w); }

private:
    Context& ctx_;
    Kind kind_;
    Options opt_;
    std::optional<DWarm> warm_;
    Rng rng_;
    Index growth_streak_ = 0;
};

struct SvtResult {
    DWarm trip;               // first `achieved` triplets, sigma already shrunk
    DBuf<double> sigma_dev;   // shrunk sigma on the device
    Index achieved_rank = 0;
    bool all_above_threshold = false;
};
/// svt (svt.hpp:216-254).
SvtResult svt(LinearOperator& w, double eps, SvdBackend& backend, RankPredictor& predictor);

// ----------------------------------------------------------------- solvers
struct SolverStats {
    Index iterations = 0;
    double wall_time_s = 0;
    std::int64_t matvec_count = 0, matvec_init = 0;
    double rel_err = -1;
    Index rank_hat = 0;
    std::int64_t e_l0 = -1, e_nnz = 0;
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
};
/// K7 microbenchmark (development): average device us of one fused ALM launch
/// on a seeded m x m problem of rank r (eonly: the end-of-solve E pass).
double alm_microbench(Context& ctx, Index m, Index r, int reps, bool eonly, double* checksum);

/// rpca_adm (solvers.hpp:72-157). d / truth / a_out / e_out are device
/// pointers with leading dimension ldd (truth, a_out, e_out may be null).
/// With `shard` (m_total = m), they hold this rank's `rows` rows starting at
/// shard->row0, and the solve runs row-sharded over the context's communicator.
SolverStats rpca_adm(Context& ctx, Index m, const double* d, Index ldd, double lambda, SvdBackend& backend,
                     const RpcaOptions& opts, const double* truth, double* a_out, double* e_out,
                     const RowShard* shard = nullptr, Index rows = 0);

struct McOptions {
    double tol_outer = 1e-4;
    Index max_iter = 500;
    Index initial_rank = 10, rank_increment = 5;
};
struct McSolution {
    DWarm uv;  // sigma = shrunk values
    SolverStats stats;
};
/// mc_svt (solvers.hpp:202-270); the observation is host CSC. With `shard`
/// (m_total = m), the CSC holds this rank's `rows` rows (row indices local to
/// the shard, nnz local), truth_ml its rows of ML; U comes back row-sharded.
McSolution mc_svt(Context& ctx, Index m, Index n, Index nnz, const std::int64_t* colptr, const std::int32_t* rowidx,
                  const double* vals, double tau, double delta, SvdBackend& backend, const McOptions& opts,
                  const double* truth_ml, const double* truth_mr, Index r_true, const RowShard* shard = nullptr,
                  Index rows = 0);

// region timer scope (Context::region_begin / region_end; a no-op unless profiling)
struct RegionGuard {
    Context& ctx;
    int id;
    RegionGuard(Context& c, int i) : ctx(c), id(i) { ctx.region_begin(id); }
    ~RegionGuard() {
        try {
            ctx.region_end(id, 0.0, 0.0);
        } catch (...) {
        }
    }
};

}  // namespace blws
