// Shared device/host infrastructure for the B200 BLWS library.
//
// Layout conventions: every matrix is column-major fp64 with an
// even leading dimension so that 16-byte cp.async / vector accesses stay
// aligned. A "stacked panel" holds an (m+n) x b block of the augmented
// operator [[0,W],[W^T,0]] (block_lanczos.hpp, augmented_operator.hpp): rows
// [0, m) are the top (W's row space, U), rows [mp, mp+n) the bottom (W's column
// space, V), with mp = round_up(m, 2); padding rows are kept at exactly zero.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace blws {

using Index = std::int64_t;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CommError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// A fresh NCCL unique id (128 bytes) for init_comm on every rank.
void comm_unique_id(void* out128);

#define BLWS_CUDA(call)                                                                         \
    do {                                                                                        \
        cudaError_t _e = (call);                                                                \
        if (_e != cudaSuccess)                                                                  \
            throw ::blws::CudaError(std::string(#call) + ": " + cudaGetErrorString(_e) + " (" + \
                                    __FILE__ + ":" + std::to_string(__LINE__) + ")");           \
    } while (0)

inline Index round_up(Index x, Index a) { return (x + a - 1) / a * a; }
inline Index ceil_div(Index x, Index a) { return (x + a - 1) / a; }

/// Per-solve device context: one stream, stream-ordered pool allocations,
/// pinned staging for the small device->host reads the control flow needs,
/// and a counter of kernel launches issued through it.
class Context {
public:
    // region timers: 0 K1, 1 EVD of T, 2 thin_qr, 3 Lanczos reseed, 4 Ritz checkpoints,
    // 5 blws_svd, 6 svt, 7 MC loop outside svt, 8 solver set-up, 9 solver epilogue
    static constexpr int kRegions = 10;
    explicit Context(int device);
    ~Context();
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    /// The stream work is enqueued on: the main stream, or the auxiliary one
    /// inside an AuxScope.
    cudaStream_t stream() const { return cur_ ? cur_ : stream_; }
    /// Row-sharded path: an NCCL communicator over `nranks`
    /// processes (one GPU each); allreduce_sum is a no-op without one.
    void init_comm(int nranks, int rank, const void* id128);
    /// Host-staged collectives (testing the sharded path with several ranks on
    /// one GPU): each collective synchronises the stream, copies the buffer to
    /// the host and calls `fn(buf, count, op, user)` (op 0 sum, 1 max), which
    /// must leave the reduced values in buf on every rank (e.g. a gloo
    /// allreduce). CUDA graphs are not captured while it is set.
    using HostAllreduceFn = int (*)(double* buf, size_t count, int op, void* user);
    void init_host_comm(int nranks, int rank, HostAllreduceFn fn, void* user);
    void allreduce_sum(double* p, size_t count);
    void allreduce_max(double* p, size_t count);
    /// recv (nranks x count) = every rank's `send` block in rank order.
    void allgather(const double* send, double* recv, size_t count);
    /// recv (count) = sum over the ranks of their send block `rank()`
    /// (send: nranks x count, used as scratch by the host-staged form).
    void reduce_scatter_sum(double* send, double* recv, size_t count);
    int nranks() const { return nranks_; }
    int rank() const { return rank_; }
    bool distributed() const { return has_comm() && nranks_ > 1; }
    bool has_comm() const { return comm_ != nullptr || host_fn_ != nullptr; }
    bool host_comm() const { return host_fn_ != nullptr; }
    /// Fork/join onto a second compute stream (see AuxScope).
    void fork_aux();
    void join_aux();
    void leave_aux() { cur_ = nullptr; }
    /// Second stream for host->device uploads that overlap queued kernels
    /// (created on first use; ordered against stream() with events).
    cudaStream_t copy_stream();
    int device() const { return device_; }
    int sm_count() const { return sms_; }

    void* alloc(size_t bytes);
    void free(void* p);
    void sync();
    /// Copies `count` doubles device->host through pinned staging and waits.
    void read(const double* dev, double* host, size_t count);
    void read_i64(const std::int64_t* dev, std::int64_t* host, size_t count);
    void write(double* dev, const double* host, size_t count);
    void note_launch(std::int64_t n = 1) { launches_ += n; }
    /// Optional CUDA-event timing of named regions (bench roofline evidence).
    void set_profiling(bool on) { profiling_ = on; }
    bool profiling() const { return profiling_; }
    void region_begin(int id);
    void region_end(int id, double flops, double bytes);
    /// total ms, count, flops, bytes of region `id` (syncs; resolves events)
    void region_stats(int id, double* ms, std::int64_t* count, double* flops, double* bytes);
    void region_reset();
    /// Regions inside a graph capture (profiling on at capture) are timed by
    /// one-thread %globaltimer stamp kernels writing into `stamps` (event
    /// record nodes cannot be used with cudaEventElapsedTime).
    struct CapturedRegion {
        int id, b, e;  // stamp indices
        double flops, bytes;
    };
    void begin_region_capture(std::uint64_t* stamps, int cap);
    std::vector<CapturedRegion> end_region_capture();
    /// After a replay has completed: add its region times to the stats.
    void add_replayed_regions(const std::vector<CapturedRegion>& regions, const std::uint64_t* stamps);
    std::int64_t launches() const { return launches_; }
    void check_launch(const char* what);

private:
    int device_ = 0;
    int sms_ = 148;
    cudaStream_t stream_ = nullptr;
    cudaStream_t copy_stream_ = nullptr;
    cudaStream_t aux_ = nullptr, cur_ = nullptr;
    bool aux_open_ = false;  // forked, not yet joined
    void* comm_ = nullptr;
    HostAllreduceFn host_fn_ = nullptr;
    void* host_user_ = nullptr;
    int nranks_ = 1, rank_ = 0;
    void host_allreduce(double* p, size_t count, int op);
    void destroy_comm() noexcept;
    cudaEvent_t fork_ev_ = nullptr, join_ev_ = nullptr;
    void* pinned_ = nullptr;
    size_t pinned_bytes_ = 0;
    std::int64_t launches_ = 0;
    bool profiling_ = false;
    struct Region {
        std::vector<cudaEvent_t> begin, end;
        double flops = 0, bytes = 0, ms = 0;
        std::int64_t count = 0;
    };
    Region regions_[kRegions];
    bool capturing_ = false;
    std::uint64_t* stamps_ = nullptr;
    int nstamps_ = 0, stamp_cap_ = 0;
    int open_[kRegions] = {};
    std::vector<CapturedRegion> captured_;
    void stamp(int idx);
    void ensure_pinned(size_t bytes);
};

/// Fork/join: work enqueued after construction runs on the context's auxiliary
/// stream, ordered after everything already queued on the main stream; main()
/// switches back to the main stream WITHOUT waiting (the second branch), and the
/// scope's end makes the main stream wait for the auxiliary branch. Independent
/// branches (the two products of a paired apply, the QRs of U and V) overlap;
/// under graph capture they become parallel branches of the graph. Buffers the
/// auxiliary branch uses must outlive the scope (declare them before it).
class AuxScope {
public:
    explicit AuxScope(Context& ctx) : ctx_(ctx) { ctx_.fork_aux(); }
    ~AuxScope() { ctx_.join_aux(); }
    void main() { ctx_.leave_aux(); }
    AuxScope(const AuxScope&) = delete;
    AuxScope& operator=(const AuxScope&) = delete;

private:
    Context& ctx_;
};

template <typename T>
class DBuf {
public:
    DBuf() = default;
    DBuf(Context& ctx, size_t count) : ctx_(&ctx), n_(count) {
        if (count) p_ = static_cast<T*>(ctx.alloc(sizeof(T) * count));
    }
    ~DBuf() { reset(); }
    DBuf(DBuf&& o) noexcept : ctx_(o.ctx_), p_(o.p_), n_(o.n_) {
        o.p_ = nullptr;
        o.n_ = 0;
    }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            reset();
            ctx_ = o.ctx_;
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    void reset() {
        if (p_ && ctx_) ctx_->free(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }

private:
    Context* ctx_ = nullptr;
    T* p_ = nullptr;
    size_t n_ = 0;
};

/// Non-owning column-major view.
struct View {
    double* p = nullptr;
    Index rows = 0, cols = 0, ld = 0;
    double* col(Index j) const { return p + j * ld; }
    View sub(Index r0, Index c0, Index nr, Index nc) const { return View{p + r0 + c0 * ld, nr, nc, ld}; }
    View left(Index k) const { return View{p, rows, k, ld}; }
    View cols_range(Index c0, Index k) const { return View{p + c0 * ld, rows, k, ld}; }
};

/// Owning column-major matrix on the device (even leading dimension).
struct DMat {
    DBuf<double> buf;
    Index rows = 0, cols = 0, ld = 0;
    DMat() = default;
    DMat(Context& ctx, Index r, Index c, bool zero = true);
    View view() const { return View{buf.get(), rows, cols, ld}; }
    double* data() const { return buf.get(); }
};

/// Geometry of a stacked (augmented) panel for an m x n operator.
struct Stack {
    Index m = 0, n = 0;
    Index mp() const { return round_up(m, 2); }
    Index ld() const { return mp() + round_up(n, 2); }
};

}  // namespace blws
