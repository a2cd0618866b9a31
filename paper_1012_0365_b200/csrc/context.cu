// Device context: stream, stream-ordered pool allocator, pinned staging.
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "ops.cuh"

namespace blws {

Context::Context(int device) : device_(device) {
    BLWS_CUDA(cudaSetDevice(device));
    BLWS_CUDA(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device));
    BLWS_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    // keep freed blocks cached in the default pool between calls
    cudaMemPool_t pool;
    BLWS_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    std::uint64_t threshold = UINT64_MAX;
    BLWS_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    ensure_pinned(1 << 20);
}

namespace {
__global__ void stamp_k(std::uint64_t* out) {
    std::uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *out = t;
}
}  // namespace

void Context::stamp(int idx) {
    if (idx >= stamp_cap_) throw std::logic_error("region stamps exhausted");
    stamp_k<<<1, 1, 0, stream()>>>(stamps_ + idx);
    check_launch("stamp_k");
}

void Context::region_begin(int id) {
    if (id < 0 || id >= kRegions) throw std::logic_error("region id out of range");
    if (capturing_) {
        if (!profiling_) return;
        open_[id] = nstamps_++;
        stamp(open_[id]);
        return;
    }
    if (!profiling_) return;
    cudaEvent_t e;
    BLWS_CUDA(cudaEventCreate(&e));
    BLWS_CUDA(cudaEventRecord(e, stream()));
    regions_[id].begin.push_back(e);
}

void Context::region_end(int id, double flops, double bytes) {
    if (id < 0 || id >= kRegions) throw std::logic_error("region id out of range");
    if (capturing_) {
        if (!profiling_) return;
        const int e = nstamps_++;
        stamp(e);
        captured_.push_back(CapturedRegion{id, open_[id], e, flops, bytes});
        return;
    }
    if (!profiling_) return;
    cudaEvent_t e;
    BLWS_CUDA(cudaEventCreate(&e));
    BLWS_CUDA(cudaEventRecord(e, stream()));
    regions_[id].end.push_back(e);
    regions_[id].flops += flops;
    regions_[id].bytes += bytes;
    regions_[id].count += 1;
}

void Context::region_stats(int id, double* ms, std::int64_t* count, double* flops, double* bytes) {
    Region& r = regions_[id];
    if (!r.begin.empty()) BLWS_CUDA(cudaEventSynchronize(r.end.back()));
    for (size_t i = 0; i < r.begin.size(); ++i) {
        float t = 0;
        BLWS_CUDA(cudaEventElapsedTime(&t, r.begin[i], r.end[i]));
        r.ms += t;
        cudaEventDestroy(r.begin[i]);
        cudaEventDestroy(r.end[i]);
    }
    r.begin.clear();
    r.end.clear();
    *ms = r.ms;
    *count = r.count;
    *flops = r.flops;
    *bytes = r.bytes;
}

void Context::begin_region_capture(std::uint64_t* stamps, int cap) {
    capturing_ = true;
    stamps_ = stamps;
    stamp_cap_ = cap;
    nstamps_ = 0;
    captured_.clear();
}

std::vector<Context::CapturedRegion> Context::end_region_capture() {
    capturing_ = false;
    stamps_ = nullptr;
    stamp_cap_ = 0;
    return std::move(captured_);
}

void Context::add_replayed_regions(const std::vector<CapturedRegion>& regions, const std::uint64_t* stamps) {
    if (!profiling_ || regions.empty()) return;
    int n = 0;
    for (const auto& c : regions) n = std::max(n, std::max(c.b, c.e) + 1);
    std::vector<std::uint64_t> h(static_cast<size_t>(n));
    BLWS_CUDA(cudaMemcpyAsync(h.data(), stamps, sizeof(std::uint64_t) * n, cudaMemcpyDeviceToHost, stream_));
    BLWS_CUDA(cudaStreamSynchronize(stream_));
    for (const auto& c : regions) {
        Region& r = regions_[c.id];
        r.ms += 1e-6 * static_cast<double>(h[static_cast<size_t>(c.e)] - h[static_cast<size_t>(c.b)]);
        r.flops += c.flops;
        r.bytes += c.bytes;
        r.count += 1;
    }
}

void Context::region_reset() {
    for (auto& r : regions_) {
        for (auto e : r.begin) cudaEventDestroy(e);
        for (auto e : r.end) cudaEventDestroy(e);
        r = Region{};
    }
}

void Context::fork_aux() {
    if (aux_open_) throw std::logic_error("fork_aux: nested fork");
    if (!aux_) {
        BLWS_CUDA(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking));
        BLWS_CUDA(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming));
        BLWS_CUDA(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming));
    }
    BLWS_CUDA(cudaEventRecord(fork_ev_, stream_));
    BLWS_CUDA(cudaStreamWaitEvent(aux_, fork_ev_, 0));
    cur_ = aux_;
    aux_open_ = true;
}

void Context::join_aux() {
    if (!aux_open_) return;
    cur_ = nullptr;
    aux_open_ = false;
    // no throw from a destructor path: record the failure for the next check
    if (cudaEventRecord(join_ev_, aux_) != cudaSuccess || cudaStreamWaitEvent(stream_, join_ev_, 0) != cudaSuccess)
        return;
}

cudaStream_t Context::copy_stream() {
    if (!copy_stream_) BLWS_CUDA(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
    return copy_stream_;
}

Context::~Context() {
    region_reset();
    destroy_comm();
    if (copy_stream_) {
        cudaStreamSynchronize(copy_stream_);
        cudaStreamDestroy(copy_stream_);
    }
    if (aux_) {
        cudaStreamSynchronize(aux_);
        cudaStreamDestroy(aux_);
        cudaEventDestroy(fork_ev_);
        cudaEventDestroy(join_ev_);
    }
    if (stream_) {
        cudaStreamSynchronize(stream_);
        cudaStreamDestroy(stream_);
    }
    if (pinned_) cudaFreeHost(pinned_);
}

void Context::ensure_pinned(size_t bytes) {
    if (bytes <= pinned_bytes_) return;
    if (pinned_) {
        BLWS_CUDA(cudaStreamSynchronize(stream_));
        BLWS_CUDA(cudaFreeHost(pinned_));
    }
    pinned_bytes_ = std::max(bytes, pinned_bytes_ * 2);
    BLWS_CUDA(cudaMallocHost(&pinned_, pinned_bytes_));
}

void* Context::alloc(size_t bytes) {
    void* p = nullptr;
    BLWS_CUDA(cudaMallocAsync(&p, bytes, stream()));
    return p;
}

void Context::free(void* p) { cudaFreeAsync(p, stream()); }

void Context::sync() { BLWS_CUDA(cudaStreamSynchronize(stream_)); }

void Context::check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void Context::read(const double* dev, double* host, size_t count) {
    if (!count) return;
    const size_t bytes = count * sizeof(double);
    if (bytes > (64u << 20)) {  // large reads go straight to pageable memory
        BLWS_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, stream_));
        sync();
        return;
    }
    ensure_pinned(bytes);
    BLWS_CUDA(cudaMemcpyAsync(pinned_, dev, bytes, cudaMemcpyDeviceToHost, stream_));
    sync();
    std::memcpy(host, pinned_, bytes);
}

void Context::read_i64(const std::int64_t* dev, std::int64_t* host, size_t count) {
    if (!count) return;
    const size_t bytes = count * sizeof(std::int64_t);
    ensure_pinned(bytes);
    BLWS_CUDA(cudaMemcpyAsync(pinned_, dev, bytes, cudaMemcpyDeviceToHost, stream_));
    sync();
    std::memcpy(host, pinned_, bytes);
}

void Context::write(double* dev, const double* host, size_t count) {
    if (!count) return;
    const size_t bytes = count * sizeof(double);
    if (bytes > (64u << 20)) {
        BLWS_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, stream_));
        sync();
        return;
    }
    ensure_pinned(bytes);
    // the staging buffer may still feed an earlier async copy
    BLWS_CUDA(cudaStreamSynchronize(stream_));
    std::memcpy(pinned_, host, bytes);
    BLWS_CUDA(cudaMemcpyAsync(dev, pinned_, bytes, cudaMemcpyHostToDevice, stream_));
}

DMat::DMat(Context& ctx, Index r, Index c, bool zero) : rows(r), cols(c), ld(std::max<Index>(round_up(r, 2), 2)) {
    buf = DBuf<double>(ctx, static_cast<size_t>(ld * std::max<Index>(c, 1)));
    if (zero) blws::zero(ctx, buf.get(), sizeof(double) * buf.size());
}

}  // namespace blws
