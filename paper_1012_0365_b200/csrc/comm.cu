// Collectives for the row-sharded path: NCCL, loaded with
// dlopen on first use so the library itself has no hard NCCL dependency (one
// process per GPU; torch's bundled libnccl.so.2 is picked up when torch is
// already loaded, else the system one).
#include <dlfcn.h>

#include <cstdlib>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "ops.cuh"

namespace blws {
namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                   cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        // BLWS_NCCL_LIB (set by the Python package to the NCCL that torch
        // bundles): loading the system libnccl first would shadow it, and a
        // later `import torch` in the same process then fails on symbols only
        // the bundled version has
        void* h = nullptr;
        if (const char* lib = std::getenv("BLWS_NCCL_LIB")) h = dlopen(lib, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("NCCL not found: ") + dlerror();
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
        api.reduce_scatter = reinterpret_cast<decltype(api.reduce_scatter)>(dlsym(h, "ncclReduceScatter"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy || !api.all_gather ||
            !api.reduce_scatter)
            err = "NCCL: missing symbols";
    });
    if (!err.empty()) throw CommError(err);
    return api;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* s = nccl().error_string ? nccl().error_string(r) : "unknown";
        throw CommError(std::string(what) + ": " + s);
    }
}

}  // namespace

void comm_unique_id(void* out128) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
}

void Context::init_comm(int nranks, int rank, const void* id128) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("init_comm: bad rank / size");
    if (comm_) throw std::invalid_argument("init_comm: communicator already set");
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    BLWS_CUDA(cudaSetDevice(device_));
    ncclComm_t c = nullptr;
    check(nccl().comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
    comm_ = c;
    nranks_ = nranks;
    rank_ = rank;
}

void Context::init_host_comm(int nranks, int rank, HostAllreduceFn fn, void* user) {
    if (nranks < 1 || rank < 0 || rank >= nranks || !fn) throw std::invalid_argument("init_host_comm: bad arguments");
    if (comm_ || host_fn_) throw std::invalid_argument("init_host_comm: communicator already set");
    host_fn_ = fn;
    host_user_ = user;
    nranks_ = nranks;
    rank_ = rank;
}

void Context::host_allreduce(double* p, size_t count, int op) {
    // stream-ordered copies (a pageable cudaMemcpy to the device may return
    // before the DMA lands, and the context's streams do not sync with it)
    std::vector<double> h(count);
    BLWS_CUDA(cudaMemcpyAsync(h.data(), p, sizeof(double) * count, cudaMemcpyDeviceToHost, stream()));
    BLWS_CUDA(cudaStreamSynchronize(stream()));
    if (host_fn_(h.data(), count, op, host_user_) != 0) throw CommError("host allreduce callback failed");
    BLWS_CUDA(cudaMemcpyAsync(p, h.data(), sizeof(double) * count, cudaMemcpyHostToDevice, stream()));
    BLWS_CUDA(cudaStreamSynchronize(stream()));  // h is freed on return
}

void Context::allreduce_sum(double* p, size_t count) {
    if (count == 0) return;
    if (host_fn_) return host_allreduce(p, count, 0);
    if (!comm_) return;
    check(nccl().all_reduce(p, p, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm_), stream()),
          "ncclAllReduce");
}

void Context::allreduce_max(double* p, size_t count) {
    if (count == 0) return;
    if (host_fn_) return host_allreduce(p, count, 1);
    if (!comm_) return;
    check(nccl().all_reduce(p, p, count, ncclDouble, ncclMax, static_cast<ncclComm_t>(comm_), stream()),
          "ncclAllReduce");
}

// recv[r count, (r+1) count) = send of rank r (recv holds nranks x count)
void Context::allgather(const double* send, double* recv, size_t count) {
    if (count == 0) return;
    if (host_fn_) {
        // through the host allreduce: every rank contributes its block into a
        // zeroed buffer (x + 0 is exact)
        zero(*this, recv, sizeof(double) * count * static_cast<size_t>(nranks_));
        BLWS_CUDA(cudaMemcpyAsync(recv + count * static_cast<size_t>(rank_), send, sizeof(double) * count,
                                  cudaMemcpyDeviceToDevice, stream()));
        return host_allreduce(recv, count * static_cast<size_t>(nranks_), 0);
    }
    if (!comm_) {
        BLWS_CUDA(cudaMemcpyAsync(recv, send, sizeof(double) * count, cudaMemcpyDeviceToDevice, stream()));
        return;
    }
    check(nccl().all_gather(send, recv, count, ncclDouble, static_cast<ncclComm_t>(comm_), stream()),
          "ncclAllGather");
}

// recv (count) = sum over the ranks of send[rank count, (rank+1) count)
void Context::reduce_scatter_sum(double* send, double* recv, size_t count) {
    if (count == 0) return;
    if (host_fn_) {
        host_allreduce(send, count * static_cast<size_t>(nranks_), 0);  // send is scratch
        BLWS_CUDA(cudaMemcpyAsync(recv, send + count * static_cast<size_t>(rank_), sizeof(double) * count,
                                  cudaMemcpyDeviceToDevice, stream()));
        return;
    }
    if (!comm_) {
        BLWS_CUDA(cudaMemcpyAsync(recv, send, sizeof(double) * count, cudaMemcpyDeviceToDevice, stream()));
        return;
    }
    check(nccl().reduce_scatter(send, recv, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm_), stream()),
          "ncclReduceScatter");
}

void Context::destroy_comm() noexcept {
    if (!comm_) return;
    try {
        nccl().comm_destroy(static_cast<ncclComm_t>(comm_));
    } catch (...) {
    }
    comm_ = nullptr;
}

}  // namespace blws
