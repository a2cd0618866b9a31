// CSC -> CSR view of the MC observation pattern on the device (SparseOperator,
// the reference's SparseOperator keeps CSC only: linear_operator.hpp:136-169).
// Deterministic: CSR entries of a row are in column order (the CSC order of
// the positions), exactly as the reference-order host transpose produced them.
//   1. colof[p] = column of CSC position p (warp per column);
//   2. (row, p) pairs sorted by row with CUB's stable LSD radix sort, so equal
//      rows keep p ascending -> perm (CSR slot -> CSC position);
//   3. colidx[q] = colof[perm[q]];
//   4. rowptr = exclusive scan of the row histogram;
// with a device check of the row indices and the values (the reference throws
// std::invalid_argument for non-finite entries, linear_operator.hpp:147).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <stdexcept>

#include "ops.cuh"

namespace blws {
namespace {

constexpr int kT = 256;
inline unsigned blocks_for(long total, long cap = 8192) {
    return static_cast<unsigned>(std::max<long>(1, std::min<long>(cap, (total + kT - 1) / kT)));
}

__global__ void colof_k(long n, const std::int64_t* __restrict__ colptr, std::int32_t* colof) {
    const long warps = (static_cast<long>(gridDim.x) * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (long j = (blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x) >> 5; j < n; j += warps)
        for (long p = colptr[j] + lane; p < colptr[j + 1]; p += 32) colof[p] = static_cast<std::int32_t>(j);
}

// positions 0..nnz-1, the row histogram and the input checks (flags: bit 0 a
// row index out of [0, m), bit 1 a non-finite value, bit 2 a column whose row
// indices do not ascend -- not an error, but the tiled SpMM needs them sorted)
__global__ void csr_prep_k(long nnz, long m, const std::int32_t* __restrict__ rowidx, const double* __restrict__ val,
                           const std::int32_t* __restrict__ colof, std::int64_t* iota, std::int64_t* counts,
                           int* flags) {
    int bad = 0;
    for (long p = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<long>(gridDim.x) * blockDim.x) {
        iota[p] = p;
        const int r = rowidx[p];
        if (r < 0 || r >= m) {
            bad |= 1;
        } else {
            atomicAdd(reinterpret_cast<unsigned long long*>(counts + r), 1ull);
        }
        if (!isfinite(val[p])) bad |= 2;
        if (p > 0 && colof[p - 1] == colof[p] && rowidx[p - 1] > r) bad |= 4;
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicOr(flags, bad);
}

__global__ void csr_colidx_k(long nnz, const std::int64_t* __restrict__ perm, const std::int32_t* __restrict__ colof,
                             std::int32_t* colidx) {
    for (long q = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; q < nnz;
         q += static_cast<long>(gridDim.x) * blockDim.x)
        colidx[q] = colof[perm[q]];
}

}  // namespace

bool build_csr_device(Context& ctx, Index m, Index n, Index nnz, const std::int64_t* colptr,
                      const std::int32_t* rowidx, const double* val, std::int64_t* rowptr, std::int32_t* colidx,
                      std::int64_t* perm, std::int32_t* colof) {
    bool rows_ascend = true;
    DBuf<int> flags(ctx, 1);
    zero(ctx, flags.get(), sizeof(int));
    zero(ctx, rowptr, sizeof(std::int64_t) * static_cast<size_t>(m + 1));
    if (n > 0) {
        colof_k<<<blocks_for(n * 32), kT, 0, ctx.stream()>>>(n, colptr, colof);
        ctx.note_launch();
        ctx.check_launch("colof_k");
    }
    if (nnz > 0) {
        if (nnz > 0x7fffffffL || m + 1 > 0x7fffffffL)
            throw std::invalid_argument("SparseOperator: more than 2^31 - 1 observed entries");
        DBuf<std::int64_t> iota(ctx, static_cast<size_t>(nnz)), counts(ctx, static_cast<size_t>(m + 1));
        DBuf<std::int32_t> keys_out(ctx, static_cast<size_t>(nnz));
        zero(ctx, counts.get(), sizeof(std::int64_t) * static_cast<size_t>(m + 1));
        csr_prep_k<<<blocks_for(nnz), kT, 0, ctx.stream()>>>(nnz, m, rowidx, val, colof, iota.get(), counts.get(),
                                                             flags.get());
        ctx.note_launch();
        ctx.check_launch("csr_prep_k");
        int hf = 0;
        BLWS_CUDA(cudaMemcpyAsync(&hf, flags.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx.stream()));
        ctx.sync();
        if (hf & 1) throw std::invalid_argument("SparseOperator: row index out of range");
        if (hf & 2) throw std::invalid_argument("SparseOperator: non-finite entries");
        rows_ascend = !(hf & 4);
        int end_bit = 1;
        while (end_bit < 31 && (1L << end_bit) < m) ++end_bit;
        size_t tsort = 0, tscan = 0;
        BLWS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tsort, rowidx, keys_out.get(), iota.get(), perm,
                                                  static_cast<int>(nnz), 0, end_bit, ctx.stream()));
        BLWS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tscan, counts.get(), rowptr, static_cast<int>(m + 1),
                                                ctx.stream()));
        DBuf<unsigned char> tmp(ctx, std::max(tsort, tscan));
        BLWS_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tsort, rowidx, keys_out.get(), iota.get(), perm,
                                                  static_cast<int>(nnz), 0, end_bit, ctx.stream()));
        BLWS_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tscan, counts.get(), rowptr, static_cast<int>(m + 1),
                                                ctx.stream()));
        ctx.note_launch(2);
        csr_colidx_k<<<blocks_for(nnz), kT, 0, ctx.stream()>>>(nnz, perm, colof, colidx);
        ctx.note_launch();
        ctx.check_launch("csr_colidx_k");
    }
    return rows_ascend;
}

}  // namespace blws
