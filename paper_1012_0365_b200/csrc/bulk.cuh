// Block-wide global -> shared copies through the bulk-copy (TMA 1D) engine:
// one instruction moves the whole range, instead of a per-thread load loop
// whose L2 round trips serialise (~50 us for a 160 KB triangle on 128 threads).
#pragma once

#include "dgemm_tma.cuh"

namespace blws {

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     gemm_tma::su32(dst)),
                 "l"(src), "r"(bytes), "r"(gemm_tma::su32(bar))
                 : "memory");
}

// dst[0, count) = src[0, count) for every thread of the block (all threads must
// call it; ends with the data visible to all of them). dst and src 16-byte
// aligned; an odd tail element is copied by thread 0. `bar` is a shared uint64_t
// used once (parity 0).
__device__ __forceinline__ void block_load_bulk(double* dst, const double* __restrict__ src, long count,
                                                uint64_t* bar) {
    const long even = count & ~1L;  // 16-byte multiple
    if (threadIdx.x == 0) {
        gemm_tma::mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        constexpr long kChunk = 1L << 15;  // doubles per bulk op (256 KB), within the tx-count range
        gemm_tma::mbar_expect_tx(bar, static_cast<uint32_t>(even * 8));
        for (long o = 0; o < even; o += kChunk)
            bulk_g2s(dst + o, src + o, static_cast<uint32_t>(min(kChunk, even - o) * 8), bar);
        if (count & 1) dst[count - 1] = src[count - 1];
    }
    gemm_tma::mbar_wait(bar, 0);
    __syncthreads();  // the scalar tail
}

}  // namespace blws
