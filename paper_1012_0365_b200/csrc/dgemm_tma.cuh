// Tall-skinny FP64 GEMM (K1's W V / W^T U, the CholQR applies, the Ritz lift)
// with TMA tile staging: C (M x N, N <= BN) = alpha op(A) B + beta C, op(A) =
// A or A^T, all column-major.
//
// * One producer warp: a single lane issues cp.async.bulk.tensor.2d loads of
//   the op(A) and B tiles of each k-tile into a STAGES-deep ring, with an
//   mbarrier per stage completing on the transaction bytes ("full") and one
//   the consumers release it with ("empty"). Out-of-range rows / k are
//   zero-filled by TMA, so edge tiles need no separate path.
// * CONS consumer warps: each owns 16 rows x BN columns of the tile and issues
//   2 x BN/8 DMMA m8n8k4 per k-step from register fragments.
// * Shared layout: 128-byte swizzled TMA boxes, 16 doubles wide (no padding).
//   The k order inside each 16-wide box is permuted per DMMA k-step (a
//   reduction order change only, identical for A and B) so that the fragment
//   loads of all three layouts ([row][k] for B and A^T, [k][row] for A) are
//   free of bank conflicts under the swizzle:
//     step 0: k = {0, 3, 12, 15}, step 1: {1, 2, 13, 14},
//     step 2: {4, 7, 8, 11},      step 3: {5, 6, 9, 10}   (lane t -> k[t]).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "dgemm.cuh"

namespace blws {
namespace gemm_tma {

// CONS consumer warps x 16 rows = BM rows per CTA; one more warp produces
template <int CONS>
constexpr int threads() {
    return 32 * (CONS + 1);
}

template <int BK, int BN, int CONS>
struct Layout {
    static constexpr int BM = 16 * CONS;
    static constexpr int A_BYTES = BM * BK * 8;  // TA: BK/16 boxes [BM][16]; !TA: BM/16 boxes [BK][16]
    static constexpr int B_BYTES = BN * BK * 8;  // BK/16 boxes [BN][16]
    static constexpr int STAGE = A_BYTES + B_BYTES;
};
template <int BK, int BN, int STAGES, int CONS>
constexpr int smem_bytes() {
    return STAGES * Layout<BK, BN, CONS>::STAGE + 1024 + 2 * STAGES * 8;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}

// permuted k of lane t at k-step s inside a 16-wide box (see the header)
__device__ __forceinline__ int kperm_tab(int s, int t) {
    switch (s * 4 + t) {  // rows: steps 0..3; columns: lanes t = 0..3
        case 0: return 0;
        case 1: return 3;
        case 2: return 12;
        case 3: return 15;
        case 4: return 1;
        case 5: return 2;
        case 6: return 13;
        case 7: return 14;
        case 8: return 4;
        case 9: return 7;
        case 10: return 8;
        case 11: return 11;
        case 12: return 5;
        case 13: return 6;
        case 14: return 9;
        default: return 10;
    }
}

/// acc[mi][ni][e] += sum_k op(A)(m0 + 16 w + 8 mi + g, k) B(k, n0 + 8 ni + 2 t + e)
template <bool TA, int BN, int BK, int STAGES, int CONS>
__global__ void __launch_bounds__(threads<CONS>(), CONS <= 4 ? 2 : 1)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, double* C,
                     long ldc, long M, long N, long K, long kchunk, double alpha, double beta, double* ws) {
    using L = Layout<BK, BN, CONS>;
    constexpr int BM = L::BM;
    extern __shared__ __align__(1024) unsigned char smraw[];
    // 1024-byte aligned base by an offset on the shared array itself (a round trip
    // through uintptr_t loses the address space: every fragment load became a
    // generic LD with 64-bit address arithmetic instead of an LDS)
    unsigned char* sm = smraw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smraw)) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * L::STAGE);
    uint64_t* empty = full + STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long m0 = static_cast<long>(blockIdx.x) * BM, n0 = static_cast<long>(blockIdx.y) * BN;
    const long kbeg = static_cast<long>(blockIdx.z) * kchunk;
    const long kend = min(K, kbeg + kchunk);
    const int ntiles = kend > kbeg ? static_cast<int>((kend - kbeg + BK - 1) / BK) : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, CONS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == CONS) {
        // ---- producer
        if (lane == 0) {
            for (int kt = 0; kt < ntiles; ++kt) {
                const int s = kt % STAGES;
                mbar_wait(empty + s, ((kt / STAGES) & 1) ^ 1);
                mbar_expect_tx(full + s, L::STAGE);
                unsigned char* as = sm + s * L::STAGE;
                unsigned char* bs = as + L::A_BYTES;
                const int k0 = static_cast<int>(kbeg + static_cast<long>(kt) * BK);
                if (TA) {
#pragma unroll
                    for (int kb = 0; kb < BK / 16; ++kb)
                        tma_2d(as + kb * (BM * 128), &tmA, full + s, k0 + 16 * kb, static_cast<int>(m0));
                } else {
#pragma unroll
                    for (int q = 0; q < BM / 16; ++q)
                        tma_2d(as + q * (BK * 128), &tmA, full + s, static_cast<int>(m0) + 16 * q, k0);
                }
#pragma unroll
                for (int kb = 0; kb < BK / 16; ++kb)
                    tma_2d(bs + kb * (BN * 128), &tmB, full + s, k0 + 16 * kb, static_cast<int>(n0));
            }
        }
        return;
    }
    // ---- consumers
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp * 16;
    // per-lane byte offsets of the fragments for each k-step s of a 16-wide box
    int brow[4];   // B and A^T boxes ([row][16 k], row-in-atom = g)
    int arow[4][2];  // A boxes ([k][16 rows]) for mi = 0, 1
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int k = kperm_tab(s, t);
        brow[s] = g * 128 + (((k >> 1) ^ g) << 4) + (k & 1) * 8;
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
            const int r = mi * 8 + g;
            arow[s][mi] = k * 128 + ((((r >> 1) ^ (k & 7)) & 7) << 4) + (r & 1) * 8;
        }
    }
    double acc[2][BN / 8][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < BN / 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < ntiles; ++kt) {
        const int s = kt % STAGES;
        mbar_wait(full + s, (kt / STAGES) & 1);
        const unsigned char* as = sm + s * L::STAGE;
        const unsigned char* bs = as + L::A_BYTES;
#pragma unroll
        for (int kb = 0; kb < BK / 16; ++kb) {
#pragma unroll
            for (int st = 0; st < 4; ++st) {
                double af[2];
#pragma unroll
                for (int mi = 0; mi < 2; ++mi) {
                    const unsigned char* p =
                        TA ? as + kb * (BM * 128) + (wm + mi * 8) * 128 + brow[st]
                           : as + warp * (BK * 128) + kb * (16 * 128) + arow[st][mi];
                    af[mi] = *reinterpret_cast<const double*>(p);
                }
#pragma unroll
                for (int ni = 0; ni < BN / 8; ++ni) {
                    const double bf = *reinterpret_cast<const double*>(bs + kb * (BN * 128) + ni * 1024 + brow[st]);
                    gemm_detail::dmma(acc[0][ni], af[0], bf);
                    gemm_detail::dmma(acc[1][ni], af[1], bf);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
    }
    double* P = ws ? ws + static_cast<long>(blockIdx.z) * M * N : nullptr;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
        const long row = m0 + wm + mi * 8 + g;
        if (row >= M) continue;
#pragma unroll
        for (int ni = 0; ni < BN / 8; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const long col = n0 + ni * 8 + 2 * t + e;
                if (col >= N) continue;
                const double v = acc[mi][ni][e];
                if (P) {
                    P[row + col * M] = v;
                } else {
                    double* c = C + row + col * ldc;
                    *c = beta == 0.0 ? alpha * v : alpha * v + beta * *c;
                }
            }
    }
}

}  // namespace gemm_tma
}  // namespace blws
