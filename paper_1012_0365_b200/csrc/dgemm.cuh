// FP64 tensor-core GEMM mainloop for sm_100a.
//
// sm_100a has no tcgen05 FP64 kind, so the FP64 tensor path is the warp-level
// DMMA `mma.sync.aligned.m8n8k4 ... f64` (SASS DMMA). Tiles of op(A) and op(B)
// are staged global->shared with 16-byte cp.async (LDGSTS) in a multi-stage
// ring; each of the 4 warps owns a 32x32 sub-tile of the 64x64 CTA tile
// (4x4 DMMA tiles, 32 fp64 accumulators per lane).
//
// All operands are column-major. TA / TB select op(X) = X^T, which changes only
// the shared-memory staging layout (the contiguous global dimension is always
// copied contiguously); shared strides are padded so that the fragment loads of
// one half-warp hit 32 distinct banks.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace blws {
namespace gemm_detail {

constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3, THREADS = 128;

template <bool TA>
struct ALayout {
    // TA=false: [BK][BM+4] (m contiguous); TA=true: [BM][BK+4] (k contiguous)
    static constexpr int LD = TA ? BK + 4 : BM + 4;
    static constexpr int SIZE = TA ? BM * (BK + 4) : BK * (BM + 4);
};
template <bool TB>
struct BLayout {
    // TB=false: [BN][BK+4] (k contiguous); TB=true: [BK][BN+4] (n contiguous)
    static constexpr int LD = TB ? BN + 4 : BK + 4;
    static constexpr int SIZE = TB ? BK * (BN + 4) : BN * (BK + 4);
};

template <bool TA, bool TB>
constexpr int smem_bytes() {
    return STAGES * (ALayout<TA>::SIZE + BLayout<TB>::SIZE) * 8;
}

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

/// Stage one BMxBK tile of op(A) and one BKxBN tile of op(B).
/// VEC = doubles per cp.async (2 -> 16 B, requires even ld and 16 B bases).
template <bool TA, bool TB, int VEC>
__device__ __forceinline__ void load_tile(double* As, double* Bs, const double* __restrict__ A, long lda,
                                          const double* __restrict__ B, long ldb, long M, long N, long m0,
                                          long n0, long k0, long kend) {
    const int tid = threadIdx.x;
    // ---- A
    if (!TA) {
        constexpr int CPR = BM / VEC;  // chunks per k-row
        for (int c = tid; c < CPR * BK; c += THREADS) {
            const int k = c / CPR, i = (c % CPR) * VEC;
            const long gi = m0 + i, gk = k0 + k;
            int nv = 0;
            if (gk < kend) nv = static_cast<int>(max(0L, min(static_cast<long>(VEC), M - gi)));
            const double* src = nv ? A + gi + gk * lda : A;
            double* dst = As + k * ALayout<TA>::LD + i;
            if (VEC == 2) cp_async16(dst, src, nv * 8); else cp_async8(dst, src, nv * 8);
        }
    } else {
        constexpr int CPR = BK / VEC;
        for (int c = tid; c < CPR * BM; c += THREADS) {
            const int i = c / CPR, k = (c % CPR) * VEC;
            const long gi = m0 + i, gk = k0 + k;
            int nv = 0;
            if (gi < M) nv = static_cast<int>(max(0L, min(static_cast<long>(VEC), kend - gk)));
            const double* src = nv ? A + gk + gi * lda : A;
            double* dst = As + i * ALayout<TA>::LD + k;
            if (VEC == 2) cp_async16(dst, src, nv * 8); else cp_async8(dst, src, nv * 8);
        }
    }
    // ---- B
    if (!TB) {
        constexpr int CPR = BK / VEC;
        for (int c = tid; c < CPR * BN; c += THREADS) {
            const int j = c / CPR, k = (c % CPR) * VEC;
            const long gj = n0 + j, gk = k0 + k;
            int nv = 0;
            if (gj < N) nv = static_cast<int>(max(0L, min(static_cast<long>(VEC), kend - gk)));
            const double* src = nv ? B + gk + gj * ldb : B;
            double* dst = Bs + j * BLayout<TB>::LD + k;
            if (VEC == 2) cp_async16(dst, src, nv * 8); else cp_async8(dst, src, nv * 8);
        }
    } else {
        constexpr int CPR = BN / VEC;
        for (int c = tid; c < CPR * BK; c += THREADS) {
            const int k = c / CPR, j = (c % CPR) * VEC;
            const long gj = n0 + j, gk = k0 + k;
            int nv = 0;
            if (gk < kend) nv = static_cast<int>(max(0L, min(static_cast<long>(VEC), N - gj)));
            const double* src = nv ? B + gj + gk * ldb : B;
            double* dst = Bs + k * BLayout<TB>::LD + j;
            if (VEC == 2) cp_async16(dst, src, nv * 8); else cp_async8(dst, src, nv * 8);
        }
    }
}

/// acc[mi][ni][e] += sum_k op(A)(m0+wm+mi*8+g, k) * op(B)(k, n0+wn+ni*8+2t+e)
/// over k in [kbeg, kend). smem must hold smem_bytes<TA,TB>().
template <bool TA, bool TB, int VEC>
__device__ __forceinline__ void mainloop(double (&acc)[4][4][2], double* smem, const double* __restrict__ A,
                                         long lda, const double* __restrict__ B, long ldb, long M, long N,
                                         long m0, long n0, long kbeg, long kend) {
    double* As = smem;
    double* Bs = smem + STAGES * ALayout<TA>::SIZE;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    const long ntiles = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ntiles)
            load_tile<TA, TB, VEC>(As + s * ALayout<TA>::SIZE, Bs + s * BLayout<TB>::SIZE, A, lda, B, ldb, M, N,
                                   m0, n0, kbeg + s * BK, kend);
        cp_commit();
    }
    for (long kt = 0; kt < ntiles; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        const long pf = kt + STAGES - 1;
        if (pf < ntiles) {
            const int ps = static_cast<int>(pf % STAGES);
            load_tile<TA, TB, VEC>(As + ps * ALayout<TA>::SIZE, Bs + ps * BLayout<TB>::SIZE, A, lda, B, ldb, M,
                                   N, m0, n0, kbeg + pf * BK, kend);
        }
        cp_commit();
        const int st = static_cast<int>(kt % STAGES);
        const double* as = As + st * ALayout<TA>::SIZE;
        const double* bs = Bs + st * BLayout<TB>::SIZE;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                const int row = wm + mi * 8 + g;
                af[mi] = TA ? as[row * ALayout<TA>::LD + kk + t] : as[(kk + t) * ALayout<TA>::LD + row];
            }
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                const int colj = wn + ni * 8 + g;
                bf[ni] = TB ? bs[(kk + t) * BLayout<TB>::LD + colj] : bs[colj * BLayout<TB>::LD + kk + t];
            }
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], af[mi], bf[ni]);
        }
    }
    cp_wait<0>();
}

}  // namespace gemm_detail
}  // namespace blws

namespace blws {
namespace gemm_ts {
// Tall-skinny output variant: the CTA covers all BN (<= 128) output columns;
// the 4 warps split BM = 64 rows (16 each), so a warp issues 2 x BN/8 DMMAs per
// k-step from 2 A and BN/8 B fragments. Used for W*X, W^T*X, X*S with b <= 128
// (and in 4 column tiles of 104 for b ~ 405). Requires 16-byte aligned operands.
using gemm_detail::cp_async16;
using gemm_detail::cp_commit;
using gemm_detail::cp_wait;
using gemm_detail::dmma;

// BK = 32 with a double buffer (95 KB per CTA, two CTAs per SM): one barrier and
// one round of cp.async per 8 k-steps. Measured against BK = 16 x 4 stages and
// BK = 24 x 3 stages at C2's K1 shapes: 245 vs 265 / 266 us per paired product.
constexpr int BM = 64, BK = 32, STAGES = 2, THREADS = 128;

template <bool TA>
struct AL {
    static constexpr int LD = TA ? BK + 4 : BM + 4;
    static constexpr int SIZE = TA ? BM * (BK + 4) : BK * (BM + 4);
};
template <int BN>
struct BL {  // op(B) = B (k contiguous): [BN][BK+4]
    static constexpr int LD = BK + 4;
    static constexpr int SIZE = BN * (BK + 4);
};
template <bool TA, int BN>
constexpr int smem_bytes() {
    return STAGES * (AL<TA>::SIZE + BL<BN>::SIZE) * 8;
}

template <bool TA, int BN>
__device__ __forceinline__ void load_tile(double* As, double* Bs, const double* __restrict__ A, long lda,
                                          const double* __restrict__ B, long ldb, long M, long N, long m0, long n0,
                                          long k0, long kend) {
    const int tid = threadIdx.x;
    if (!TA) {
        constexpr int CPR = BM / 2;
        for (int c = tid; c < CPR * BK; c += THREADS) {
            const int k = c / CPR, i = (c % CPR) * 2;
            const long gi = m0 + i, gk = k0 + k;
            int nv = 0;
            if (gk < kend) nv = static_cast<int>(max(0L, min(2L, M - gi)));
            cp_async16(As + k * AL<TA>::LD + i, nv ? A + gi + gk * lda : A, nv * 8);
        }
    } else {
        constexpr int CPR = BK / 2;
        for (int c = tid; c < CPR * BM; c += THREADS) {
            const int i = c / CPR, k = (c % CPR) * 2;
            const long gi = m0 + i, gk = k0 + k;
            int nv = 0;
            if (gi < M) nv = static_cast<int>(max(0L, min(2L, kend - gk)));
            cp_async16(As + i * AL<TA>::LD + k, nv ? A + gk + gi * lda : A, nv * 8);
        }
    }
    constexpr int CPR = BK / 2;
    for (int c = tid; c < CPR * BN; c += THREADS) {
        const int j = c / CPR, k = (c % CPR) * 2;
        const long gj = n0 + j, gk = k0 + k;
        int nv = 0;
        if (gj < N) nv = static_cast<int>(max(0L, min(2L, kend - gk)));
        cp_async16(Bs + j * BL<BN>::LD + k, nv ? B + gk + gj * ldb : B, nv * 8);
    }
}

// DMMA without `volatile`: register effects only, so the compiler may interleave
// it with the cp.async prefetch and the fragment loads
__device__ __forceinline__ void dmma_nv(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

// Interior tile (all BM rows of op(A) inside M, the whole BK inside the k range):
// no clamping; B columns beyond N are zero-filled (their validity is fixed per CTA).
template <bool TA, int BN>
__device__ __forceinline__ void load_tile_fast(double* As, double* Bs, const double* __restrict__ A, long lda,
                                               const double* __restrict__ B, long ldb, long N, long m0, long n0,
                                               long k0) {
    const int tid = threadIdx.x;
    if (!TA) {
        constexpr int CPR = BM / 2;
#pragma unroll
        for (int c = tid; c < CPR * BK; c += THREADS) {
            const int k = c / CPR, i = (c % CPR) * 2;
            cp_async16(As + k * AL<TA>::LD + i, A + (m0 + i) + (k0 + k) * lda, 16);
        }
    } else {
        constexpr int CPR = BK / 2;
#pragma unroll
        for (int c = tid; c < CPR * BM; c += THREADS) {
            const int i = c / CPR, k = (c % CPR) * 2;
            cp_async16(As + i * AL<TA>::LD + k, A + (k0 + k) + (m0 + i) * lda, 16);
        }
    }
    constexpr int CPR = BK / 2;
#pragma unroll
    for (int c = tid; c < CPR * BN; c += THREADS) {
        const int j = c / CPR, k = (c % CPR) * 2;
        const bool ok = n0 + j < N;
        cp_async16(Bs + j * BL<BN>::LD + k, ok ? B + (k0 + k) + (n0 + j) * ldb : B, ok ? 16 : 0);
    }
}

constexpr bool kPrefetchLate = false;  // measured: issuing the prefetch first is faster for W V

/// acc[mi][ni][e] += op(A)(m0 + 16w + 8mi + g, k) * B(k, n0 + 8ni + 2t + e)
template <bool TA, int BN>
__device__ __forceinline__ void mainloop(double (&acc)[2][BN / 8][2], double* smem, const double* __restrict__ A,
                                         long lda, const double* __restrict__ B, long ldb, long M, long N, long m0,
                                         long n0, long kbeg, long kend) {
    double* As = smem;
    double* Bs = smem + STAGES * AL<TA>::SIZE;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp * 16;
    const long ntiles = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
    const bool rows_in = m0 + BM <= M;
    auto stage_tile = [&](long tile, int slot) {
        const long k0 = kbeg + tile * BK;
        if (rows_in && k0 + BK <= kend)
            load_tile_fast<TA, BN>(As + slot * AL<TA>::SIZE, Bs + slot * BL<BN>::SIZE, A, lda, B, ldb, N, m0, n0, k0);
        else
            load_tile<TA, BN>(As + slot * AL<TA>::SIZE, Bs + slot * BL<BN>::SIZE, A, lda, B, ldb, M, N, m0, n0, k0,
                              kend);
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ntiles) stage_tile(s, s);
        cp_commit();
    }
    for (long kt = 0; kt < ntiles; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        const int st = static_cast<int>(kt % STAGES);
        const double* as = As + st * AL<TA>::SIZE;
        const double* bs = Bs + st * BL<BN>::SIZE;
        const long pf = kt + STAGES - 1;
        if (!kPrefetchLate) {
            if (pf < ntiles) stage_tile(pf, static_cast<int>(pf % STAGES));
            cp_commit();
        }
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[2];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) {
                const int row = wm + mi * 8 + g;
                af[mi] = TA ? as[row * AL<TA>::LD + kk + t] : as[(kk + t) * AL<TA>::LD + row];
            }
#pragma unroll
            for (int ni = 0; ni < BN / 8; ++ni) {
                const double bf = bs[(ni * 8 + g) * BL<BN>::LD + kk + t];
                dmma(acc[0][ni], af[0], bf);
                dmma(acc[1][ni], af[1], bf);
            }
            if (kPrefetchLate && kk == 0) {
                // prefetch after the first k-step, so the copies overlap the math
                // (the slot written was consumed two iterations ago: safe after the barrier)
                if (pf < ntiles) stage_tile(pf, static_cast<int>(pf % STAGES));
                cp_commit();
            }
        }
    }
    cp_wait<0>();
}

}  // namespace gemm_ts
}  // namespace blws
