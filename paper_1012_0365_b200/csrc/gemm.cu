// DMMA GEMM kernels (K1 block products W*X / W^T*X, K2 Grams, K5 Ritz lift).
#include <algorithm>
#include <cstdlib>

#include "dgemm.cuh"
#include "dgemm_tma.cuh"
#include "ops.cuh"

namespace blws {
using namespace gemm_detail;

namespace {

/// Plain GEMM: partial = true writes the raw split-K partial sum into
/// ws + blockIdx.z * M * N (ld M); otherwise C = alpha*acc + beta*C.
template <bool TA, bool TB, int VEC>
__global__ void __launch_bounds__(THREADS) dgemm_kernel(const double* __restrict__ A, long lda,
                                                        const double* __restrict__ B, long ldb, double* C, long ldc,
                                                        long M, long N, long K, long kchunk, double alpha,
                                                        double beta, double* ws) {
    extern __shared__ __align__(16) double smem[];
    const long m0 = static_cast<long>(blockIdx.x) * BM, n0 = static_cast<long>(blockIdx.y) * BN;
    const long kbeg = static_cast<long>(blockIdx.z) * kchunk;
    const long kend = min(K, kbeg + kchunk);
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    mainloop<TA, TB, VEC>(acc, smem, A, lda, B, ldb, M, N, m0, n0, kbeg, kend);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    double* P = ws ? ws + static_cast<long>(blockIdx.z) * M * N : nullptr;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
        const long row = m0 + wm + mi * 8 + g;
        if (row >= M) continue;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const long col = n0 + wn + ni * 8 + 2 * t + e;
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

/// C = alpha * sum_z ws[z] + beta * C  (ws slices are M x N, ld M)
__global__ void splitk_reduce(const double* __restrict__ ws, long M, long N, int S, double alpha, double beta,
                              double* C, long ldc) {
    const long total = M * N;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        // slices summed in order; their loads issued 8 at a time (a plain loop
        // left one global latency per slice on the chain: 11 us for a 62-slice
        // 100 x 100 Gram)
        double s = 0.0;
        int z = 0;
        for (; z + 8 <= S; z += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = ws[(z + q) * total + idx];
#pragma unroll
            for (int q = 0; q < 8; ++q) s += v[q];
        }
        for (; z < S; ++z) s += ws[z * total + idx];
        const long i = idx % M, j = idx / M;
        double* c = C + i + j * ldc;
        *c = beta == 0.0 ? alpha * s : alpha * s + beta * *c;
    }
}

void launch_splitk_reduce(Context& ctx, const double* ws, long M, long N, int S, double alpha, double beta, double* C,
                          long ldc) {
    const long total = M * N;
    splitk_reduce<<<static_cast<unsigned>(std::min<long>(2048, (total + 255) / 256)), 256, 0, ctx.stream()>>>(
        ws, M, N, S, alpha, beta, C, ldc);
    ctx.note_launch();
    ctx.check_launch("splitk_reduce");
}

__global__ void scale_kernel(double* C, long ldc, long M, long N, double beta) {
    const long total = M * N;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx % M, j = idx / M;
        C[i + j * ldc] = beta == 0.0 ? 0.0 : beta * C[i + j * ldc];
    }
}

template <bool TA, bool TB, int VEC>
void launch(Context& ctx, dim3 grid, const double* A, long lda, const double* B, long ldb, double* C, long ldc,
            long M, long N, long K, long kchunk, double alpha, double beta, double* ws) {
    constexpr int bytes = smem_bytes<TA, TB>();
    static bool configured = false;  // per-instantiation, per process
    if (!configured) {
        BLWS_CUDA(cudaFuncSetAttribute(dgemm_kernel<TA, TB, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        configured = true;
    }
    dgemm_kernel<TA, TB, VEC><<<grid, THREADS, bytes, ctx.stream()>>>(A, lda, B, ldb, C, ldc, M, N, K, kchunk, alpha,
                                                                      beta, ws);
    ctx.note_launch();
    ctx.check_launch("dgemm_kernel");
}

template <int VEC>
void dispatch(Context& ctx, bool ta, bool tb, dim3 grid, const double* A, long lda, const double* B, long ldb,
              double* C, long ldc, long M, long N, long K, long kchunk, double alpha, double beta, double* ws) {
    if (!ta && !tb) launch<false, false, VEC>(ctx, grid, A, lda, B, ldb, C, ldc, M, N, K, kchunk, alpha, beta, ws);
    else if (ta && !tb) launch<true, false, VEC>(ctx, grid, A, lda, B, ldb, C, ldc, M, N, K, kchunk, alpha, beta, ws);
    else if (!ta && tb) launch<false, true, VEC>(ctx, grid, A, lda, B, ldb, C, ldc, M, N, K, kchunk, alpha, beta, ws);
    else launch<true, true, VEC>(ctx, grid, A, lda, B, ldb, C, ldc, M, N, K, kchunk, alpha, beta, ws);
}

template <bool TA, int BN>
__global__ void __launch_bounds__(gemm_ts::THREADS) dgemm_ts_kernel(const double* __restrict__ A, long lda,
                                                                    const double* __restrict__ B, long ldb, double* C,
                                                                    long ldc, long M, long N, long K, long kchunk,
                                                                    double alpha, double beta, double* ws) {
    extern __shared__ __align__(16) double smem[];
    const long m0 = static_cast<long>(blockIdx.x) * gemm_ts::BM, n0 = static_cast<long>(blockIdx.y) * BN;
    const long kbeg = static_cast<long>(blockIdx.z) * kchunk;
    const long kend = min(K, kbeg + kchunk);
    double acc[2][BN / 8][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < BN / 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    gemm_ts::mainloop<TA, BN>(acc, smem, A, lda, B, ldb, M, N, m0, n0, kbeg, kend);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    double* P = ws ? ws + static_cast<long>(blockIdx.z) * M * N : nullptr;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
        const long row = m0 + warp * 16 + mi * 8 + g;
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

template <bool TA, int BN>
int ts_occupancy(int dev) {
    static int occ[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (!occ[dev & 7]) {
        constexpr int bytes = gemm_ts::smem_bytes<TA, BN>();
        BLWS_CUDA(cudaFuncSetAttribute(dgemm_ts_kernel<TA, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        int o = 0;
        BLWS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, dgemm_ts_kernel<TA, BN>, gemm_ts::THREADS, bytes));
        occ[dev & 7] = std::max(o, 1);
    }
    return occ[dev & 7];
}

// ---- TMA variant (dgemm_tma.cuh): tensor maps encoded per call through the
// driver entry point (no libcuda link dependency), passed as __grid_constant__.
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_tiled() {
    static const EncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeTiled>(nullptr);
        return reinterpret_cast<EncodeTiled>(p);
    }();
    return fn;
}

// column-major `outer` x ... matrix seen as a 2D tensor {inner, outer} with row
// stride ld; boxes of {16 (128 B, swizzled), box_outer}
bool tensor_map(CUtensorMap* map, const double* base, long inner, long outer, long ld, int box_outer) {
    const EncodeTiled fn = encode_tiled();
    if (!fn || reinterpret_cast<uintptr_t>(base) % 16 != 0 || (ld * 8) % 16 != 0 || inner < 1 || outer < 1)
        return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
    const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(box_outer)};
    const cuuint32_t es[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr int kTmaBK = 32, kTmaStages = 2, kTmaCons = 4;

template <bool TA, int BN>
bool launch_tma(Context& ctx, const double* A, long lda, const double* B, long ldb, double* C, long ldc, long M,
                long N, long K, double alpha, double beta) {
    static const bool enabled = [] {
        const char* e = std::getenv("BLWS_TMA");
        return !(e && e[0] == '0');
    }();
    if (!enabled || M > (1L << 31) - 64 || K > (1L << 31) - 64) return false;
    CUtensorMap ta, tb;
    // op(A) tile: TA -> A is K x M (k contiguous) boxes {16 k, 64 rows}; else M x K boxes {16 rows, BK k}
    constexpr int BM = gemm_tma::Layout<kTmaBK, BN, kTmaCons>::BM, THREADS = gemm_tma::threads<kTmaCons>();
    if (!(TA ? tensor_map(&ta, A, K, M, lda, BM) : tensor_map(&ta, A, M, K, lda, kTmaBK))) return false;
    if (!tensor_map(&tb, B, K, N, ldb, BN)) return false;
    constexpr int bytes = gemm_tma::smem_bytes<kTmaBK, BN, kTmaStages, kTmaCons>();
    auto kern = gemm_tma::dgemm_tma_kernel<TA, BN, kTmaBK, kTmaStages, kTmaCons>;
    static int occ = 0;
    if (!occ) {
        BLWS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        BLWS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, bytes));
        occ = std::max(occ, 1);
    }
    const long mt = ceil_div(M, BM), nt = ceil_div(N, BN);
    const long ktiles = ceil_div(K, kTmaBK);
    const long slots = static_cast<long>(ctx.sm_count()) * occ;
    long S = 1;  // split-K so the CTA count fills whole waves (as launch_ts)
    const long tiles = mt * nt;
    if (tiles < 2 * slots) {
        const long smax = std::max<long>(1, std::min<long>(64, ktiles / 4));
        double best = 1e30;
        for (long s = 1; s <= smax; ++s) {
            const long waves = ceil_div(tiles * s, slots);
            const double cost = static_cast<double>(waves) / s + (s > 1 ? 0.02 : 0.0);
            if (cost < best - 1e-12) {
                best = cost;
                S = s;
            }
        }
    }
    const long kchunk = ceil_div(ktiles, S) * kTmaBK;
    S = ceil_div(K, kchunk);
    DBuf<double> ws;
    if (S > 1) ws = DBuf<double>(ctx, static_cast<size_t>(S * M * N));
    dim3 grid(static_cast<unsigned>(mt), static_cast<unsigned>(nt), static_cast<unsigned>(S));
    kern<<<grid, THREADS, bytes, ctx.stream()>>>(ta, tb, C, ldc, M, N, K, kchunk, alpha, beta,
                                                           S > 1 ? ws.get() : nullptr);
    ctx.note_launch();
    ctx.check_launch("dgemm_tma_kernel");
    if (S > 1) {
        const long total = M * N;
        launch_splitk_reduce(ctx, ws.get(), M, N, static_cast<int>(S), alpha, beta, C, ldc);
    }
    return true;
}

template <bool TA, int BN>
void launch_ts(Context& ctx, const double* A, long lda, const double* B, long ldb, double* C, long ldc, long M,
               long N, long K, double alpha, double beta) {
    if (launch_tma<TA, BN>(ctx, A, lda, B, ldb, C, ldc, M, N, K, alpha, beta)) return;
    const int occ = ts_occupancy<TA, BN>(ctx.device());
    const long mt = ceil_div(M, gemm_ts::BM), nt = ceil_div(N, BN);
    const long ktiles = ceil_div(K, gemm_ts::BK);
    const long slots = static_cast<long>(ctx.sm_count()) * occ;
    // split-K so the CTA count fills whole waves (each split >= 8 k-tiles)
    long S = 1;
    const long tiles = mt * nt;
    if (tiles < 2 * slots) {
        const long smax = std::max<long>(1, std::min<long>(64, ktiles / 8));
        double best = 1e30;
        for (long s = 1; s <= smax; ++s) {
            const long ctas = tiles * s;
            const long waves = ceil_div(ctas, slots);
            // time ~ waves * (work per CTA) ~ waves / s ; prefer full waves
            const double cost = static_cast<double>(waves) / s + (s > 1 ? 0.02 : 0.0);
            if (cost < best - 1e-12) {
                best = cost;
                S = s;
            }
        }
    }
    const long kchunk = ceil_div(ktiles, S) * gemm_ts::BK;
    S = ceil_div(K, kchunk);
    DBuf<double> ws;
    if (S > 1) ws = DBuf<double>(ctx, static_cast<size_t>(S * M * N));
    constexpr int bytes = gemm_ts::smem_bytes<TA, BN>();
    dim3 grid(static_cast<unsigned>(mt), static_cast<unsigned>(nt), static_cast<unsigned>(S));
    dgemm_ts_kernel<TA, BN><<<grid, gemm_ts::THREADS, bytes, ctx.stream()>>>(A, lda, B, ldb, C, ldc, M, N, K, kchunk,
                                                                             alpha, beta, S > 1 ? ws.get() : nullptr);
    ctx.note_launch();
    ctx.check_launch("dgemm_ts_kernel");
    if (S > 1) {
        const long total = M * N;
        launch_splitk_reduce(ctx, ws.get(), M, N, static_cast<int>(S), alpha, beta, C, ldc);
    }
}

template <bool TA>
bool try_ts(Context& ctx, const double* A, long lda, const double* B, long ldb, double* C, long ldc, long M, long N,
            long K, double alpha, double beta) {
    // column tile: smallest of {32, 64, 104, 128} covering ceil(N / ntiles);
    // 64-wide column tiles when the row tiles alone leave SMs idle and K is too
    // short for split-K to fill them (the CholQR applies X R^{-1}: 4000 x 100
    // 18.0 -> 14.7 us)
    long ntiles = ceil_div(N, 128);
    if (N > 64 && K < 1024 && ceil_div(M, 64L) * ntiles < 2L * ctx.sm_count()) ntiles = ceil_div(N, 64);
    const long per = ceil_div(N, ntiles);
    if (per <= 32) launch_ts<TA, 32>(ctx, A, lda, B, ldb, C, ldc, M, N, K, alpha, beta);
    else if (per <= 64) launch_ts<TA, 64>(ctx, A, lda, B, ldb, C, ldc, M, N, K, alpha, beta);
    else if (per <= 104) launch_ts<TA, 104>(ctx, A, lda, B, ldb, C, ldc, M, N, K, alpha, beta);
    else launch_ts<TA, 128>(ctx, A, lda, B, ldb, C, ldc, M, N, K, alpha, beta);
    return true;
}

}  // namespace

// the 2D tensor map of the TMA GEMM, for other TMA-fed kernels (K7)
bool tma_map_2d(CUtensorMap* map, const double* base, long inner, long outer, long ld, int box_outer) {
    return tensor_map(map, base, inner, outer, ld, box_outer);
}

void gemm(Context& ctx, bool ta, bool tb, Index M, Index N, Index K, double alpha, const double* A, Index lda,
          const double* B, Index ldb, double beta, double* C, Index ldc) {
    if (M <= 0 || N <= 0) return;
    if (K <= 0 || alpha == 0.0) {
        const long total = M * N;
        scale_kernel<<<static_cast<unsigned>(std::min<long>(1024, (total + 255) / 256)), 256, 0, ctx.stream()>>>(
            C, ldc, M, N, beta);
        ctx.note_launch();
        ctx.check_launch("scale_kernel");
        return;
    }
    const bool aligned16 = (lda % 2 == 0) && (ldb % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                           (reinterpret_cast<uintptr_t>(B) % 16 == 0);
    // tall-skinny outputs (M >> N, the BLWS panels): one CTA spans all columns
    if (aligned16 && !tb && M >= 256 && M >= 4 * N) {
        if (ta)
            try_ts<true>(ctx, A, lda, B, ldb, C, ldc, M, N, K, alpha, beta);
        else
            try_ts<false>(ctx, A, lda, B, ldb, C, ldc, M, N, K, alpha, beta);
        return;
    }
    const Index tiles = ceil_div(M, BM) * ceil_div(N, BN);
    const Index ktiles = ceil_div(K, BK);
    // enough CTAs for ~2 waves of 3 resident CTAs/SM, each split >= 8 k-tiles
    const Index want = 3 * static_cast<Index>(ctx.sm_count());
    Index S = 1;
    if (tiles < want) S = std::min<Index>(ceil_div(want, tiles), std::max<Index>(1, ktiles / 8));
    S = std::max<Index>(1, std::min<Index>(S, 64));
    const Index kchunk = ceil_div(ktiles, S) * BK;
    S = ceil_div(K, kchunk);
    const bool aligned = (lda % 2 == 0) && (ldb % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(B) % 16 == 0);
    dim3 grid(static_cast<unsigned>(ceil_div(M, BM)), static_cast<unsigned>(ceil_div(N, BN)),
              static_cast<unsigned>(S));
    DBuf<double> ws;
    if (S > 1) ws = DBuf<double>(ctx, static_cast<size_t>(S * M * N));
    if (aligned)
        dispatch<2>(ctx, ta, tb, grid, A, lda, B, ldb, C, ldc, M, N, K, kchunk, alpha, beta, ws.get());
    else
        dispatch<1>(ctx, ta, tb, grid, A, lda, B, ldb, C, ldc, M, N, K, kchunk, alpha, beta, ws.get());
    if (S > 1) {
        const long total = M * N;
        launch_splitk_reduce(ctx, ws.get(), M, N, static_cast<int>(S), alpha, beta, C, ldc);
    }
}

}  // namespace blws

// ---------------------------------------------------------------------------
// FP64 peak microbenchmarks (roofline denominator; MEASURED_PEAKS.json has no
// FP64 figure). mode 0: DMMA m8n8k4 chains; mode 1: DFMA chains.
namespace blws {
namespace {

__global__ void __launch_bounds__(256) fp64_dmma_peak_k(double* sink, int iters) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) gemm_detail::dmma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) sink[0] = s;
}

__global__ void __launch_bounds__(256) fp64_dfma_peak_k(double* sink, int iters) {
    double acc[8];
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.678) sink[0] = s;
}

}  // namespace

// L2 throughput probes (the bound of the gather-form sparse kernels K8 / K9):
// mode 0 streams a 16 MB L2-resident buffer in 512-byte warp segments; mode 1
// gathers random rows of `row` doubles (lanes over the row, as K8 / K9 read X /
// U rows) from a rows x row matrix of 4 MB. Bytes counted = bytes requested.
__global__ void l2_probe_k(const double* __restrict__ buf, long n, int row, int mode, int iters, double* sink) {
    const int lane = threadIdx.x & 31;
    const long gw = (blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x) >> 5;
    const long nw = (static_cast<long>(gridDim.x) * blockDim.x) >> 5;
    double acc = 0.0;
    if (mode == 0) {
        const long segs = n / 64;  // 64 doubles per warp segment (2 per lane, 16 B loads)
        for (int it = 0; it < iters; ++it)
            for (long sgm = (gw + it * 7919) % segs, c = 0; c < 4; ++c, sgm = (sgm + nw) % segs) {
                const double2 v = reinterpret_cast<const double2*>(buf + sgm * 64)[lane];
                acc += v.x + v.y;
            }
    } else {
        // 8 independent rows in flight per warp (as K9's unrolled 32-position batch)
        const long rows = n / row;
        unsigned long long z = 0x9e3779b97f4a7c15ull * static_cast<unsigned long long>(gw + 1);
        for (int it = 0; it < iters / 2; ++it) {
            double part[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                z = z * 6364136223846793005ull + 1442695040888963407ull;
                const long i = static_cast<long>((z >> 33) % static_cast<unsigned long long>(rows));
                const double* a = buf + i * row;
                double t = 0.0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int c = lane + 32 * q;
                    if (c < row) t += a[c];
                }
                part[u] = t;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += part[u];
        }
    }
    if (acc == 12345.678) sink[0] = acc;  // keeps the loads
}

double l2_probe_gbps(Context& ctx, int mode, int row) {
    const long n = mode == 0 ? (16L << 20) / 8 : (4L << 20) / 8;
    DBuf<double> buf(ctx, static_cast<size_t>(n)), sink(ctx, 1);
    zero(ctx, buf.get(), sizeof(double) * n);
    const int blocks = ctx.sm_count() * 8, threads = 256, iters = 400;
    cudaEvent_t e0, e1;
    BLWS_CUDA(cudaEventCreate(&e0));
    BLWS_CUDA(cudaEventCreate(&e1));
    double best = 0;
    for (int rep = 0; rep < 4; ++rep) {
        BLWS_CUDA(cudaEventRecord(e0, ctx.stream()));
        l2_probe_k<<<blocks, threads, 0, ctx.stream()>>>(buf.get(), n, row, mode, iters, sink.get());
        BLWS_CUDA(cudaEventRecord(e1, ctx.stream()));
        BLWS_CUDA(cudaEventSynchronize(e1));
        ctx.note_launch();
        float ms = 0;
        BLWS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        const double warps = static_cast<double>(blocks) * threads / 32.0;
        const double bytes = mode == 0 ? warps * iters * 4 * 512.0 : warps * (iters / 2) * 8 * 8.0 * row;
        if (rep > 0) best = std::max(best, bytes / (ms * 1e-3) / 1e9);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

double fp64_peak_tflops(Context& ctx, int mode) {
    DBuf<double> sink(ctx, 1);
    const int blocks = ctx.sm_count() * 4, threads = 256, iters = 20000;
    cudaEvent_t e0, e1;
    BLWS_CUDA(cudaEventCreate(&e0));
    BLWS_CUDA(cudaEventCreate(&e1));
    double best = 0;
    for (int rep = 0; rep < 3; ++rep) {
        BLWS_CUDA(cudaEventRecord(e0, ctx.stream()));
        if (mode == 0)
            fp64_dmma_peak_k<<<blocks, threads, 0, ctx.stream()>>>(sink.get(), iters);
        else
            fp64_dfma_peak_k<<<blocks, threads, 0, ctx.stream()>>>(sink.get(), iters);
        BLWS_CUDA(cudaEventRecord(e1, ctx.stream()));
        BLWS_CUDA(cudaEventSynchronize(e1));
        ctx.note_launch();
        float ms = 0;
        BLWS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        // DMMA: 8x8x4 = 256 FMA per warp-instruction; DFMA: 1 FMA per thread-instruction
        const double warps = static_cast<double>(blocks) * threads / 32.0;
        const double flops = mode == 0 ? warps * iters * 8 * 256 * 2.0
                                       : static_cast<double>(blocks) * threads * iters * 8 * 2.0;
        best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

}  // namespace blws
