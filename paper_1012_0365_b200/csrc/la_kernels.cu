// Level-1 / small dense / GEMV / sparse kernels of the BLWS hot path.
#include <algorithm>
#include <cmath>

#include <climits>
#include <cstdlib>
#include <cstring>

#include "bulk.cuh"
#include "ops.cuh"

namespace blws {

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(long total, int threads = kThreads, long cap = 4096) {
    return static_cast<unsigned>(std::max<long>(1, std::min<long>(cap, (total + threads - 1) / threads)));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

/// Block-wide sum; result valid in thread 0. blockDim.x multiple of 32, <= 1024.
__device__ double block_sum(double v) {
    __shared__ double sh[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    v = threadIdx.x < nw ? sh[threadIdx.x] : 0.0;
    if (wid == 0) v = warp_sum(v);
    return v;
}

__global__ void fill_k(double* x, long rows, long cols, long ld, double v) {
    const long total = rows * cols;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x)
        x[idx % rows + (idx / rows) * ld] = v;
}

__global__ void zero_k(unsigned* p, size_t words) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < words;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = 0u;
}

__global__ void copy_k(double* d, long ldd, const double* s, long lds, long rows, long cols, double alpha) {
    const long total = rows * cols;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx % rows, j = idx / rows;
        d[i + j * ldd] = alpha == 1.0 ? s[i + j * lds] : alpha * s[i + j * lds];
    }
}

__global__ void axpy_k(double* y, long ldy, const double* x, long ldx, long rows, long cols, double alpha) {
    const long total = rows * cols;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx % rows, j = idx / rows;
        y[i + j * ldy] += alpha * x[i + j * ldx];
    }
}

__global__ void sumsq_partial_k(const double* x, long rows, long cols, long ld, int minus_identity,
                                double* partial) {
    const long total = rows * cols;
    double s = 0.0;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx % rows, j = idx / rows;
        double v = x[i + j * ld];
        if (minus_identity && i == j) v -= 1.0;
        s += v * v;
    }
    s = block_sum(s);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void reduce_k(const double* partial, long count, double* out) {
    double s = 0.0;
    for (long i = threadIdx.x; i < count; i += blockDim.x) s += partial[i];
    s = block_sum(s);
    if (threadIdx.x == 0) out[0] = s;
}

__global__ void symmetrize_k(double* d, long ldd, const double* s, long lds, long n) {
    const long total = n * n;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx % n, j = idx / n;
        d[i + j * ldd] = 0.5 * (s[i + j * lds] + s[j + i * lds]);
    }
}

__global__ void place_k(double* d, long ldd, const double* s, long lds, long rows, long cols, int transpose) {
    const long total = rows * cols;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx % rows, j = idx / rows;
        if (transpose)
            d[j + i * ldd] = s[i + j * lds];
        else
            d[i + j * ldd] = s[i + j * lds];
    }
}

__global__ void scale_cols_k(double* d, long ldd, const double* s, long lds, long rows, long cols,
                             const double* sc) {
    const long total = rows * cols;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx % rows, j = idx / rows;
        d[i + j * ldd] = s[i + j * lds] * sc[j];
    }
}

__global__ void gather_cols_k(double* d, long ldd, const double* s, long lds, long rows, long cols, const int* ix) {
    const long total = rows * cols;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx % rows, j = idx / rows;
        d[i + j * ldd] = s[i + static_cast<long>(ix[j]) * lds];
    }
}

// Right-looking upper Cholesky, one CTA. G is staged in shared memory when it
// fits (n <= 160), else updated in place in global memory (L1/L2 resident).
constexpr long kCholSmem = 160 * 160;
__global__ void __launch_bounds__(1024) potrf_k(double* g, long n, long ld, int* status, double* diag) {
    extern __shared__ __align__(16) double sm[];
    double* rj = sm;  // row j of R (n doubles)
    const bool on_chip = n * n <= kCholSmem;
    double* a = on_chip ? sm + n : g;
    const long la = on_chip ? n : ld;
    __shared__ int fail;
    if (threadIdx.x == 0) fail = 0;
    if (on_chip)
        for (long idx = threadIdx.x; idx < n * n; idx += blockDim.x) a[idx] = g[idx % n + (idx / n) * ld];
    __syncthreads();
    for (long j = 0; j < n; ++j) {
        const double piv = a[j + j * la];
        if (!(piv > 0.0) || !isfinite(piv)) {
            if (threadIdx.x == 0) fail = static_cast<int>(j + 1);
            break;
        }
        const double rjj = sqrt(piv);
        __syncthreads();
        for (long k = j + 1 + threadIdx.x; k < n; k += blockDim.x) {
            const double r = a[j + k * la] / rjj;
            a[j + k * la] = r;
            rj[k] = r;
        }
        if (threadIdx.x == 0) a[j + j * la] = rjj;
        __syncthreads();
        // trailing update of the upper triangle, warp per column k, lanes over i <= k
        {
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
            const int jj = static_cast<int>(j), nn = static_cast<int>(n);
            for (int k = jj + 1 + wid; k < nn; k += nw) {
                const double rk = rj[k];
                double* col = a + static_cast<long>(k) * la;
                for (int i = jj + 1 + lane; i <= k; i += 32) col[i] -= rj[i] * rk;
            }
        }
        __syncthreads();
    }
    __syncthreads();
    if (threadIdx.x == 0) status[0] = fail;
    if (fail) return;
    double mn = INFINITY, mx = 0.0;
    for (long idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        const long i = idx % n, k = idx / n;
        const double v = i > k ? 0.0 : a[i + k * la];
        g[i + k * ld] = v;
        if (i == k) {
            mn = fmin(mn, v);
            mx = fmax(mx, v);
        }
    }
    __shared__ double smn[32], smx[32];
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        smn[threadIdx.x >> 5] = mn;
        smx[threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w2 = 1; w2 < static_cast<int>(blockDim.x >> 5); ++w2) {
            mn = fmin(mn, smn[w2]);
            mx = fmax(mx, smx[w2]);
        }
        diag[0] = mn;
        diag[1] = mx;
    }
}

// Inverse of an upper-triangular R: R staged in shared memory per CTA (when it
// fits), one warp per column, column-oriented back substitution on a
// per-warp shared vector (x = e_j; for i = j..0: x_i /= R_ii; x_{<i} -= R_{<i,i} x_i).
constexpr long kTrtriSmem = 150 * 150;
constexpr int kTrtriWarps = 8;
__global__ void trtri_k(double* out, long ldo, const double* r, long ldr, long n) {
    extern __shared__ __align__(16) double sm[];
    const bool on_chip = n * n <= kTrtriSmem;
    double* xs = sm;  // kTrtriWarps * n
    const double* R = r;
    long lr = ldr;
    if (on_chip) {
        double* rs = sm + kTrtriWarps * n;
        for (long idx = threadIdx.x; idx < n * n; idx += blockDim.x) rs[idx] = r[idx % n + (idx / n) * ldr];
        R = rs;
        lr = n;
        __syncthreads();
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* x = xs + warp * n;
    const int nn = static_cast<int>(n), l = static_cast<int>(lr);
    for (int j = blockIdx.x * kTrtriWarps + warp; j < nn; j += gridDim.x * kTrtriWarps) {
        for (int i = lane; i <= j; i += 32) x[i] = (i == j) ? 1.0 : 0.0;
        __syncwarp();
        for (int i = j; i >= 0; --i) {
            const double xi = x[i] / R[i + i * l];
            const double* rc = R + i * l;
            for (int k = lane; k < i; k += 32) x[k] -= rc[k] * xi;
            __syncwarp();
            if (lane == 0) x[i] = xi;
            __syncwarp();
        }
        double* o = out + static_cast<long>(j) * ldo;
        for (int i = lane; i < nn; i += 32) o[i] = i <= j ? x[i] : 0.0;
        __syncwarp();
    }
}

__global__ void add_diag_k(double* g, long ld, long n, const double* s) {
    const double v = s[0];
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long>(gridDim.x) * blockDim.x)
        g[i + i * ld] += v;
}

__global__ void count_diag_k(const double* r, long ld, long n, const double* sumsq, double scale,
                             std::int64_t* out) {
    const double tau = scale * sqrt(sumsq[0]);
    long c = 0;
    for (long i = threadIdx.x; i < n; i += blockDim.x) c += (r[i + i * ld] > tau) ? 1 : 0;
    double s = block_sum(static_cast<double>(c));
    if (threadIdx.x == 0) out[0] = static_cast<std::int64_t>(s + 0.5);
}

// y_partial[split][i] = sum_{j in split} A[i,j] x[j]
__global__ void gemv_n_partial(const double* __restrict__ A, long lda, long rows, long cols, long cchunk,
                               const double* __restrict__ x, double* partial) {
    const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    const long j0 = blockIdx.y * cchunk, j1 = min(cols, j0 + cchunk);
    if (i >= rows) return;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    long j = j0;
    for (; j + 3 < j1; j += 4) {
        s0 += A[i + j * lda] * x[j];
        s1 += A[i + (j + 1) * lda] * x[j + 1];
        s2 += A[i + (j + 2) * lda] * x[j + 2];
        s3 += A[i + (j + 3) * lda] * x[j + 3];
    }
    for (; j < j1; ++j) s0 += A[i + j * lda] * x[j];
    partial[blockIdx.y * rows + i] = (s0 + s1) + (s2 + s3);
}

__global__ void gemv_n_finish(const double* partial, int S, long rows, double alpha, double beta, double* y) {
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < rows;
         i += static_cast<long>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int z = 0; z < S; ++z) s += partial[z * rows + i];
        y[i] = beta == 0.0 ? alpha * s : alpha * s + beta * y[i];
    }
}

// partial[split][j] = sum_{i in split} A[i,j] x[i]; one block per (column, split)
__global__ void gemv_t_partial(const double* __restrict__ A, long lda, long rows, long cols, long rchunk,
                               const double* __restrict__ x, double* partial) {
    const long j = blockIdx.x;
    const long i0 = blockIdx.y * rchunk, i1 = min(rows, i0 + rchunk);
    const double* a = A + j * lda;
    double s = 0.0;
    for (long i = i0 + threadIdx.x; i < i1; i += blockDim.x) s += a[i] * x[i];
    s = block_sum(s);
    if (threadIdx.x == 0) partial[blockIdx.y * cols + j] = s;
}

__global__ void dot_partial_k(long n, const double* x, const double* y, double* partial) {
    double s = 0.0;
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long>(gridDim.x) * blockDim.x)
        s += x[i] * y[i];
    s = block_sum(s);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// X (rows x b, col-major, ld) -> XT row-major (rows x b)
__global__ void to_row_major_k(const double* X, long ld, long rows, long b, double* xt) {
    const long total = rows * b;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long c = idx / rows, i = idx % rows;
        xt[i * b + c] = X[i + c * ld];
    }
}

// K8: warp per row, lanes over the b output columns (SLOTS x 32 >= b). The
// row's nonzeros are taken 32 at a time: (column, value) pairs loaded coalesced,
// shuffled out one by one; the X-row gathers of a batch are independent, so
// several are in flight (two interleaved accumulators per slot, fixed order).
#ifndef K8_UNROLL
#define K8_UNROLL 32
#endif
constexpr int kK8Unroll = K8_UNROLL;
#ifndef K8_DEFAULT_MODE
#define K8_DEFAULT_MODE 0  // 0 gather, 1 tiled when it pays
#endif
template <int SLOTS>
__global__ void csr_spmm_k(long rows, const std::int64_t* __restrict__ rowptr, const std::int32_t* __restrict__ colidx,
                           const double* __restrict__ val, long b, const double* __restrict__ xt, double* Y,
                           long ldy) {
    const long warps = (static_cast<long>(gridDim.x) * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (long i = (blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x) >> 5; i < rows; i += warps) {
        const long p0 = rowptr[i], p1 = rowptr[i + 1];
        double acc[SLOTS][2];
#pragma unroll
        for (int q = 0; q < SLOTS; ++q) acc[q][0] = acc[q][1] = 0.0;
        // per slot, the lane's column of X^T as a byte pointer: an X-row element is then one
        // 32 x 32 -> 64-bit multiply-add away (col * 8b). Lanes past b read column b - 1 and
        // accumulate values that are never stored, so the loads and FMAs carry no predicate
        // (the predicated form cost ~25 instructions per nonzero: 64-bit index arithmetic and
        // a register-pair move after every predicated DFMA; ncu r02i)
        const char* xl[SLOTS];
#pragma unroll
        for (int q = 0; q < SLOTS; ++q)
            xl[q] = reinterpret_cast<const char*>(xt + min(static_cast<long>(lane + 32 * q), b - 1));
        const unsigned bbytes = static_cast<unsigned>(b) * 8u;
        for (long pb = p0; pb < p1; pb += 32) {
            const long p = pb + lane;
            const int cj = p < p1 ? colidx[p] : 0;
            const double vj = p < p1 ? val[p] : 0.0;  // padding entries contribute 0
#pragma unroll(kK8Unroll)
            for (int t = 0; t < 32; ++t) {
                const unsigned long long ro =
                    static_cast<unsigned long long>(static_cast<unsigned>(__shfl_sync(0xffffffffu, cj, t))) * bbytes;
                const double v = __shfl_sync(0xffffffffu, vj, t);
#pragma unroll
                for (int q = 0; q < SLOTS; ++q)
                    acc[q][t & 1] = fma(v, *reinterpret_cast<const double*>(xl[q] + ro), acc[q][t & 1]);
            }
        }
#pragma unroll
        for (int q = 0; q < SLOTS; ++q) {
            const long c = lane + 32 * q;
            if (c < b) Y[i + c * ldy] = acc[q][0] + acc[q][1];
        }
    }
}

// K8, tiled. The gather kernel above re-reads a whole X row from L2 for every
// nonzero (8 b bytes per nonzero: L2-bound). Here a CTA owns a group of rows
// (kK8Warps consumer warps x RPW rows each, accumulators in registers) and
// streams X through shared memory in tiles of T rows: bulk copies into a
// kK8Stages-deep mbarrier ring, issued by one producer warp. The column indices
// of a row ascend, so the row's nonzeros inside the current tile are the next
// ones at its cursor. Each row keeps a 32-entry (column, value) batch in
// registers, aligned as in csr_spmm_k, and entry t goes into accumulator t & 1:
// the same sums in the same order as the gather kernel. L2 traffic drops from
// 8 b nnz to (row groups) x 8 b ncols.
constexpr int kK8Warps = 15;  // + the producer warp = 512 threads (128 registers each)
constexpr int kK8Stages = 3;
constexpr int kK8MaxRpw = 6;
constexpr int kK8TileBytes = 64 * 1024;

// the row's (column, value) stream comes from DRAM and is read once: the batch
// after the one just loaded is pulled into L1, the one after that into L2, so
// a reload does not stall its warp for a DRAM round trip
__device__ __forceinline__ void k8_prefetch(const std::int32_t* colidx, const double* val, long base, int left,
                                            int lane) {
#ifndef K8T_NO_PREFETCH
    if (lane + 32 < left) {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(colidx + base + 32 + lane));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(val + base + 32 + lane));
    }
    if (lane + 64 < left) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(colidx + base + 64 + lane));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(val + base + 64 + lane));
    }
#endif
}

template <int SLOTS, int RPW>
__global__ void __launch_bounds__((kK8Warps + 1) * 32, 1)
    csr_spmm_tiled_k(long rows, long ncols, const std::int64_t* __restrict__ rowptr,
                     const std::int32_t* __restrict__ colidx, const double* __restrict__ val, int b,
                     const double* __restrict__ xt, double* Y, long ldy, int T, long ngroups, long rpc) {
    extern __shared__ __align__(128) unsigned char k8_smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(k8_smem);
    uint64_t* empty = full + kK8Stages;
    double* tiles = reinterpret_cast<double*>(k8_smem + 128);
    const long tile_elems = static_cast<long>(T) * b;  // 8 T b is a multiple of 128 (T % 16 == 0)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long ntiles = (ncols + T - 1) / T;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kK8Stages; ++s) {
            gemm_tma::mbar_init(full + s, 1);
            gemm_tma::mbar_init(empty + s, kK8Warps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    long it = 0;  // tiles this CTA has streamed: ring slot it % stages, use it / stages
    if (warp == kK8Warps) {  // producer
        if (lane == 0) {
            for (long g = blockIdx.x; g < ngroups; g += gridDim.x)
                for (long c = 0; c < ntiles; ++c, ++it) {
                    const int s = static_cast<int>(it % kK8Stages);
                    const long use = it / kK8Stages;
                    if (use > 0) gemm_tma::mbar_wait(empty + s, static_cast<uint32_t>((use - 1) & 1));
                    const long r0 = c * T;
                    const long cnt = min(static_cast<long>(T), ncols - r0) * b;
                    const long even = cnt & ~1L;  // bulk copies move 16-byte multiples
                    double* dst = tiles + s * tile_elems;
                    const double* src = xt + r0 * b;
                    if (cnt & 1) dst[cnt - 1] = src[cnt - 1];  // ordered by the arrive below (release)
                    gemm_tma::mbar_expect_tx(full + s, static_cast<uint32_t>(even * 8));
                    if (even > 0) bulk_g2s(dst, src, static_cast<uint32_t>(even * 8), full + s);
                }
        }
        return;
    }
    for (long g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const long gr0 = g * rpc, gr1 = min(rows, gr0 + rpc);
        double acc[RPW][SLOTS][2];
        long base[RPW];  // position of the batch's entry 0
        int left[RPW];   // entries of the row from base on
        int off[RPW];    // entries of the batch already consumed
        int cj[RPW];
        double vj[RPW];
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
#pragma unroll
            for (int q = 0; q < SLOTS; ++q) acc[r][q][0] = acc[r][q][1] = 0.0;
            const long i = gr0 + warp + static_cast<long>(r) * kK8Warps;
            base[r] = i < gr1 ? rowptr[i] : 0;
            left[r] = i < gr1 ? static_cast<int>(rowptr[i + 1] - base[r]) : 0;
            off[r] = 0;
            cj[r] = lane < left[r] ? colidx[base[r] + lane] : INT_MAX;
            vj[r] = lane < left[r] ? val[base[r] + lane] : 0.0;
            k8_prefetch(colidx, val, base[r], left[r], lane);
        }
        for (long c = 0; c < ntiles; ++c, ++it) {
            const int s = static_cast<int>(it % kK8Stages);
            gemm_tma::mbar_wait(full + s, static_cast<uint32_t>((it / kK8Stages) & 1));
            const double* xs = tiles + s * tile_elems;
            const int j0 = static_cast<int>(c * T);
            const int j1 = static_cast<int>(min(ncols, static_cast<long>(j0) + T));
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
                while (true) {
                    // ascending columns: the entries inside the tile are a run starting at off
                    const int cnt = __popc(__ballot_sync(0xffffffffu, lane >= off[r] && cj[r] < j1));
                    int t = off[r];
                    const int te = t + cnt;
#define K8_STEP(P, TT)                                                                      \
    {                                                                                       \
        const int col = __shfl_sync(0xffffffffu, cj[r], (TT)) - j0;                         \
        const double v = __shfl_sync(0xffffffffu, vj[r], (TT));                             \
        const double* xr = xs + col * b;                                                    \
        _Pragma("unroll") for (int q = 0; q < SLOTS; ++q) {                                 \
            const int cc = lane + 32 * q;                                                   \
            if (cc < b) acc[r][q][P] = fma(v, xr[cc], acc[r][q][P]);                        \
        }                                                                                   \
    }
                    if (t < te && (t & 1)) {
                        K8_STEP(1, t);
                        ++t;
                    }
                    for (; t + 3 < te; t += 4) {  // straight-line: the four entries' loads go out together
                        K8_STEP(0, t);
                        K8_STEP(1, t + 1);
                        K8_STEP(0, t + 2);
                        K8_STEP(1, t + 3);
                    }
                    if (t + 1 < te) {
                        K8_STEP(0, t);
                        K8_STEP(1, t + 1);
                        t += 2;
                    }
                    if (t < te) K8_STEP(0, t);
#undef K8_STEP
                    off[r] = te;
                    if (te == 32 && left[r] > 32) {  // batch used up, the row goes on
                        base[r] += 32;
                        left[r] -= 32;
                        off[r] = 0;
                        cj[r] = lane < left[r] ? colidx[base[r] + lane] : INT_MAX;
                        vj[r] = lane < left[r] ? val[base[r] + lane] : 0.0;
                        k8_prefetch(colidx, val, base[r], left[r], lane);
                    } else {
                        break;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) gemm_tma::mbar_arrive(empty + s);
        }
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const long i = gr0 + warp + static_cast<long>(r) * kK8Warps;
            if (i < gr1) {
#pragma unroll
                for (int q = 0; q < SLOTS; ++q) {
                    const int cc = lane + 32 * q;
                    if (cc < b) Y[i + cc * ldy] = acc[r][q][0] + acc[r][q][1];
                }
            }
        }
    }
}

// narrow blocks (b <= NB <= 8, e.g. the Lanczos vector products): lanes over
// the row's nonzeros, NB per-lane accumulators, xor-tree warp reductions
template <int NB>
__global__ void csr_spmm_narrow_k(long rows, const std::int64_t* __restrict__ rowptr,
                                  const std::int32_t* __restrict__ colidx, const double* __restrict__ val, long b,
                                  const double* __restrict__ xt, double* Y, long ldy) {
    const long warps = (static_cast<long>(gridDim.x) * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (long i = (blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x) >> 5; i < rows; i += warps) {
        const long p1 = rowptr[i + 1];
        double acc[NB];
#pragma unroll
        for (int c = 0; c < NB; ++c) acc[c] = 0.0;
        for (long p = rowptr[i] + lane; p < p1; p += 32) {
            const double v = val[p];
            const double* xr = xt + static_cast<long>(colidx[p]) * b;
#pragma unroll
            for (int c = 0; c < NB; ++c)
                if (c < b) acc[c] = fma(v, xr[c], acc[c]);
        }
#pragma unroll
        for (int c = 0; c < NB; ++c) {
            for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
            if (lane == c && c < b) Y[i + c * ldy] = acc[c];
        }
    }
}

// the generic path for wide blocks (b > 128): lanes over chunks of the columns
__global__ void csr_spmm_wide_k(long rows, const std::int64_t* __restrict__ rowptr,
                                const std::int32_t* __restrict__ colidx, const double* __restrict__ val, long b,
                                const double* __restrict__ xt, double* Y, long ldy) {
    const long warps = (static_cast<long>(gridDim.x) * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (long i = (blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x) >> 5; i < rows; i += warps) {
        const long p0 = rowptr[i], p1 = rowptr[i + 1];
        for (long c = lane; c < b; c += 32) {
            double a0 = 0.0, a1 = 0.0;
            long p = p0;
            for (; p + 1 < p1; p += 2) {
                a0 = fma(val[p], xt[static_cast<long>(colidx[p]) * b + c], a0);
                a1 = fma(val[p + 1], xt[static_cast<long>(colidx[p + 1]) * b + c], a1);
            }
            if (p < p1) a0 = fma(val[p], xt[static_cast<long>(colidx[p]) * b + c], a0);
            Y[i + c * ldy] = a0 + a1;
        }
    }
}

__global__ void pack_rows_k(const double* __restrict__ x, long ld, long rows, long cols, double* __restrict__ out) {
    const long total = rows * cols;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx / cols, c = idx % cols;
        out[idx] = x[i + c * ld];
    }
}

__global__ void unpack_rows_k(const double* __restrict__ in, long rows, long cols, double* __restrict__ x, long ld) {
    const long total = rows * cols;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx / cols, c = idx % cols;
        x[i + c * ld] = in[idx];
    }
}

__global__ void gather_vals_k(long nnz, double* dst, const double* src, const std::int64_t* perm) {
    for (long p = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<long>(gridDim.x) * blockDim.x)
        dst[p] = src[perm[p]];
}

}  // namespace

#define LAUNCH(ctx, name) \
    do {                   \
        (ctx).note_launch(); \
        (ctx).check_launch(name); \
    } while (0)

void zero(Context& ctx, void* p, size_t bytes) {
    if (bytes == 0) return;
    if (bytes % 4) throw std::invalid_argument("zero: size must be a multiple of 4 bytes");
    const size_t words = bytes / 4;
    zero_k<<<grid_for(static_cast<Index>(words)), kThreads, 0, ctx.stream()>>>(static_cast<unsigned*>(p), words);
    LAUNCH(ctx, "zero");
}

void fill(Context& ctx, View x, double v) {
    if (x.rows * x.cols == 0) return;
    fill_k<<<grid_for(x.rows * x.cols), kThreads, 0, ctx.stream()>>>(x.p, x.rows, x.cols, x.ld, v);
    LAUNCH(ctx, "fill");
}

void copy(Context& ctx, View d, View s, double alpha) {
    if (d.rows * d.cols == 0) return;
    copy_k<<<grid_for(d.rows * d.cols), kThreads, 0, ctx.stream()>>>(d.p, d.ld, s.p, s.ld, d.rows, d.cols, alpha);
    LAUNCH(ctx, "copy");
}

void axpy(Context& ctx, View y, View x, double alpha) {
    if (y.rows * y.cols == 0) return;
    axpy_k<<<grid_for(y.rows * y.cols), kThreads, 0, ctx.stream()>>>(y.p, y.ld, x.p, x.ld, y.rows, y.cols, alpha);
    LAUNCH(ctx, "axpy");
}

static void sumsq_impl(Context& ctx, View x, int minus_identity, double* out) {
    const unsigned blocks = grid_for(x.rows * x.cols, kThreads, 1024);
    DBuf<double> part(ctx, blocks);
    sumsq_partial_k<<<blocks, kThreads, 0, ctx.stream()>>>(x.p, x.rows, x.cols, x.ld, minus_identity, part.get());
    LAUNCH(ctx, "sumsq_partial");
    reduce_k<<<1, 1024, 0, ctx.stream()>>>(part.get(), blocks, out);
    LAUNCH(ctx, "reduce");
}

void sumsq(Context& ctx, View x, double* out) { sumsq_impl(ctx, x, 0, out); }
void sumsq_minus_identity(Context& ctx, View x, double* out) { sumsq_impl(ctx, x, 1, out); }

void reduce_partials(Context& ctx, const double* partials, Index count, double* out) {
    reduce_k<<<1, 1024, 0, ctx.stream()>>>(partials, count, out);
    LAUNCH(ctx, "reduce");
}

void symmetrize(Context& ctx, View d, View s) {
    symmetrize_k<<<grid_for(s.rows * s.rows), kThreads, 0, ctx.stream()>>>(d.p, d.ld, s.p, s.ld, s.rows);
    LAUNCH(ctx, "symmetrize");
}

void place_block(Context& ctx, View d, View s, bool transpose) {
    place_k<<<grid_for(s.rows * s.cols), kThreads, 0, ctx.stream()>>>(d.p, d.ld, s.p, s.ld, s.rows, s.cols,
                                                                      transpose ? 1 : 0);
    LAUNCH(ctx, "place_block");
}

void scale_columns(Context& ctx, View d, View s, const double* sc) {
    if (s.rows * s.cols == 0) return;
    scale_cols_k<<<grid_for(s.rows * s.cols), kThreads, 0, ctx.stream()>>>(d.p, d.ld, s.p, s.ld, s.rows, s.cols, sc);
    LAUNCH(ctx, "scale_columns");
}

void gather_columns(Context& ctx, View d, View s, const int* ix) {
    if (d.rows * d.cols == 0) return;
    gather_cols_k<<<grid_for(d.rows * d.cols), kThreads, 0, ctx.stream()>>>(d.p, d.ld, s.p, s.ld, d.rows, d.cols,
                                                                            ix);
    LAUNCH(ctx, "gather_columns");
}

void potrf_upper(Context& ctx, View g, int* status, double* diag) {
    static bool cfg = false;
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(potrf_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        cfg = true;
    }
    const long n = g.rows;
    const size_t smem = static_cast<size_t>((n + (n * n <= kCholSmem ? n * n : 0)) * 8);
    potrf_k<<<1, 1024, smem, ctx.stream()>>>(g.p, n, g.ld, status, diag);
    LAUNCH(ctx, "potrf");
}

void trtri_upper(Context& ctx, View out, View r) {
    static bool cfg = false;
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(trtri_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        cfg = true;
    }
    const long n = r.rows;
    const size_t smem = static_cast<size_t>((kTrtriWarps * n + (n * n <= kTrtriSmem ? n * n : 0)) * 8);
    const unsigned blocks = static_cast<unsigned>(std::max<long>(1, std::min<long>(32, (n + kTrtriWarps - 1) / kTrtriWarps)));
    trtri_k<<<blocks, kTrtriWarps * 32, smem, ctx.stream()>>>(out.p, out.ld, r.p, r.ld, n);
    LAUNCH(ctx, "trtri");
}

void trmm_upper(Context& ctx, View c, View a, View b) {
    gemm(ctx, false, false, a.rows, b.cols, a.cols, 1.0, a.p, a.ld, b.p, b.ld, 0.0, c.p, c.ld);
}

void add_diagonal(Context& ctx, View g, const double* s) {
    add_diag_k<<<grid_for(g.rows), kThreads, 0, ctx.stream()>>>(g.p, g.ld, g.rows, s);
    LAUNCH(ctx, "add_diagonal");
}

void count_diag_above(Context& ctx, View r, const double* ss, double scale, std::int64_t* out) {
    count_diag_k<<<1, 256, 0, ctx.stream()>>>(r.p, r.ld, r.rows, ss, scale, out);
    LAUNCH(ctx, "count_diag");
}

void gemv(Context& ctx, bool trans, Index rows, Index cols, double alpha, const double* A, Index lda,
          const double* x, double beta, double* y) {
    const int sms = ctx.sm_count();
    if (!trans) {
        if (rows <= 0) return;
        const long rb = (rows + kThreads - 1) / kThreads;
        long S = std::max<long>(1, std::min<long>((8L * sms + rb - 1) / rb, std::max<long>(1, cols / 64)));
        const long cchunk = (cols + S - 1) / S;
        S = std::max<long>(1, (cols + cchunk - 1) / cchunk);
        DBuf<double> part(ctx, static_cast<size_t>(S * rows));
        if (cols > 0) {
            gemv_n_partial<<<dim3(static_cast<unsigned>(rb), static_cast<unsigned>(S)), kThreads, 0, ctx.stream()>>>(
                A, lda, rows, cols, cchunk, x, part.get());
            LAUNCH(ctx, "gemv_n_partial");
        } else {
            S = 0;
        }
        gemv_n_finish<<<grid_for(rows), kThreads, 0, ctx.stream()>>>(part.get(), static_cast<int>(S), rows, alpha, beta,
                                                                     y);
        LAUNCH(ctx, "gemv_n_finish");
    } else {
        if (cols <= 0) return;
        long S = std::max<long>(1, std::min<long>((8L * sms + cols - 1) / cols, std::max<long>(1, rows / 1024)));
        const long rchunk = (rows + S - 1) / S;
        S = std::max<long>(1, (rows + rchunk - 1) / rchunk);
        DBuf<double> part(ctx, static_cast<size_t>(S * cols));
        if (rows > 0) {
            gemv_t_partial<<<dim3(static_cast<unsigned>(cols), static_cast<unsigned>(S)), 128, 0, ctx.stream()>>>(
                A, lda, rows, cols, rchunk, x, part.get());
            LAUNCH(ctx, "gemv_t_partial");
        } else {
            S = 0;
        }
        gemv_n_finish<<<grid_for(cols), kThreads, 0, ctx.stream()>>>(part.get(), static_cast<int>(S), cols, alpha, beta,
                                                                     y);
        LAUNCH(ctx, "gemv_t_finish");
    }
}

void dot(Context& ctx, Index n, const double* x, const double* y, double* out) {
    const unsigned blocks = grid_for(n, kThreads, 512);
    DBuf<double> part(ctx, blocks);
    dot_partial_k<<<blocks, kThreads, 0, ctx.stream()>>>(n, x, y, part.get());
    LAUNCH(ctx, "dot_partial");
    reduce_k<<<1, 1024, 0, ctx.stream()>>>(part.get(), blocks, out);
    LAUNCH(ctx, "reduce");
}

namespace {

// BLWS_K8=gather keeps the L2 gather kernel, BLWS_K8=tiled forces the tiled one
// wherever it can run; default: tiled when the X re-streaming is well below
// the gather traffic
int k8_mode() {
    static const int mode = [] {
        const char* e = std::getenv("BLWS_K8");
        if (e && std::strcmp(e, "gather") == 0) return 0;
        if (e && std::strcmp(e, "tiled") == 0) return 2;
        return K8_DEFAULT_MODE;
    }();
    return mode;
}

template <int SLOTS, int RPW>
void launch_k8_tiled(Context& ctx, unsigned grid, size_t smem, Index rows, Index ncols, const std::int64_t* rowptr,
                     const std::int32_t* colidx, const double* val, Index b, const double* xt, double* Y, Index ldy,
                     int T, long ngroups, long rpc) {
    static bool once = [] {
        BLWS_CUDA(cudaFuncSetAttribute(csr_spmm_tiled_k<SLOTS, RPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       128 + kK8Stages * kK8TileBytes));
        return true;
    }();
    (void)once;
    csr_spmm_tiled_k<SLOTS, RPW><<<grid, (kK8Warps + 1) * 32, smem, ctx.stream()>>>(
        rows, ncols, rowptr, colidx, val, static_cast<int>(b), xt, Y, ldy, T, ngroups, rpc);
}

template <int SLOTS>
void launch_k8_tiled_rpw(int rpw, Context& ctx, unsigned grid, size_t smem, Index rows, Index ncols,
                         const std::int64_t* rowptr, const std::int32_t* colidx, const double* val, Index b,
                         const double* xt, double* Y, Index ldy, int T, long ngroups, long rpc) {
#define K8_CASE(R)                                                                                              \
    case R:                                                                                                     \
        launch_k8_tiled<SLOTS, R>(ctx, grid, smem, rows, ncols, rowptr, colidx, val, b, xt, Y, ldy, T, ngroups, \
                                  rpc);                                                                         \
        break;
    switch (rpw) {
        K8_CASE(1) K8_CASE(2) K8_CASE(3) K8_CASE(4) K8_CASE(5) K8_CASE(6)
        default: throw std::logic_error("csr_spmm_tiled: rows per warp");
    }
#undef K8_CASE
}

// true when the tiled kernel ran
bool csr_spmm_tiled(Context& ctx, Index rows, const std::int64_t* rowptr, const std::int32_t* colidx,
                    const double* val, Index ncols, Index b, const double* xt, double* Y, Index ldy, Index nnz) {
    const int mode = k8_mode();
    if (mode == 0 || nnz < 0 || b <= 8 || b > 64 || ncols >= INT_MAX) return false;
    const long sms = ctx.sm_count();
    // row groups: a multiple of the SM count, at most kK8Warps * kK8MaxRpw rows each
    const long per = static_cast<long>(kK8Warps) * kK8MaxRpw;
    const long ngroups = sms * ((rows + sms * per - 1) / (sms * per));
    const long rpc = (rows + ngroups - 1) / ngroups;
    const int rpw = static_cast<int>((rpc + kK8Warps - 1) / kK8Warps);
    // every group streams X once: worth it when that is well below one X row per nonzero
    if (mode == 1 && nnz < 4 * ngroups * ncols) return false;
    int T = static_cast<int>((kK8TileBytes / (8 * b)) & ~15L);
    T = static_cast<int>(std::min<long>(T, (ncols + 15) & ~15L));
    const size_t smem = 128 + static_cast<size_t>(kK8Stages) * T * b * 8;
    const unsigned grid = static_cast<unsigned>(std::min(ngroups, sms));
    if (b <= 32)
        launch_k8_tiled_rpw<1>(rpw, ctx, grid, smem, rows, ncols, rowptr, colidx, val, b, xt, Y, ldy, T, ngroups, rpc);
    else
        launch_k8_tiled_rpw<2>(rpw, ctx, grid, smem, rows, ncols, rowptr, colidx, val, b, xt, Y, ldy, T, ngroups, rpc);
    return true;
}

}  // namespace

void csr_spmm(Context& ctx, Index rows, const std::int64_t* rowptr, const std::int32_t* colidx, const double* val,
              Index ncols, Index b, const double* X, Index ldx, double* Y, Index ldy, double* xt, Index nnz) {
    if (rows <= 0 || b <= 0) return;
    to_row_major_k<<<grid_for(ncols * b), kThreads, 0, ctx.stream()>>>(X, ldx, ncols, b, xt);
    LAUNCH(ctx, "to_row_major");
    if (csr_spmm_tiled(ctx, rows, rowptr, colidx, val, ncols, b, xt, Y, ldy, nnz)) {
        LAUNCH(ctx, "csr_spmm_tiled");
        return;
    }
    const long warps_needed = rows;
    const unsigned blocks = static_cast<unsigned>(std::min<long>(8L * 1024, (warps_needed * 32 + kThreads - 1) / kThreads));
    if (b == 1)
        csr_spmm_narrow_k<1><<<blocks, kThreads, 0, ctx.stream()>>>(rows, rowptr, colidx, val, b, xt, Y, ldy);
    else if (b <= 4)
        csr_spmm_narrow_k<4><<<blocks, kThreads, 0, ctx.stream()>>>(rows, rowptr, colidx, val, b, xt, Y, ldy);
    else if (b <= 8)
        csr_spmm_narrow_k<8><<<blocks, kThreads, 0, ctx.stream()>>>(rows, rowptr, colidx, val, b, xt, Y, ldy);
    else if (b <= 32)
        csr_spmm_k<1><<<blocks, kThreads, 0, ctx.stream()>>>(rows, rowptr, colidx, val, b, xt, Y, ldy);
    else if (b <= 64)
        csr_spmm_k<2><<<blocks, kThreads, 0, ctx.stream()>>>(rows, rowptr, colidx, val, b, xt, Y, ldy);
    else if (b <= 128)
        csr_spmm_k<4><<<blocks, kThreads, 0, ctx.stream()>>>(rows, rowptr, colidx, val, b, xt, Y, ldy);
    else
        csr_spmm_wide_k<<<blocks, kThreads, 0, ctx.stream()>>>(rows, rowptr, colidx, val, b, xt, Y, ldy);
    LAUNCH(ctx, "csr_spmm");
}

void pack_rows(Context& ctx, View x, double* dst) {
    if (x.rows <= 0 || x.cols <= 0) return;
    pack_rows_k<<<grid_for(x.rows * x.cols), kThreads, 0, ctx.stream()>>>(x.p, x.ld, x.rows, x.cols, dst);
    LAUNCH(ctx, "pack_rows");
}

void unpack_rows(Context& ctx, const double* src, View dst) {
    if (dst.rows <= 0 || dst.cols <= 0) return;
    unpack_rows_k<<<grid_for(dst.rows * dst.cols), kThreads, 0, ctx.stream()>>>(src, dst.rows, dst.cols, dst.p, dst.ld);
    LAUNCH(ctx, "unpack_rows");
}

void gather_values(Context& ctx, Index nnz, double* dst, const double* src, const std::int64_t* perm) {
    if (nnz <= 0) return;
    gather_vals_k<<<grid_for(nnz), kThreads, 0, ctx.stream()>>>(nnz, dst, src, perm);
    LAUNCH(ctx, "gather_values");
}

}  // namespace blws
