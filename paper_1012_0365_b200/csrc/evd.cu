// Symmetric EVD of the projected block-tridiagonal T (K4), top `want` pairs.
//
// The reference diagonalises T = BlockTridiagonal::embed() completely with
// Eigen's SelfAdjointEigenSolver (block_lanczos.hpp:144 -> small_dense.hpp:36)
// and then keeps at most r leading positive pairs (block_lanczos.hpp:235-248).
// Here only the top `want` (= r) pairs are produced:
//   1. sytrd_k: Householder tridiagonalisation (LAPACK dsytd2, lower), one CTA,
//      the lower triangle packed in shared memory (global for large n);
//   2. tridiag_eig_top: bisection + inverse iteration on (d, e) (tridiag.cu);
//   3. ormtr_k: back-transformation Z = H_0 ... H_{n-3} Y, one warp per
//      eigenvector, no inter-warp synchronisation.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <string>

#include "bulk.cuh"
#include "ops.cuh"

namespace blws {
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRowsPerLane = 8;  // n <= 256 on this path (32 * 8 trailing rows per warp)
constexpr int kColsPerWarp = 16;    // 256 columns / 16 warps
constexpr long kSmemBudget = 220 * 1024;

__device__ __forceinline__ int loff(int j, int n) { return j * n - ((j * (j - 1)) >> 1); }  // start of column j
__device__ __forceinline__ int lidx(int i, int j, int n) {                                 // (i >= j), n <= 4096
    return loff(j, n) + (i - j);
}

__device__ double block_sum_1024(double v, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = 0.0;
    const int nw = blockDim.x >> 5;
    for (int w = 0; w < nw; ++w) s += red[w];
    return s;
}

// In: T (n x n, ld) symmetric. Out: d (n), e (n-1), packed lower with the
// reflectors below the diagonal (v[0] = 1 implicit) in `lp`, tau (n).
template <bool SH>
__global__ void __launch_bounds__(kThreads) sytrd_k(const double* __restrict__ t, long ld, int n,
                                                    double* lp, double* d, double* e, double* tau) {
    constexpr bool on_chip = SH;
    extern __shared__ __align__(16) double sm[];
    double* v = sm;               // n
    double* p = v + n;            // n
    double* pcol = p + n;         // n
    double* red = pcol + n;       // 32
    double* pw = red + 32;        // kWarps * n private partials (n <= 256 only)
    double* a = on_chip ? pw + (n <= 32 * kMaxRowsPerLane ? kWarps * n : 0) : lp;
    const long np = static_cast<long>(n) * (n + 1) / 2;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // load the lower triangle, column by column (warp per column)
    for (int j = wid; j < n; j += nw)
        for (int i = j + lane; i < n; i += 32) a[lidx(i, j, n)] = 0.5 * (t[i + j * ld] + t[j + i * ld]);
    __syncthreads();
    for (int k = 0; k < n - 2; ++k) {
        const int w = n - k - 1;  // trailing order, rows k+1 .. n-1
        double* x = a + lidx(k + 1, k, n);
        double s = 0.0;
        for (int i = 1 + threadIdx.x; i < w; i += blockDim.x) s += x[i] * x[i];
        const double sigma2 = block_sum_1024(s, red);
        const double alpha = x[0];
        double tk = 0.0, beta = alpha;
        if (sigma2 > 0.0) {
            beta = -copysign(sqrt(alpha * alpha + sigma2), alpha);
            tk = (beta - alpha) / beta;
            const double scl = 1.0 / (alpha - beta);
            for (int i = threadIdx.x; i < w; i += blockDim.x) v[i] = i == 0 ? 1.0 : x[i] * scl;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            e[k] = beta;
            tau[k] = tk;
            d[k] = a[lidx(k, k, n)];
        }
        if (tk == 0.0) {
            // H = I: store a zero reflector, nothing to update
            for (int i = threadIdx.x; i < w; i += blockDim.x) x[i] = 0.0;
            __syncthreads();
            continue;
        }
        // p = tau * A22 v from column reads only (conflict-free): warp `wid`
        // owns columns j = wid, wid+nw, ...; per column it forms the dot of the
        // strictly-lower part with v (-> pcol[j]) and accumulates L(:,j) v_j into
        // a private per-lane register vector (rows i = lane + 32 t).
        if (n > 32 * kMaxRowsPerLane) {
            // large orders: warp per row, row part strided (global-memory path)
            for (int i = wid; i < w; i += nw) {
                const int gi = k + 1 + i;
                double acc = 0.0;
                for (int j = lane; j < w; j += 32) {
                    const int gj = k + 1 + j;
                    const double aij = gi >= gj ? a[lidx(gi, gj, n)] : a[lidx(gj, gi, n)];
                    acc += aij * v[j];
                }
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (lane == 0) p[i] = tk * acc;
            }
        } else {
            // v, restricted to this lane's rows, in registers
            double vr[kMaxRowsPerLane], acc[kMaxRowsPerLane], dp[kColsPerWarp];
#pragma unroll
            for (int q = 0; q < kMaxRowsPerLane; ++q) {
                const int i = lane + 32 * q;
                vr[q] = i < w ? v[i] : 0.0;
                acc[q] = 0.0;
            }
#pragma unroll
            for (int c = 0; c < kColsPerWarp; ++c) {
                dp[c] = 0.0;
                const int j = wid + c * kWarps;
                if (j < w) {
                    const double* col = a + lidx(k + 1 + j, k + 1 + j, n) - j;  // col[i] = A(k+1+i, k+1+j)
                    const double vj = v[j];
#pragma unroll
                    for (int q = 0; q < kMaxRowsPerLane; ++q) {
                        const int i = lane + 32 * q;
                        if (i >= j && i < w) {
                            const double lij = col[i];
                            acc[q] = fma(lij, vj, acc[q]);
                            if (i > j) dp[c] = fma(lij, vr[q], dp[c]);
                        }
                    }
                }
            }
            // batched reduction of the kColsPerWarp (=16) column dots over the warp:
            // each stage halves the values per lane (16 -> 8 -> 4 -> 2 -> 1)
#pragma unroll
            for (int stage = 0; stage < 4; ++stage) {
                const int half = kColsPerWarp >> (stage + 1);
                const int o = 16 >> stage;
                const bool hi = (lane & o) != 0;
#pragma unroll
                for (int c = 0; c < half; ++c) {
                    const double send = hi ? dp[c] : dp[c + half];
                    const double keep = hi ? dp[c + half] : dp[c];
                    dp[c] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            dp[0] += __shfl_xor_sync(0xffffffffu, dp[0], 1);
            {
                const int c = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
                const int j = wid + c * kWarps;
                if ((lane & 1) == 0 && j < w) pcol[j] = dp[0];
            }
#pragma unroll
            for (int q = 0; q < kMaxRowsPerLane; ++q) {
                const int i = lane + 32 * q;
                if (i < w) pw[wid * n + i] = acc[q];
            }
            __syncthreads();
            for (int i = threadIdx.x; i < w; i += blockDim.x) {
                double sacc = pcol[i];
                for (int ww = 0; ww < nw; ++ww) sacc += pw[ww * n + i];
                p[i] = tk * sacc;
            }
        }
        __syncthreads();
        double pv = 0.0;
        for (int i = threadIdx.x; i < w; i += blockDim.x) pv += p[i] * v[i];
        const double K = 0.5 * tk * block_sum_1024(pv, red);
        for (int i = threadIdx.x; i < w; i += blockDim.x) p[i] -= K * v[i];  // p <- w
        __syncthreads();
        // A22 -= v w^T + w v^T (lower), warp per column
        if (n <= 32 * kMaxRowsPerLane) {
            double vr[kMaxRowsPerLane], wr[kMaxRowsPerLane];
#pragma unroll
            for (int q = 0; q < kMaxRowsPerLane; ++q) {
                const int i = lane + 32 * q;
                vr[q] = i < w ? v[i] : 0.0;
                wr[q] = i < w ? p[i] : 0.0;
            }
#pragma unroll
            for (int c = 0; c < kColsPerWarp; ++c) {
                const int j = wid + c * kWarps;
                if (j >= w) break;
                const double vj = v[j], wj = p[j];
                double* col = a + lidx(k + 1 + j, k + 1 + j, n) - j;
#pragma unroll
                for (int q = 0; q < kMaxRowsPerLane; ++q) {
                    const int i = lane + 32 * q;
                    if (i >= j && i < w) col[i] -= fma(vr[q], wj, wr[q] * vj);
                }
            }
        } else {
            for (int j = wid; j < w; j += nw) {
                const int gj = k + 1 + j;
                const double vj = v[j], wj = p[j];
                double* col = a + lidx(gj, gj, n) - j;  // so col[i] = A(k+1+i, gj) for i >= j
                for (int i = j + lane; i < w; i += 32) col[i] -= v[i] * wj + p[i] * vj;
            }
        }
        __syncthreads();
        // keep the reflector below the diagonal of column k
        for (int i = threadIdx.x; i < w; i += blockDim.x) x[i] = v[i];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (n >= 2) {
            d[n - 2] = a[lidx(n - 2, n - 2, n)];
            e[n - 2] = a[lidx(n - 1, n - 2, n)];
            tau[n - 2] = 0.0;
        }
        d[n - 1] = a[lidx(n - 1, n - 1, n)];
        tau[n - 1] = 0.0;
    }
    if (on_chip)
        for (long idx = threadIdx.x; idx < np; idx += blockDim.x) lp[idx] = a[idx];
}

// Z = H_0 H_1 ... H_{n-3} Y, column j of Y per warp; H_k = I - tau_k v_k v_k^T
// acting on rows k+1..n-1 with v_k stored in packed column k (v[0] = 1).
// Reflectors are staged through shared memory in chunks shared by the CTA.
constexpr int kOrmWarps = 8;
constexpr int kOrmChunk = 8;
__global__ void __launch_bounds__(kOrmWarps * 32) ormtr_k(const double* __restrict__ lp, const double* __restrict__ tau,
                                                          int n, int want, double* z, long ldz) {
    extern __shared__ __align__(16) double sm[];
    double* vs = sm;                           // kOrmChunk * n
    double* zs = sm + kOrmChunk * n;           // kOrmWarps * n
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long j = static_cast<long>(blockIdx.x) * kOrmWarps + warp;
    const bool active = j < want;
    double* zc = zs + warp * n;
    if (active)
        for (int i = lane; i < n; i += 32) zc[i] = z[i + j * ldz];
    for (int k0 = n - 3; k0 >= 0; k0 -= kOrmChunk) {
        const int k1 = max(0, k0 - kOrmChunk + 1);  // chunk covers k = k0 .. k1 (descending)
        __syncthreads();
        for (int kk = k1; kk <= k0; ++kk) {
            const int w = n - kk - 1;
            const double* src = lp + lidx(kk + 1, kk, n);
            double* dst = vs + (k0 - kk) * n;
            for (int i = threadIdx.x; i < w; i += blockDim.x) dst[i] = i == 0 ? 1.0 : src[i];
        }
        __syncthreads();
        if (!active) continue;
        for (int kk = k0; kk >= k1; --kk) {
            const double tk = tau[kk];
            if (tk == 0.0) continue;
            const double* vk = vs + (k0 - kk) * n;
            const int w = n - kk - 1;
            double s = 0.0;
            for (int i = lane; i < w; i += 32) s += vk[i] * zc[kk + 1 + i];
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            const double f = tk * s;
            for (int i = lane; i < w; i += 32) zc[kk + 1 + i] -= f * vk[i];
            __syncwarp();
        }
    }
    if (active)
        for (int i = lane; i < n; i += 32) z[i + j * ldz] = zc[i];
}

// Z = H_0 ... H_{n-3} Y straight from global memory (large orders, where the
// shared-memory staging of ormtr_k does not fit): one warp per eigenvector,
// reflectors and the vector read through L2.
__global__ void __launch_bounds__(kOrmWarps * 32) ormtr_global_k(const double* __restrict__ lp,
                                                                 const double* __restrict__ tau, int n, int want,
                                                                 double* z, long ldz) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long j = static_cast<long>(blockIdx.x) * kOrmWarps + warp;
    if (j >= want) return;
    double* zc = z + j * ldz;
    for (int k = n - 3; k >= 0; --k) {
        const double tk = tau[k];
        if (tk == 0.0) continue;
        const int w = n - k - 1;
        const double* vk = lp + lidx(k + 1, k, n);  // vk[0] = 1 (stored)
        double s = 0.0;
        for (int i = lane; i < w; i += 32) s = fma(i == 0 ? 1.0 : vk[i], zc[k + 1 + i], s);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const double f = tk * s;
        for (int i = lane; i < w; i += 32) zc[k + 1 + i] -= f * (i == 0 ? 1.0 : vk[i]);
        __syncwarp();
    }
}

// Z = H_0 ... H_{n-3} Y with every reflector resident in shared memory (the
// packed lower triangle, n <= 208) and each eigenvector in registers of one
// warp (row i = lane + 32 q): no block barrier after the load, one warp
// reduction per reflector. 4 warps per block (one per scheduler).
constexpr int kOrmFullWarps = 4;
template <int QN>
__global__ void __launch_bounds__(kOrmFullWarps * 32) ormtr_full_k(const double* __restrict__ lp,
                                                                    const double* __restrict__ tau, int n, int want,
                                                                    double* z, long ldz) {
    extern __shared__ __align__(16) double sm[];
    double* ts = sm;      // n
    double* a = sm + n;   // packed lower triangle with the reflectors
    const long np = static_cast<long>(n) * (n + 1) / 2;
    for (long idx = threadIdx.x; idx < np; idx += blockDim.x) a[idx] = lp[idx];
    for (int i = threadIdx.x; i < n; i += blockDim.x) ts[i] = tau[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long j = static_cast<long>(blockIdx.x) * kOrmFullWarps + warp;
    if (j >= want) return;
    double zr[QN];
#pragma unroll
    for (int q = 0; q < QN; ++q) {
        const int i = lane + 32 * q;
        zr[q] = i < n ? z[i + j * ldz] : 0.0;
    }
    for (int k = n - 3; k >= 0; --k) {
        const double tk = ts[k];
        if (tk == 0.0) continue;
        const double* col = a + lidx(k, k, n) - k;  // col[i] = reflector entry of row i (i > k)
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int i = lane + 32 * q;
            if (i > k && i < n) s = fma(col[i], zr[q], s);
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const double f = tk * s;
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int i = lane + 32 * q;
            if (i > k && i < n) zr[q] = fma(-f, col[i], zr[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < QN; ++q) {
        const int i = lane + 32 * q;
        if (i < n) z[i + j * ldz] = zr[q];
    }
}

// The same product with the reflectors taken G at a time in compact WY form
// (LAPACK dlarft, forward / columnwise): H_lo H_lo+1 ... H_lo+G-1 = I - V T V^T,
// so each eigenvector needs ceil((n-2) / G) sequential steps, each with G
// independent dot products reduced together, instead of n - 2 steps with one
// warp reduction each (the reduction latency was the whole cost). The T factors
// (G x G upper triangular per group, from the pairwise v_i^T v_j and tau) are
// formed once per block in shared memory. Group g = 0 holds the highest
// reflector indices (applied first).
template <int QN, int G>
__global__ void __launch_bounds__(kOrmFullWarps * 32) ormtr_wy_k(const double* __restrict__ lp,
                                                                  const double* __restrict__ tau, int n, int want,
                                                                  double* z, long ldz) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bar;
    const long np = static_cast<long>(n) * (n + 1) / 2;
    double* a = sm;                 // packed lower triangle with the reflectors
    double* ts = sm + (np + 1) / 2 * 2;  // n (16-byte aligned)
    double* tf = ts + n;            // groups x G x G
    const int nref = n - 2;   // reflectors 0 .. n-3
    const int groups = (nref + G - 1) / G;
    for (int i = threadIdx.x; i < n; i += blockDim.x) ts[i] = tau[i];
    block_load_bulk(a, lp, np, &bar);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // ---- T factors, one group per warp at a time
    for (int g = warp; g < groups; g += kOrmFullWarps) {
        const int hi = nref - g * G, lo = max(0, hi - G), cnt = hi - lo;
        double d[G][G];  // d[l][j] = v_l^T v_j (l < j), rows > lo + j
#pragma unroll
        for (int l = 0; l < G; ++l)
#pragma unroll
            for (int j = 0; j < G; ++j) d[l][j] = 0.0;
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int i = lane + 32 * q;
            double vr[G];
#pragma unroll
            for (int l = 0; l < G; ++l) {
                const int k = lo + l;
                vr[l] = (l < cnt && i > k && i < n) ? a[lidx(k, k, n) - k + i] : 0.0;
            }
#pragma unroll
            for (int j = 1; j < G; ++j)
#pragma unroll
                for (int l = 0; l < j; ++l) d[l][j] = fma(vr[l], vr[j], d[l][j]);
        }
#pragma unroll
        for (int j = 1; j < G; ++j)
#pragma unroll
            for (int l = 0; l < j; ++l)
                for (int o = 16; o > 0; o >>= 1) d[l][j] += __shfl_xor_sync(0xffffffffu, d[l][j], o);
        if (lane == 0) {
            double* T = tf + static_cast<long>(g) * G * G;  // T[i + j G]
#pragma unroll
            for (int j = 0; j < G; ++j) {
                const double tj = j < cnt ? ts[lo + j] : 0.0;
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    double w = 0.0;
                    if (i < j) {
#pragma unroll
                        for (int l = 0; l < G; ++l)
                            if (l >= i && l < j) w = fma(T[i + l * G], d[l][j], w);
                    }
                    T[i + j * G] = i < j ? -tj * w : (i == j ? tj : 0.0);
                }
            }
        }
    }
    __syncthreads();
    const long jv = static_cast<long>(blockIdx.x) * kOrmFullWarps + warp;
    if (jv >= want) return;
    double zr[QN];
#pragma unroll
    for (int q = 0; q < QN; ++q) {
        const int i = lane + 32 * q;
        zr[q] = i < n ? z[i + jv * ldz] : 0.0;
    }
    for (int g = 0; g < groups; ++g) {
        const int hi = nref - g * G, lo = max(0, hi - G), cnt = hi - lo;
        double sv[G], vq[QN][G];
#pragma unroll
        for (int l = 0; l < G; ++l) sv[l] = 0.0;
#pragma unroll
        for (int q = 0; q < QN; ++q) {
            const int i = lane + 32 * q;
#pragma unroll
            for (int l = 0; l < G; ++l) {
                const int k = lo + l;
                // slots whose rows are all <= lo hold no reflector entries (warp-uniform)
                vq[q][l] = (32 * q + 31 > lo && l < cnt && i > k && i < n) ? a[lidx(k, k, n) - k + i] : 0.0;
                sv[l] = fma(vq[q][l], zr[q], sv[l]);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int l = 0; l < G; ++l) sv[l] += __shfl_xor_sync(0xffffffffu, sv[l], o);
        const double* T = tf + static_cast<long>(g) * G * G;
        double u[G];  // u = T s (upper triangular)
#pragma unroll
        for (int i = 0; i < G; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int j = i; j < G; ++j) acc = fma(T[i + j * G], sv[j], acc);
            u[i] = acc;
        }
#pragma unroll
        for (int q = 0; q < QN; ++q)
#pragma unroll
            for (int l = 0; l < G; ++l) zr[q] = fma(-u[l], vq[q][l], zr[q]);
    }
#pragma unroll
    for (int q = 0; q < QN; ++q) {
        const int i = lane + 32 * q;
        if (i < n) z[i + jv * ldz] = zr[q];
    }
}

#ifndef BLWS_ORM_G
#define BLWS_ORM_G 4
#endif
template <int QN>
bool launch_ormtr_wy(Context& ctx, const double* lp, const double* tau, int n, int want, View z) {
    constexpr int G = BLWS_ORM_G;
    const int groups = (n - 2 + G - 1) / G;
    const size_t bytes =
        (static_cast<size_t>(n) + 1 + static_cast<size_t>(n) * (n + 1) / 2 + static_cast<size_t>(groups) * G * G) *
        sizeof(double);
    if (bytes > 220u * 1024u) return false;
    static bool cfg = false;
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(ormtr_wy_k<QN, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        cfg = true;
    }
    ormtr_wy_k<QN, G><<<static_cast<unsigned>((want + kOrmFullWarps - 1) / kOrmFullWarps), kOrmFullWarps * 32, bytes,
                        ctx.stream()>>>(lp, tau, n, want, z.p, z.ld);
    ctx.note_launch();
    ctx.check_launch("ormtr_wy_k");
    return true;
}

template <int QN>
bool launch_ormtr_full(Context& ctx, const double* lp, const double* tau, int n, int want, View z) {
    const size_t bytes = (static_cast<size_t>(n) + static_cast<size_t>(n) * (n + 1) / 2) * sizeof(double);
    if (bytes > 220u * 1024u) return false;
    static bool cfg = false;
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(ormtr_full_k<QN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        cfg = true;
    }
    ormtr_full_k<QN><<<static_cast<unsigned>((want + kOrmFullWarps - 1) / kOrmFullWarps), kOrmFullWarps * 32, bytes,
                       ctx.stream()>>>(lp, tau, n, want, z.p, z.ld);
    ctx.note_launch();
    ctx.check_launch("ormtr_full_k");
    return true;
}

bool ormtr_full(Context& ctx, const double* lp, const double* tau, int n, int want, View z) {
    static const bool wy = [] {
        const char* e = std::getenv("BLWS_ORMTR");
        return !(e && std::string(e) == "single");
    }();
    if (wy && n >= 3) {
        switch ((n + 31) / 32) {
            case 1: if (launch_ormtr_wy<1>(ctx, lp, tau, n, want, z)) return true; break;
            case 2: if (launch_ormtr_wy<2>(ctx, lp, tau, n, want, z)) return true; break;
            case 3: if (launch_ormtr_wy<3>(ctx, lp, tau, n, want, z)) return true; break;
            case 4: if (launch_ormtr_wy<4>(ctx, lp, tau, n, want, z)) return true; break;
            case 5: if (launch_ormtr_wy<5>(ctx, lp, tau, n, want, z)) return true; break;
            case 6: if (launch_ormtr_wy<6>(ctx, lp, tau, n, want, z)) return true; break;
            case 7: if (launch_ormtr_wy<7>(ctx, lp, tau, n, want, z)) return true; break;
            default: break;
        }
    }
    switch ((n + 31) / 32) {
        case 1: return launch_ormtr_full<1>(ctx, lp, tau, n, want, z);
        case 2: return launch_ormtr_full<2>(ctx, lp, tau, n, want, z);
        case 3: return launch_ormtr_full<3>(ctx, lp, tau, n, want, z);
        case 4: return launch_ormtr_full<4>(ctx, lp, tau, n, want, z);
        case 5: return launch_ormtr_full<5>(ctx, lp, tau, n, want, z);
        case 6: return launch_ormtr_full<6>(ctx, lp, tau, n, want, z);
        case 7: return launch_ormtr_full<7>(ctx, lp, tau, n, want, z);
        default: return false;
    }
}

}  // namespace

bool sytrd_cluster(Context& ctx, View t, double* lp, double* d, double* e, double* tau, bool auto_pick);
bool sytrd_fused(Context& ctx, View t, double* lp, double* d, double* e, double* tau);

void sym_evd_top(Context& ctx, View t, Index want, double* values, View vectors) {
    const int n = static_cast<int>(t.rows);
    if (n <= 0 || want <= 0) return;
    static const bool trace = std::getenv("BLWS_EVD_TRACE") != nullptr;
    if (trace) std::fprintf(stderr, "sym_evd_top n=%d want=%lld\n", n, static_cast<long long>(want));
    if (n == 1) {
        BLWS_CUDA(cudaMemcpyAsync(values, t.p, sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream()));
        fill(ctx, vectors.left(1), 1.0);
        return;
    }
    if (sytrd2_fits(n)) return sym_evd_top_two_stage(ctx, t, want, values, vectors);
    const long np = static_cast<long>(n) * (n + 1) / 2;
    const long head = (3L * n + 32 + (n <= 32 * kMaxRowsPerLane ? static_cast<long>(kWarps) * n : 0)) * 8;
    const bool on_chip = head + np * 8 <= kSmemBudget;
    DBuf<double> lp(ctx, static_cast<size_t>(np)), d(ctx, static_cast<size_t>(n)), e(ctx, static_cast<size_t>(n)),
        tau(ctx, static_cast<size_t>(n));
    static bool cfg = false;
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(sytrd_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
        BLWS_CUDA(cudaFuncSetAttribute(sytrd_k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
        cfg = true;
    }
    const int smem = static_cast<int>(head + (on_chip ? np * 8 : 0));
    if (!sytrd_cluster(ctx, t, lp.get(), d.get(), e.get(), tau.get(), false) &&
        !sytrd_fused(ctx, t, lp.get(), d.get(), e.get(), tau.get()) &&
        !sytrd_cluster(ctx, t, lp.get(), d.get(), e.get(), tau.get(), true)) {
    if (on_chip)
        sytrd_k<true><<<1, kThreads, smem, ctx.stream()>>>(t.p, t.ld, n, lp.get(), d.get(), e.get(), tau.get());
    else
        sytrd_k<false><<<1, kThreads, smem, ctx.stream()>>>(t.p, t.ld, n, lp.get(), d.get(), e.get(), tau.get());
    ctx.note_launch();
    ctx.check_launch("sytrd_k");
    }
    tridiag_eig_top(ctx, n, d.get(), e.get(), want, values, vectors);
    static bool cfg2 = false;
    if (!cfg2) {
        BLWS_CUDA(cudaFuncSetAttribute(ormtr_k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
        cfg2 = true;
    }
    if (ormtr_full(ctx, lp.get(), tau.get(), n, static_cast<int>(want), vectors)) return;
    const int smem2 = (kOrmChunk + kOrmWarps) * n * 8;
    if (smem2 > kSmemBudget) {
        ormtr_global_k<<<static_cast<unsigned>((want + kOrmWarps - 1) / kOrmWarps), kOrmWarps * 32, 0,
                         ctx.stream()>>>(lp.get(), tau.get(), n, static_cast<int>(want), vectors.p, vectors.ld);
        ctx.note_launch();
        ctx.check_launch("ormtr_global_k");
        return;
    }
    ormtr_k<<<static_cast<unsigned>((want + kOrmWarps - 1) / kOrmWarps), kOrmWarps * 32, smem2, ctx.stream()>>>(
        lp.get(), tau.get(), n, static_cast<int>(want), vectors.p, vectors.ld);
    ctx.note_launch();
    ctx.check_launch("ormtr_k");
}

// full_svd_small (small_dense.hpp:72-87) on the device, from the symmetric
// embedding (theorem 1, block_lanczos.hpp): the top p = min(m, n) eigenpairs of
// [[0, W], [W^T, 0]] are (sigma_i, [u_i; v_i] / sqrt(2)). Exact to ~eps ||W||
// for distinct nonzero sigma (a zero or repeated singular value mixes the
// +/- pairs; the reference's BDCSVD has no such caveat).
void full_svd_small(Context& ctx, View w, double* sigma, View u, View v) {
    const Index m = w.rows, n = w.cols, p = std::min(m, n), d = m + n;
    if (d > 4096) throw std::invalid_argument("full_svd_small: m + n exceeds the small-dense limit (4096)");
    DMat t(ctx, d, d, true);
    place_block(ctx, t.view().sub(0, m, m, n), w, false);
    place_block(ctx, t.view().sub(m, 0, n, m), w, true);
    DMat vecs(ctx, d, p, false);
    sym_evd_top(ctx, t.view(), p, sigma, vecs.view());
    copy(ctx, u, View{vecs.data(), m, p, vecs.ld}, std::sqrt(2.0));
    copy(ctx, v, View{vecs.data() + m, n, p, vecs.ld}, std::sqrt(2.0));
}

}  // namespace blws
