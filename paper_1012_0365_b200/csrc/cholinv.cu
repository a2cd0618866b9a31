// Fused Cholesky + triangular inverse for CholQR (K3): G = R^T R, Rinv = R^{-1}.
// With skip_rel > 0 a Gram that is a scaled identity to ||G - cI||_F <=
// skip_rel c (c = tr(G) / n) returns R = sqrt(c) I, Rinv = I / sqrt(c) instead
// (the CholQR pass skip, decided on the device); tr(G) is optionally written out.
//
// thin_qr (core/qr.hpp:24-47) becomes CholQR2 on the device; each pass needs
// chol(G) and R^{-1} of a b x b Gram (b <= ~411). One CTA does both:
//   * right-looking Cholesky: per column one warp scales the pivot row, then
//     every warp updates its trailing columns (two barriers per column);
//   * R^{-1} by recursive doubling, X = [[XA, -XA B XC], [0, XC]] over block
//     sizes k = 1, 2, 4, ...; from k = 8 on, the two products per level run on
//     DMMA m8n8k4 fragments (measured: 70k -> 34k cycles at b = 104).
// Compact loops on purpose: fully unrolled register-resident blocks made the
// code large enough to thrash the instruction cache (measured 30 us at b=32).
// Staged in shared memory when it fits (b <= 116); the SH template parameter
// keeps those accesses LDS/STS instead of generic loads.
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "ops.cuh"

namespace blws {
__device__ double g_chol_probe[4];  // phase cycle counts of the last chol_inv call (profiling)
namespace {

/// a[idx] for a runtime idx in [0, 32) as a 5-level select tree (depth 5
/// instead of a 32-long dependent select chain).
__device__ __forceinline__ double pick32(const double (&a)[32], int idx) {
    double v16[16], v8[8], v4[4], v2[2];
#pragma unroll
    for (int j = 0; j < 16; ++j) v16[j] = (idx & 16) ? a[j + 16] : a[j];
#pragma unroll
    for (int j = 0; j < 8; ++j) v8[j] = (idx & 8) ? v16[j + 8] : v16[j];
#pragma unroll
    for (int j = 0; j < 4; ++j) v4[j] = (idx & 4) ? v8[j + 4] : v8[j];
#pragma unroll
    for (int j = 0; j < 2; ++j) v2[j] = (idx & 2) ? v4[j + 2] : v4[j];
    return (idx & 1) ? v2[1] : v2[0];
}

constexpr int kCT = 1024;  // one thread per element of a 32x32 diagonal block

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}
constexpr long kSmemBudget = 216 * 1024;

// block-wide sum (all threads get the result); red: 32 doubles
__device__ __forceinline__ double chol_block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = lane < nw ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

template <bool SH>
__global__ void __launch_bounds__(kCT) chol_inv_k(double* g, long ldg, double* rinv, long ldri, int n,
                                                  double* scratch, int* status, double* diag, double skip_rel,
                                                  double* trace_out) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int fail;
    __shared__ double red[32];
    const int ld = n | 1;  // odd stride: conflict-free row access
    double* A = SH ? sm : scratch;
    double* X = A + static_cast<long>(ld) * n;
    double* rowj = X + static_cast<long>(ld) * n;  // n
    double* dinv = rowj + n;                         // n
    double* rowbuf = dinv + n;                       // 32 row entries + 2 pivot slots
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) fail = 0;
    long long t0 = clock64();
    for (int j = wid; j < n; j += nw)
        for (int i = lane; i < n; i += 32) A[i + j * ld] = g[i + j * ldg];
    __syncthreads();
    // trace (= ||X||_F^2 for a Gram) and the scaled-identity test of the CholQR
    // pass skip: ||G - c I||_F <= skip_rel c with c = tr(G) / n gives R = sqrt(c) I
    double tr = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) tr += A[i + i * ld];
    tr = chol_block_sum(tr, red);
    if (trace_out && threadIdx.x == 0) *trace_out = tr;
    if (skip_rel > 0.0 && tr > 0.0 && isfinite(tr)) {
        const double c = tr / n;
        double off = 0.0;
        for (int j = wid; j < n; j += nw)
            for (int i = lane; i < n; i += 32) {
                const double x = A[i + j * ld] - (i == j ? c : 0.0);
                off = fma(x, x, off);
            }
        off = chol_block_sum(off, red);
        if (off <= skip_rel * skip_rel * c * c) {
            const double rc = sqrt(c), ric = 1.0 / rc;
            for (int j = wid; j < n; j += nw)
                for (int i = lane; i < n; i += 32) {
                    g[i + j * ldg] = i == j ? rc : 0.0;
                    if (rinv) rinv[i + j * ldri] = i == j ? ric : 0.0;
                }
            if (threadIdx.x == 0) {
                status[0] = 0;
                diag[0] = rc;
                diag[1] = rc;
            }
            return;
        }
    }
    long long t1 = clock64();
    // ---- right-looking Cholesky, trailing matrix in registers: thread t owns
    // upper-triangle entries e = t + kCT * q (q < kOwn) in column-major packed
    // order. Per column: the pivot owner publishes R(k,k); row-k owners publish
    // R(k, j); every owner updates its (i, j) with k < i <= j.
    // ---- blocked right-looking Cholesky (32-wide panels)
    long long td = 0, tp = 0, tsy = 0;
    for (int kb = 0; kb < n && !fail; kb += 32) {
        const int nb = min(32, n - kb);
        long long c0 = clock64();
        {
            // diagonal block: thread t owns element (i, j) = (t % 32, t / 32) of the
            // 32x32 block in a register (all 1024 threads); two barriers per pivot
            const int ti = threadIdx.x & 31, tj = threadIdx.x >> 5;
            const bool own = ti < nb && tj < nb && ti <= tj;
            double a = own ? A[(kb + ti) + (kb + tj) * ld] : 0.0;
            if (ti == 0 && tj == 0) rowbuf[32] = a;  // pivot 0
            __syncthreads();
            for (int k = 0; k < nb; ++k) {
                const double piv = rowbuf[32 + (k & 1)];
                const bool bad = !(piv > 0.0) || !isfinite(piv);
                const double rs = bad ? 1.0 : rsqrt(piv);
                if (own && ti == k) {
                    a = (tj == k) ? piv * rs : a * rs;
                    rowbuf[tj] = a;
                }
                if (threadIdx.x == 0) {
                    dinv[kb + k] = rs;
                    if (bad && fail == 0) fail = kb + k + 1;
                }
                __syncthreads();
                if (own && ti > k) {
                    a = fma(-rowbuf[ti], rowbuf[tj], a);
                    if (ti == k + 1 && tj == k + 1) rowbuf[32 + ((k + 1) & 1)] = a;
                }
                __syncthreads();
            }
            if (ti < nb && tj < nb) A[(kb + ti) + (kb + tj) * ld] = own ? a : 0.0;
        }
        __syncthreads();
        long long c1 = clock64();
        td += c1 - c0;
        if (fail) break;
        const int rest = n - kb - nb;
        if (rest <= 0) break;
        // panel rows: R12 = R11^{-T} A12, forward substitution, warp per column, lane = row
        for (int j = kb + nb + wid; j < n; j += nw) {
            double x = lane < nb ? A[kb + lane + j * ld] : 0.0;
            for (int ii = 0; ii < nb; ++ii) {
                const double xi = __shfl_sync(0xffffffffu, x, ii) * dinv[kb + ii];
                if (lane == ii) x = xi;
                if (lane > ii && lane < nb) x -= A[kb + ii + (kb + lane) * ld] * xi;
            }
            if (lane < nb) A[kb + lane + j * ld] = x;
        }
        __syncthreads();
        long long c2 = clock64();
        tp += c2 - c1;
        // trailing SYRK (upper): A22 -= R12^T R12, warp per column, lanes over rows
        for (int j = kb + nb + wid; j < n; j += nw) {
            const double* cj = A + kb + j * ld;
            for (int i2 = kb + nb + lane; i2 <= j; i2 += 32) {
                const double* ci = A + kb + i2 * ld;
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                int k = 0;
                for (; k + 3 < nb; k += 4) {
                    s0 = fma(ci[k], cj[k], s0);
                    s1 = fma(ci[k + 1], cj[k + 1], s1);
                    s2 = fma(ci[k + 2], cj[k + 2], s2);
                    s3 = fma(ci[k + 3], cj[k + 3], s3);
                }
                for (; k < nb; ++k) s0 = fma(ci[k], cj[k], s0);
                A[i2 + j * ld] -= (s0 + s1) + (s2 + s3);
            }
        }
        __syncthreads();
        tsy += clock64() - c2;
    }
    long long t2 = clock64();
    if (threadIdx.x == 0) status[0] = fail;
    if (fail) return;
    // ---- R^{-1} by recursive doubling: X_{2k-block} = [[XA, -XA B XC], [0, XC]]
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        const int i = idx % n, j = idx / n;
        X[i + j * ld] = i == j ? dinv[i] : 0.0;
    }
    __syncthreads();
    for (int lk = 0; (1 << lk) < n; ++lk) {
        const int k = 1 << lk;  // power of two: index math by shifts / masks
        const int pairs = (n + 2 * k - 1) / (2 * k);
        if (k >= 8) {
            // DMMA m8n8k4 on 8x8 fragments (lane g = lane / 4, t = lane % 4):
            // phase 1, T = B XC into X's upper-right block (no read/write overlap);
            // phase 2, X_UR = -XA T in place: a warp owns a column block and walks the
            // row blocks top-down -- XA is upper triangular, so row block fr reads
            // T rows >= 8 fr only, none of which it has overwritten yet.
            const int g = lane >> 2, t4 = lane & 3;
            const int kf = k >> 3;  // fragments per side
            auto ldx = [&](const double* M, int r, int c) { return (r < n && c < n) ? M[r + c * ld] : 0.0; };
            for (int task = wid; task < pairs * kf * kf; task += nw) {
                const int p = task / (kf * kf), fr = (task / kf) % kf, fc = task % kf;
                const int o = p * 2 * k, r0 = o + 8 * fr, c0 = o + k + 8 * fc;
                if (c0 >= n) continue;
                double acc[2] = {0.0, 0.0}, acc2[2] = {0.0, 0.0};
                const int tend = min(o + k + 8 * fc + 8, n);  // XC[t][c] = 0 for t > c
                int t = o + k;
                for (; t + 4 < tend; t += 8) {
                    dmma884(acc, ldx(A, r0 + g, t + t4), ldx(X, t + t4, c0 + g));
                    dmma884(acc2, ldx(A, r0 + g, t + 4 + t4), ldx(X, t + 4 + t4, c0 + g));
                }
                for (; t < tend; t += 4) dmma884(acc, ldx(A, r0 + g, t + t4), ldx(X, t + t4, c0 + g));
                const int r = r0 + g;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = c0 + 2 * t4 + e;
                    if (r < n && c < n) X[r + c * ld] = acc[e] + acc2[e];
                }
            }
            __syncthreads();
            for (int task = wid; task < pairs * kf; task += nw) {
                const int p = task / kf, fc = task % kf;
                const int o = p * 2 * k, c0 = o + k + 8 * fc;
                if (c0 >= n) continue;
                for (int fr = 0; fr < kf; ++fr) {
                    const int r0 = o + 8 * fr;
                    double acc[2] = {0.0, 0.0}, acc2[2] = {0.0, 0.0};
                    const int tend = min(o + k, n);
                    int t = r0;  // XA[r][t] = 0 for t < r
                    for (; t + 4 < tend; t += 8) {
                        dmma884(acc, ldx(X, r0 + g, t + t4), ldx(X, t + t4, c0 + g));
                        dmma884(acc2, ldx(X, r0 + g, t + 4 + t4), ldx(X, t + 4 + t4, c0 + g));
                    }
                    for (; t < tend; t += 4) dmma884(acc, ldx(X, r0 + g, t + t4), ldx(X, t + t4, c0 + g));
                    __syncwarp();
                    const int r = r0 + g;
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int c = c0 + 2 * t4 + e;
                        if (r < n && c < n) X[r + c * ld] = -(acc[e] + acc2[e]);
                    }
                    __syncwarp();
                }
            }
            __syncthreads();
            continue;
        }
        const int total = pairs * k * k;
        // phase 1: T = B XC into X's upper-right block (B = R[o:o+k, o+k:o+2k])
        for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
            const int p = idx >> (2 * lk), rr = idx & (k - 1), cc = (idx >> lk) & (k - 1);
            const int o = p * 2 * k, r = o + rr, c = o + k + cc;
            if (c >= n) continue;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int t = o + k;
            for (; t + 3 <= c; t += 4) {
                s0 = fma(A[r + t * ld], X[t + c * ld], s0);
                s1 = fma(A[r + (t + 1) * ld], X[t + 1 + c * ld], s1);
                s2 = fma(A[r + (t + 2) * ld], X[t + 2 + c * ld], s2);
                s3 = fma(A[r + (t + 3) * ld], X[t + 3 + c * ld], s3);
            }
            for (; t <= c; ++t) s0 = fma(A[r + t * ld], X[t + c * ld], s0);
            X[r + c * ld] = (s0 + s1) + (s2 + s3);
        }
        __syncthreads();
        // phase 2: X_UR = -XA T (read all into registers, sync, write)
        for (int base = 0; base < total; base += 4 * kCT) {
            double out[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int idx = base + q * kCT + threadIdx.x;
                out[q] = 0.0;
                if (idx >= total) continue;
                const int p = idx >> (2 * lk), rr = idx & (k - 1), cc = (idx >> lk) & (k - 1);
                const int o = p * 2 * k, r = o + rr, c = o + k + cc;
                if (c >= n) continue;
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                int t = r;
                for (; t + 3 < o + k; t += 4) {
                    s0 = fma(X[r + t * ld], X[t + c * ld], s0);
                    s1 = fma(X[r + (t + 1) * ld], X[t + 1 + c * ld], s1);
                    s2 = fma(X[r + (t + 2) * ld], X[t + 2 + c * ld], s2);
                    s3 = fma(X[r + (t + 3) * ld], X[t + 3 + c * ld], s3);
                }
                for (; t < o + k; ++t) s0 = fma(X[r + t * ld], X[t + c * ld], s0);
                out[q] = -((s0 + s1) + (s2 + s3));
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int idx = base + q * kCT + threadIdx.x;
                if (idx >= total) continue;
                const int p = idx >> (2 * lk), rr = idx & (k - 1), cc = (idx >> lk) & (k - 1);
                const int o = p * 2 * k, r = o + rr, c = o + k + cc;
                if (c < n) X[r + c * ld] = out[q];
            }
            __syncthreads();
        }
    }
    __syncthreads();
    long long t3 = clock64();
    double mn = INFINITY, mx = 0.0;
    for (int j = wid; j < n; j += nw)
        for (int i = lane; i < n; i += 32) {
            const double v = i > j ? 0.0 : A[i + j * ld];
            g[i + j * ldg] = v;
            if (rinv) rinv[i + j * ldri] = i > j ? 0.0 : X[i + j * ld];
            if (i == j) {
                mn = fmin(mn, v);
                mx = fmax(mx, v);
            }
        }
    __shared__ double smn[32], smx[32];
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
        smn[wid] = mn;
        smx[wid] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w2 = 1; w2 < nw; ++w2) {
            mn = fmin(mn, smn[w2]);
            mx = fmax(mx, smx[w2]);
        }
        diag[0] = mn;
        diag[1] = mx;
        g_chol_probe[0] = static_cast<double>(td) + 1e-6 * static_cast<double>(tp);  // diag . panel(1e6 scale)
        g_chol_probe[4 % 4] = static_cast<double>(td);
        g_chol_probe[1] = static_cast<double>(t2 - t1);
        g_chol_probe[2] = static_cast<double>(t3 - t2);
        g_chol_probe[3] = static_cast<double>(tp) * 1e6 + static_cast<double>(tsy);
    }
}

}  // namespace

void chol_inv_upper(Context& ctx, View g, View rinv, int* status, double* diag, double skip_rel,
                    double* trace_out) {
    const int n = static_cast<int>(g.rows);
    static const bool blocked = [] {
        const char* e = std::getenv("BLWS_CHOL_BLOCKED");
        return !(e && e[0] == '0');
    }();
    if (blocked && chol_blocked_fits(n)) return chol_inv_blocked(ctx, g, rinv, status, diag, trace_out);
    const long ld = n | 1;
    const long bytes = (2L * ld * n + 2L * n + 34) * 8;
    const bool on_chip = bytes <= kSmemBudget;
    static bool cfg = false;
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(chol_inv_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
        cfg = true;
    }
    if (on_chip) {
        chol_inv_k<true><<<1, kCT, bytes, ctx.stream()>>>(g.p, g.ld, rinv.p, rinv.ld, n, nullptr, status, diag,
                                                         skip_rel, trace_out);
    } else {
        DBuf<double> scratch(ctx, static_cast<size_t>(2L * ld * n + 2L * n + 34));
        chol_inv_k<false><<<1, kCT, 0, ctx.stream()>>>(g.p, g.ld, rinv.p, rinv.ld, n, scratch.get(), status,
                                               diag, skip_rel, trace_out);
    }
    ctx.note_launch();
    ctx.check_launch("chol_inv_k");
}

}  // namespace blws

namespace blws {
void chol_probe_read(double* out) { BLWS_CUDA(cudaMemcpyFromSymbol(out, g_chol_probe, 4 * sizeof(double))); }
}  // namespace blws
