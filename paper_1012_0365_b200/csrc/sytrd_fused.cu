// Householder tridiagonalisation of T (K4, stage 1), LAPACK dsytd2 (lower)
// semantics, one CTA, for orders n <= 208 (the packed lower triangle on chip).
//
// Single-pass formulation: every step reads and writes each trailing element
// once, and no phase runs on a single warp. Step k (v_k known):
//   [S]  sweep over columns j >= k+1: apply the pending rank-2 update of step
//        k-1 to each element, then accumulate p = A22 v_k from the updated
//        value -- rows in per-lane registers (row i = lane + 32 q), columns as
//        per-warp dots (column j = wid + 16 c), reduced by a batched transpose;
//        (each warp also reduces its share of v^T A v, so K = tau^2/2 v^T A v
//        needs no block reduction of its own);
//   [P]  one row per thread: p_i = tau_k (column dot + row partials), w_i =
//        p_i - K v_i; look-ahead: apply update k to column k+1 (element i per
//        thread; w_{k+1} formed by every thread from broadcast reads) and its
//        sum of squares below the subdiagonal;
//   [P3] every thread forms beta, tau_{k+1}, v_{k+1} and stores its reflector
//        element; three block barriers per step.
// Thread ownership in [S] is static: row i >= column j needs q >= c / 2, so
// the unrolled loops cover exactly that slot triangle; only the q = c / 2 slot
// carries a lane predicate. v and w are double-buffered by step parity and zero
// outside the trailing range (the pending update is a no-op there).
// Output equals sytrd_k's layout (packed lower + reflectors, d, e, tau).
#include "ops.cuh"

#ifdef SYTRD_PROBE  // per-phase cycle accounting (tools/probes/sytrd_probe.cu only)
__device__ unsigned long long g_sytrd_phase[8];
__device__ unsigned int g_sytrd_sweep[256];  // sweep cycles per step (thread 0)
#define PHASE_MARK(id)                                                       \
    do {                                                                     \
        if (threadIdx.x == 0) {                                              \
            const long long t_ = clock64();                                  \
            s_phase[id] += static_cast<unsigned long long>(t_ - tp_);        \
            tp_ = t_;                                                        \
        }                                                                    \
    } while (0)
#else
#define PHASE_MARK(id) \
    do {               \
    } while (0)
#endif

namespace blws {
namespace {

constexpr int kFT = 512;  // 16 warps
constexpr int kFW = kFT / 32;

__device__ __forceinline__ int floff(int j, int n) { return j * n - ((j * (j - 1)) >> 1); }

// 1/sqrt(x), 1/x for positive / nonzero normal x: MUFU approximation + Newton
// (within an ulp; every BLWS path uses the same kernel)
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    y = y * fma(-hx * y, y, 1.5);
    y = y * fma(-hx * y, y, 1.5);
    return y;
}
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = y * fma(-x, y, 2.0);
    y = y * fma(-x, y, 2.0);
    return fma(y, fma(-x, y, 1.0), y);
}

__device__ __forceinline__ double warp_sum(double x) {
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// [P3] shared by the prologue and the loop: from the sum of squares `s2` of
// column c below the subdiagonal (already updated) and alpha = A(c+1, c), form
// the reflector; thread i (= row) writes v[i] and the packed reflector.
__device__ __forceinline__ void form_reflector(double* a, int n, int c, double s2, double xi, double* v, double* d,
                                               double* e, double* tau, double* tau_out) {
    const int i = threadIdx.x;
    double* colc = a + floff(c, n);  // colc[r - c] = A(r, c)
    // the scalar chain on every thread, branch-free: MUFU rsqrt / rcp refined by
    // Newton steps (no IEEE div / sqrt slow-path calls, no lane-0 divergence
    // and shuffle broadcast; measured 1361 -> see DESIGN cycles per step)
    const double alpha = colc[1];
    const double nrm2 = fma(alpha, alpha, s2);
    const bool refl = s2 > 0.0;
    const double rn = rsqrt_nr(refl ? nrm2 : 1.0);         // 1 / ||x||
    const double sg = alpha >= 0.0 ? 1.0 : -1.0;           // copysign(1, alpha) for finite alpha
    const double beta = refl ? -sg * nrm2 * rn : alpha;    // -sign(alpha) ||x||
    const double tk = refl ? fma(alpha, sg * rn, 1.0) : 0.0;  // (beta - alpha) / beta = 1 + alpha sign / ||x||
    const double scl = refl ? rcp_nr(alpha - beta) : 0.0;
    if (i < n) {
        double vi = 0.0;
        if (i > c) vi = tk == 0.0 ? 0.0 : (i == c + 1 ? 1.0 : xi * scl);
        v[i] = vi;
        if (i > c) colc[i - c] = vi;  // the reflector below the diagonal of column c
    }
    if (i == 0) {
        d[c] = colc[0];
        e[c] = beta;
        tau[c] = tk;
    }
    *tau_out = tk;
}

// PAIR (orders 209..224, where 16 per-warp row partials do not fit next to the
// triangle): warps w and w + 8 combine their row partials through one extra
// barrier, so the partial buffer holds 8 rows instead of 16.
template <int QN, bool PAIR>
__global__ void __launch_bounds__(kFT) sytrd_fused_k(const double* __restrict__ t, long ld, int n, double* lp,
                                                     double* d, double* e, double* tau) {
    constexpr int NP = 32 * QN;  // padded vector length (<= kFT)
    constexpr int CN = 2 * QN;   // column classes per warp
    constexpr int PWN = PAIR ? kFW / 2 : kFW;
    extern __shared__ __align__(16) double sm[];
    double* vb = sm;             // 2 x NP: v_k by parity
    double* wb = vb + 2 * NP;    // NP: w_k (w_{k-1} is dead once the sweep of step k is done)
    double* pcol = wb + NP;      // NP: column-dot part of p, then p
    double* red = pcol + NP;     // 64
    double* pw = red + 64;       // PWN x NP: row part of p per warp (pair)
    double* a = pw + PWN * NP;   // packed lower triangle
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int row = threadIdx.x;  // [P] phases: one row per thread
#ifdef SYTRD_PROBE
    __shared__ unsigned long long s_phase[8];
    __shared__ unsigned s_sweep[256];
    if (threadIdx.x < 8) s_phase[threadIdx.x] = 0;
    long long tp_ = clock64();
#endif

    for (int j = wid; j < n; j += kFW)
        for (int i = j + lane; i < n; i += 32) a[floff(j, n) + (i - j)] = 0.5 * (t[i + j * ld] + t[j + i * ld]);
    for (int i = threadIdx.x; i < 3 * NP; i += kFT) vb[i] = 0.0;  // vb and wb
    __syncthreads();
    // prologue: reflector of column 0
    double tk;
    {
        const double xi = row < n ? a[row] : 0.0;  // column 0 packed at offset 0
        double s2 = warp_sum(row >= 2 && row < n ? xi * xi : 0.0);
        if (lane == 0) {
            red[wid] = s2;
            red[32 + wid] = 0.0;  // the [P] s2 share of warps without live rows stays 0
        }
        __syncthreads();
        s2 = warp_sum(lane < kFW ? red[lane] : 0.0);
        form_reflector(a, n, 0, s2, xi, vb, d, e, tau, &tk);
        __syncthreads();
    }

    PHASE_MARK(0);
    for (int k = 0; k < n - 2; ++k) {
        const int par = k & 1;
        const double* v = vb + par * NP;         // v_k
        const double* vo = vb + (1 - par) * NP;  // v_{k-1}
        const double* wo = wb;                   // w_{k-1}
        double* wn = wb;                         // w_k (written after the sweep barrier)
        double* vn = vb + (1 - par) * NP;        // v_{k+1} (overwrites v_{k-1} after [S])
        // ---- [S] fused sweep: pending update k-1, then p = A22 v_k
        {
            double vr[QN], vor[QN], wor[QN], acc[QN], dp[CN];
#pragma unroll
            for (int q = 0; q < QN; ++q) {
                const int i = lane + 32 * q;
                vr[q] = v[i];
                vor[q] = vo[i];
                wor[q] = wo[i];
                acc[q] = 0.0;
            }
            double qv = 0.0;  // this lane's share of v^T A v (A = the updated A22)
#pragma unroll
            for (int c = 0; c < CN; ++c) {
                dp[c] = 0.0;
                const int j = wid + 16 * c;
                if (j <= k || j >= n) continue;  // warp-uniform
                const double vj = v[j], voj = vo[j], woj = wo[j];
                double* col = a + floff(j, n) - j;  // col[i] = A(i, j)
                // all loads of the column first (independent; a store of one slot
                // would otherwise order the next slot's load behind it), then the
                // arithmetic, then the stores
                double xs[QN];
#pragma unroll
                for (int q = c / 2; q < QN; ++q) {
                    const int i = lane + 32 * q;
                    const bool ok = (q != c / 2 || i >= j) && (q != QN - 1 || i < n);
                    xs[q] = ok ? col[i] : 0.0;
                }
#pragma unroll
                for (int q = c / 2; q < QN; ++q) {
                    const int i = lane + 32 * q;
                    const bool ok = (q != c / 2 || i >= j) && (q != QN - 1 || i < n);
                    const double x = ok ? fma(-vor[q], woj, fma(-wor[q], voj, xs[q])) : 0.0;
                    xs[q] = x;
                    acc[q] = fma(x, vj, acc[q]);
                    if (i > j) dp[c] = fma(x, vr[q], dp[c]);
                }
#pragma unroll
                for (int q = c / 2; q < QN; ++q) {
                    const int i = lane + 32 * q;
                    const bool ok = (q != c / 2 || i >= j) && (q != QN - 1 || i < n);
                    if (ok) col[i] = xs[q];
                }
                qv = fma(vj, dp[c], qv);  // v^T A v, strictly-lower half through column j
            }
            // column dots: batched transpose-reduce of the CN (<= 16) values
            double r[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) r[c] = c < CN ? dp[c] : 0.0;
#pragma unroll
            for (int stage = 0; stage < 4; ++stage) {
                const int half = 8 >> stage, o = 16 >> stage;
                const bool hi = (lane & o) != 0;
#pragma unroll
                for (int c = 0; c < half; ++c) {
                    const double send = hi ? r[c] : r[c + half];
                    const double keep = hi ? r[c + half] : r[c];
                    r[c] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            r[0] += __shfl_xor_sync(0xffffffffu, r[0], 1);
            const int cc = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
            const int jj = wid + 16 * cc;
            if ((lane & 1) == 0 && cc < CN && jj > k && jj < n) pcol[jj] = r[0];
#pragma unroll
            for (int q = 0; q < QN; ++q) qv = fma(vr[q], acc[q], qv);  // lower half incl. the diagonal
            qv = warp_sum(qv);
            if (lane == 0) red[wid] = qv;  // per-warp share: K needs no separate reduction
            if (!PAIR) {
#pragma unroll
                for (int q = 0; q < QN; ++q) pw[wid * NP + lane + 32 * q] = acc[q];
            } else {
                if (wid >= PWN) {
#pragma unroll
                    for (int q = 0; q < QN; ++q) pw[(wid - PWN) * NP + lane + 32 * q] = acc[q];
                }
                __syncthreads();
                if (wid < PWN) {
#pragma unroll
                    for (int q = 0; q < QN; ++q) pw[wid * NP + lane + 32 * q] += acc[q];
                }
            }
        }
#ifdef SYTRD_PROBE
        if (threadIdx.x == 0 && k < 256) s_sweep[k] = static_cast<unsigned>(clock64() - tp_);
#endif
        PHASE_MARK(1);
        __syncthreads();
        PHASE_MARK(2);
        // ---- [P] K = tau/2 p^T v = tau^2/2 v^T A v (per-warp shares); p_i, w_i;
        //      look-ahead update of column k+1 (w_{k+1} formed by every thread
        //      from broadcast reads) and its squared norm below the subdiagonal
        // warps whose rows are all >= n have no [P] / [P3] work (their s2 share
        // in red[32 + wid] was zeroed in the prologue)
        const bool rows_live = 32 * wid < n;
        const int c1 = k + 1;
        double xi = 0.0;
        if (rows_live) {
        double vav = 0.0;
#pragma unroll
        for (int ww = 0; ww < kFW; ++ww) vav += red[ww];
        const double K = 0.5 * tk * tk * vav;
        double p = 0.0;
        if (row > k && row < n) {
            double sacc = pcol[row];
#pragma unroll
            for (int ww = 0; ww < PWN; ++ww) sacc += pw[ww * NP + row];
            p = tk * sacc;
        }
        const double vi = row < NP ? v[row] : 0.0;
        const double wi = fma(-K, vi, p);
        if (row < NP) wn[row] = wi;
        double pc = pcol[c1];
#pragma unroll
        for (int ww = 0; ww < PWN; ++ww) pc += pw[ww * NP + c1];
        const double vc = v[c1];
        const double wc = fma(-K, vc, tk * pc);  // w_{k+1}, identical in every thread
        if (row >= c1 && row < n) {
            double* col1 = a + floff(c1, n) - c1;
            xi = fma(-vi, wc, fma(-wi, vc, col1[row]));
            col1[row] = xi;
        }
        const double s2 = warp_sum(row >= c1 + 2 && row < n ? xi * xi : 0.0);
        if (lane == 0) red[32 + wid] = s2;  // second half: red[0..] holds the v^T A v shares
        }
        PHASE_MARK(5);
        __syncthreads();
        // ---- [P3] reflector of column k+1 (if any)
        if (k + 1 < n - 2 && rows_live) {
            const double s2 = warp_sum(lane < kFW ? red[32 + lane] : 0.0);
            form_reflector(a, n, c1, s2, xi, vn, d, e, tau, &tk);
        }
        PHASE_MARK(6);
        __syncthreads();
        PHASE_MARK(7);
    }
    // the last update (step n-3) is already applied to column n-2 by the
    // look-ahead; column n-1 (one element) still needs it
    if (threadIdx.x == 0 && n >= 2) {
        const int kl = n - 3;
        double* c2 = a + floff(n - 2, n);  // c2[0] = A(n-2, n-2), c2[1] = A(n-1, n-2)
        double* c1 = a + floff(n - 1, n);  // c1[0] = A(n-1, n-1)
        if (kl >= 0) {
            const double* vl = vb + (kl & 1) * NP;
            const double* wl = wb;
            c1[0] -= fma(vl[n - 1], wl[n - 1], wl[n - 1] * vl[n - 1]);
        }
        d[n - 2] = c2[0];
        e[n - 2] = c2[1];
        tau[n - 2] = 0.0;
        d[n - 1] = c1[0];
        tau[n - 1] = 0.0;
    }
    __syncthreads();
    const long np = static_cast<long>(n) * (n + 1) / 2;
    for (long idx = threadIdx.x; idx < np; idx += kFT) lp[idx] = a[idx];
#ifdef SYTRD_PROBE
    if (threadIdx.x < 8) g_sytrd_phase[threadIdx.x] = s_phase[threadIdx.x];
    for (int i = threadIdx.x; i < 256; i += kFT) g_sytrd_sweep[i] = s_sweep[i];
#endif
}

constexpr size_t kFusedSmemMax = 226 * 1024;  // the 227 KB per-block opt-in limit less 1 KB static

template <int QN, bool PAIR>
size_t fused_smem(int n) {
    constexpr int NP = 32 * QN;
    const long pwn = PAIR ? kFW / 2 : kFW;
    return (4L * NP + 64 + pwn * NP + static_cast<long>(n) * (n + 1) / 2) * 8;
}

template <int QN, bool PAIR>
bool launch_fused_v(Context& ctx, View t, int n, double* lp, double* d, double* e, double* tau) {
    const size_t bytes = fused_smem<QN, PAIR>(n);
    if (bytes > kFusedSmemMax) return false;
    static bool cfg = false;
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(sytrd_fused_k<QN, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kFusedSmemMax)));
        cfg = true;
    }
    sytrd_fused_k<QN, PAIR><<<1, kFT, bytes, ctx.stream()>>>(t.p, t.ld, n, lp, d, e, tau);
    ctx.note_launch();
    ctx.check_launch("sytrd_fused_k");
    return true;
}

template <int QN>
bool launch_fused(Context& ctx, View t, int n, double* lp, double* d, double* e, double* tau) {
    if (fused_smem<QN, false>(n) <= kFusedSmemMax) return launch_fused_v<QN, false>(ctx, t, n, lp, d, e, tau);
    return launch_fused_v<QN, true>(ctx, t, n, lp, d, e, tau);
}

}  // namespace

bool sytrd_fused(Context& ctx, View t, double* lp, double* d, double* e, double* tau) {
    const int n = static_cast<int>(t.rows);
    if (n < 3) return false;
    switch ((n + 31) / 32) {
        case 1: return launch_fused<1>(ctx, t, n, lp, d, e, tau);
        case 2: return launch_fused<2>(ctx, t, n, lp, d, e, tau);
        case 3: return launch_fused<3>(ctx, t, n, lp, d, e, tau);
        case 4: return launch_fused<4>(ctx, t, n, lp, d, e, tau);
        case 5: return launch_fused<5>(ctx, t, n, lp, d, e, tau);
        case 6: return launch_fused<6>(ctx, t, n, lp, d, e, tau);
        case 7: return launch_fused<7>(ctx, t, n, lp, d, e, tau);
        default: return false;
    }
}

}  // namespace blws
