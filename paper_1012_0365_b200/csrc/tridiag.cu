// Top eigenpairs of the Lanczos tridiagonal T_k (K11) for the Ritz
// checkpoints of the cold reseed path.
//
// The reference calls sym_evd_tridiagonal (small_dense.hpp:46-62) at every
// checkpoint (lanczos.hpp:191-207) and uses only the leading pairs: |lambda_1|
// for the scale, the last eigenvector components for the residual estimates,
// and the leading `avail` vectors for the lift (lanczos.hpp:241-244). So only
// the top `want` pairs are computed here:
//   * eigenvalues: Sturm-count bisection, one warp per eigenvalue, 32-way
//     multisection per step (LAPACK dstebz semantics, pivmin safeguard);
//   * eigenvectors: inverse iteration on LU (partial pivoting) of T - lambda I,
//     with modified Gram-Schmidt against earlier members of the same cluster
//     (LAPACK dstein's cluster rule: gap <= 1e-3 * ||T||_1).
#include <algorithm>
#include <cmath>
#include <vector>

#include "ops.cuh"

namespace blws {
namespace {

// Eigenvalues closer than this (relative to ||T||_1) are inverse-iterated
// together with modified Gram-Schmidt (LAPACK dstein uses 1e-3; outside a
// cluster the loss of orthogonality is <= eps ||T|| / gap <= 2e-11).
constexpr double kClusterTol = 1e-5;

// Bisection interval, pivmin and ||T||_1 (dstebz's Gershgorin set-up), on the
// device so the eigensolver needs no host round trip. params: gl, gu, pivmin,
// onenrm (0 => T == 0), the power-of-two scale 2^-E >= 1 / ||T||_1.
constexpr int kBoundsThreads = 512;
__global__ void __launch_bounds__(kBoundsThreads) tridiag_bounds_k(const double* __restrict__ d,
                                                                    const double* __restrict__ e, int n,
                                                                    double* params) {
    __shared__ double red[4][kBoundsThreads / 32];
    double gl = INFINITY, gu = -INFINITY, emax2 = 0.0, onenrm = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double el = i > 0 ? fabs(e[i - 1]) : 0.0, er = i < n - 1 ? fabs(e[i]) : 0.0;
        gl = fmin(gl, d[i] - el - er);
        gu = fmax(gu, d[i] + el + er);
        onenrm = fmax(onenrm, fabs(d[i]) + el + er);
        if (i < n - 1) emax2 = fmax(emax2, e[i] * e[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
        gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
        onenrm = fmax(onenrm, __shfl_xor_sync(0xffffffffu, onenrm, o));
        emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][wid] = gl;
        red[1][wid] = gu;
        red[2][wid] = onenrm;
        red[3][wid] = emax2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
            gl = fmin(gl, red[0][w]);
            gu = fmax(gu, red[1][w]);
            onenrm = fmax(onenrm, red[2][w]);
            emax2 = fmax(emax2, red[3][w]);
        }
        const double safmin = 2.2250738585072014e-308;
        const double pivmin = safmin * fmax(1.0, emax2);
        const double tnorm = fmax(fabs(gl), fabs(gu));
        params[0] = gl - (2.0 * 2.220446049250313e-16 * tnorm * n + 2.0 * pivmin);
        params[1] = gu + (2.0 * 2.220446049250313e-16 * tnorm * n + 2.0 * pivmin);
        params[2] = pivmin;
        params[3] = onenrm;  // exact zero flags T == 0
        int ex = 0;
        frexp(onenrm, &ex);  // onenrm < 2^ex
        params[4] = onenrm > 0.0 ? ldexp(1.0, -ex) : 1.0;
    }
}

// Number of eigenvalues < x: sign changes of the Sturm sequence
// p_i = det(T_i - x I) = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2}, evaluated
// division-free (a dependent FMA per step instead of a ~130-cycle divide) on T
// scaled by an exact power of two s with ||sT||_1 <= 1, so |p| grows at most
// 3x per step. Inputs (shared memory): ds = s d, e2s = (s e)^2, or -1 where
// (s e)^2 < 2^-200, which splits T (the recurrence restarts; an eigenvalue
// perturbation <= 2^-100 ||T||). A zero p_i becomes -2^-200 p_{i-1} (dstebz's
// -pivmin pivot, in scaled units). Every 4 steps the pair is renormalised by an
// exact power of two; per step max(|p_i|, |p_{i+1}|) >= (e^2 / 4) max(|p_{i-1}|,
// |p_i|) >= 2^-202 of it, so nothing reaches the subnormal range in between.
// Sturm counts at P shifts at once: P independent
// chains interleaved -- one chain is latency-bound -- sharing the loads of
// (ds, e2s).
template <int P>
__device__ __forceinline__ void sturm_count_multi(const double* ds, const double* e2s, int n, const double (&xs)[P],
                                                  int (&cnt)[P]) {
    constexpr double kRepl = 0x1p-200;
    double p0[P], p1[P];
    const double d0 = ds[0];
#pragma unroll
    for (int q = 0; q < P; ++q) {
        p0[q] = 1.0;
        const double t = d0 - xs[q];
        p1[q] = t == 0.0 ? -kRepl : t;
        cnt[q] = p1[q] < 0.0;
    }
#pragma unroll 4
    for (int i = 1; i < n; ++i) {
        const double e2 = e2s[i - 1], di = ds[i];
        const bool split = e2 < 0.0;
        const double me2 = -fmax(e2, 0.0);
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const double p1s = split ? 1.0 : p1[q];
            double p2 = fma(di - xs[q], p1s, me2 * p0[q]);
            p2 = p2 == 0.0 ? -kRepl * p1s : p2;
            // sign change of two nonzero values: the sign bits differ (integer
            // pipe; the FP64 pipe is the bottleneck of this loop)
            cnt[q] += static_cast<unsigned>(__double2hiint(p2) ^ __double2hiint(p1s)) >> 31;
            p0[q] = p1s;
            p1[q] = p2;
        }
        if ((i & 3) == 0) {
#pragma unroll
            for (int q = 0; q < P; ++q) {
                // renormalise (p0, p1) so the larger magnitude is in [1, 2): the
                // larger exponent field of the two, by integer max
                const int e0 = (__double2hiint(p0[q]) >> 20) & 0x7ff, e1 = (__double2hiint(p1[q]) >> 20) & 0x7ff;
                const int ex = max(e0, e1);
                const double sc = __hiloint2double((2046 - ex) << 20, 0);
                p0[q] *= sc;
                p1[q] *= sc;
            }
        }
    }
}

// The same counts with the zero-pivot replacement taken off the dependent
// chain: the chain per step is the split select and one FMA. A step that hits
// an exact zero sets `zero` and the caller redoes the round with
// sturm_count_multi (dstebz's -pivmin rule), so the counts always equal it.
template <int P>
__device__ __forceinline__ void sturm_count_fast(const double* ds, const double* e2s, int n, const double (&xs)[P],
                                                 int (&cnt)[P], bool& zero) {
    double p0[P], p1[P];
    const double d0 = ds[0];
    bool z = false;
#pragma unroll
    for (int q = 0; q < P; ++q) {
        p0[q] = 1.0;
        p1[q] = d0 - xs[q];
        z |= p1[q] == 0.0;
        cnt[q] = p1[q] < 0.0;
    }
#pragma unroll 4
    for (int i = 1; i < n; ++i) {
        const double e2 = e2s[i - 1], di = ds[i];
        const bool split = e2 < 0.0;
        const double me2 = -fmax(e2, 0.0);
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const double p1s = split ? 1.0 : p1[q];
            const double p2 = fma(di - xs[q], p1s, me2 * p0[q]);
            z |= p2 == 0.0;
            cnt[q] += static_cast<unsigned>(__double2hiint(p2) ^ __double2hiint(p1s)) >> 31;
            p0[q] = p1s;
            p1[q] = p2;
        }
        if ((i & 3) == 0) {
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const int e0 = (__double2hiint(p0[q]) >> 20) & 0x7ff, e1 = (__double2hiint(p1[q]) >> 20) & 0x7ff;
                const int ex = max(e0, e1);
                const double sc = __hiloint2double((2046 - ex) << 20, 0);
                p0[q] *= sc;
                p1[q] *= sc;
            }
        }
    }
    zero = z;
}

// One block of kBisThreads per wanted eigenvalue (j-th largest = ascending
// index n-1-j), kBisPts-way multisection per round: every thread evaluates
// kBisP shifts, the first shift whose count exceeds the index is found by a
// block min, and [lo, hi] shrinks by kBisPts + 1 per round (8 rounds from the
// Gershgorin interval to the dstebz tolerance, against 11 for the former
// 32-way one-warp search). The loop is bound by the FP64 pipe of the SMSP
// running it, so the block's 4 warps (one per SMSP) each run one chain: 4
// interleaved chains per thread (512-way, 6 rounds) measured slower (140 vs
// 118 us at C2). LAPACK dstebz semantics, pivmin safeguard.
// (256 / 512 threads, 256- / 512-way: 69 / 94 vs 60 us at order 200, r02f)
constexpr int kBisThreads = 128, kBisP = 1, kBisPts = kBisThreads * kBisP;
template <bool SH>
__global__ void __launch_bounds__(kBisThreads) bisect_k(const double* __restrict__ d, const double* __restrict__ e,
                                                         int n, int want, const double* __restrict__ params,
                                                         double* values, double* gscratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double gl = params[0], gu = params[1], pivmin = params[2], scale = params[4];
    const bool zero = params[3] == 0.0;
    extern __shared__ __align__(16) double tsm[];
    __shared__ int sfirst[2][kBisThreads / 32];
    double* ds = SH ? tsm : gscratch + 2L * n * blockIdx.x;  // n: s d
    double* e2s = ds + n;                                    // n: (s e)^2, -1 marks a split
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        ds[i] = d[i] * scale;
        if (i < n - 1) {
            const double es = e[i] * scale;
            const double e2 = es * es;
            e2s[i] = e2 < 0x1p-200 ? -1.0 : e2;
        }
    }
    __syncthreads();
    for (int j = blockIdx.x; j < want; j += gridDim.x) {
        if (zero) {  // T == 0: eigenvalues exactly zero
            if (threadIdx.x == 0) values[j] = 0.0;
            continue;
        }
        const int k = n - 1 - j;  // want lambda_k (ascending): count(lo) <= k < count(hi)
        double lo = gl, hi = gu;
        for (int it = 0; it < 16; ++it) {
            const double w = hi - lo;
            const double tol = 2.0 * 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi)) + 2.0 * pivmin;
            if (w <= tol) break;  // block-uniform
            double xs[kBisP];
            int c[kBisP];
#pragma unroll
            for (int q = 0; q < kBisP; ++q) {
                const int idx = threadIdx.x * kBisP + q;
                xs[q] = (lo + w * static_cast<double>(idx + 1) / static_cast<double>(kBisPts + 1)) * scale;
            }
            bool hit = false;
            sturm_count_fast<kBisP>(ds, e2s, n, xs, c, hit);
            if (__syncthreads_or(hit)) sturm_count_multi<kBisP>(ds, e2s, n, xs, c);  // an exact zero pivot
            int first = kBisPts;
#pragma unroll
            for (int q = kBisP - 1; q >= 0; --q)
                if (c[q] >= k + 1) first = threadIdx.x * kBisP + q;
            first = __reduce_min_sync(0xffffffffu, first);
            if (lane == 0) sfirst[it & 1][wid] = first;
            __syncthreads();  // the other parity slot is free: one barrier per round
#pragma unroll
            for (int ww = 0; ww < kBisThreads / 32; ++ww) first = min(first, sfirst[it & 1][ww]);
            auto xat = [&](int idx) { return lo + w * static_cast<double>(idx + 1) / static_cast<double>(kBisPts + 1); };
            if (first == kBisPts) {
                lo = xat(kBisPts - 1);
            } else {
                const double xh = xat(first);
                if (first > 0) lo = xat(first - 1);
                hi = xh;
            }
        }
        if (threadIdx.x == 0) {
            const double lam = 0.5 * (lo + hi);
            values[j] = fabs(lam) <= 4.0 * pivmin ? 0.0 : lam;
        }
        __syncthreads();
    }
}

__device__ __forceinline__ double hash_uniform(unsigned long long seed, long i) {
    unsigned long long z = seed + 0x9e3779b97f4a7c15ull * static_cast<unsigned long long>(i + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

// Inverse iteration, one warp per cluster. Clusters are the maximal runs of the
// wanted eigenvalues (descending) with consecutive gaps <= ortol; warp s takes
// the cluster starting at s, if one does (found here, no host round trip).
// One warp per block: the LU of T - lambda I, the right-hand side, the iterate
// and (d, e) live in shared memory (9 n doubles); the serial recurrences carry
// their state in registers (lane 0), loads are independent of the chain.
constexpr int kInvitMaxN = 2048;  // shared-memory path; larger orders use global scratch
constexpr int kCh = 8;            // recurrence steps per load / store chunk

// 1 / x for the LU pivots: MUFU rcp + Newton (within an ulp) in the normal
// range, IEEE division outside it (the rcp approximation flushes subnormals)
__device__ __forceinline__ double rcp_pivot(double x) {
    const double ax = fabs(x);
    if (!(ax >= 1e-290 && ax <= 1e290)) return x != 0.0 ? 1.0 / x : 0.0;
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = y * fma(-x, y, 2.0);
    y = y * fma(-x, y, 2.0);
    return fma(y, fma(-x, y, 1.0), y);
}
template <bool SH>
__global__ void __launch_bounds__(32) inverse_iteration_k(const double* __restrict__ d_g,
                                                           const double* __restrict__ e_g, int n,
                                                           const double* __restrict__ values, int want,
                                                           const double* __restrict__ params, double* vecs, long ldv,
                                                           double* gscratch) {
    extern __shared__ __align__(16) double ism[];
    const int warps = gridDim.x;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x;
    const double onenrm_raw = params[3];
    if (onenrm_raw == 0.0) {
        // T == 0: the unit vectors e_{n-1-j} (as Eigen returns)
        for (int j = gw; j < want; j += warps)
            for (int i = lane; i < n; i += 32) vecs[static_cast<long>(j) * ldv + i] = i == n - 1 - j ? 1.0 : 0.0;
        return;
    }
    double* d = SH ? ism : gscratch + 9L * n * blockIdx.x;
    double* e = d + n;   // e[n-1] = 0
    double* u0 = e + n;  // reciprocal pivots
    double* u1 = u0 + n;
    double* u2 = u1 + n;
    double* lm = u2 + n;
    double* piv = lm + n;
    double* y = piv + n;
    double* x = y + n;
    for (int i = lane; i < n; i += 32) {
        d[i] = d_g[i];
        e[i] = i < n - 1 ? e_g[i] : 0.0;
    }
    __syncwarp();
    const double onenrm = fmax(onenrm_raw, 1e-300);
    const double eps = 2.220446049250313e-16;
    const double eps3 = eps * onenrm;
    const double ortol = kClusterTol * onenrm;
    for (int c0 = gw; c0 < want; c0 += warps) {
        if (c0 > 0 && !(values[c0 - 1] - values[c0] > ortol)) continue;  // not a cluster start
        int c1 = c0 + 1;
        while (c1 < want && !(values[c1 - 1] - values[c1] > ortol)) ++c1;
        double xjm = 0.0;
        for (int j = c0; j < c1; ++j) {
            double xj = values[j];
            if (j > c0) {
                // descending order inside the cluster: keep shifts strictly separated
                const double pertol = 10.0 * fabs(eps * xj);
                if (xjm - xj < pertol) xj = xjm - pertol;
            }
            xjm = xj;
            double* xg = vecs + static_cast<long>(j) * ldv;
            for (int i = lane; i < n; i += 32) x[i] = hash_uniform(0x5eedull + static_cast<unsigned long long>(j), i);
            if (lane == 0) {
                // LU of T - xj I with partial pivoting (dstein's dlagtf), reciprocal pivots.
                // Chunks of kCh steps: the chunk's loads are issued ahead of its
                // dependent chain and its stores after it; the pivot reciprocal is
                // one MUFU rcp + Newton (no IEEE division on the chain).
                double a = d[0] - xj, b = e[0];
                auto lu_step = [&](int k, double ck, double dk1, double bn) {
                    const double an = dk1 - xj;
                    const bool sw = !(fabs(a) >= fabs(ck));
                    const double num = sw ? a : ck, den = sw ? ck : a;  // den is the pivot
                    const double rden = rcp_pivot(den);
                    const double l = den != 0.0 ? num * rden : 0.0;
                    u0[k] = fabs(den) < eps3 ? (den >= 0.0 ? 1.0 / eps3 : -1.0 / eps3) : rden;
                    u1[k] = sw ? an : b;
                    u2[k] = sw ? bn : 0.0;
                    lm[k] = l;
                    piv[k] = sw ? 1.0 : 0.0;
                    const double na = sw ? fma(-l, an, b) : fma(-l, b, an);
                    b = sw ? -l * bn : bn;
                    a = na;
                };
                int k0 = 0;
                for (; k0 + kCh <= n - 1; k0 += kCh) {  // full chunks: loads first, straight-line chain
                    double ek[kCh], dn[kCh], en[kCh];
#pragma unroll
                    for (int u = 0; u < kCh; ++u) {
                        ek[u] = e[k0 + u];
                        dn[u] = d[k0 + u + 1];
                        en[u] = e[k0 + u + 1];
                    }
#pragma unroll
                    for (int u = 0; u < kCh; ++u) lu_step(k0 + u, ek[u], dn[u], en[u]);
                }
                for (; k0 < n - 1; ++k0) lu_step(k0, e[k0], d[k0 + 1], e[k0 + 1]);
                u0[n - 1] = fabs(a) < eps3 ? (a >= 0.0 ? 1.0 / eps3 : -1.0 / eps3) : 1.0 / a;
                u1[n - 1] = 0.0;  // read (times zero) by the back substitution
                u2[n - 1] = 0.0;
            }
            __syncwarp();
            // dstein: iterate until the solution grows past sqrt(0.1 / n), then once more
            const double dtpcrt = sqrt(0.1 / n);
            int extra = 0;
            for (int it = 0; it < 5; ++it) {
                // scale rhs: ||x||_1 -> n * onenrm * max(eps, |u_nn|) as in dstein
                double s1 = 0.0;
                for (int i = lane; i < n; i += 32) s1 += fabs(x[i]);
                for (int o = 16; o > 0; o >>= 1) s1 += __shfl_xor_sync(0xffffffffu, s1, o);
                const double scl = static_cast<double>(n) * onenrm * fmax(eps, fabs(1.0 / u0[n - 1])) / fmax(s1, 1e-300);
                for (int i = lane; i < n; i += 32) y[i] = x[i] * scl;
                __syncwarp();
                if (lane == 0) {
                    // forward: L^{-1} P y, state in registers; chunked like the LU
                    // (y[k+1..] are not written before they are read)
                    double cur = y[0];
                    auto fwd = [&](int k, double nxt, double lv, double pv) {
                        const bool sw = pv != 0.0;
                        const double lo = sw ? nxt : cur, hi = sw ? cur : nxt;
                        cur = fma(-lv, lo, hi);
                        return lo;
                    };
                    int k0 = 0;
                    for (; k0 + kCh <= n - 1; k0 += kCh) {
                        double yn[kCh], lv[kCh], pv[kCh], out[kCh];
#pragma unroll
                        for (int u = 0; u < kCh; ++u) {
                            yn[u] = y[k0 + u + 1];
                            lv[u] = lm[k0 + u];
                            pv[u] = piv[k0 + u];
                        }
#pragma unroll
                        for (int u = 0; u < kCh; ++u) out[u] = fwd(k0 + u, yn[u], lv[u], pv[u]);
#pragma unroll
                        for (int u = 0; u < kCh; ++u) y[k0 + u] = out[u];
                    }
                    for (; k0 < n - 1; ++k0) {
                        const double lo = fwd(k0, y[k0 + 1], lm[k0], piv[k0]);
                        y[k0] = lo;
                    }
                    y[n - 1] = cur;
                    // backward: U^{-1}
                    double x1 = 0.0, x2 = 0.0;  // x[k+1], x[k+2]
                    auto bwd = [&](double a0, double a1, double a2, double yv) {
                        const double v = fma(-a2, x2, fma(-a1, x1, yv)) * a0;
                        x2 = x1;
                        x1 = v;
                        return v;
                    };
                    int k1 = n - 1;
                    for (; k1 - kCh + 1 >= 0; k1 -= kCh) {
                        double a0[kCh], a1[kCh], a2[kCh], yv[kCh], out[kCh];
#pragma unroll
                        for (int u = 0; u < kCh; ++u) {
                            a0[u] = u0[k1 - u];
                            a1[u] = u1[k1 - u];
                            a2[u] = u2[k1 - u];
                            yv[u] = y[k1 - u];
                        }
#pragma unroll
                        for (int u = 0; u < kCh; ++u) out[u] = bwd(a0[u], a1[u], a2[u], yv[u]);
#pragma unroll
                        for (int u = 0; u < kCh; ++u) x[k1 - u] = out[u];
                    }
                    for (; k1 >= 0; --k1) x[k1] = bwd(u0[k1], u1[k1], u2[k1], y[k1]);
                }
                __syncwarp();
                // MGS against earlier members of the cluster that are within ortol
                for (int p = c0; p < j; ++p) {
                    if (fabs(values[p] - values[j]) > ortol) continue;
                    const double* xp = vecs + static_cast<long>(p) * ldv;
                    double dp = 0.0;
                    for (int i = lane; i < n; i += 32) dp += xp[i] * x[i];
                    for (int o = 16; o > 0; o >>= 1) dp += __shfl_xor_sync(0xffffffffu, dp, o);
                    for (int i = lane; i < n; i += 32) x[i] -= dp * xp[i];
                    __syncwarp();
                }
                // normalise (2-norm), largest component positive
                double s2 = 0.0, amax = -1.0;
                int imax = 0;
                for (int i = lane; i < n; i += 32) {
                    s2 += x[i] * x[i];
                    if (fabs(x[i]) > amax) {
                        amax = fabs(x[i]);
                        imax = i;
                    }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
                    const double am2 = __shfl_xor_sync(0xffffffffu, amax, o);
                    const int im2 = __shfl_xor_sync(0xffffffffu, imax, o);
                    if (am2 > amax || (am2 == amax && im2 < imax)) {
                        amax = am2;
                        imax = im2;
                    }
                }
                const double sgn = x[imax] < 0.0 ? -1.0 : 1.0;
                const double inv = sgn / sqrt(s2);
                __syncwarp();
                for (int i = lane; i < n; i += 32) x[i] *= inv;
                __syncwarp();
                if (amax >= dtpcrt && ++extra >= 2) break;
            }
            for (int i = lane; i < n; i += 32) xg[i] = x[i];
            __syncwarp();
        }
    }
}

}  // namespace

void tridiag_eig_top(Context& ctx, Index n_, const double* d, const double* e, Index want_, double* values,
                     View vectors) {
    const int n = static_cast<int>(n_), want = static_cast<int>(want_);
    if (n <= 0 || want <= 0) return;
    // three launches, no host round trip (the bounds stay on the device)
    DBuf<double> params(ctx, 5);
    tridiag_bounds_k<<<1, kBoundsThreads, 0, ctx.stream()>>>(d, e, n, params.get());
    ctx.note_launch();
    ctx.check_launch("tridiag_bounds_k");
    // bisection: one warp per eigenvalue and per block (latency-bound chains,
    // spread over the SMs instead of sharing schedulers)
    static bool cfg = false;
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(bisect_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
        BLWS_CUDA(cudaFuncSetAttribute(inverse_iteration_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       9 * kInvitMaxN * static_cast<int>(sizeof(double))));
        cfg = true;
    }
    const bool small = n <= kInvitMaxN;  // both kernels stage their vectors in shared memory
    DBuf<double> gscratch;
    if (!small) gscratch = DBuf<double>(ctx, static_cast<size_t>(want) * 9 * n);
    if (small)
        bisect_k<true><<<static_cast<unsigned>(want), kBisThreads, 2 * n * sizeof(double), ctx.stream()>>>(
            d, e, n, want, params.get(), values, nullptr);
    else
        bisect_k<false><<<static_cast<unsigned>(want), kBisThreads, 0, ctx.stream()>>>(d, e, n, want, params.get(), values,
                                                                             gscratch.get());
    ctx.note_launch();
    ctx.check_launch("bisect_k");
    // inverse iteration: one warp per candidate cluster start, one warp per block
    if (small)
        inverse_iteration_k<true><<<static_cast<unsigned>(want), 32, 9 * n * sizeof(double), ctx.stream()>>>(
            d, e, n, values, want, params.get(), vectors.p, vectors.ld, nullptr);
    else
        inverse_iteration_k<false><<<static_cast<unsigned>(want), 32, 0, ctx.stream()>>>(
            d, e, n, values, want, params.get(), vectors.p, vectors.ld, gscratch.get());
    ctx.note_launch();
    ctx.check_launch("inverse_iteration_k");
}

}  // namespace blws
