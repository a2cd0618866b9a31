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

// Number of eigenvalues < x: sign changes of the Sturm sequence
// p_i = det(T_i - x I), p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2}
// (division-free: two dependent FMAs per step instead of a division), with
// exact power-of-two rescaling against over/underflow. A zero p_i takes the
// sign opposite to p_{i-1} (dstebz's pivmin convention in the ratio form).
__device__ __forceinline__ int sturm_count(const double* d, const double* e, int n, double x, double pivmin) {
    double p0 = 1.0, p1 = d[0] - x;
    if (p1 == 0.0) p1 = -pivmin;
    int cnt = p1 < 0.0;
    for (int i = 1; i < n; ++i) {
        const double e2 = e[i - 1] * e[i - 1];
        double p2 = fma(d[i] - x, p1, -e2 * p0);
        if (p2 == 0.0) p2 = p1 > 0.0 ? -pivmin * fabs(p1) : pivmin * fabs(p1);
        cnt += (p2 < 0.0) != (p1 < 0.0);
        const double a = fabs(p2);
        if (a > 0x1p+600) {
            p1 *= 0x1p-600;
            p2 *= 0x1p-600;
        } else if (a < 0x1p-600) {
            p1 *= 0x1p+600;
            p2 *= 0x1p+600;
        }
        p0 = p1;
        p1 = p2;
    }
    return cnt;
}

// Bisection interval, pivmin and ||T||_1 (dstebz's Gershgorin set-up), on the
// device so the eigensolver needs no host round trip. params: gl, gu, pivmin,
// onenrm (0 => T == 0).
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
    }
}

// one warp per wanted eigenvalue; j-th largest = ascending index n-1-j
__global__ void bisect_k(const double* __restrict__ d, const double* __restrict__ e, int n, int want,
                         const double* __restrict__ params, double* values) {
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const double gl = params[0], gu = params[1], pivmin = params[2];
    const bool zero = params[3] == 0.0;
    for (int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < want; j += warps) {
        if (zero) {  // T == 0: eigenvalues exactly zero
            if (lane == 0) values[j] = 0.0;
            continue;
        }
        const int k = n - 1 - j;  // want lambda_k (ascending): count(lo) <= k < count(hi)
        double lo = gl, hi = gu;
        for (int it = 0; it < 40; ++it) {
            const double w = hi - lo;
            const double tol = 2.0 * 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi)) + 2.0 * pivmin;
            if (w <= tol) break;
            const double x = lo + w * static_cast<double>(lane + 1) / 33.0;
            const int c = sturm_count(d, e, n, x, pivmin);
            const unsigned above = __ballot_sync(0xffffffffu, c >= k + 1);
            if (above == 0u) {
                lo = __shfl_sync(0xffffffffu, x, 31);
            } else {
                const int l = __ffs(above) - 1;
                const double xh = __shfl_sync(0xffffffffu, x, l);
                const double xl = __shfl_sync(0xffffffffu, x, l > 0 ? l - 1 : 0);
                if (l > 0) lo = xl;
                hi = xh;
            }
        }
        if (lane == 0) {
            const double lam = 0.5 * (lo + hi);
            values[j] = fabs(lam) <= 4.0 * pivmin ? 0.0 : lam;
        }
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
__global__ void inverse_iteration_k(const double* __restrict__ d, const double* __restrict__ e, int n,
                                    const double* __restrict__ values, int want, const double* __restrict__ params,
                                    double* vecs, long ldv, double* scratch) {
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const double onenrm_raw = params[3];
    if (onenrm_raw == 0.0) {
        // T == 0: the unit vectors e_{n-1-j} (as Eigen returns)
        for (int j = gw; j < want; j += warps)
            for (int i = lane; i < n; i += 32) vecs[static_cast<long>(j) * ldv + i] = i == n - 1 - j ? 1.0 : 0.0;
        return;
    }
    const double onenrm = fmax(onenrm_raw, 1e-300);
    const double eps = 2.220446049250313e-16;
    const double eps3 = eps * onenrm;
    const double ortol = kClusterTol * onenrm;
    double* u0 = scratch + static_cast<long>(gw) * 6 * n;
    double* u1 = u0 + n;
    double* u2 = u1 + n;
    double* lm = u2 + n;
    double* piv = lm + n;
    double* y = piv + n;
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
            double* x = vecs + static_cast<long>(j) * ldv;
            if (lane == 0) {
                // LU of T - xj I with partial pivoting
                double a = d[0] - xj, b = n > 1 ? e[0] : 0.0;
                for (int k = 0; k < n - 1; ++k) {
                    const double ck = e[k];
                    const double an = d[k + 1] - xj;
                    const double bn = k + 1 < n - 1 ? e[k + 1] : 0.0;
                    if (fabs(a) >= fabs(ck)) {
                        const double l = a != 0.0 ? ck / a : 0.0;
                        u0[k] = a;
                        u1[k] = b;
                        u2[k] = 0.0;
                        lm[k] = l;
                        piv[k] = 0.0;
                        a = an - l * b;
                        b = bn;
                    } else {
                        const double l = a / ck;
                        u0[k] = ck;
                        u1[k] = an;
                        u2[k] = bn;
                        lm[k] = l;
                        piv[k] = 1.0;
                        a = b - l * an;
                        b = -l * bn;
                    }
                }
                u0[n - 1] = a;
                for (int k = 0; k < n; ++k) {
                    if (fabs(u0[k]) < eps3) u0[k] = u0[k] >= 0.0 ? eps3 : -eps3;
                    y[k] = 1.0 / u0[k];  // reciprocal pivots (y is reused as rhs below)
                }
                for (int k = 0; k < n; ++k) u0[k] = y[k];
                for (long i = 0; i < n; ++i) x[i] = hash_uniform(0x5eedull + static_cast<unsigned long long>(j), i);
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
                __syncwarp();
                if (lane == 0) {
                    for (int i = 0; i < n; ++i) y[i] = x[i] * scl;
                    for (int k = 0; k < n - 1; ++k) {
                        if (piv[k] != 0.0) {
                            const double tmp = y[k];
                            y[k] = y[k + 1];
                            y[k + 1] = tmp;
                        }
                        y[k + 1] -= lm[k] * y[k];
                    }
                    for (int k = n - 1; k >= 0; --k) {
                        double v = y[k];
                        if (k + 1 < n) v -= u1[k] * x[k + 1];
                        if (k + 2 < n) v -= u2[k] * x[k + 2];
                        x[k] = v * u0[k];
                    }
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
        }
    }
}

}  // namespace

void tridiag_eig_top(Context& ctx, Index n_, const double* d, const double* e, Index want_, double* values,
                     View vectors) {
    const int n = static_cast<int>(n_), want = static_cast<int>(want_);
    if (n <= 0 || want <= 0) return;
    // three launches, no host round trip (the bounds stay on the device)
    DBuf<double> params(ctx, 4);
    tridiag_bounds_k<<<1, kBoundsThreads, 0, ctx.stream()>>>(d, e, n, params.get());
    ctx.note_launch();
    ctx.check_launch("tridiag_bounds_k");
    const int threads = 256, wpb = threads / 32;
    const int blocks = (want + wpb - 1) / wpb;
    bisect_k<<<static_cast<unsigned>(blocks), threads, 0, ctx.stream()>>>(d, e, n, want, params.get(), values);
    ctx.note_launch();
    ctx.check_launch("bisect_k");
    DBuf<double> scratch(ctx, static_cast<size_t>(blocks) * wpb * 6 * n);
    inverse_iteration_k<<<static_cast<unsigned>(blocks), threads, 0, ctx.stream()>>>(
        d, e, n, values, want, params.get(), vectors.p, vectors.ld, scratch.get());
    ctx.note_launch();
    ctx.check_launch("inverse_iteration_k");
}

}  // namespace blws
