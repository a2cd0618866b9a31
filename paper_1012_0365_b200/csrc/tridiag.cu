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
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
    double p0 = 1.0, p1 = d[0] - x;
    if (p1 == 0.0) p1 = -pivmin;
    int cnt = p1 < 0.0;
    for (int i = 1; i < n; ++i) {
        double p2 = fma(d[i] - x, p1, -e2[i - 1] * p0);
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

// one warp per wanted eigenvalue; j-th largest = ascending index n-1-j
__global__ void bisect_k(const double* __restrict__ d, const double* __restrict__ e2, int n, int want, double gl,
                         double gu, double pivmin, double* values) {
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < want; j += warps) {
        const int k = n - 1 - j;  // want lambda_k (ascending): count(lo) <= k < count(hi)
        double lo = gl, hi = gu;
        for (int it = 0; it < 40; ++it) {
            const double w = hi - lo;
            const double tol = 2.0 * 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi)) + 2.0 * pivmin;
            if (w <= tol) break;
            const double x = lo + w * static_cast<double>(lane + 1) / 33.0;
            const int c = sturm_count(d, e2, n, x, pivmin);
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

// Inverse iteration, one warp per cluster (clusters are contiguous runs of the
// wanted eigenvalues in descending order: [cstart[c], cstart[c+1])).
__global__ void inverse_iteration_k(const double* __restrict__ d, const double* __restrict__ e, int n,
                                    const double* __restrict__ values, const int* __restrict__ cstart, int nclusters,
                                    double onenrm, double* vecs, long ldv, double* scratch) {
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const double eps = 2.220446049250313e-16;
    const double eps3 = eps * onenrm;
    const double ortol = kClusterTol * onenrm;
    double* u0 = scratch + static_cast<long>(gw) * 6 * n;
    double* u1 = u0 + n;
    double* u2 = u1 + n;
    double* lm = u2 + n;
    double* piv = lm + n;
    double* y = piv + n;
    for (int c = gw; c < nclusters; c += warps) {
        double xjm = 0.0;
        for (int j = cstart[c]; j < cstart[c + 1]; ++j) {
            double xj = values[j];
            if (j > cstart[c]) {
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
                for (int p = cstart[c]; p < j; ++p) {
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
    // host copy of (d, e) for the bounds (n <= 4096: small)
    std::vector<double> hd(n), he(std::max(n - 1, 1), 0.0);
    ctx.read(d, hd.data(), n);
    if (n > 1) ctx.read(e, he.data(), n - 1);
    double gl = INFINITY, gu = -INFINITY, emax2 = 0.0, onenrm = 0.0;
    for (int i = 0; i < n; ++i) {
        const double el = i > 0 ? std::fabs(he[i - 1]) : 0.0, er = i < n - 1 ? std::fabs(he[i]) : 0.0;
        gl = std::min(gl, hd[i] - el - er);
        gu = std::max(gu, hd[i] + el + er);
        onenrm = std::max(onenrm, std::fabs(hd[i]) + el + er);
        if (i < n - 1) emax2 = std::max(emax2, he[i] * he[i]);
    }
    if (onenrm == 0.0) {
        // T == 0: eigenvalues exactly zero, eigenvectors the unit vectors (as Eigen returns)
        BLWS_CUDA(cudaMemsetAsync(values, 0, sizeof(double) * want, ctx.stream()));
        fill(ctx, vectors.left(want), 0.0);
        std::vector<double> one(1, 1.0);
        for (int j = 0; j < want; ++j) ctx.write(vectors.p + (n - 1 - j) + static_cast<long>(j) * vectors.ld, one.data(), 1);
        return;
    }
    const double safmin = 2.2250738585072014e-308;
    const double pivmin = safmin * std::max(1.0, emax2);
    const double tnorm = std::max(std::fabs(gl), std::fabs(gu));
    gl -= 2.0 * 2.220446049250313e-16 * tnorm * n + 2.0 * pivmin;
    gu += 2.0 * 2.220446049250313e-16 * tnorm * n + 2.0 * pivmin;
    onenrm = std::max(onenrm, 1e-300);

    std::vector<double> he2(std::max(n - 1, 1), 0.0);
    for (int i = 0; i + 1 < n; ++i) he2[i] = he[i] * he[i];
    DBuf<double> e2(ctx, static_cast<size_t>(std::max(n - 1, 1)));
    ctx.write(e2.get(), he2.data(), std::max(n - 1, 1));

    const int threads = 256, wpb = threads / 32;
    bisect_k<<<static_cast<unsigned>((want + wpb - 1) / wpb), threads, 0, ctx.stream()>>>(d, e2.get(), n, want, gl, gu,
                                                                                          pivmin, values);
    ctx.note_launch();
    ctx.check_launch("bisect_k");

    std::vector<double> hv(want);
    ctx.read(values, hv.data(), want);
    std::vector<int> cs;
    cs.push_back(0);
    const double ortol = kClusterTol * onenrm;
    for (int j = 1; j < want; ++j)
        if (hv[j - 1] - hv[j] > ortol) cs.push_back(j);
    cs.push_back(want);
    const int ncl = static_cast<int>(cs.size()) - 1;
    DBuf<int> dcs(ctx, cs.size());
    BLWS_CUDA(cudaMemcpyAsync(dcs.get(), cs.data(), sizeof(int) * cs.size(), cudaMemcpyHostToDevice, ctx.stream()));
    ctx.sync();
    const int blocks = (ncl + wpb - 1) / wpb;
    DBuf<double> scratch(ctx, static_cast<size_t>(blocks) * wpb * 6 * n);
    inverse_iteration_k<<<static_cast<unsigned>(blocks), threads, 0, ctx.stream()>>>(
        d, e, n, values, dcs.get(), ncl, onenrm, vectors.p, vectors.ld, scratch.get());
    ctx.note_launch();
    ctx.check_launch("inverse_iteration_k");
}

}  // namespace blws
