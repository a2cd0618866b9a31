// Two-stage Householder tridiagonalisation of T (K4) for orders up to ~200,
// one CTA, the packed lower triangle in shared memory throughout.
//
// The one-stage sytrd_fused_k needs a symmetric matrix-vector product with
// the whole trailing matrix for every one of its n - 2 reflectors, so its n
// steps are each a block-wide sweep + three barriers (~6k cycles per step at
// order 200). Here:
//   stage 1 (dense -> band, bandwidth kB = 8, LAPACK dsytrd_sy2sb semantics):
//     per 8-column panel, warp 0 factors the panel below the band (Householder
//     QR, in shared memory), all warps form the compact-WY T factor and update
//     the trailing matrix A22 <- Q^T A22 Q = A22 - W V^T - V W^T with
//     X = A22 V T, W = X - V (T^T V^T X) / 2, both products and the rank-16
//     update on DMMA m8n8k4 tiles of the packed triangle;
//   stage 2 (band -> tridiagonal, bulge chasing): sweep c annihilates column c
//     below the subdiagonal with a length-8 reflector, then chases the bulge
//     it creates down the band, one reflector per 8-row block (task (c, t)).
//     A task touches an 8 x 8 diagonal block, the 8 x 8 block below it and the
//     bulge columns to its left. Task (c, t) may run once (c - 1, t + 2) is
//     done (the footprints of (c, t) and (c - 1, t + 3) are disjoint), so the
//     sweeps run as a wavefront over the 16 warps, one warp per sweep, with
//     per-sweep progress counters in shared memory. Each task is one warp's
//     straight-line code: one shared-memory round trip for all its operands.
// Output: d, e (the tridiagonal), the stage-1 panels (V_p, T_p) and the
// stage-2 reflectors for the back-transformation bt2_k.
//
// Measured at order 200 (r02g, BLWS_EVD2_PROF=1): stage 1 1.69M cycles (panel
// QR on warp 0 1.17M, ~6k per reflector; WY update 0.50M), stage 2 1.59M cycles
// (a task is ~2.5k cycles of dependent shared-memory / shuffle / FP64 latency
// and the wavefront's critical path is ~3n tasks), so sym_evd_top takes 2.03 ms
// against 0.74 ms on the one-stage path. Opt-in (BLWS_EVD2=1) and tested.
//
// Z = Q1 Q2 Y (bt2_k): the stage-2 reflectors of one sweep act on disjoint
// rows, so they are applied sweep by sweep (last first), then the stage-1
// panels by compact WY; one CTA per 8 eigenvectors, everything staged on chip.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "ops.cuh"

namespace blws {
namespace {

constexpr int kB = 8;        // band width of stage 1
constexpr int kT = 512;      // 16 warps
constexpr int kWn = kT / 32;
constexpr int kVtxWarps = 4;  // warps forming V^T X

__device__ __forceinline__ int pk(int i, int j, int n) { return j * n - ((j * (j - 1)) >> 1) + (i - j); }  // i >= j
__device__ __forceinline__ double sym_at(const double* a, int i, int j, int n) {
    return i >= j ? a[pk(i, j, n)] : a[pk(j, i, n)];
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

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

// dlarfg from (alpha, s2 = ||x(2:)||^2): beta, tau and the scale of x(2:)
__device__ __forceinline__ void house_scalars(double alpha, double s2, double& beta, double& tau, double& scl) {
    const bool refl = s2 > 0.0;
    const double nrm2 = fma(alpha, alpha, s2);
    const double rn = rsqrt_nr(refl ? nrm2 : 1.0);
    const double sg = alpha >= 0.0 ? 1.0 : -1.0;
    beta = refl ? -sg * nrm2 * rn : alpha;
    tau = refl ? fma(alpha, sg * rn, 1.0) : 0.0;
    scl = refl ? rcp_nr(alpha - beta) : 0.0;
}

// number of stage-2 tasks of sweep c (reflectors of length >= 2)
__host__ __device__ __forceinline__ int sweep_tasks(int n, int c) { return (n - 2 - c + kB - 1) / kB; }

struct S2Layout {
    int n, hp, np;
    // offsets in doubles
    long a, v, y, x, part, g, t, m, vtx, tau, base, prog, total;
};

__host__ __device__ inline S2Layout s2_layout(int n) {
    S2Layout L{};
    L.n = n;
    L.hp = (n + 7) / 8 * 8;
    L.np = n * (n + 1) / 2;
    long o = 0;
    L.a = o;
    o += (L.np + 1) / 2 * 2;
    L.v = o;
    o += L.hp * kB;
    L.y = o;
    o += L.hp * kB;
    L.x = o;
    o += L.hp * kB;
    L.part = o;
    o += kVtxWarps * 64;
    L.g = o;
    o += 64;
    L.t = o;
    o += 64;
    L.m = o;
    o += 64;
    L.vtx = o;
    o += 64;
    L.tau = o;
    o += kB;
    L.base = o;  // ints: n (2 per double slot)
    o += (n + 1) / 2 + 1;
    L.prog = o;  // ints
    o += (n + 1) / 2 + 1;
    L.total = o;
    return L;
}

// ---------------------------------------------------------------- stage 2 task
// One warp: lane = (grp, i), grp = lane >> 3 (0..3), i = lane & 7.
__device__ __forceinline__ void chase_task(double* a, int n, int col, int s, int L, double* rv, double* rt) {
    const int lane = threadIdx.x & 31, grp = lane >> 3, i = lane & 7;
    const bool ri = i < L;
    __syncwarp();
    // every operand first (one shared-memory round trip)
    const double xi = ri ? a[pk(s + i, col, n)] : 0.0;
    // bulge columns col+1 .. s-1 (left apply), this lane: columns col+1+grp, col+5+grp
    const int jb0 = col + 1 + grp, jb1 = col + 5 + grp;
    const bool hb0 = ri && jb0 < s, hb1 = ri && jb1 < s;
    double b0 = hb0 ? a[pk(s + i, jb0, n)] : 0.0;
    double b1 = hb1 ? a[pk(s + i, jb1, n)] : 0.0;
    // diagonal block: D[i][2grp], D[i][2grp+1]
    const int j0 = 2 * grp, j1 = 2 * grp + 1;
    const bool hd0 = ri && j0 < L, hd1 = ri && j1 < L;
    double d0 = hd0 ? sym_at(a, s + i, s + j0, n) : 0.0;
    double d1 = hd1 ? sym_at(a, s + i, s + j1, n) : 0.0;
    // block below: rows s+L+i (< n and < s+L+kB), columns s+j0, s+j1
    const int rb = s + L + i;
    const bool hr = rb < n;
    const bool hk0 = hr && j0 < L, hk1 = hr && j1 < L;
    double k0 = hk0 ? a[pk(rb, s + j0, n)] : 0.0;
    double k1 = hk1 ? a[pk(rb, s + j1, n)] : 0.0;
    // reflector of x = A[s:s+L, col]
    double s2 = (ri && i >= 1) ? xi * xi : 0.0;
    s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
    s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
    s2 += __shfl_xor_sync(0xffffffffu, s2, 4);
    const double alpha = __shfl_sync(0xffffffffu, xi, lane & 24);
    double beta, tau, scl;
    house_scalars(alpha, s2, beta, tau, scl);
    const double vi = i == 0 ? 1.0 : (ri ? xi * scl : 0.0);
    const double vj0 = __shfl_sync(0xffffffffu, vi, j0), vj1 = __shfl_sync(0xffffffffu, vi, j1);
    // (2) left apply to the bulge columns: dots over i within the group
    double p0 = vi * b0, p1 = vi * b1;
    // (3) w = tau D v: partial over this lane's two columns, then over the groups
    double pw = fma(d0, vj0, d1 * vj1);
    // (4) y = K v for the block below: same pattern
    double py = fma(k0, vj0, k1 * vj1);
#pragma unroll
    for (int o = 1; o <= 4; o <<= 1) {
        p0 += __shfl_xor_sync(0xffffffffu, p0, o);
        p1 += __shfl_xor_sync(0xffffffffu, p1, o);
    }
    pw += __shfl_xor_sync(0xffffffffu, pw, 8);
    py += __shfl_xor_sync(0xffffffffu, py, 8);
    pw += __shfl_xor_sync(0xffffffffu, pw, 16);
    py += __shfl_xor_sync(0xffffffffu, py, 16);
    double wi = tau * pw;
    double kk = vi * wi;
    kk += __shfl_xor_sync(0xffffffffu, kk, 1);
    kk += __shfl_xor_sync(0xffffffffu, kk, 2);
    kk += __shfl_xor_sync(0xffffffffu, kk, 4);
    wi = fma(-0.5 * tau * kk, vi, wi);
    const double wj0 = __shfl_sync(0xffffffffu, wi, j0), wj1 = __shfl_sync(0xffffffffu, wi, j1);
    // stores
    if (hb0) a[pk(s + i, jb0, n)] = fma(-tau * p0, vi, b0);
    if (hb1) a[pk(s + i, jb1, n)] = fma(-tau * p1, vi, b1);
    if (hd0 && i >= j0) a[pk(s + i, s + j0, n)] = d0 - fma(vi, wj0, wi * vj0);
    if (hd1 && i >= j1) a[pk(s + i, s + j1, n)] = d1 - fma(vi, wj1, wi * vj1);
    if (hk0) a[pk(rb, s + j0, n)] = fma(-tau * py, vj0, k0);
    if (hk1) a[pk(rb, s + j1, n)] = fma(-tau * py, vj1, k1);
    if (grp == 0) {
        if (ri) a[pk(s + i, col, n)] = i == 0 ? beta : 0.0;
        rv[i] = vi;
        if (i == 0) *rt = tau;
    }
}

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(kT) sytrd2_k(const double* __restrict__ tin, long ld, int n, double* d, double* e,
                                               double* pv, double* pt, double* rv, double* rt, int prof) {
    long long tp0 = clock64(), tqr = 0, tup = 0;
    extern __shared__ __align__(16) double sm[];
    const S2Layout Ly = s2_layout(n);
    double* a = sm + Ly.a;
    double* V = sm + Ly.v;  // hp x 8, column-major (ld hp)
    double* Y = sm + Ly.y;
    double* X = sm + Ly.x;
    double* part = sm + Ly.part;
    double* G = sm + Ly.g;
    double* Tm = sm + Ly.t;
    double* M = sm + Ly.m;
    double* VtX = sm + Ly.vtx;
    double* taus = sm + Ly.tau;
    int* base = reinterpret_cast<int*>(sm + Ly.base);
    volatile int* prog = reinterpret_cast<volatile int*>(sm + Ly.prog);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int hp = Ly.hp;

    for (int j = wid; j < n; j += kWn)
        for (int i = j + lane; i < n; i += 32) a[pk(i, j, n)] = 0.5 * (tin[i + j * ld] + tin[j + i * ld]);
    for (int c = tid; c < n; c += kT) {
        int b = 0;
        for (int q = 0; q < c; ++q) b += sweep_tasks(n, q);
        base[c] = b;
        prog[c] = 0;
    }
    __syncthreads();

    const long long tp1 = clock64();
    // ------------------------------------------------------------ stage 1
    int panel = 0;
    for (int c0 = 0; c0 + kB < n - 1; c0 += kB, ++panel) {
        const int r0 = c0 + kB, h = n - r0, nt = (h + 7) / 8, hpp = nt * 8;
        // (a) panel QR on warp 0, in place (rows r0.., columns c0..c0+7)
        const long long tq0 = clock64();
        if (wid == 0) {
            for (int k = 0; k < kB; ++k) {
                // column k of the panel, rows k..h-1 (panel-relative)
                const int cj = c0 + k;
                double s2 = 0.0;
                for (int r = k + 1 + lane; r < h; r += 32) {
                    const double x = a[pk(r0 + r, cj, n)];
                    s2 = fma(x, x, s2);
                }
                __syncwarp();  // reconverge before the shuffles (else the BRA.DIV slow path)
                for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
                const double alpha = k < h ? a[pk(r0 + k, cj, n)] : 0.0;
                double beta, tau, scl;
                house_scalars(alpha, s2, beta, tau, scl);
                // v (rows k..h-1), stored in V; column k of A <- beta e_k
                for (int r = lane; r < hpp; r += 32) {
                    double v = 0.0;
                    if (r == k && k < h) v = 1.0;
                    else if (r > k && r < h) v = a[pk(r0 + r, cj, n)] * scl;
                    V[r + k * hp] = v;
                }
                __syncwarp();
                for (int r = k + lane; r < h; r += 32) a[pk(r0 + r, cj, n)] = r == k ? beta : 0.0;
                if (lane == 0) taus[k] = tau;
                // apply H = I - tau v v^T to the panel columns k+1..7
                double dj[kB];
#pragma unroll
                for (int j = 0; j < kB; ++j) dj[j] = 0.0;
                for (int r = k + lane; r < h; r += 32) {
                    const double v = V[r + k * hp];
#pragma unroll
                    for (int j = 1; j < kB; ++j)
                        if (j > k) dj[j] = fma(v, a[pk(r0 + r, c0 + j, n)], dj[j]);
                }
                __syncwarp();
#pragma unroll
                for (int j = 1; j < kB; ++j) {
                    if (j <= k) continue;
                    for (int o = 16; o > 0; o >>= 1) dj[j] += __shfl_xor_sync(0xffffffffu, dj[j], o);
                }
                for (int r = k + lane; r < h; r += 32) {
                    const double v = V[r + k * hp];
#pragma unroll
                    for (int j = 1; j < kB; ++j)
                        if (j > k) {
                            double* p = a + pk(r0 + r, c0 + j, n);
                            *p = fma(-tau * dj[j], v, *p);
                        }
                }
                __syncwarp();
            }
        }
        __syncthreads();
        const long long tq1 = clock64();
        tqr += tq1 - tq0;
        // (b) G = V^T V (strict upper), then T (thread j of warp 0 owns row j of T)
        for (int pr = wid; pr < 28; pr += kWn) {
            // simple decode: pairs in row-major order of the strict upper triangle
            int rem = pr, j = 0;
            while (rem >= kB - 1 - j) {
                rem -= kB - 1 - j;
                ++j;
            }
            const int k = j + 1 + rem;
            double sacc = 0.0;
            for (int r = lane; r < h; r += 32) sacc = fma(V[r + j * hp], V[r + k * hp], sacc);
            __syncwarp();
            for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
            if (lane == 0) G[j * kB + k] = sacc;
        }
        __syncthreads();
        if (tid < kB) {
            const int j = tid;
            double trow[kB];
#pragma unroll
            for (int k = 0; k < kB; ++k) trow[k] = 0.0;
#pragma unroll
            for (int k = 0; k < kB; ++k) {
                if (k == j) trow[k] = taus[k];
                if (k > j) {
                    double sacc = 0.0;
#pragma unroll
                    for (int l = 0; l < kB; ++l)
                        if (l >= j && l < k) sacc = fma(trow[l], G[l * kB + k], sacc);
                    trow[k] = -taus[k] * sacc;
                }
            }
#pragma unroll
            for (int k = 0; k < kB; ++k) Tm[j * kB + k] = trow[k];
        }
        __syncthreads();
        // (c) Y = V T (hpp x 8)
        for (int idx = tid; idx < hpp * kB; idx += kT) {
            const int r = idx % hpp, jj = idx / hpp;
            double sacc = 0.0;
#pragma unroll
            for (int l = 0; l < kB; ++l)
                if (l <= jj) sacc = fma(V[r + l * hp], Tm[l * kB + jj], sacc);
            Y[r + jj * hp] = sacc;
        }
        __syncthreads();
        // (d) X = A22 Y on DMMA: warp per 8-row tile
        {
            const int g = lane >> 2, tg = lane & 3;
            for (int I = wid; I < nt; I += kWn) {
                double c0f[2] = {0.0, 0.0}, c1f[2] = {0.0, 0.0};
                const int ri = I * 8 + g;
                for (int K = 0; K < hpp / 4; K += 2) {
                    const int k0 = K * 4 + tg, k1 = k0 + 4;
                    const double a0 = (ri < h && k0 < h) ? sym_at(a, r0 + ri, r0 + k0, n) : 0.0;
                    const double bb0 = Y[k0 + g * hp];
                    dmma(c0f, a0, bb0);
                    if (K + 1 < hpp / 4) {
                        const double a1 = (ri < h && k1 < h) ? sym_at(a, r0 + ri, r0 + k1, n) : 0.0;
                        const double bb1 = Y[k1 + g * hp];
                        dmma(c1f, a1, bb1);
                    }
                }
                X[ri + (2 * tg) * hp] = c0f[0] + c1f[0];
                X[ri + (2 * tg + 1) * hp] = c0f[1] + c1f[1];
            }
        }
        __syncthreads();
        // (e) VtX = V^T X (8 x 8): kVtxWarps warps split K, partials reduced by 64 threads
        if (wid < kVtxWarps) {
            const int g = lane >> 2, tg = lane & 3;
            double cf[2] = {0.0, 0.0};
            for (int K = wid; K < hpp / 4; K += kVtxWarps) {
                const int kr = K * 4 + tg;
                dmma(cf, V[kr + g * hp], X[kr + g * hp]);
            }
            part[wid * 64 + g * 8 + 2 * tg] = cf[0];
            part[wid * 64 + g * 8 + 2 * tg + 1] = cf[1];
        }
        __syncthreads();
        if (tid < 64) {
            double sacc = 0.0;
#pragma unroll
            for (int w = 0; w < kVtxWarps; ++w) sacc += part[w * 64 + tid];
            VtX[tid] = sacc;
        }
        __syncthreads();
        if (tid < 64) {  // M = T^T VtX
            const int i = tid >> 3, j = tid & 7;
            double sacc = 0.0;
#pragma unroll
            for (int k = 0; k < kB; ++k)
                if (k <= i) sacc = fma(Tm[k * kB + i], VtX[k * kB + j], sacc);
            M[i * kB + j] = sacc;
        }
        __syncthreads();
        // (f) W = X - V M / 2 (into Y)
        for (int idx = tid; idx < hpp * kB; idx += kT) {
            const int r = idx % hpp, jj = idx / hpp;
            double sacc = 0.0;
#pragma unroll
            for (int l = 0; l < kB; ++l) sacc = fma(V[r + l * hp], M[l * kB + jj], sacc);
            Y[r + jj * hp] = fma(-0.5, sacc, X[r + jj * hp]);
        }
        __syncthreads();
        // (g) A22 -= W V^T + V W^T on the lower 8 x 8 tiles
        {
            const int g = lane >> 2, tg = lane & 3;
            const int ntile = nt * (nt + 1) / 2;
            for (int tI = wid; tI < ntile; tI += kWn) {
                int I = 0, rem = tI;
                while (rem > I) {
                    rem -= I + 1;
                    ++I;
                }
                const int J = rem;  // J <= I
                const int ri = I * 8 + g;
                const int cj0 = J * 8 + 2 * tg, cj1 = cj0 + 1;
                const bool s0 = ri < h && cj0 < h && ri >= cj0, s1 = ri < h && cj1 < h && ri >= cj1;
                double cf[2];
                cf[0] = s0 ? a[pk(r0 + ri, r0 + cj0, n)] : 0.0;
                cf[1] = s1 ? a[pk(r0 + ri, r0 + cj1, n)] : 0.0;
                const int rj = J * 8 + g;  // B operand row (the n index)
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                    dmma(cf, -Y[ri + (kk * 4 + tg) * hp], V[rj + (kk * 4 + tg) * hp]);
                    dmma(cf, -V[ri + (kk * 4 + tg) * hp], Y[rj + (kk * 4 + tg) * hp]);
                }
                if (s0) a[pk(r0 + ri, r0 + cj0, n)] = cf[0];
                if (s1) a[pk(r0 + ri, r0 + cj1, n)] = cf[1];
            }
        }
        // export the panel for the back-transformation: V (h x 8, ld n), T (8 x 8)
        for (int idx = tid; idx < h * kB; idx += kT) {
            const int r = idx % h, jj = idx / h;
            pv[static_cast<long>(panel) * n * kB + r + jj * n] = V[r + jj * hp];
        }
        if (tid < 64) pt[panel * 64 + tid] = Tm[tid];
        __syncthreads();
        tup += clock64() - tq1;
    }
    const long long tp2 = clock64();

    // ------------------------------------------------------------ stage 2
    long long tsw0 = 0, twait = 0;
    for (int c = wid; c < n - 2; c += kWn) {
        const long long tsa = clock64();
        const int nt_c = sweep_tasks(n, c);
        const int nt_p = c > 0 ? sweep_tasks(n, c - 1) : 0;
        int col = c, s = c + 1;
        for (int t = 0; t < nt_c; ++t) {
            if (c > 0) {
                const int need = min(t + 3, nt_p);
                const long long tw = clock64();
                if (lane == 0)
                    while (prog[c - 1] < need) {
                    }
                twait += clock64() - tw;
                __syncwarp();
                __threadfence_block();
            }
            const int L = min(kB, n - s);
            const int idx = base[c] + t;
            chase_task(a, n, col, s, L, rv + static_cast<long>(idx) * kB, rt + idx);
            __syncwarp();
            __threadfence_block();
            if (lane == 0) prog[c] = t + 1;
            col = s;
            s += L;
        }
        if (c == 0) tsw0 = clock64() - tsa;
    }
    __syncthreads();
    if (prof && tid == 0)
        printf("sytrd2 n=%d: load %lld, stage1 %lld (qr %lld, update %lld), stage2 %lld cycles; sweep0 %lld (%d tasks), "
               "warp0 wait %lld\n", n, tp1 - tp0, tp2 - tp1, tqr, tup, clock64() - tp2, tsw0, sweep_tasks(n, 0), twait);
    for (int i = tid; i < n; i += kT) {
        d[i] = a[pk(i, i, n)];
        e[i] = i + 1 < n ? a[pk(i + 1, i, n)] : 0.0;
    }
}

// ---------------------------------------------------------------- back-transformation
constexpr int kBtCols = 8;
constexpr int kBtT = 256;

__global__ void __launch_bounds__(kBtT) bt2_k(int n, int want, const double* __restrict__ pv,
                                              const double* __restrict__ pt, const double* __restrict__ rv,
                                              const double* __restrict__ rt, int ntask, int npanel, double* z,
                                              long ldz) {
    extern __shared__ __align__(16) double sm[];
    double* zs = sm;                     // kBtCols x n (column j at zs + j * n)
    double* st = zs + kBtCols * n;       // staging: reflectors, then panels
    __shared__ double U[64], TU[64];
    const int tid = threadIdx.x;
    const int col0 = blockIdx.x * kBtCols, nc = min(kBtCols, want - col0);
    for (int idx = tid; idx < kBtCols * n; idx += kBtT) {
        const int j = idx / n, r = idx % n;
        zs[idx] = j < nc ? z[r + static_cast<long>(col0 + j) * ldz] : 0.0;
    }
    double* sv = st;
    double* stau = st + static_cast<long>(ntask) * kB;
    for (long idx = tid; idx < static_cast<long>(ntask) * kB; idx += kBtT) sv[idx] = rv[idx];
    for (int idx = tid; idx < ntask; idx += kBtT) stau[idx] = rt[idx];
    __syncthreads();
    // Q2: sweeps last to first; the tasks of one sweep touch disjoint rows
    {
        int base = ntask;
        for (int c = n - 3; c >= 0; --c) {
            const int ntc = sweep_tasks(n, c);
            base -= ntc;
            const int t = tid / kBtCols, j = tid % kBtCols;
            if (t < ntc) {
                const int s = c + 1 + t * kB, L = min(kB, n - s);
                const double* v = sv + static_cast<long>(base + t) * kB;
                const double tau = stau[base + t];
                double* zc = zs + j * n + s;
                double dot = 0.0;
#pragma unroll
                for (int i = 0; i < kB; ++i)
                    if (i < L) dot = fma(v[i], zc[i], dot);
                dot *= tau;
#pragma unroll
                for (int i = 0; i < kB; ++i)
                    if (i < L) zc[i] = fma(-dot, v[i], zc[i]);
            }
            __syncthreads();
        }
    }
    // Q1: panels last to first, z[r0:, :] -= V T (V^T z[r0:, :])
    for (int p = npanel - 1; p >= 0; --p) {
        const int r0 = (p + 1) * kB, h = n - r0;
        const double* vp = pv + static_cast<long>(p) * n * kB;
        double* vs = st;  // h x 8 staged
        for (int idx = tid; idx < h * kB; idx += kBtT) {
            const int r = idx % h, jj = idx / h;
            vs[idx] = vp[r + jj * n];
        }
        __syncthreads();
        {  // U = V^T z (8 x 8): 4 threads per entry
            const int ent = tid >> 2, q = tid & 3;
            const int jj = ent >> 3, cc = ent & 7;
            double sacc = 0.0;
            for (int r = q; r < h; r += 4) sacc = fma(vs[r + jj * h], zs[cc * n + r0 + r], sacc);
            sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
            sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
            if (q == 0) U[jj * 8 + cc] = sacc;
        }
        __syncthreads();
        if (tid < 64) {
            const int i = tid >> 3, cc = tid & 7;
            double sacc = 0.0;
#pragma unroll
            for (int k = 0; k < kB; ++k)
                if (k >= i) sacc = fma(pt[p * 64 + i * kB + k], U[k * 8 + cc], sacc);
            TU[i * 8 + cc] = sacc;
        }
        __syncthreads();
        for (int idx = tid; idx < h * kBtCols; idx += kBtT) {
            const int r = idx % h, cc = idx / h;
            double sacc = 0.0;
#pragma unroll
            for (int k = 0; k < kB; ++k) sacc = fma(vs[r + k * h], TU[k * 8 + cc], sacc);
            zs[cc * n + r0 + r] -= sacc;
        }
        __syncthreads();
    }
    for (int idx = tid; idx < nc * n; idx += kBtT) {
        const int j = idx / n, r = idx % n;
        z[r + static_cast<long>(col0 + j) * ldz] = zs[idx];
    }
}

int total_tasks(int n) {
    int s = 0;
    for (int c = 0; c + 2 < n; ++c) s += sweep_tasks(n, c);
    return s;
}
int total_panels(int n) {
    int p = 0;
    for (int c0 = 0; c0 + kB < n - 1; c0 += kB) ++p;
    return p;
}

constexpr long kSmemMax = 226 * 1024;

}  // namespace

bool sytrd2_fits(Index n) {
    const char* env = std::getenv("BLWS_EVD2");  // read per call: tests switch it in-process
    const int mode = env ? std::atoi(env) : -1;
    if (mode == 0 || n < 16 || std::getenv("BLWS_SYTRD")) return false;  // BLWS_SYTRD picks a one-stage variant
    const long s1 = s2_layout(static_cast<int>(n)).total * 8;
    const long s2 = (static_cast<long>(kBtCols) * n + static_cast<long>(total_tasks(static_cast<int>(n))) * (kB + 1)) * 8;
    if (s1 > kSmemMax || s2 > kSmemMax) return false;
    return mode == 1;  // opt-in: slower than sytrd_fused_k at every order measured
}

void sym_evd_top_two_stage(Context& ctx, View t, Index want, double* values, View vectors) {
    const int n = static_cast<int>(t.rows);
    const int ntask = total_tasks(n), npanel = total_panels(n);
    DBuf<double> d(ctx, static_cast<size_t>(n)), e(ctx, static_cast<size_t>(n));
    DBuf<double> pv(ctx, static_cast<size_t>(std::max(1, npanel)) * n * kB), pt(ctx, static_cast<size_t>(std::max(1, npanel)) * 64);
    DBuf<double> rv(ctx, static_cast<size_t>(std::max(1, ntask)) * kB), rt(ctx, static_cast<size_t>(std::max(1, ntask)));
    const long s1 = s2_layout(n).total * 8;
    static bool cfg = false;
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(sytrd2_k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemMax)));
        BLWS_CUDA(cudaFuncSetAttribute(bt2_k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemMax)));
        cfg = true;
    }
    sytrd2_k<<<1, kT, s1, ctx.stream()>>>(t.p, t.ld, n, d.get(), e.get(), pv.get(), pt.get(), rv.get(), rt.get(),
                                                std::getenv("BLWS_EVD2_PROF") != nullptr);
    ctx.note_launch();
    ctx.check_launch("sytrd2_k");
    tridiag_eig_top(ctx, n, d.get(), e.get(), want, values, vectors);
    const long s2 = (static_cast<long>(kBtCols) * n + static_cast<long>(ntask) * (kB + 1)) * 8;
    const int w = static_cast<int>(want);
    bt2_k<<<static_cast<unsigned>((w + kBtCols - 1) / kBtCols), kBtT, s2, ctx.stream()>>>(
        n, w, pv.get(), pt.get(), rv.get(), rt.get(), ntask, npanel, vectors.p, vectors.ld);
    ctx.note_launch();
    ctx.check_launch("bt2_k");
}

}  // namespace blws
