// One CholQR pass factor (K3) for b <= 112: R = chol(G) (upper, G = R^T R),
// Rinv = R^{-1}, and optionally R_total = R * R_prev (the R of CholQR2 is
// R2 R1) with the rank count of diag(R_total) > 1e-12 ||X||_F -- one launch,
// one CTA of 512 threads, everything on chip.
//
// The factorisation is chosen on the device from ||G - cI||_F (c = tr(G)/n):
//   * <= 1e-14 c  (a scaled identity, e.g. the Gram of an orthonormal panel):
//     R = sqrt(c) I (the pass skip of chol_inv_upper);
//   * <= 1e-9 c   (the second CholQR pass of a well-conditioned panel):
//     with E = G/c - I and F = strict_upper(E) + diag(E)/2 (so F + F^T = E),
//     R = sqrt(c) (I + F) and Rinv = (I - F) / sqrt(c). Then
//     R^T R = G + c F^T F and R Rinv = I - F^2: both off by ||E||^2 <= 1e-18,
//     below rounding, so Q = X Rinv is orthonormal to working accuracy;
//   * otherwise a blocked right-looking Cholesky (16-wide blocks): warp 0
//     factors each diagonal block in registers and inverts it, the panel
//     R12 = R11^{-T} A12 and the trailing update A22 -= R12^T R12 run on DMMA
//     m8n8k4 fragments over all 16 warps. R^{-1} follows by blocked back
//     substitution, one warp per 8-column strip (no block barriers), also on
//     DMMA.
// R^{-1} is kept in the lower triangle of the same shared array (transposed)
// plus a diagonal vector, so R and R^{-1} fit one n x (n+1) tile.
// Status semantics are chol_inv_upper's: status 0 / j+1 for the first bad
// pivot, diag = min / max diag(R), trace_out = tr(G).
#include <cmath>

#include "ops.cuh"

#ifdef BLWS_CHOLQR_PROF  // phase clocks of the last launch (tools/probes/cholqr_prof.sh builds only)
namespace blws {
__device__ long long g_cholqr_prof[24];
}
#define CQ_MARK(id)                                                 \
    do {                                                            \
        if (threadIdx.x == 0) blws::g_cholqr_prof[id] = clock64();  \
    } while (0)
#else
#define CQ_MARK(id) \
    do {            \
    } while (0)
#endif

namespace blws {
namespace {

constexpr int kQT = 512;       // 16 warps
constexpr int kQW = kQT / 32;
constexpr int kQMax = 112;     // largest padded order on chip
constexpr int kPL = 17;        // panel / scratch leading dimension (odd: conflict-free fragment loads)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// 1/sqrt(x) and 1/x for positive normal x: the MUFU approximation (~2^-22)
// refined by two Newton steps (~2^-88 before rounding). No slow-path call, so
// the warp-0 register arrays are not spilled around it; the result is within
// an ulp, not correctly rounded -- every CholQR path uses these same kernels.
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

__device__ __forceinline__ double qr_block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = lane < kQW ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

struct Tile {
    double* a;   // NP x LD: R in the upper triangle, R^{-1} transposed in the strict lower
    double* xd;  // diag(R^{-1})
    int ld;
    __device__ double r(int i, int j) const { return i <= j ? a[i + j * ld] : 0.0; }
    __device__ double x(int i, int j) const { return i < j ? a[j + i * ld] : (i == j ? xd[i] : 0.0); }
    __device__ void setx(int i, int j, double v) const {
        if (i < j) a[j + i * ld] = v;
        else if (i == j) xd[i] = v;
    }
};

__global__ void __launch_bounds__(kQT) cholqr_factor_k(double* g, long ldg, double* rinv, long ldri, int n, int np,
                                                       const double* r_prev, long ldp, double* r_out, long ldo,
                                                       int* status, double* diag, double* trace_out,
                                                       const double* trace_ref, std::int64_t* rank_out) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[32];
    __shared__ int fail;
    const int ld = np + 1;
    double* A = sm;
    double* P = A + np * ld;       // 16 x np panel, ld kPL
    double* S = P + kPL * np;      // per-warp 16 x 8 scratch, ld kPL
    double* xd = S + kQW * 8 * kPL;
    const Tile T{A, xd, ld};
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g8 = lane >> 2, t4 = lane & 3;
    if (threadIdx.x == 0) fail = 0;
    CQ_MARK(0);

    // ---- load (padding: identity), trace, distance to a scaled identity
    // column j per warp, rows lane + 32 r per lane; each batch issues its 16
    // loads (clamped, always in bounds) before any store, so they overlap
    // instead of paying one global latency each. The off-diagonal part of
    // ||G - cI||_F^2 is summed from the registers on the way.
    double offd = 0.0;
    for (int j0 = wid; j0 < np; j0 += 4 * kQW) {
        double v[4][4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int jc = min(j0 + c * kQW, n - 1);
#pragma unroll
            for (int r = 0; r < 4; ++r) v[c][r] = __ldg(g + min(lane + 32 * r, n - 1) + static_cast<long>(jc) * ldg);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int j = j0 + c * kQW;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = lane + 32 * r;
                if (i < np && j < np) A[i + j * ld] = (i < n && j < n) ? v[c][r] : (i == j ? 1.0 : 0.0);
                if (i < n && j < n && i != j) offd = fma(v[c][r], v[c][r], offd);
            }
        }
    }
    __syncthreads();
    double tr = 0.0;
    for (int i = threadIdx.x; i < n; i += kQT) tr += A[i + i * ld];
    tr = qr_block_sum(tr, red);
    if (trace_out && threadIdx.x == 0) *trace_out = tr;
    const double c = tr / n;
    for (int i = threadIdx.x; i < n; i += kQT) {
        const double v = A[i + i * ld] - c;
        offd = fma(v, v, offd);
    }
    const double off = qr_block_sum(offd, red);
    const bool finite = isfinite(tr) && isfinite(off) && tr > 0.0;
    CQ_MARK(1);
    const int mode = !finite ? 3 : off <= 1e-28 * c * c ? 0 : off <= 1e-18 * c * c ? 1 : 2;

    if (mode == 3) {
        if (threadIdx.x == 0) {
            status[0] = 1;
            diag[0] = diag[1] = 0.0;
        }
        return;
    }
    if (mode <= 1 && !(r_prev && r_out)) {
        // R = sqrt(c) (I + F), Rinv = (I - F) / sqrt(c); F = 0 for the skip.
        // Elementwise in G, so every output goes straight from the staged G to
        // global memory (the same arithmetic as the on-chip branch below, so
        // both give identical bits); only R_total = R R_prev needs the tile.
        const double rc = sqrt(c), ric = 1.0 / rc, ic = 1.0 / c;
        const double tau = rank_out ? 1e-12 * sqrt(trace_ref ? trace_ref[0] : tr) : 0.0;
        double mn = INFINITY, mx = 0.0, cnt = 0.0;
        for (int j = wid; j < n; j += kQW) {
            double rv[4], xv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = lane + 32 * r;
                double f = 0.0;
                if (mode == 1 && i <= j) f = i == j ? 0.5 * fma(A[i + j * ld], ic, -1.0) : A[i + j * ld] * ic;
                rv[r] = i == j ? rc * (1.0 + f) : (i < j ? rc * f : 0.0);
                xv[r] = i == j ? ric * (1.0 - f) : (i < j ? -ric * f : 0.0);
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = lane + 32 * r;
                if (i < n) {
                    if (rinv) rinv[i + j * ldri] = xv[r];
                    g[i + j * ldg] = rv[r];
                }
                if (i == j) {
                    mn = fmin(mn, rv[r]);
                    mx = fmax(mx, rv[r]);
                    if (rank_out) {
                        double d = rv[r];
                        if (r_prev) d *= r_prev[j + static_cast<long>(j) * ldp];
                        cnt += d > tau ? 1.0 : 0.0;
                    }
                }
            }
        }
        if (rank_out) {
            cnt = qr_block_sum(cnt, red);
            if (threadIdx.x == 0) rank_out[0] = static_cast<std::int64_t>(cnt + 0.5);
        }
        for (int o = 16; o > 0; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        __syncthreads();  // red[] is free again
        if (lane == 0) {
            red[wid] = mn;
            red[kQW + wid] = mx;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w2 = 1; w2 < kQW; ++w2) {
                mn = fmin(mn, red[w2]);
                mx = fmax(mx, red[kQW + w2]);
            }
            status[0] = 0;
            diag[0] = mn;
            diag[1] = mx;
        }
        CQ_MARK(19);
        return;
    }
    if (mode <= 1) {
        // the same R and Rinv on chip, for the R_total product below
        const double rc = sqrt(c), ric = 1.0 / rc, ic = 1.0 / c;
        __syncthreads();
        for (int j = wid; j < np; j += kQW)
            for (int i = lane; i <= j; i += 32) {
                double f = 0.0;
                if (mode == 1 && j < n) f = i == j ? 0.5 * fma(A[i + j * ld], ic, -1.0) : A[i + j * ld] * ic;
                if (j >= n) {  // padding stays the identity
                    A[i + j * ld] = i == j ? 1.0 : 0.0;
                    T.setx(i, j, i == j ? 1.0 : 0.0);
                } else if (i == j) {
                    A[i + j * ld] = rc * (1.0 + f);
                    xd[i] = ric * (1.0 - f);
                } else {
                    A[i + j * ld] = rc * f;
                    T.setx(i, j, -ric * f);
                }
            }
        __syncthreads();
    } else {
        // ---- blocked right-looking Cholesky, 16-wide diagonal blocks
        const int nb = np / 16;
        __syncthreads();
        for (int kb = 0; kb < nb; ++kb) {
            const int o = 16 * kb;
            if (kb < 7) CQ_MARK(2 + 2 * kb);
            if (wid == 0) {
                // diagonal block on warp 0, in registers: lane j < 16 holds column j.
                // __syncwarp reconverges the warp so every shuffle below takes the
                // converged fast path (measured: 133k -> see DESIGN cycles per block)
                __syncwarp();
                const bool act = lane < 16;
                double cc[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) cc[i] = (act && i <= lane) ? A[(o + i) + (o + lane) * ld] : 0.0;
                int bad = 0;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const double piv = __shfl_sync(0xffffffffu, cc[k], k);
                    const bool bk = !(piv > 0.0) || !isfinite(piv);
                    if (bk && bad == 0) bad = o + k + 1;
                    const double inv = bk ? 1.0 : rsqrt_nr(piv);
                    cc[k] = lane == k ? piv * inv : cc[k] * inv;  // r_kj in lane j >= k
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        if (i <= k) continue;  // compile-time after unrolling
                        const double rki = __shfl_sync(0xffffffffu, cc[k], i);
                        cc[i] = (act && lane >= i) ? fma(-rki, cc[k], cc[i]) : cc[i];
                    }
                }
                // inverse of the block: lane j solves R11 x = e_j by back substitution
                double xx[16];
#pragma unroll
                for (int ii = 0; ii < 16; ++ii) {
                    const int i = 15 - ii;
                    const double irii = rcp_nr(__shfl_sync(0xffffffffu, cc[i], i));
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        if (k <= i) continue;
                        const double rik = __shfl_sync(0xffffffffu, cc[i], k);
                        if ((k & 1) == 0) s0 = fma(rik, xx[k], s0);
                        else s1 = fma(rik, xx[k], s1);
                    }
                    xx[i] = lane == i ? irii : (lane > i ? -(s0 + s1) * irii : 0.0);
                }
                if (act) {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (i <= lane) {
                            A[(o + i) + (o + lane) * ld] = cc[i];
                            T.setx(o + i, o + lane, xx[i]);
                        }
                }
                if (lane == 0 && bad) fail = bad;
            }
            __syncthreads();
            if (kb < 7) CQ_MARK(3 + 2 * kb);
            if (fail) break;
            const int w = np - o - 16;  // trailing width
            if (w <= 0) break;
            // panel R12 = R11^{-T} A12 -> P (16 x w): fragments (2 row halves) x (w / 8)
            for (int f = wid; f < 2 * (w / 8); f += kQW) {
                const int rh = f & 1, cf = f >> 1;
                double acc[2] = {0.0, 0.0};
#pragma unroll
                for (int k0 = 0; k0 < 16; k0 += 4) {
                    // A operand: R11^{-T}[8 rh + g][k] = Rinv11[k][8 rh + g]
                    const double av = T.x(o + k0 + t4, o + 8 * rh + g8);
                    const double bv = A[(o + k0 + t4) + (o + 16 + 8 * cf + g8) * ld];
                    dmma(acc, av, bv);
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) P[(8 * rh + g8) + (8 * cf + 2 * t4 + e) * kPL] = acc[e];
            }
            __syncthreads();
            // R12 into A; trailing update A22 -= P^T P on the upper 8x8 fragments
            for (int idx = threadIdx.x; idx < 16 * w; idx += kQT) {
                const int r = idx & 15, cl = idx >> 4;
                A[(o + r) + (o + 16 + cl) * ld] = P[r + cl * kPL];
            }
            const int wf = w / 8;
            for (int f = wid; f < wf * wf; f += kQW) {
                const int fi = f / wf, fj = f % wf;
                if (fi > fj) continue;
                double acc[2] = {0.0, 0.0};
#pragma unroll
                for (int k0 = 0; k0 < 16; k0 += 4)
                    dmma(acc, P[(k0 + t4) + (8 * fi + g8) * kPL], P[(k0 + t4) + (8 * fj + g8) * kPL]);
                const int i = o + 16 + 8 * fi + g8;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = o + 16 + 8 * fj + 2 * t4 + e;
                    A[i + j * ld] -= acc[e];
                }
            }
            __syncthreads();
        }
        if (fail) {
            if (threadIdx.x == 0) {
                status[0] = fail;
                diag[0] = diag[1] = 0.0;
            }
            return;
        }
        CQ_MARK(16);
        // ---- R^{-1}: strip (J, h) = columns 16 J + 8 h .. +8, rows block I = J-1 .. 0:
        //      X_IJ = -Rinv_II (sum_{K=I+1..J} R_IK X_KJ)
        for (int strip = wid; strip < 2 * nb; strip += kQW) {
            const int J = strip >> 1, h = strip & 1;
            const int c0 = 16 * J + 8 * h;
            double* Sw = S + wid * 8 * kPL;
            for (int I = J - 1; I >= 0; --I) {
                double s0[2] = {0.0, 0.0}, s1[2] = {0.0, 0.0};
                for (int k0 = 16 * (I + 1); k0 < 16 * J + 8 * h + 8; k0 += 4) {
                    const double bv = T.x(k0 + t4, c0 + g8);
                    dmma(s0, T.r(16 * I + g8, k0 + t4), bv);
                    dmma(s1, T.r(16 * I + 8 + g8, k0 + t4), bv);
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    Sw[g8 + (2 * t4 + e) * kPL] = s0[e];
                    Sw[8 + g8 + (2 * t4 + e) * kPL] = s1[e];
                }
                __syncwarp();
                double x0[2] = {0.0, 0.0}, x1[2] = {0.0, 0.0};
#pragma unroll
                for (int k0 = 0; k0 < 16; k0 += 4) {
                    const double bv = Sw[(k0 + t4) + g8 * kPL];
                    dmma(x0, T.x(16 * I + g8, 16 * I + k0 + t4), bv);
                    dmma(x1, T.x(16 * I + 8 + g8, 16 * I + k0 + t4), bv);
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    T.setx(16 * I + g8, c0 + 2 * t4 + e, -x0[e]);
                    T.setx(16 * I + 8 + g8, c0 + 2 * t4 + e, -x1[e]);
                }
                __syncwarp();
            }
        }
        __syncthreads();
    }

    CQ_MARK(17);
    // ---- outputs: R (upper, in place of G), Rinv, diag range, R_total, rank
    double mn = INFINITY, mx = 0.0;
    for (int j = wid; j < n; j += kQW)
        for (int i = lane; i < n; i += 32) {
            const double v = T.r(i, j);
            if (rinv) rinv[i + j * ldri] = T.x(i, j);
            if (i == j) {
                mn = fmin(mn, v);
                mx = fmax(mx, v);
            }
        }
    if (r_prev && (r_out || rank_out)) {
        // R_prev's upper triangle replaces R^{-1} (already written out) in the
        // lower-triangle storage: T.x(k, j) now reads R_prev(k, j)
        __syncthreads();
        for (int j0 = wid; j0 < np; j0 += 4 * kQW) {
            double v[4][4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int jc = min(j0 + c * kQW, n - 1);
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    v[c][r] = __ldg(r_prev + min(lane + 32 * r, n - 1) + static_cast<long>(jc) * ldp);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int j = j0 + c * kQW;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int i = lane + 32 * r;
                    if (i <= j && j < np) T.setx(i, j, (j < n) ? v[c][r] : (i == j ? 1.0 : 0.0));
                }
            }
        }
        __syncthreads();
    }
    if (r_prev && r_out) {
        // R_total = R * R_prev on the upper 8x8 fragments
        const int nf = np / 8;
        for (int f = wid; f < nf * nf; f += kQW) {
            const int fi = f / nf, fj = f % nf;
            if (fi > fj) continue;
            double acc[2] = {0.0, 0.0};
            const int col = 8 * fj + g8;
            for (int k0 = 8 * fi; k0 < 8 * fj + 8; k0 += 4) {
                const int k = k0 + t4;
                dmma(acc, T.r(8 * fi + g8, k), T.x(k, col));
            }
            const int i = 8 * fi + g8;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int j = 8 * fj + 2 * t4 + e;
                if (i <= j && j < n) r_out[i + static_cast<long>(j) * ldo] = acc[e];
            }
            if (fi < fj) {  // the strictly lower mirror fragment is zero
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = 8 * fj + 2 * t4 + e;
                    if (i < n && j < n) r_out[j + static_cast<long>(i) * ldo] = 0.0;
                }
            }
        }
        // zero the strictly lower part of the diagonal fragments
        for (int idx = threadIdx.x; idx < n * 8; idx += kQT) {
            const int j = idx / 8, i = 8 * (j / 8) + (idx & 7);
            if (i > j && i < n) r_out[i + static_cast<long>(j) * ldo] = 0.0;
        }
    }
    if (rank_out) {
        const double tau = 1e-12 * sqrt(trace_ref ? trace_ref[0] : tr);
        double cnt = 0.0;
        for (int j = threadIdx.x; j < n; j += kQT) {
            double d = T.r(j, j);
            if (r_prev) d *= T.x(j, j);
            cnt += d > tau ? 1.0 : 0.0;
        }
        cnt = qr_block_sum(cnt, red);
        if (threadIdx.x == 0) rank_out[0] = static_cast<std::int64_t>(cnt + 0.5);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    __shared__ double smn[kQW], smx[kQW];
    if (lane == 0) {
        smn[wid] = mn;
        smx[wid] = mx;
    }
    CQ_MARK(18);
    __syncthreads();  // every read of A above is done before R overwrites G below
    for (int j = wid; j < n; j += kQW)
        for (int i = lane; i < n; i += 32) g[i + j * ldg] = T.r(i, j);
    if (threadIdx.x == 0) {
        for (int w2 = 1; w2 < kQW; ++w2) {
            mn = fmin(mn, smn[w2]);
            mx = fmax(mx, smx[w2]);
        }
        status[0] = 0;
        diag[0] = mn;
        diag[1] = mx;
    }
    CQ_MARK(19);
}

}  // namespace

bool cholqr_factor_fits(Index n) { return n >= 1 && n <= kQMax; }

void cholqr_factor(Context& ctx, View g, View rinv, const double* r_prev, Index ldp, View* r_out, int* status,
                   double* diag, double* trace_out, const double* trace_ref, std::int64_t* rank_out) {
    const int n = static_cast<int>(g.rows);
    const int np = static_cast<int>(round_up(n, 16));
    const int ld = np + 1;
    const size_t bytes = sizeof(double) * (static_cast<size_t>(np) * ld + kPL * np + kQW * 8 * kPL + np);
    static bool cfg = false;
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(cholqr_factor_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sizeof(double) * (kQMax * (kQMax + 1) + kPL * kQMax +
                                                                          kQW * 8 * kPL + kQMax))));
        cfg = true;
    }
    cholqr_factor_k<<<1, kQT, bytes, ctx.stream()>>>(g.p, g.ld, rinv.p, rinv.ld, n, np, r_prev, ldp,
                                                     r_out ? r_out->p : nullptr, r_out ? r_out->ld : 1, status,
                                                     diag, trace_out, trace_ref, rank_out);
    ctx.note_launch();
    ctx.check_launch("cholqr_factor_k");
}

#ifdef BLWS_CHOLQR_PROF
extern "C" void blws_debug_cholqr_prof(long long* out) {
    cudaMemcpyFromSymbol(out, g_cholqr_prof, 24 * sizeof(long long));
}
#endif
}  // namespace blws
