// Row-owned cooperative Lanczos steps (lanczos.hpp:112-138 + full CGS2,
// :123-126) with the basis resident in shared memory. One CTA per SM; CTA b
// owns the panel rows [b*RB, (b+1)*RB) for the whole launch and keeps ITS rows
// of the first CS basis columns in shared memory (row-major tile[i][p]); the
// basis is append-only, so a step adds one column to every tile and the CGS2
// products never re-read those columns from L2. Columns >= CS (a basis larger
// than the GPU's aggregate shared memory) are read from global memory,
// coalesced: each CTA keeps its rows of them in a contiguous copy (rebuilt by
// the prologue, extended as columns are appended), so the CGS2 passes stream
// them sequentially. Per step l (grid barriers marked |):
//   [A] paired apply on 2D tiles of W (tr rows x tc columns): W q_bot partials
//       per (column tile, row), W^T q_top partials per (row tile, column);
//       q_l is r / beta of the previous step (or basis column l0)          |
//   [B] owned rows: r = sum of the tile partials (fixed order); alpha partial |
//   [C] alpha; r' = r - alpha q_l - beta q_{l-1} (owned rows, in shared
//       memory); per-CTA partials of Q^T r' over the owned rows             |
//   [D] coefficient sums over the CTAs (a warp per column)                  |
//   [E] r'' = r' - Q c; partials of Q^T r''                                 |
//   [F] coefficient sums                                                    |
//   [G] r''' = r'' - Q c; ||r'''||^2 partial; r''' to global                |
//   then beta, the breakdown latch of lanczos_finalize_k and q_{l+1} = r'''/beta
//   (owned rows into the tile and the basis) open the next step's [A].
// Deterministic: every reduction is a fixed-order sum.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "ops.cuh"

namespace cg = cooperative_groups;

namespace blws {
namespace {

constexpr int kRT = 384;  // threads per CTA (one CTA per SM)
constexpr int kRW = kRT / 32;
constexpr int kSpillMLP = 16;  // spilled-basis loads in flight per lane in r -= Q c

struct RowArgs {
    const double* w;
    long ldw, m, n, mp, ld;
    double* q;  // basis, ldq x cap
    long ldq;
    double* r;  // residual (global copy, read by the apply), ld
    double* alpha;
    double* lastbeta;
    double* coup;
    double* state;  // [0] first broken step or -1, [1] tau
    double* coef;   // cap
    double* ptop;   // Cb x m
    double* pbot;   // Rb x n
    double* pcol;   // G x cap
    double* pscal;  // G
    long cap, dim, l0, l1;
    long Rb, Cb, tr, tc;  // apply tiles
    long RB, CS;          // owned rows per CTA, resident basis columns
    double* spill;        // G x (cap - CS) x RB: each CTA's rows of the spilled columns, contiguous
    long scap;            // cap - CS (>= 1)
#ifdef COOP_PROBE
    unsigned long long* probe;
#endif
};

#ifdef COOP_PROBE
unsigned long long* g_rows_probe = nullptr;
__device__ __forceinline__ unsigned long long rtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define ROWS_MARK(k)                                        \
    if (blockIdx.x == 0 && threadIdx.x == 0) {              \
        const unsigned long long now_ = rtimer();           \
        a.probe[k] += now_ - probe_last;                    \
        probe_last = now_;                                  \
    }
#else
#define ROWS_MARK(k)
#endif

__device__ __forceinline__ double wsum(double x) {
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// 32 per-lane column partials -> lane c holds the warp's sum for column c
__device__ __forceinline__ double transpose_reduce(double (&bp)[32], int lane) {
#pragma unroll
    for (int stage = 0; stage < 5; ++stage) {
        const int half = 16 >> stage, o = 16 >> stage;
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int c = 0; c < half; ++c) {
            const double send = hi ? bp[c] : bp[c + half];
            const double keep = hi ? bp[c + half] : bp[c];
            bp[c] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return bp[0];
}

// fixed-order sum of G partials (warp 0 loads, broadcast through shared memory)
__device__ __forceinline__ double partials_sum(const double* part, long G, double* slot) {
    if (threadIdx.x < 32) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const long g = threadIdx.x + 32L * u;
            v[u] = g < G ? part[g] : 0.0;
        }
        double s = 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u) s += v[u];
        s = wsum(s);
        if (threadIdx.x == 0) *slot = s;
    }
    __syncthreads();
    const double v = *slot;
    __syncthreads();
    return v;
}

__global__ void __launch_bounds__(kRT, 1) lanczos_rows_k(RowArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    const long G = gridDim.x, b = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long RB = a.RB, CS = a.CS;
    const long o0 = b * RB, nown = max(0L, min(a.ld, o0 + RB) - o0);
    double* tile = sm;                  // RB x CS, row-major
    double* cf = tile + RB * CS;        // cap
    double* rs = cf + a.cap;            // RB: the residual of the owned rows
    double* qc = rs + RB;               // RB: q_l
    double* qp = qc + RB;               // RB: q_{l-1}
    double* acc2 = qp + RB;             // RB: spill sums
    double* sp = acc2 + RB;             // 2 x kRW x 32 (the apply alternates halves)
    double* slot = sp + 2 * kRW * 32;   // 1
    double* spb = a.spill + b * a.scap * RB;  // this CTA's spilled columns: spb[(p - CS) * RB + ii]
    // ---- prologue: owned rows of basis columns [0, l0] into the tile; q_l0, q_l0-1
    {
        const long cols = min(a.l0 + 1, CS);
        for (long e = threadIdx.x; nown > 0 && e < nown * cols; e += kRT) {
            const long i = e % nown, p = e / nown;
            tile[i * CS + p] = a.q[(o0 + i) + p * a.ldq];
        }
        // spilled columns [CS, l0] into this CTA's contiguous copy (rebuilt every
        // launch; rows past the owned range are zero, as is rs there)
        for (long e = threadIdx.x; CS + e / RB <= a.l0; e += kRT) {
            const long i = e % RB, p = CS + e / RB;
            spb[(p - CS) * RB + i] = i < nown ? a.q[(o0 + i) + p * a.ldq] : 0.0;
        }
        for (long i = threadIdx.x; i < RB; i += kRT) rs[i] = 0.0;
        for (long i = threadIdx.x; i < nown; i += kRT) {
            qc[i] = a.q[(o0 + i) + a.l0 * a.ldq];
            qp[i] = a.l0 > 0 ? a.q[(o0 + i) + (a.l0 - 1) * a.ldq] : 0.0;
        }
    }
    const double* qsrc = a.q + a.l0 * a.ldq;  // the direction the apply reads
    double qscale = 1.0;
    bool qzero = false;
    __syncthreads();
#ifdef COOP_PROBE
    unsigned long long probe_last = rtimer();
#endif
    for (long l = a.l0; l < a.l1; ++l) {
        const long c = l + 1;  // basis columns 0..l
        // ---- [A] paired apply over this CTA's tile of W
        if (b < a.Rb * a.Cb) {
            const long rb = b / a.Cb, cb = b % a.Cb;
            const long i0 = rb * a.tr, i1 = min(a.m, i0 + a.tr);
            const long j0 = cb * a.tc, j1 = min(a.n, j0 + a.tc);
            const long i = i0 + threadIdx.x;
            const bool hasrow = i < i1;
            const double* wrow = a.w + min(i, a.m - 1);  // clamped: loads stay unconditional
            const double yi = hasrow && !qzero ? qsrc[i] * qscale : 0.0;
            double acc = 0.0;
            int par = 0;  // the column-partial buffer alternates by chunk: one barrier per chunk
            for (long jc = j0; jc < j1; jc += 32, par ^= 1) {
                const long jl = jc + lane;
                const double xl = jl < j1 && !qzero ? qsrc[a.mp + jl] * qscale : 0.0;
                double bp[32];
#pragma unroll
                for (int cc = 0; cc < 32; ++cc) bp[cc] = wrow[min(jc + cc, j1 - 1) * a.ldw];
#pragma unroll
                for (int cc = 0; cc < 32; ++cc) {
                    acc = fma(bp[cc], __shfl_sync(0xffffffffu, xl, cc), acc);  // x = 0 past j1
                    bp[cc] = jc + cc < j1 ? bp[cc] * yi : 0.0;
                }
                const double colp = transpose_reduce(bp, lane);
                double* spp = sp + par * (kRW * 32);
                spp[wid * 32 + lane] = colp;
                __syncthreads();
                if (wid == 0 && jl < j1) {
                    double s = 0.0;
#pragma unroll
                    for (int w = 0; w < kRW; ++w) s += spp[w * 32 + lane];
                    a.pbot[rb * a.n + jl] = s;
                }
            }
            __syncthreads();  // warp 0's last partial read precedes any reuse of sp
            if (hasrow) a.ptop[cb * a.m + i] = acc;
        }
        grid.sync();
        ROWS_MARK(0)
        // ---- [B] owned rows: r = sum of the tile partials; alpha partial
        for (long ii = wid; ii < nown; ii += kRW) {
            const long i = o0 + ii;
            double s = 0.0;
            if (i < a.m) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const long g = lane + 32L * u;
                    v[u] = g < a.Cb ? a.ptop[g * a.m + i] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) s += v[u];
            } else if (i >= a.mp) {
                for (long g = lane; g < a.Rb; g += 32) s += a.pbot[g * a.n + (i - a.mp)];
            }
            s = wsum(s);
            if (lane == 0) rs[ii] = s;  // padding rows: 0
        }
        __syncthreads();
        if (wid == 0) {
            double pa = 0.0;
            for (long ii = lane; ii < nown; ii += 32) pa = fma(qc[ii], rs[ii], pa);
            pa = wsum(pa);
            if (lane == 0) a.pscal[b] = pa;
        }
        grid.sync();
        ROWS_MARK(1)
        // ---- [C] alpha; three-term recurrence on the owned rows; Q^T r' partials
        const double alpha = partials_sum(a.pscal, G, slot);
        const double beta_prev = l > 0 ? a.coup[l] : 0.0;
        if (b == 0 && threadIdx.x == 0) a.alpha[l] = alpha;
        for (long ii = threadIdx.x; ii < nown; ii += kRT) {
            double v = rs[ii] - alpha * qc[ii];
            if (l > 0) v -= beta_prev * qp[ii];
            rs[ii] = v;
        }
        __syncthreads();
        // Q^T r over the owned rows: resident columns a thread per column, spilled
        // columns a warp per 32 (lanes over the owned rows, transpose-reduced)
        auto qt_partials = [&]() {
            const long cr = min(c, CS);
            for (long p = threadIdx.x; p < cr; p += kRT) {
                double s0 = 0.0, s1 = 0.0;
                long ii = 0;
                for (; ii + 1 < nown; ii += 2) {
                    s0 = fma(tile[ii * CS + p], rs[ii], s0);
                    s1 = fma(tile[(ii + 1) * CS + p], rs[ii + 1], s1);
                }
                if (ii < nown) s0 = fma(tile[ii * CS + p], rs[ii], s0);
                a.pcol[p * G + b] = s0 + s1;
            }
            // spilled columns: a thread per column over the contiguous copy (RB even,
            // 16-byte loads; rows past the owned range are zero in both operands)
            for (long p = CS + threadIdx.x; p < c; p += kRT) {
                const double2* col = reinterpret_cast<const double2*>(spb + (p - CS) * RB);
                double s0 = 0.0, s1 = 0.0;
#pragma unroll 7
                for (long h = 0; h < RB / 2; ++h) {
                    const double2 v = col[h];
                    s0 = fma(v.x, rs[2 * h], s0);
                    s1 = fma(v.y, rs[2 * h + 1], s1);
                }
                a.pcol[p * G + b] = s0 + s1;
            }
        };
        // coefficient p = fixed-order sum over the CTAs of pcol[., p]; a warp per column
        auto col_sums = [&]() {
            const long gw = b * kRW + wid, nw = G * kRW;
            for (long p = gw; p < c; p += nw) {
                const double* col = a.pcol + p * G;
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const long g = lane + 32L * u;
                    v[u] = g < G ? col[g] : 0.0;
                }
                double s = 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u) s += v[u];
                s = wsum(s);
                if (lane == 0) a.coef[p] = s;
            }
        };
        // rs -= Q coef over the owned rows (resident part a warp per row with lanes
        // over the columns; spilled part lanes over rows, warps over columns)
        auto sub_qc = [&]() {
            for (long p = threadIdx.x; p < c; p += kRT) cf[p] = a.coef[p];
            __syncthreads();
            const long cr = min(c, CS);
            for (long ii = wid; ii < nown; ii += kRW) {
                const double* trow = tile + ii * CS;
                double t0 = 0.0, t1 = 0.0;
                long p = lane;
                for (; p + 32 < cr; p += 64) {
                    t0 = fma(trow[p], cf[p], t0);
                    t1 = fma(trow[p + 32], cf[p + 32], t1);
                }
                if (p < cr) t0 = fma(trow[p], cf[p], t0);
                const double t = wsum(t0 + t1);
                if (lane == 0) acc2[ii] = t;
            }
            __syncthreads();
            if (c > CS) {
                // each warp: columns CS + wid, CS + wid + kRW, ...; lanes over rows
                for (long i0 = 0; i0 < nown; i0 += 32) {
                    const long ii = i0 + lane;
                    double t0 = 0.0, t1 = 0.0;
                    {
                        // columns CS + wid + kRW * k; kSpillMLP loads in flight (clamped, zero weight past c)
                        const double* src = spb + (min(ii, nown - 1) - CS * RB);
                        for (long p0 = CS + wid; p0 < c; p0 += kSpillMLP * kRW) {
                            double v[kSpillMLP];
#pragma unroll
                            for (int u = 0; u < kSpillMLP; ++u) v[u] = src[min(p0 + u * kRW, c - 1) * RB];
#pragma unroll
                            for (int u = 0; u < kSpillMLP; ++u) {
                                const long p = p0 + u * kRW;
                                const double cv = p < c ? cf[p] : 0.0;
                                if (u & 1)
                                    t1 = fma(v[u], cv, t1);
                                else
                                    t0 = fma(v[u], cv, t0);
                            }
                        }
                    }
                    sp[wid * 32 + lane] = t0 + t1;
                    __syncthreads();
                    if (wid == 0 && ii < nown) {
                        double s = 0.0;
#pragma unroll
                        for (int w = 0; w < kRW; ++w) s += sp[w * 32 + lane];
                        acc2[ii] += s;
                    }
                    __syncthreads();
                }
            }
            for (long ii = threadIdx.x; ii < nown; ii += kRT) rs[ii] -= acc2[ii];
            __syncthreads();
        };
        qt_partials();
        grid.sync();
        ROWS_MARK(2)
        // ---- [D]
        col_sums();
        grid.sync();
        ROWS_MARK(3)
        // ---- [E]
        sub_qc();
        qt_partials();
        grid.sync();
        ROWS_MARK(4)
        // ---- [F]
        col_sums();
        grid.sync();
        ROWS_MARK(5)
        // ---- [G]
        sub_qc();
        if (wid == 0) {
            double pb = 0.0;
            for (long ii = lane; ii < nown; ii += 32) pb = fma(rs[ii], rs[ii], pb);
            pb = wsum(pb);
            if (lane == 0) a.pscal[b] = pb;
        }
        for (long ii = threadIdx.x; ii < nown; ii += kRT) a.r[o0 + ii] = rs[ii];
        const double state0 = a.state[0];  // read before this step's latch update
        grid.sync();
        ROWS_MARK(6)
        // ---- beta, breakdown latch, q_{l+1} (owned rows) for the next step
        const double rsq = partials_sum(a.pscal, G, slot);
        const double beta = sqrt(rsq);
        const double tau = l == 0 ? 1e-12 * fabs(alpha) : a.state[1];
        const bool already = state0 >= 0.0;
        const bool now = beta <= tau || (l + 1) >= a.dim;
        const bool broken = already || now;
        if (b == 0 && threadIdx.x == 0) {
            if (l == 0) a.state[1] = tau;
            if (!already && now) a.state[0] = static_cast<double>(l);
            a.lastbeta[l] = beta;
            if (!broken && l + 1 < a.cap) a.coup[l + 1] = beta;
        }
        if (l + 1 < a.cap) {
            const double inv = broken ? 0.0 : 1.0 / beta;
            if (l + 1 >= CS)
                for (long ii = nown + threadIdx.x; ii < RB; ii += kRT) spb[(l + 1 - CS) * RB + ii] = 0.0;
            for (long ii = threadIdx.x; ii < nown; ii += kRT) {
                const double v = broken ? 0.0 : rs[ii] * inv;
                a.q[(o0 + ii) + (l + 1) * a.ldq] = v;
                if (l + 1 < CS)
                    tile[ii * CS + (l + 1)] = v;
                else
                    spb[(l + 1 - CS) * RB + ii] = v;
                qp[ii] = qc[ii];
                qc[ii] = v;
            }
            qsrc = a.r;
            qscale = inv;
            qzero = broken;
        }
        __syncthreads();
        ROWS_MARK(7)
    }
}

size_t rows_smem_fixed(long RB, long cap) { return sizeof(double) * (cap + 4 * RB + 2 * kRW * 32 + 8); }

}  // namespace

bool lanczos_rows_steps(Context& ctx, const double* w, Index ldw, Index m, Index n, Index mp, double* q, Index ldq,
                        double* r, double* alpha, double* lastbeta, double* coup, double* state, double* coef,
                        Index cap, Index dim, Index l0, Index l1) {
    static int coop = -1, smem_max = 0;
    if (coop < 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrCooperativeLaunch, ctx.device());
        cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx.device());
        coop = v;
    }
    if (!coop || l1 <= l0) return false;
    const long G = std::min<long>(ctx.sm_count(), 512);
    const long ld = mp + n;
    const long RB = ((ld + G - 1) / G + 1) & ~1L;  // even: 16-byte rows of the spill copy
    const long budget = static_cast<long>(smem_max) - 1024;
    const long fixed = static_cast<long>(rows_smem_fixed(RB, cap));
    if (fixed > budget) return false;
    const long CS = std::min<long>(cap, (budget - fixed) / (8 * RB));
    const size_t smem = rows_smem_fixed(RB, cap) + sizeof(double) * RB * CS;
    static size_t attr = 0;
    if (smem > attr) {
        BLWS_CUDA(cudaFuncSetAttribute(lanczos_rows_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem_max)));
        attr = static_cast<size_t>(smem_max);
    }
    int occ = 0;
    BLWS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lanczos_rows_k, kRT, smem));
    if (occ < 1) return false;
    // apply tiles: at most kRT rows each, as many column tiles as the grid affords
    const long Rb = std::max<long>(1, (m + kRT - 1) / kRT);
    if (Rb > G) return false;
    const long Cb = std::max<long>(1, std::min<long>(G / Rb, n));
    const long tr = (m + Rb - 1) / Rb, tc = (n + Cb - 1) / Cb;
    DBuf<double> ptop(ctx, static_cast<size_t>(Cb * m)), pbot(ctx, static_cast<size_t>(Rb * n)),
        pcol(ctx, static_cast<size_t>(G * cap)), pscal(ctx, static_cast<size_t>(G));
    const long scap = std::max<long>(1, cap - CS);
    DBuf<double> spill(ctx, static_cast<size_t>(G * scap * RB));
    RowArgs args{w, ldw, m, n, mp, ld, q, ldq, r, alpha, lastbeta, coup, state, coef, ptop.get(), pbot.get(),
                 pcol.get(), pscal.get(), cap, dim, l0, l1, Rb, Cb, tr, tc, RB, CS, spill.get(), scap
#ifdef COOP_PROBE
                 , g_rows_probe
#endif
    };
    void* kargs[] = {&args};
    BLWS_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lanczos_rows_k), dim3(static_cast<unsigned>(G)),
                                          dim3(kRT), kargs, smem, ctx.stream()));
    ctx.note_launch();
    ctx.check_launch("lanczos_rows_k");
    return true;
}

}  // namespace blws
