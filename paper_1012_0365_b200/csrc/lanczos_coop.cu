// Cooperative persistent Lanczos steps (lanczos.hpp:112-138 + full CGS2,
// :123-126) for a dense, unsharded operator with m <= 4096: one launch runs a
// whole step range; grid-wide barriers replace the ~17 kernel boundaries of a
// step (each step of a C1/C3-size reseed was launch-bound: ~120 us of ~17 tiny
// kernels for ~30 us of work). Per step l (q_l is already in the basis):
//   [1] paired apply: block b owns a column range of W and all m rows; per
//       chunk of 32 columns each lane accumulates W q_bot over its rows (4..16
//       rows, registers) and per-column partials of W^T q_top, transpose-reduced
//       per warp and summed over the 8 warps -> r_bot complete; W q_bot partials
//       per block -> ptop;                                         grid barrier
//   [2] r_top = sum of the block partials (fixed order); alpha partials;    barrier
//   [3] alpha (every thread, fixed order); r -= alpha q_l + beta q_{l-1};   barrier
//   [4] CGS pass: c_p = q_p . r (a block per 4 basis columns, the warps
//       splitting the rows);                                              barrier
//   [5] r -= Q c (four lanes per row, interleaved basis columns);         barrier
//   [6] second pass: c = Q^T r;                                           barrier
//   [7] r -= Q c and ||r||^2 partials;                                    barrier
//   [8] beta, the breakdown latch of lanczos_finalize_k, q_{l+1} = r / beta
//       written straight into the basis;                                  barrier
// Deterministic: every reduction is a fixed-order sum.
#include <cooperative_groups.h>

#include <algorithm>

#include "ops.cuh"

namespace cg = cooperative_groups;

namespace blws {
namespace {

constexpr int kCoopThreads = 256;
constexpr int kCoopWarps = kCoopThreads / 32;

struct CoopArgs {
    const double* w;
    long ldw, m, n, mp, ld;  // panel: top rows [0, m), bottom [mp, mp + n), ld = mp + n
    double* q;               // basis, ldq x cap (column l+1 receives the next direction)
    long ldq;
    double* r;               // residual, ld
    double* alpha;
    double* lastbeta;
    double* coup;
    double* state;           // [0] first broken step or -1, [1] tau
    double* coef;            // cap
    double* ptop;            // gridDim.x x m
    double* pscal;           // gridDim.x
    long cap, dim, l0, l1;
#ifdef COOP_PROBE
    unsigned long long* probe;  // per-phase ns, block 0's view (tools/probes/coop_probe.cu)
#endif
};

#ifdef COOP_PROBE
unsigned long long* g_coop_probe = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define COOP_MARK(k)                                        \
    if (blockIdx.x == 0 && threadIdx.x == 0) {              \
        const unsigned long long now_ = gtimer();           \
        a.probe[k] += now_ - probe_last;                    \
        probe_last = now_;                                  \
    }
#else
#define COOP_MARK(k)
#endif

__device__ __forceinline__ double warp_sum(double x) {
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// block sum in a fixed order (every thread gets the result)
__device__ __forceinline__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kCoopWarps; ++w) s += red[w];
    return s;
}

// sum of the G block partials, the same fixed order in every block (warp 0 loads
// them lane-strided, shuffle-reduces, broadcasts through shared memory)
__device__ __forceinline__ double grid_partials_sum(const double* part, long G, double* slot) {
    if (threadIdx.x < 32) {
        // all loads in flight first (G <= 32 * 16), then a fixed-order sum
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const long g = threadIdx.x + 32L * u;
            v[u] = g < G ? part[g] : 0.0;
        }
        double s = 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u) s += v[u];
        s = warp_sum(s);
        if (threadIdx.x == 0) *slot = s;
    }
    __syncthreads();
    const double v = *slot;
    __syncthreads();
    return v;
}

template <int R>
__global__ void __launch_bounds__(kCoopThreads) lanczos_coop_k(CoopArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double sp[kCoopWarps][32];
    __shared__ double red[kCoopWarps];
    __shared__ double s_scalar;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long G = gridDim.x, b = blockIdx.x;
    const long gtid = b * kCoopThreads + threadIdx.x, gthreads = G * kCoopThreads;
    const long gwarp = b * kCoopWarps + wid, gwarps = G * kCoopWarps;
    const long cpb = (a.n + G - 1) / G;  // columns of W per block
    int lanes_per_row = 4;  // r -= Q c: lanes per row, a power of two the grid can feed
    while (lanes_per_row < 32 && (gthreads / (2 * lanes_per_row)) >= a.ld) lanes_per_row <<= 1;
    const long j0 = b * cpb, j1 = min(a.n, j0 + cpb);
#ifdef COOP_PROBE
    unsigned long long probe_last = gtimer();
#endif
    for (long l = a.l0; l < a.l1; ++l) {
        const double* ql = a.q + l * a.ldq;
        const double* qtop = ql;
        const double* qbot = ql + a.mp;
        // ---- [1] paired apply over this block's columns
        {
            double acc[R], yr[R];
#pragma unroll
            for (int t = 0; t < R; ++t) {
                const long i = wid * 32 + lane + static_cast<long>(kCoopThreads) * t;
                yr[t] = i < a.m ? qtop[i] : 0.0;
                acc[t] = 0.0;
            }
            for (long jc = j0; jc < j1; jc += 32) {
                double bp[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    bp[c] = 0.0;
                    const long j = jc + c;
                    if (j < j1) {  // uniform
                        const double xj = qbot[j];
                        const double* col = a.w + j * a.ldw;
#pragma unroll
                        for (int t = 0; t < R; ++t) {
                            const long i = wid * 32 + lane + static_cast<long>(kCoopThreads) * t;
                            const double v = i < a.m ? col[i] : 0.0;
                            acc[t] = fma(v, xj, acc[t]);
                            bp[c] = fma(v, yr[t], bp[c]);
                        }
                    }
                }
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
                sp[wid][lane] = bp[0];  // column jc + lane, this warp's rows
                __syncthreads();
                if (wid == 0 && jc + lane < j1) {
                    double s = 0.0;
#pragma unroll
                    for (int w = 0; w < kCoopWarps; ++w) s += sp[w][lane];
                    a.r[a.mp + jc + lane] = s;  // W^T q_top: all rows are in this block
                }
                __syncthreads();
            }
#pragma unroll
            for (int t = 0; t < R; ++t) {
                const long i = wid * 32 + lane + static_cast<long>(kCoopThreads) * t;
                if (i < a.m) a.ptop[b * a.m + i] = acc[t];
            }
        }
        grid.sync();
        COOP_MARK(0)
        // ---- [2] r_top = sum of the block partials (four lanes per row, eight
        //      independent accumulators each, fixed-order quad combine); alpha partials
        double pa = 0.0;
        {
            const int sub = lane & 3;
            const long gw = gtid >> 5, nwarps = gthreads >> 5;
            for (long wb = gw * 8; wb < a.m; wb += nwarps * 8) {  // warp-uniform bounds
                const long i = wb + (lane >> 2);
                double v8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                if (i < a.m) {
                    long g = sub;
                    for (; g + 28 < G; g += 32) {
#pragma unroll
                        for (int u = 0; u < 8; ++u) v8[u] += a.ptop[(g + 4 * u) * a.m + i];
                    }
                    for (; g < G; g += 4) v8[0] += a.ptop[g * a.m + i];
                }
                double v = ((v8[0] + v8[1]) + (v8[2] + v8[3])) + ((v8[4] + v8[5]) + (v8[6] + v8[7]));
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                if (i < a.m && sub == 0) {
                    a.r[i] = v;
                    pa = fma(ql[i], v, pa);
                }
            }
            for (long i = a.m + gtid; i < a.ld; i += gthreads) {
                if (i < a.mp) {
                    a.r[i] = 0.0;  // padding row
                } else {
                    pa = fma(ql[i], a.r[i], pa);
                }
            }
        }
        pa = block_sum(pa, red);
        if (threadIdx.x == 0) a.pscal[b] = pa;
        grid.sync();
        COOP_MARK(1)
        // ---- [3] alpha; three-term recurrence
        const double alpha = grid_partials_sum(a.pscal, G, &s_scalar);
        const double beta_prev = l > 0 ? a.coup[l] : 0.0;
        if (gtid == 0) a.alpha[l] = alpha;
        const double* qp = l > 0 ? a.q + (l - 1) * a.ldq : a.q;
        for (long i = gtid; i < a.ld; i += gthreads) {
            double v = a.r[i] - alpha * ql[i];
            if (l > 0) v -= beta_prev * qp[i];
            a.r[i] = v;
        }
        grid.sync();
        COOP_MARK(2)
        // ---- [4]-[7] full CGS2 against columns 0..l
        const long c = l + 1;
        double pb = 0.0;
        for (int pass = 0; pass < 2; ++pass) {
            // c_p = q_p . r: block b takes p = b, b + G, ... four at a time; the 8 warps
            // split the rows, lanes accumulate independently, warps combine in smem
            for (long p0 = b * 4; p0 < c; p0 += G * 4) {
                double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
                for (long i = wid * 32 + lane; i < a.ld; i += kCoopThreads) {
                    const double ri = a.r[i];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (p0 + u < c) s4[u] = fma(a.q[i + (p0 + u) * a.ldq], ri, s4[u]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) s4[u] = warp_sum(s4[u]);
                __syncthreads();
                if (lane == 0) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) sp[wid][u] = s4[u];
                }
                __syncthreads();
                if (threadIdx.x < 4 && p0 + threadIdx.x < c) {
                    double t = 0.0;
#pragma unroll
                    for (int w = 0; w < kCoopWarps; ++w) t += sp[w][threadIdx.x];
                    a.coef[p0 + threadIdx.x] = t;
                }
            }
            grid.sync();
            COOP_MARK(3 + 2 * pass)
            // r -= Q c: lpr lanes per row (as many as the grid affords, 4..32), each
            // every lpr-th basis column with four independent accumulators; the lane
            // group combines by shuffles in a fixed order
            const int lpr = lanes_per_row;
            const int sub = lane & (lpr - 1);
            const int rows_per_warp = 32 / lpr;
            const long gw = gtid >> 5, nwarps = gthreads >> 5;
            for (long wb = gw * rows_per_warp; wb < a.ld; wb += nwarps * rows_per_warp) {  // warp-uniform
                const long i = wb + lane / lpr;
                double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
                if (i < a.ld) {
                    long p = sub;
                    for (; p + 3 * lpr < c; p += 4 * lpr) {
                        t0 = fma(a.q[i + p * a.ldq], a.coef[p], t0);
                        t1 = fma(a.q[i + (p + lpr) * a.ldq], a.coef[p + lpr], t1);
                        t2 = fma(a.q[i + (p + 2 * lpr) * a.ldq], a.coef[p + 2 * lpr], t2);
                        t3 = fma(a.q[i + (p + 3 * lpr) * a.ldq], a.coef[p + 3 * lpr], t3);
                    }
                    for (; p < c; p += lpr) t0 = fma(a.q[i + p * a.ldq], a.coef[p], t0);
                }
                double t = (t0 + t1) + (t2 + t3);
                for (int o = 1; o < lpr; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                if (i < a.ld && sub == 0) {
                    const double v = a.r[i] - t;
                    a.r[i] = v;
                    if (pass == 1) pb = fma(v, v, pb);
                }
            }
            if (pass == 0) {
                grid.sync();
                COOP_MARK(4)
            }
        }
        pb = block_sum(pb, red);
        const double state0 = a.state[0];  // read before this step's latch update
        if (threadIdx.x == 0) a.pscal[b] = pb;
        grid.sync();
        COOP_MARK(6)
        // ---- [8] beta, breakdown latch, next direction into the basis
        const double rsq = grid_partials_sum(a.pscal, G, &s_scalar);
        const double beta = sqrt(rsq);
        const double tau = l == 0 ? 1e-12 * fabs(alpha) : a.state[1];
        const bool already = state0 >= 0.0;
        const bool now = beta <= tau || (l + 1) >= a.dim;
        const bool broken = already || now;
        if (gtid == 0) {
            if (l == 0) a.state[1] = tau;
            if (!already && now) a.state[0] = static_cast<double>(l);
            a.lastbeta[l] = beta;
            if (!broken && l + 1 < a.cap) a.coup[l + 1] = beta;
        }
        if (l + 1 < a.cap) {
            double* qn = a.q + (l + 1) * a.ldq;
            const double inv = broken ? 0.0 : 1.0 / beta;
            for (long i = gtid; i < a.ld; i += gthreads) qn[i] = broken ? 0.0 : a.r[i] * inv;
        }
        grid.sync();
        COOP_MARK(7)
    }
}

template <int R>
bool launch_coop(Context& ctx, CoopArgs& args) {
    static int occ = -1;
    if (occ < 0) {
        int o = 0;
        BLWS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, lanczos_coop_k<R>, kCoopThreads, 0));
        occ = o;
    }
    if (occ < 1) return false;
    // the whole GPU: blocks past the last column contribute zero partials to the
    // apply, and every block works in the reorthogonalisation phases
    const long G = std::min<long>(static_cast<long>(ctx.sm_count()) * std::min(occ, 2), 512);  // <= 32 x 16 partials
    DBuf<double> ptop(ctx, static_cast<size_t>(G * args.m)), pscal(ctx, static_cast<size_t>(G));
    args.ptop = ptop.get();
    args.pscal = pscal.get();
#ifdef COOP_PROBE
    args.probe = g_coop_probe;
#endif
    void* kargs[] = {&args};
    BLWS_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lanczos_coop_k<R>), dim3(static_cast<unsigned>(G)),
                                          dim3(kCoopThreads), kargs, 0, ctx.stream()));
    ctx.note_launch();
    ctx.check_launch("lanczos_coop_k");
    return true;
}

}  // namespace

bool lanczos_coop_steps(Context& ctx, const double* w, Index ldw, Index m, Index n, Index mp, double* q, Index ldq,
                        double* r,
                        double* alpha, double* lastbeta, double* coup, double* state, double* coef, Index cap,
                        Index dim, Index l0, Index l1) {
    static int coop = -1;
    if (coop < 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrCooperativeLaunch, ctx.device());
        coop = v;
    }
    if (!coop || m > 16 * kCoopThreads || l1 <= l0) return false;
    CoopArgs args{w, ldw, m, n, mp, mp + n, q, ldq, r, alpha, lastbeta, coup, state, coef, nullptr, nullptr,
                  cap, dim, l0, l1};
    const int rows = static_cast<int>((m + kCoopThreads - 1) / kCoopThreads);
    if (rows <= 1) return launch_coop<1>(ctx, args);
    if (rows <= 2) return launch_coop<2>(ctx, args);
    if (rows <= 4) return launch_coop<4>(ctx, args);
    if (rows <= 8) return launch_coop<8>(ctx, args);
    return launch_coop<16>(ctx, args);
}

}  // namespace blws
