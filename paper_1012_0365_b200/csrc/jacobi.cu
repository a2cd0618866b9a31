// Symmetric EVD of the projected block-tridiagonal T (K4), two-sided cyclic
// Jacobi with the parallel round-robin ordering.
//
// The reference diagonalises T = BlockTridiagonal::embed() with Eigen's
// SelfAdjointEigenSolver (block_lanczos.hpp:144 -> small_dense.hpp:24-43);
// its test oracle is a cyclic Jacobi sweep (tests/oracles.hpp:28-78). T is
// symmetric indefinite with near +-sigma pairs, so a two-sided Jacobi (no
// shift needed) is used, as SURVEY.md finding 3 recommends.
//
// Stage 1 (one CTA): T's upper triangle lives packed in shared memory; each
// round applies n/2 disjoint rotations as 2x2 block updates J_P^T A J_Q and
// appends (c, s) to a rotation log in global memory. Stage 2 (many CTAs):
// every row of V = J_1 J_2 ... is independent, so warps replay the log on
// their own row in parallel. Stage 3 sorts descending.
#include <algorithm>
#include <cmath>

#include "ops.cuh"

namespace blws {
namespace {

constexpr int kMaxSweeps = 40;
constexpr int kJacobiThreads = 1024;
constexpr long kSmemBudget = 220 * 1024;  // dynamic shared bytes for stage 1

__device__ __forceinline__ long pidx(long i, long j) {
    // packed upper triangle, column-major: (i <= j)
    return i <= j ? j * (j + 1) / 2 + i : i * (i + 1) / 2 + j;
}

/// Player at position x of round r in the circle method over N (even) slots.
__device__ __forceinline__ int player(int x, int r, int N) { return x == 0 ? 0 : 1 + (x - 1 + r) % (N - 1); }

__global__ void __launch_bounds__(kJacobiThreads) jacobi_k(const double* __restrict__ t, long ld, int n,
                                                           int on_chip, double* gpacked, double2* log,
                                                           int* rounds_out, double* diag_out) {
    extern __shared__ __align__(16) double sm[];
    const long np = static_cast<long>(n) * (n + 1) / 2;
    const int N = n + (n & 1);
    const int half = N / 2;
    double* rc = sm;
    double* rs = rc + half;
    double* rt = rs + half;
    int* rp = reinterpret_cast<int*>(rt + half);
    int* rq = rp + half;
    double* a = on_chip ? reinterpret_cast<double*>(rq + half) : gpacked;  // 32*half bytes: 8-aligned
    __shared__ double red[32];
    __shared__ int flag;

    for (long idx = threadIdx.x; idx < np; idx += blockDim.x) {
        long j = static_cast<long>((sqrt(8.0 * static_cast<double>(idx) + 1.0) - 1.0) * 0.5);
        while (j * (j + 1) / 2 > idx) --j;
        while ((j + 1) * (j + 2) / 2 <= idx) ++j;
        const long i = idx - j * (j + 1) / 2;
        a[idx] = t[i + j * ld];
    }
    __syncthreads();
    // ||A||_F (invariant under the rotations)
    double fs = 0.0;
    for (long idx = threadIdx.x; idx < static_cast<long>(n) * n; idx += blockDim.x) {
        const long i = idx % n, j = idx / n;
        const double v = t[i + j * ld];
        fs += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) fs += __shfl_xor_sync(0xffffffffu, fs, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = fs;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];
        red[0] = sqrt(s);
    }
    __syncthreads();
    const double fro = red[0];
    const double abs_floor = 1e-17 * fro;

    int rounds = 0;
    for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
        // convergence: any non-negligible off-diagonal entry left?
        if (threadIdx.x == 0) flag = 0;
        __syncthreads();
        for (long idx = threadIdx.x; idx < np; idx += blockDim.x) {
            long j = static_cast<long>((sqrt(8.0 * static_cast<double>(idx) + 1.0) - 1.0) * 0.5);
            while (j * (j + 1) / 2 > idx) --j;
            while ((j + 1) * (j + 2) / 2 <= idx) ++j;
            const long i = idx - j * (j + 1) / 2;
            if (i == j) continue;
            const double apq = fabs(a[idx]);
            if (apq == 0.0 || apq <= abs_floor) continue;
            const double app = fabs(a[pidx(i, i)]), aqq = fabs(a[pidx(j, j)]);
            const double g = 100.0 * apq;
            if (app + g == app && aqq + g == aqq) continue;
            flag = 1;
        }
        __syncthreads();
        if (!flag) break;
        for (int r = 0; r < N - 1; ++r) {
            // rotation parameters for the N/2 disjoint pairs of this round
            for (int k = threadIdx.x; k < half; k += blockDim.x) {
                int p = player(k, r, N), q = player(N - 1 - k, r, N);
                if (p > q) {
                    const int tmp = p;
                    p = q;
                    q = tmp;
                }
                double c = 1.0, s = 0.0, tt = 0.0;
                if (q < n) {
                    const double apq = a[pidx(p, q)];
                    const double app = a[pidx(p, p)], aqq = a[pidx(q, q)];
                    const double g = 100.0 * fabs(apq);
                    const bool negligible = apq == 0.0 || fabs(apq) <= abs_floor ||
                                            (fabs(app) + g == fabs(app) && fabs(aqq) + g == fabs(aqq));
                    if (!negligible) {
                        const double theta = (aqq - app) / (2.0 * apq);
                        if (fabs(theta) > 1e150)
                            tt = 0.5 / theta;
                        else
                            tt = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                        c = 1.0 / sqrt(tt * tt + 1.0);
                        s = tt * c;
                    } else {
                        tt = 0.0;
                    }
                }
                rc[k] = c;
                rs[k] = s;
                rt[k] = tt;
                rp[k] = p;
                rq[k] = q;
                log[static_cast<long>(rounds) * half + k] = make_double2(c, s);
            }
            __syncthreads();
            // 2x2 block updates J_P^T A J_Q over pair blocks P <= Q
            const long nblocks = static_cast<long>(half) * (half + 1) / 2;
            for (long idx = threadIdx.x; idx < nblocks; idx += blockDim.x) {
                long Q = static_cast<long>((sqrt(8.0 * static_cast<double>(idx) + 1.0) - 1.0) * 0.5);
                while (Q * (Q + 1) / 2 > idx) --Q;
                while ((Q + 1) * (Q + 2) / 2 <= idx) ++Q;
                const long P = idx - Q * (Q + 1) / 2;
                const int p1 = rp[P], q1 = rq[P], p2 = rp[Q], q2 = rq[Q];
                if (P == Q) {
                    if (q1 >= n) continue;
                    const double apq = a[pidx(p1, q1)];
                    const double tt = rt[P];
                    if (rs[P] == 0.0) {
                        // negligible: zero it exactly (NR-style termination)
                        const double g = 100.0 * fabs(apq);
                        const double app = a[pidx(p1, p1)], aqq = a[pidx(q1, q1)];
                        if (apq != 0.0 && (fabs(apq) <= abs_floor || (fabs(app) + g == fabs(app) && fabs(aqq) + g == fabs(aqq))))
                            a[pidx(p1, q1)] = 0.0;
                        continue;
                    }
                    a[pidx(p1, p1)] -= tt * apq;
                    a[pidx(q1, q1)] += tt * apq;
                    a[pidx(p1, q1)] = 0.0;
                    continue;
                }
                const double c1 = rc[P], s1 = rs[P], c2 = rc[Q], s2 = rs[Q];
                const bool v1 = q1 < n, v2 = q2 < n;
                const double x00 = a[pidx(p1, p2)];
                const double x01 = v2 ? a[pidx(p1, q2)] : 0.0;
                const double x10 = v1 ? a[pidx(q1, p2)] : 0.0;
                const double x11 = (v1 && v2) ? a[pidx(q1, q2)] : 0.0;
                const double y00 = c2 * x00 - s2 * x01, y01 = s2 * x00 + c2 * x01;
                const double y10 = c2 * x10 - s2 * x11, y11 = s2 * x10 + c2 * x11;
                a[pidx(p1, p2)] = c1 * y00 - s1 * y10;
                if (v2) a[pidx(p1, q2)] = c1 * y01 - s1 * y11;
                if (v1) a[pidx(q1, p2)] = s1 * y00 + c1 * y10;
                if (v1 && v2) a[pidx(q1, q2)] = s1 * y01 + c1 * y11;
            }
            __syncthreads();
            ++rounds;
        }
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) diag_out[i] = a[pidx(i, i)];
    if (threadIdx.x == 0) rounds_out[0] = rounds;
}

/// V = I * J_1 * ... * J_R, one warp per row. Log chunks are staged in shared.
constexpr int kReplayWarps = 8;
constexpr int kChunkMax = 16;  // rounds per staged log chunk

__global__ void __launch_bounds__(kReplayWarps * 32) jacobi_replay_k(const double2* __restrict__ log,
                                                                     const int* rounds_ptr, int n, int kChunk,
                                                                     int rows_on_chip, double* v, long ldv,
                                                                     double* rowbuf) {
    extern __shared__ __align__(16) double sm[];
    const int N = n + (n & 1);
    const int half = N / 2;
    double2* lg = reinterpret_cast<double2*>(sm);  // kChunk * half
    double* rowsm = sm + static_cast<long>(kChunk) * half * 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long row = static_cast<long>(blockIdx.x) * kReplayWarps + warp;
    double* x = rows_on_chip ? rowsm + static_cast<long>(warp) * N : rowbuf + row * N;
    const int R = rounds_ptr[0];
    if (row < n)
        for (int i = lane; i < N; i += 32) x[i] = (i == row) ? 1.0 : 0.0;
    for (int r0 = 0; r0 < R; r0 += kChunk) {
        const int nr = min(kChunk, R - r0);
        __syncthreads();
        for (long idx = threadIdx.x; idx < static_cast<long>(nr) * half; idx += blockDim.x)
            lg[idx] = log[static_cast<long>(r0) * half + idx];
        __syncthreads();
        if (row >= n) continue;
        for (int rr = 0; rr < nr; ++rr) {
            const int r = r0 + rr;
            for (int k = lane; k < half; k += 32) {
                int p = player(k, r % (N - 1), N), q = player(N - 1 - k, r % (N - 1), N);
                if (p > q) {
                    const int tmp = p;
                    p = q;
                    q = tmp;
                }
                const double2 cs = lg[static_cast<long>(rr) * half + k];
                if (cs.y == 0.0) continue;
                const double xp = x[p], xq = x[q];
                x[p] = cs.x * xp - cs.y * xq;
                x[q] = cs.y * xp + cs.x * xq;
            }
            __syncwarp();
        }
    }
    if (row < n)
        for (int i = lane; i < n; i += 32) v[row + static_cast<long>(i) * ldv] = x[i];
}

/// Descending order with index tie-break; permute values and vector columns.
__global__ void sort_desc_k(const double* vals, int n, int* order) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double vi = vals[i];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const double vj = vals[j];
            if (vj > vi || (vj == vi && j < i)) ++rank;
        }
        order[rank] = i;
    }
}

__global__ void permute_k(const double* vals, const int* order, int n, double* out_vals, const double* vin,
                          long ldi, double* vout, long ldo) {
    const long total = static_cast<long>(n) * n;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx % n, j = idx / n;
        const int src = order[j];
        vout[i + j * ldo] = vin[i + static_cast<long>(src) * ldi];
        if (i == 0) out_vals[j] = vals[src];
    }
}

}  // namespace

int sym_evd_jacobi(Context& ctx, View t, double* values, View vectors) {
    const int n = static_cast<int>(t.rows);
    if (n <= 0) return 0;
    const int N = n + (n & 1);
    const int half = N / 2;
    if (half > 2048) throw std::invalid_argument("sym_evd_jacobi: order too large");
    const long np = static_cast<long>(n) * (n + 1) / 2;
    const long max_rounds = static_cast<long>(kMaxSweeps) * (N - 1);
    DBuf<double2> log(ctx, static_cast<size_t>(max_rounds * half));
    const long head = static_cast<long>(half) * 32 + 16;
    const bool on_chip = head + np * 8 <= kSmemBudget;
    DBuf<double> gpacked(ctx, on_chip ? 1 : static_cast<size_t>(np));
    DBuf<int> rounds(ctx, 1);
    DBuf<double> diag(ctx, static_cast<size_t>(n));
    if (head > kSmemBudget) throw std::invalid_argument("sym_evd_jacobi: order too large");
    const int smem1 = static_cast<int>(head + (on_chip ? np * 8 : 0));
    static bool cfg = false;
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(jacobi_k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
        BLWS_CUDA(cudaFuncSetAttribute(jacobi_replay_k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
        cfg = true;
    }
    jacobi_k<<<1, kJacobiThreads, smem1, ctx.stream()>>>(t.p, t.ld, n, on_chip ? 1 : 0, gpacked.get(), log.get(),
                                                         rounds.get(), diag.get());
    ctx.note_launch();
    ctx.check_launch("jacobi_k");

    DMat vraw(ctx, n, n, false);
    const int chunk = static_cast<int>(std::max<long>(1, std::min<long>(kChunkMax, (64L * 1024) / (16L * half))));
    const long lg_doubles = static_cast<long>(chunk) * half * 2;
    const bool rows_on_chip = (lg_doubles + static_cast<long>(kReplayWarps) * N) * 8 <= kSmemBudget;
    const int smem2 = static_cast<int>((lg_doubles + (rows_on_chip ? static_cast<long>(kReplayWarps) * N : 0)) * 8);
    const unsigned blocks = static_cast<unsigned>((n + kReplayWarps - 1) / kReplayWarps);
    DBuf<double> rowbuf(ctx, rows_on_chip ? 1 : static_cast<size_t>(blocks) * kReplayWarps * N);
    jacobi_replay_k<<<blocks, kReplayWarps * 32, smem2, ctx.stream()>>>(
        log.get(), rounds.get(), n, chunk, rows_on_chip ? 1 : 0, vraw.data(), vraw.ld, rowbuf.get());
    ctx.note_launch();
    ctx.check_launch("jacobi_replay_k");

    DBuf<int> order(ctx, static_cast<size_t>(n));
    sort_desc_k<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx.stream()>>>(diag.get(), n, order.get());
    ctx.note_launch();
    permute_k<<<static_cast<unsigned>(std::min<long>(1024, (static_cast<long>(n) * n + 255) / 256)), 256, 0,
                ctx.stream()>>>(diag.get(), order.get(), n, values, vraw.data(), vraw.ld, vectors.p, vectors.ld);
    ctx.note_launch();
    ctx.check_launch("jacobi sort/permute");
    return 0;
}

}  // namespace blws
