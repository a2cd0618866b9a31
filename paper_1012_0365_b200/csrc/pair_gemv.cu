// Paired GEMV of the Lanczos step (K10): top = W x, bot = W^T y
// in ONE pass over W (the augmented apply of lanczos.hpp:112-138 reads W for
// both products; separately it is two full HBM reads, 8 m n bytes each).
//
// Grid: row blocks of 512 rows x column groups. A warp owns 64 rows (lane
// rows r = lane + 32 q, q < 2) with y in registers; it walks the group's
// columns in chunks of 32 (a full chunk's 64 loads issued before use): per
// column, 2 coalesced loads, W x into 2 register
// accumulators, W^T y partials into 32 per-lane accumulators that one
// transpose-reduction (31 shuffle-adds) turns into per-column warp sums; the 8
// warps combine through shared memory. Partials per row block (bot) and per
// column group (top) go to small global buffers and pair_gemv_reduce_k adds
// them in a fixed order (deterministic).
#include <algorithm>

#include "ops.cuh"

namespace blws {
namespace {

constexpr int kPgThreads = 256;           // 8 warps
constexpr int kPgWarps = kPgThreads / 32;
constexpr int kPgRowsPerLane = 2;
constexpr int kPgRows = kPgWarps * 32 * kPgRowsPerLane;  // 512 rows per block

__global__ void __launch_bounds__(kPgThreads) pair_gemv_k(const double* __restrict__ w, long ld, long m, long n,
                                                          long cols_per_group, const double* __restrict__ x,
                                                          const double* __restrict__ y, double* __restrict__ ptop,
                                                          double* __restrict__ pbot) {
    __shared__ double sp[2][kPgWarps][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long rb = blockIdx.x, cg = blockIdx.y;
    const long row0 = rb * kPgRows + static_cast<long>(wid) * 32 * kPgRowsPerLane;
    const long j0 = cg * cols_per_group, j1 = min(n, j0 + cols_per_group);
    double yr[kPgRowsPerLane], acc[kPgRowsPerLane];
    bool ok[kPgRowsPerLane];
#pragma unroll
    for (int q = 0; q < kPgRowsPerLane; ++q) {
        const long r = row0 + lane + 32 * q;
        ok[q] = r < m;
        yr[q] = ok[q] ? y[r] : 0.0;
        acc[q] = 0.0;
    }
    // 16-byte path: lane owns rows (r2, r2 + 1); both must exist (else the scalar path)
    const long r2 = row0 + 2 * lane;
    const bool vec2 = (ld % 2 == 0) && ((reinterpret_cast<unsigned long long>(w) & 15) == 0) &&
                      (row0 + 64 <= m);  // warp-uniform: the warp's 64 rows are all inside
    const bool ok2 = r2 + 1 < m;
    const double2 y2 = make_double2(ok2 ? y[r2] : 0.0, ok2 ? y[r2 + 1] : 0.0);
    if (vec2) {  // the vector path accumulates rows (r2, r2 + 1) instead of (lane, lane + 32)
        acc[0] = acc[1] = 0.0;
    }
    int buf = 0;
    for (long jc = j0; jc < j1; jc += 32) {
        double bp[32];
        if (jc + 32 <= j1 && vec2) {
            // full chunk, branch-free: each lane loads its 2 adjacent rows as one
            // 16-byte load, all 32 loads of the chunk in flight before use
            double2 v[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const double* col = w + (jc + c) * ld;
                v[c] = ok2 ? __ldg(reinterpret_cast<const double2*>(col + r2)) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const double xj = __ldg(x + jc + c);
                acc[0] = fma(v[c].x, xj, acc[0]);
                acc[1] = fma(v[c].y, xj, acc[1]);
                bp[c] = fma(v[c].y, y2.y, v[c].x * y2.x);
            }
        } else {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                bp[c] = 0.0;
                const long j = jc + c;
                if (j < j1) {  // warp-uniform (tail chunk / unaligned only)
                    const double xj = x[j];
                    const double* col = w + j * ld;
#pragma unroll
                    for (int q = 0; q < kPgRowsPerLane; ++q) {
                        const long r = vec2 ? r2 + q : row0 + lane + 32 * q;
                        const bool okr = vec2 ? ok2 : ok[q];
                        const double yq = vec2 ? (q == 0 ? y2.x : y2.y) : yr[q];
                        const double vv = okr ? col[r] : 0.0;
                        acc[q] = fma(vv, xj, acc[q]);
                        bp[c] = fma(vv, yq, bp[c]);
                    }
                }
            }
        }
        // transpose-reduce: lane l ends with the warp sum of column l of the chunk
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
        sp[buf][wid][lane] = bp[0];  // the reduction leaves column `lane` on lane `lane`
        __syncthreads();
        if (wid == 0) {
            double s = 0.0;
#pragma unroll
            for (int ww = 0; ww < kPgWarps; ++ww) s += sp[buf][ww][lane];
            const long j = jc + lane;
            if (j < j1) pbot[rb * n + j] = s;
        }
        buf ^= 1;  // the next chunk writes the other buffer: one barrier per chunk
    }
#pragma unroll
    for (int q = 0; q < kPgRowsPerLane; ++q) {
        const long r = vec2 ? r2 + q : row0 + lane + 32 * q;
        if (vec2 ? ok2 : ok[q]) ptop[cg * m + r] = acc[q];
    }
}

__global__ void pair_gemv_reduce_k(const double* __restrict__ ptop, long ngroups, long m, double* __restrict__ top,
                                   const double* __restrict__ pbot, long nblocks, long n, double* __restrict__ bot) {
    const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    if (i < m) {
        double s = 0.0;
        for (long g = 0; g < ngroups; ++g) s += ptop[g * m + i];
        top[i] = s;
    }
    if (i < n) {
        double s = 0.0;
        for (long b = 0; b < nblocks; ++b) s += pbot[b * n + i];
        bot[i] = s;
    }
}

}  // namespace

void pair_gemv(Context& ctx, Index m, Index n, const double* w, Index ld, const double* x, const double* y,
               double* top, double* bot) {
    if (m <= 0 || n <= 0) return;
    const long nblocks = (m + kPgRows - 1) / kPgRows;
    // column groups (multiples of 32 columns): at least ~4 CTAs per SM, and the
    // count that wastes least of the last wave (one resident CTA per SM at the
    // register count of the 16-byte path)
    const long sms = ctx.sm_count();
    const long gmax = std::max<long>(1, std::min<long>((n + 31) / 32, 128));
    const long gmin = std::min<long>(gmax, std::max<long>(1, (4 * sms + nblocks - 1) / nblocks));
    long groups = 1, cpg = ((n + 31) / 32) * 32;
    double best = -1.0;
    for (long g = gmin; g <= gmax; ++g) {  // small problems: gmin == gmax (every 32-column chunk its own group)
        const long c = ((n + g - 1) / g + 31) / 32 * 32;
        const long gg = (n + c - 1) / c;
        const long ctas = nblocks * gg;
        const double eff = static_cast<double>(ctas) / static_cast<double>(((ctas + sms - 1) / sms) * sms);
        if (eff > best + 1e-9) {
            best = eff;
            groups = gg;
            cpg = c;
        }
        if (eff > 0.985) break;
    }
    DBuf<double> ptop(ctx, static_cast<size_t>(groups * m)), pbot(ctx, static_cast<size_t>(nblocks * n));
    pair_gemv_k<<<dim3(static_cast<unsigned>(nblocks), static_cast<unsigned>(groups)), kPgThreads, 0,
                  ctx.stream()>>>(w, ld, m, n, cpg, x, y, ptop.get(), pbot.get());
    ctx.note_launch();
    ctx.check_launch("pair_gemv_k");
    const long mx = std::max<long>(m, n);
    pair_gemv_reduce_k<<<static_cast<unsigned>((mx + 255) / 256), 256, 0, ctx.stream()>>>(
        ptop.get(), groups, m, top, pbot.get(), nblocks, n, bot);
    ctx.note_launch();
    ctx.check_launch("pair_gemv_reduce_k");
}

}  // namespace blws
