// Blocked CholQR factor for Grams wider than one CTA's on-chip factor (K3 for
// 112 < n <= 1024; the C5 panels are b ~ 400-411, C3's transients ~528).
//
// G = R^T R (upper R) by right-looking blocks of <= 112 columns:
//   R_kk, R_kk^{-1}  <- cholqr_factor_k on the diagonal block (one CTA, on chip)
//   R_k,(k+1:)       <- R_kk^{-T} G_k,(k+1:)            (multi-CTA GEMM)
//   G_(k+1:),(k+1:)  -= R_k,(k+1:)^T R_k,(k+1:)          (multi-CTA GEMM)
// and R^{-1} by block back substitution, X_ij = -R_ii^{-1} sum_{k=i+1..j} R_ik X_kj,
// also on the GEMM. The one-CTA chol_inv_k streamed every trailing update of an
// n = 400 Gram through one SM (3.15 ms); here the O(n^3) work spreads over the GPU
// and only the 112-wide diagonal factors stay on one CTA each.
// Outputs as chol_inv_upper: G <- R (upper, zero lower), rinv <- R^{-1} (upper,
// zero lower), status 0 / first bad pivot + 1, diag = min / max diag(R),
// trace_out = tr(G). No whole-matrix skip mode: a near-identity Gram (the second
// CholQR pass) takes cholqr_factor_k's near-identity path block by block.
#include <algorithm>

#include "ops.cuh"

namespace blws {
namespace {

constexpr int kBlk = 112;  // cholqr_factor_fits

__global__ void blk_trace_k(const double* __restrict__ g, long ld, int n, double* out) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += g[i + i * ld];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ double red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
        out[0] = t;
    }
}

// strictly lower triangle of an n x n column-major matrix -> 0
__global__ void blk_zero_lower_k(double* a, long ld, int n) {
    const long total = static_cast<long>(n) * n;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx % n, j = idx / n;
        if (i > j) a[i + j * ld] = 0.0;
    }
}

// per-block statuses / diag ranges -> the matrix's (first failing pivot, global index)
__global__ void blk_combine_k(const int* __restrict__ bst, const double* __restrict__ bdg, int nb, int bsz,
                              int* status, double* diag) {
    if (threadIdx.x != 0) return;
    int st = 0;
    double mn = INFINITY, mx = 0.0;
    for (int k = 0; k < nb; ++k) {
        if (st == 0 && bst[k] != 0) st = k * bsz + bst[k];
        mn = fmin(mn, bdg[2 * k]);
        mx = fmax(mx, bdg[2 * k + 1]);
    }
    status[0] = st;
    diag[0] = mn;
    diag[1] = mx;
}

}  // namespace

bool chol_blocked_fits(Index n) { return n > kBlk && n <= 1024; }

void chol_inv_blocked(Context& ctx, View g, View rinv, int* status, double* diag, double* trace_out) {
    const int n = static_cast<int>(g.rows);
    const int nb = (n + kBlk - 1) / kBlk;
    const int bsz = (n + nb - 1) / nb;  // equal blocks (<= kBlk), the last one shorter
    const long ld = g.ld, ldr = rinv.ld;
    if (trace_out) {
        blk_trace_k<<<1, 256, 0, ctx.stream()>>>(g.p, ld, n, trace_out);
        ctx.note_launch();
    }
    DBuf<int> bst(ctx, static_cast<size_t>(nb));
    DBuf<double> bdg(ctx, static_cast<size_t>(2 * nb));
    DBuf<double> tmp(ctx, static_cast<size_t>(bsz) * n);
    for (int k = 0; k < nb; ++k) {
        const int o = k * bsz, b = std::min(bsz, n - o), w = n - o - b;
        View akk = g.sub(o, o, b, b), rkk = rinv.sub(o, o, b, b);
        cholqr_factor(ctx, akk, rkk, nullptr, 0, nullptr, bst.get() + k, bdg.get() + 2 * k, nullptr, nullptr, nullptr);
        if (w <= 0) continue;
        // panel R_k,(k+1:) = R_kk^{-T} G_k,(k+1:) (through tmp: the GEMM may not alias)
        const double* gkj = g.p + o + static_cast<long>(o + b) * ld;
        gemm(ctx, true, false, b, w, b, 1.0, rkk.p, ldr, gkj, ld, 0.0, tmp.get(), b);
        copy(ctx, g.sub(o, o + b, b, w), View{tmp.get(), b, w, b});
        // trailing G_(k+1:),(k+1:) -= P^T P
        double* gtt = g.p + (o + b) + static_cast<long>(o + b) * ld;
        gemm(ctx, true, false, w, w, b, -1.0, tmp.get(), b, tmp.get(), b, 1.0, gtt, ld);
    }
    blk_zero_lower_k<<<static_cast<unsigned>(std::min<long>(1024, (static_cast<long>(n) * n + 255) / 256)), 256, 0,
                       ctx.stream()>>>(g.p, ld, n);
    ctx.note_launch();
    // R^{-1}: diagonal blocks from the factors; X_ij = -R_ii^{-1} (sum_{k=i+1..j} R_ik X_kj), i descending
    blk_zero_lower_k<<<static_cast<unsigned>(std::min<long>(1024, (static_cast<long>(n) * n + 255) / 256)), 256, 0,
                       ctx.stream()>>>(rinv.p, ldr, n);
    ctx.note_launch();
    for (int j = 1; j < nb; ++j) {
        const int oj = j * bsz, bj = std::min(bsz, n - oj);
        for (int i = j - 1; i >= 0; --i) {
            const int oi = i * bsz, bi = std::min(bsz, n - oi), o1 = oi + bi, kk = oj + bj - o1;
            // tmp (bi x bj) = R[oi.., o1..oj+bj) X[o1..oj+bj, oj..]
            gemm(ctx, false, false, bi, bj, kk, 1.0, g.p + oi + static_cast<long>(o1) * ld, ld,
                 rinv.p + o1 + static_cast<long>(oj) * ldr, ldr, 0.0, tmp.get(), bi);
            gemm(ctx, false, false, bi, bj, bi, -1.0, rinv.p + oi + static_cast<long>(oi) * ldr, ldr, tmp.get(), bi, 0.0,
                 rinv.p + oi + static_cast<long>(oj) * ldr, ldr);
        }
    }
    blk_combine_k<<<1, 32, 0, ctx.stream()>>>(bst.get(), bdg.get(), nb, bsz, status, diag);
    ctx.note_launch();
    ctx.check_launch("chol_inv_blocked");
}

}  // namespace blws
