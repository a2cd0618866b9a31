// SvdBackend / svt and the RPCA (inexact ALM) and MC (SVT) solvers.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>

#include "dgemm.cuh"
#include "dgemm_tma.cuh"
#include "host.hpp"
#include "ops.cuh"

namespace blws {
bool tma_map_2d(CUtensorMap* map, const double* base, long inner, long outer, long ld, int box_outer);
}  // namespace blws

namespace blws {

// ================================================================== svt
RankPredictor predict_rank(RankPredictor p, Index achieved, bool all_above) {
    const Index next = achieved + (all_above ? p.increment : 1);
    p.r = std::clamp<Index>(next, 1, p.max_rank);
    p.history.push_back(p.r);
    return p;
}

SvdBackend::SvdBackend(Context& ctx, Kind k, Options o) : ctx_(ctx), kind_(k), opt_(o), rng_(o.seed) {}

namespace {
// dense m x n copy of a CSC operator (ExactFull on a sparse W)
__global__ void csc_to_dense_k(long n, const std::int64_t* colptr, const std::int32_t* rowidx, const double* val,
                               double* out, long ld) {
    for (long j = blockIdx.x; j < n; j += gridDim.x)
        for (long q = colptr[j] + threadIdx.x; q < colptr[j + 1]; q += blockDim.x) out[rowidx[q] + j * ld] = val[q];
}
}  // namespace

// svt.hpp:104-186
SvdBackend::Triplets SvdBackend::compute(LinearOperator& w, Index r) {
    const Index p = std::min(global_rows(w), w.cols());
    if (r < 1 || r > p) throw std::invalid_argument("SvdBackend: bad r");
    Triplets t;
    if (kind_ == Kind::ExactFull) {
        // svt.hpp:108-116: full SVD of the dense W, top r triplets
        if (w.row_sharded()) throw std::invalid_argument("SvdBackend: ExactFull on a row-sharded operator");
        const Index m = w.rows(), n = w.cols();
        DMat wd;
        View wv;
        if (auto* dop = dynamic_cast<DenseOperator*>(&w)) {
            wv = dop->w();
        } else if (auto* sop = dynamic_cast<SparseOperator*>(&w)) {
            wd = DMat(ctx_, m, n, true);
            csc_to_dense_k<<<static_cast<unsigned>(std::min<Index>(n, 4096)), 128, 0, ctx_.stream()>>>(
                n, sop->colptr_csc(), sop->rowidx_csc(), sop->val_csc(), wd.data(), wd.ld);
            ctx_.note_launch();
            ctx_.check_launch("csc_to_dense");
            wv = wd.view();
        } else {
            throw std::invalid_argument("SvdBackend: ExactFull needs a dense or sparse operator");
        }
        DWarm all = make_warm(ctx_, m, n, p);
        DBuf<double> sig(ctx_, static_cast<size_t>(p));
        full_svd_small(ctx_, wv, sig.get(), all.u(), all.v());
        std::vector<double> hs(static_cast<size_t>(p));
        ctx_.read(sig.get(), hs.data(), static_cast<size_t>(p));
        t.own = copy_warm(ctx_, all, r);
        t.own.sigma.assign(hs.begin(), hs.begin() + r);
        t.converged = r;
        return t;
    }
    if (kind_ == Kind::Lanczos) {
        LanczosOptions lo;
        lo.tol = opt_.ritz_tol;
        lo.max_k = opt_.max_k;
        lo.seed = rng_.next_u64();
        auto svd = lanczos_partial_svd(w, r, lo);
        t.own = std::move(svd.uv);
        t.converged = svd.stats.converged;
        t.hit_cap = !svd.stats.all_converged;
        return t;
    }
    const Index held = warm_ ? warm_->rank() : 0;
    if (held < r) {
        const Index margin = opt_.seed_margin * (Index(1) << std::min<Index>(growth_streak_, 5));
        ++growth_streak_;
        const Index r_seed = std::min(p, r + margin);
        LanczosOptions lo;
        lo.tol = opt_.ritz_tol;
        lo.max_k = opt_.max_k;
        lo.seed = rng_.next_u64();
        auto svd = lanczos_partial_svd(w, r_seed, lo);
        DWarm ws = std::move(svd.uv);
        if (ws.rank() < r_seed)
            ws = adapt_subspace(ctx_, ws.rank() > 0 ? &ws : nullptr, r_seed, w.rows(), w.cols(), rng_,
                                w.row_sharded() ? &w.shard() : nullptr);
        warm_ = std::move(ws);
        t.held = &*warm_;
        t.converged = svd.stats.converged;
        t.hit_cap = !svd.stats.all_converged;
        return t;
    }
    if (r < held) growth_streak_ = 0;
    if (held > r + 2 * opt_.seed_margin)
        warm_ = adapt_subspace(ctx_, &*warm_, r + opt_.seed_margin, w.rows(), w.cols(), rng_,
                               w.row_sharded() ? &w.shard() : nullptr);
    auto res = blws_svd(w, *warm_, opt_.block_steps, warm_->rank(), rng_);
    warm_ = std::move(res.warm);
    t.held = &*warm_;
    t.converged = res.padded ? std::min(r, warm_->rank()) : warm_->rank();
    return t;
}

// svt.hpp:216-254
SvtResult svt(LinearOperator& w, double eps, SvdBackend& backend, RankPredictor& predictor) {
    if (eps < 0.0) throw std::invalid_argument("svt: negative threshold");
    Context& ctx = w.ctx();
    RegionGuard region(ctx, 6);
    const Index p = std::min(global_rows(w), w.cols());
    Index r = std::clamp<Index>(predictor.r, 1, p);
    SvdBackend::Triplets t;
    bool all_above = false;
    while (true) {
        t = backend.compute(w, r);
        const DWarm& tr = t.get();
        const Index have = tr.rank();
        const bool smallest_above = have > 0 && tr.sigma[static_cast<size_t>(have - 1)] > eps;
        if (!smallest_above || std::max(r, have) >= p) {
            all_above = smallest_above;
            break;
        }
        r = std::min<Index>(std::max(r, have) + predictor.increment, p);
    }
    const DWarm& tr = t.get();
    if (t.hit_cap && t.converged == 0 && tr.rank() > 0 && tr.sigma[0] > eps) {
        std::ostringstream msg;
        msg << "svt: partial SVD backend hit its step cap with no converged triplet (requested " << r << " of " << p
            << ")";
        throw NumericalError(msg.str());
    }
    Index achieved = 0;
    while (achieved < tr.rank() && tr.sigma[static_cast<size_t>(achieved)] > eps) ++achieved;
    SvtResult out;
    out.trip = copy_warm(ctx, tr, achieved);
    for (Index j = 0; j < achieved; ++j) out.trip.sigma[static_cast<size_t>(j)] -= eps;
    out.sigma_dev = DBuf<double>(ctx, static_cast<size_t>(std::max<Index>(achieved, 1)));
    if (achieved > 0) ctx.write(out.sigma_dev.get(), out.trip.sigma.data(), achieved);
    out.achieved_rank = achieved;
    out.all_above_threshold = all_above;
    predictor = predict_rank(predictor, achieved, all_above);
    return out;
}

// ============================================================ device kernels
namespace {

constexpr int kT = 256;
inline unsigned gridn(long total, long cap = 4096) {
    return static_cast<unsigned>(std::max<long>(1, std::min<long>(cap, (total + kT - 1) / kT)));
}

__device__ __forceinline__ double shrink_d(double x, double eps) { return x > eps ? x - eps : (x < -eps ? x + eps : 0.0); }

// W = D - E + Y / mu (solvers.hpp:112), non-finite flag
__global__ void form_w_k(const double* D, const double* E, const double* Y, double* W, long m, long n, long ld,
                         double mu, int* bad) {
    const long total = m * n;
    int b = 0;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long o = idx % m + (idx / m) * ld;
        const double w = D[o] - E[o] + Y[o] / mu;
        W[o] = w;
        b |= !isfinite(w);
    }
    if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

// Y = D / s
__global__ void scale_into_k(const double* D, double* Y, long m, long n, long ld, double s) {
    const long total = m * n;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long o = idx % m + (idx / m) * ld;
        Y[o] = D[o] / s;
    }
}

__global__ void maxabs_partial_k(const double* x, long m, long n, long ld, double* partial) {
    const long total = m * n;
    double v = 0.0;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x)
        v = fmax(v, fabs(x[idx % m + (idx / m) * ld]));
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) v = fmax(v, sh[w]);
        partial[blockIdx.x] = v;
    }
}

// e_l0 = #|E| > tol, nnz = #E != 0 (solvers.hpp:400-409)
__global__ void e_counts_k(const double* E, long m, long n, long ld, double tol, unsigned long long* out) {
    const long total = m * n;
    unsigned long long l0 = 0, nz = 0;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const double v = E[idx % m + (idx / m) * ld];
        l0 += fabs(v) > tol;
        nz += v != 0.0;
    }
    for (int o = 16; o > 0; o >>= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        nz += __shfl_xor_sync(0xffffffffu, nz, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, l0);
        atomicAdd(out + 1, nz);
    }
}

/// K7: fused rank-r reconstruction + ALM update (solvers.hpp:114-124):
///   a = (U diag(s)) V^T            (DMMA mainloop, K = r)
///   e = shrink(D - a + Y/mu, lambda/mu); res = D - a - e; Y' = Y + mu res
///   W = D - e + Y'/mu_next;  partial ||res||^2, non-finite(W)
/// One pass over D, Y (read) and Y', W (write): 32 B per element. Y and Y' are
/// different buffers (ping-pong), so E is never stored during the iterations:
/// after the last one the EONLY instance recomputes the same tile from the
/// same inputs (U, V, D, Y, mu of that iteration -- bitwise the same a and e)
/// and stores E alone (solvers.hpp:133-146 needs E only at the end).
/// m x n: the rows held here (a row shard of a square RPCA problem, or all of it).
template <bool EONLY>
__global__ void __launch_bounds__(gemm_detail::THREADS) alm_fused_k(const double* __restrict__ us, long ldu,
                                                                   const double* __restrict__ v, long ldv, long m,
                                                                   long n, long r, const double* __restrict__ D,
                                                                   const double* __restrict__ Y,
                                                                   double* __restrict__ Yout, double* __restrict__ W,
                                                                   double* __restrict__ E, long ld, double mu,
                                                                   double mu_next, double lambda_mu, double* partial,
                                                                   int* bad) {
    using namespace gemm_detail;
    extern __shared__ __align__(16) double smem[];
    const long m0 = static_cast<long>(blockIdx.x) * BM, n0 = static_cast<long>(blockIdx.y) * BN;
    // The streamed operands of the epilogue (this tile's columns of D and Y)
    // are pulled into L2 by bulk prefetches issued before the DMMA mainloop, so
    // their HBM reads overlap the reconstruction instead of following it.
    {
        const int c = threadIdx.x & (BN - 1);
        const long col = n0 + c;
        if (col < n && (ld & 1) == 0) {
            const double* base = (threadIdx.x < BN ? D : Y) + m0 + col * ld;
            const unsigned bytes = static_cast<unsigned>(((min(static_cast<long>(BM), m - m0) * 8) + 15) & ~15L);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(base), "r"(bytes) : "memory");
        }
    }
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    mainloop<false, true, 2>(acc, smem, us, ldu, v, ldv, m, n, m0, n0, 0, r);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    double ss = 0.0;
    int nonfinite = 0;
    const double inv_mu = 1.0 / mu, inv_mu_next = 1.0 / mu_next;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
        const long row = m0 + wm + mi * 8 + g;
        if (row >= m) continue;
        // a row group's 8 D and 8 Y values are loaded before any store, so the
        // loads are in flight together (one L2 round trip per row group)
        double dv[4][2], yv[4][2];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int e2 = 0; e2 < 2; ++e2) {
                const long col = n0 + wn + ni * 8 + 2 * t + e2;
                const long o = row + col * ld;
                dv[ni][e2] = col < n ? D[o] : 0.0;
                yv[ni][e2] = col < n ? Y[o] : 0.0;
            }
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int e2 = 0; e2 < 2; ++e2) {
                const long col = n0 + wn + ni * 8 + 2 * t + e2;
                if (col >= n) continue;
                const long o = row + col * ld;
                const double a = acc[mi][ni][e2];
                const double d = dv[ni][e2];
                const double y = yv[ni][e2];
                const double dma = d - a;
                const double e = shrink_d(dma + y * inv_mu, lambda_mu);
                if (EONLY) {
                    E[o] = e;
                    continue;
                }
                const double res = dma - e;
                const double yn = y + mu * res;
                const double w = (d - e) + yn * inv_mu_next;
                Yout[o] = yn;
                W[o] = w;
                ss += res * res;
                nonfinite |= !isfinite(w);
            }
    }
    if constexpr (!EONLY) {
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        __shared__ double sh[4];
        __syncthreads();
        if (lane == 0) sh[warp] = ss;
        if (__syncthreads_or(nonfinite) && threadIdx.x == 0) atomicOr(bad, 1);
        if (threadIdx.x == 0)
            partial[blockIdx.x + static_cast<long>(blockIdx.y) * gridDim.x] = (sh[0] + sh[1]) + (sh[2] + sh[3]);
    }
}

// K7 with TMA-fed operands (the default; alm_fused_k above is the fallback for
// unaligned panels). a = us v^T has both operands with the row index
// contiguous, so both tiles are staged as [BK k][16 rows] boxes (128-byte
// swizzle) and the consumers read DMMA fragments with the conflict-free
// permuted-k addressing of the tall-skinny GEMM (dgemm_tma.cuh).
//
// Persistent, two CTAs per SM walking the 64 x 32 tiles blockIdx.x, +
// gridDim.x, ... A producer warp streams, per tile, the tile's D and Y (eight
// [32 cols][16 rows] swizzled boxes, 32 KB) and then the U / V k-tiles (a
// 4-stage ring of BK = 16), so the tile's D / Y arrive during its DMMA phase.
// Two CTAs per SM give each scheduler two consumer warps. Measured at C3
// (ncu, one ALM iteration): 80.5 us (cp.async, epilogue loads from HBM) ->
// 77.5 (TMA operands, L2 prefetch) -> 68.2 (D / Y staged, 64 x 64, 2 stages;
// the consumers then waited mostly on the operand ring) -> 65.4 us here, DMMA
// pipe 46% active. The consumers' epilogue therefore reads D and Y from shared
// memory -- no global-load latency after the DMMA phase -- and its stores of
// Y, E, W drain while the next tile's DMMAs run.
#ifndef K7_DYBUF
#define K7_DYBUF 1
#endif
#ifndef K7_STAGES
#define K7_STAGES 4
#endif
#ifndef K7_BN
#define K7_BN 32
#endif
#ifndef K7_KFIRST
#define K7_KFIRST 1
#endif
namespace k7 {
constexpr int CONS = 4, BM = 16 * CONS, BN = K7_BN, BK = 16, STAGES = K7_STAGES, DYBUF = K7_DYBUF;
constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8, STAGE = A_BYTES + B_BYTES;
constexpr int DY_BYTES = 2 * BM * BN * 8;  // D and Y of one tile
constexpr int SMEM = STAGES * STAGE + DYBUF * DY_BYTES + 1024 + 2 * (STAGES + 2) * 8;  // 81 KB: two CTAs per SM
constexpr int THREADS = 32 * (CONS + 1);
}  // namespace k7

template <bool EONLY>
__global__ void __launch_bounds__(k7::THREADS, 2) alm_tma_k(const __grid_constant__ CUtensorMap tmU,
                                                             const __grid_constant__ CUtensorMap tmV,
                                                             const __grid_constant__ CUtensorMap tmD,
                                                             const __grid_constant__ CUtensorMap tmY, long m, long n,
                                                             long r, double* __restrict__ Yout, double* __restrict__ W,
                                                             double* __restrict__ E, long ld, double mu,
                                                             double mu_next, double lambda_mu, double* partial,
                                                             int* bad) {
    using namespace k7;
    using namespace gemm_tma;
    extern __shared__ __align__(1024) unsigned char smraw[];
    // 1024-byte aligned base by an offset on the shared array itself (a round trip
    // through uintptr_t loses the address space: every fragment load became a
    // generic LD with 64-bit address arithmetic instead of an LDS)
    unsigned char* sm = smraw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smraw)) & 1023u)) & 1023u);
    unsigned char* dyb = sm + STAGES * STAGE;  // DYBUF x (D 32 KB, Y 32 KB)
    uint64_t* full = reinterpret_cast<uint64_t*>(dyb + DYBUF * DY_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* dyfull = empty + STAGES;  // 2
    uint64_t* dyempty = dyfull + 2;     // 2
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long mt = (m + BM - 1) / BM, nt = (n + BN - 1) / BN, tiles = mt * nt;
    const int ktiles = static_cast<int>((r + BK - 1) / BK);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, CONS);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(dyfull + s, 1);
            mbar_init(dyempty + s, CONS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == CONS) {
        // ---- producer
        if (lane == 0) {
            long q = 0;  // ring sequence number over the CTA's (tile, k-tile) stream
            long j = 0;  // local tile counter (D / Y buffer j & 1)
            for (long tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++j) {
                const int m0 = static_cast<int>((tile % mt) * BM), n0 = static_cast<int>((tile / mt) * BN);
                const int bsel = static_cast<int>(j % DYBUF);
                auto issue_dy = [&] {
                    mbar_wait(dyempty + bsel, static_cast<uint32_t>(((j / DYBUF) & 1) ^ 1));
                    mbar_expect_tx(dyfull + bsel, DY_BYTES);
                    unsigned char* dst = dyb + bsel * DY_BYTES;
#pragma unroll
                    for (int qq = 0; qq < BM / 16; ++qq) {
                        tma_2d(dst + qq * (BN * 128), &tmD, dyfull + bsel, m0 + 16 * qq, n0);
                        tma_2d(dst + DY_BYTES / 2 + qq * (BN * 128), &tmY, dyfull + bsel, m0 + 16 * qq, n0);
                    }
                };
                if (!K7_KFIRST) issue_dy();
                for (int kt = 0; kt < ktiles; ++kt, ++q) {
                    const int s = static_cast<int>(q % STAGES);
                    mbar_wait(empty + s, static_cast<uint32_t>(((q / STAGES) & 1) ^ 1));
                    mbar_expect_tx(full + s, STAGE);
                    unsigned char* as = sm + s * STAGE;
                    unsigned char* bs = as + A_BYTES;
                    const int k0 = kt * BK;
#pragma unroll
                    for (int qq = 0; qq < BM / 16; ++qq) tma_2d(as + qq * (BK * 128), &tmU, full + s, m0 + 16 * qq, k0);
#pragma unroll
                    for (int qq = 0; qq < BN / 16; ++qq) tma_2d(bs + qq * (BK * 128), &tmV, full + s, n0 + 16 * qq, k0);
                }
                if (K7_KFIRST) issue_dy();
            }
        }
        return;
    }
    // ---- consumers: warp w owns rows [16 w, 16 w + 16) x all 64 columns of a tile
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp * 16;
    int off[4][2];  // [k][16 rows] box offsets of rows (8 mi + g) at k-step s
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int k = kperm_tab(s, t);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int rr = h * 8 + g;
            off[s][h] = k * 128 + ((((rr >> 1) ^ (k & 7)) & 7) << 4) + (rr & 1) * 8;
        }
    }
    const double inv_mu = 1.0 / mu, inv_mu_next = 1.0 / mu_next;
    long q = 0, j = 0;
    for (long tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++j) {
        const long m0 = (tile % mt) * BM, n0 = (tile / mt) * BN;
        double acc[2][BN / 8][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int jj = 0; jj < BN / 8; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
        for (int kt = 0; kt < ktiles; ++kt, ++q) {
            const int s = static_cast<int>(q % STAGES);
            mbar_wait(full + s, static_cast<uint32_t>((q / STAGES) & 1));
            const unsigned char* as = sm + s * STAGE + warp * (BK * 128);
            const unsigned char* bs = sm + s * STAGE + A_BYTES;
            // k boxes entirely past r are zero-filled: skip their DMMAs
            const int kbn = static_cast<int>(min(static_cast<long>(BK / 16), (r - kt * BK + 15) / 16));
#pragma unroll
            for (int kb = 0; kb < BK / 16; ++kb) {
                if (kb >= kbn) break;
#pragma unroll
                for (int st = 0; st < 4; ++st) {
                    double af[2];
#pragma unroll
                    for (int mi = 0; mi < 2; ++mi)
                        af[mi] = *reinterpret_cast<const double*>(as + kb * (16 * 128) + off[st][mi]);
#pragma unroll
                    for (int ni = 0; ni < BN / 8; ++ni) {
                        const double bf = *reinterpret_cast<const double*>(bs + (ni >> 1) * (BK * 128) +
                                                                           kb * (16 * 128) + off[st][ni & 1]);
                        gemm_detail::dmma(acc[0][ni], af[0], bf);
                        gemm_detail::dmma(acc[1][ni], af[1], bf);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
        // ---- epilogue: D and Y of this warp's 16 rows from its [64 cols][16 rows] boxes
        const int bsel = static_cast<int>(j % DYBUF);
        mbar_wait(dyfull + bsel, static_cast<uint32_t>((j / DYBUF) & 1));
        const unsigned char* dbox = dyb + bsel * DY_BYTES + warp * (BN * 128);
        const unsigned char* ybox = dbox + DY_BYTES / 2;
        double ss = 0.0;
        int nonfinite = 0;
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
            const int rr = mi * 8 + g;
            const long row = m0 + wm + rr;
#pragma unroll
            for (int ni = 0; ni < BN / 8; ++ni)
#pragma unroll
                for (int e2 = 0; e2 < 2; ++e2) {
                    const int c = ni * 8 + 2 * t + e2;
                    const long col = n0 + c;
                    const int so = c * 128 + ((((rr >> 1) ^ (c & 7)) & 7) << 4) + (rr & 1) * 8;
                    const double d = *reinterpret_cast<const double*>(dbox + so);
                    const double y = *reinterpret_cast<const double*>(ybox + so);
                    if (row >= m || col >= n) continue;
                    const long o = row + col * ld;
                    const double a = acc[mi][ni][e2];
                    const double dma = d - a;
                    const double e = shrink_d(dma + y * inv_mu, lambda_mu);
                    if (EONLY) {
                        E[o] = e;
                        continue;
                    }
                    const double res = dma - e;
                    const double yn = y + mu * res;
                    const double w = (d - e) + yn * inv_mu_next;
                    Yout[o] = yn;
                    W[o] = w;
                    ss += res * res;
                    nonfinite |= !isfinite(w);
                }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(dyempty + bsel);
        if constexpr (!EONLY) {
            // one partial per (tile, warp): no consumer barrier in the epilogue
            for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            nonfinite = __any_sync(0xffffffffu, nonfinite);
            if (lane == 0) {
                partial[tile * CONS + warp] = ss;
                if (nonfinite) atomicOr(bad, 1);
            }
        }
    }
}

// K9: a_p = sum_c us[i,c] v[j,c] over CSC positions p (solvers.hpp:181-196, :247);
// resid_p = obs_p - a_p; per-block partial ||resid||^2. A warp takes 32
// consecutive positions; lanes run over the rank dimension, so every U / V row
// read is one coalesced segment; a transpose-reduction leaves the full dot of
// position t on lane t (fixed order).
template <int SLOTS>
__global__ void mc_sampled_k(long nnz, const std::int32_t* __restrict__ rowidx, const std::int32_t* __restrict__ colof,
                             const double* __restrict__ ust, const double* __restrict__ vt, long r,
                             const double* __restrict__ obs, double* resid, double* partial) {
    const int lane = threadIdx.x & 31;
    const long gw = (blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x) >> 5;
    const long nw = (static_cast<long>(gridDim.x) * blockDim.x) >> 5;
    double ss = 0.0;
    for (long p0 = gw * 32; p0 < nnz; p0 += nw * 32) {  // warp-uniform
        const long p = p0 + lane;
        const long myi = p < nnz ? rowidx[p] : 0, myj = p < nnz ? colof[p] : 0;
        double pd[32];
        // CSC order: the 32 positions usually share one column (~1000 observed
        // entries per column at C4); then V's row is loaded once into registers
        // and only the U rows are gathered (same products, same order)
        const long j0 = __shfl_sync(0xffffffffu, myj, 0);
        if (__all_sync(0xffffffffu, p >= nnz || myj == j0)) {
            double vv[SLOTS];
#pragma unroll
            for (int q = 0; q < SLOTS; ++q) {
                const long c = lane + 32 * q;
                vv[q] = c < r ? vt[j0 * r + c] : 0.0;
            }
#pragma unroll
            for (int t = 0; t < 32; ++t) {
                const long i = __shfl_sync(0xffffffffu, myi, t);
                const double* a = ust + i * r;
                double d = 0.0;
#pragma unroll
                for (int q = 0; q < SLOTS; ++q) {
                    const long c = lane + 32 * q;
                    if (c < r) d = fma(a[c], vv[q], d);
                }
                pd[t] = d;
            }
        } else {
#pragma unroll
            for (int t = 0; t < 32; ++t) {
                const long i = __shfl_sync(0xffffffffu, myi, t), j = __shfl_sync(0xffffffffu, myj, t);
                const double* a = ust + i * r;
                const double* bb = vt + j * r;
                double d = 0.0;
#pragma unroll
                for (int q = 0; q < SLOTS; ++q) {
                    const long c = lane + 32 * q;
                    if (c < r) d = fma(a[c], bb[c], d);
                }
                pd[t] = d;
            }
        }
#pragma unroll
        for (int stage = 0; stage < 5; ++stage) {
            const int half = 16 >> stage, o = 16 >> stage;
            const bool hi = (lane & o) != 0;
#pragma unroll
            for (int t = 0; t < half; ++t) {
                const double send = hi ? pd[t] : pd[t + half];
                const double keep = hi ? pd[t + half] : pd[t];
                pd[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        if (p < nnz) {  // lane t holds the dot of position p0 + t
            const double res = obs[p] - pd[0];
            resid[p] = res;
            ss = fma(res, res, ss);
        }
    }
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    __shared__ double sh[32];
    if (lane == 0) sh[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += sh[w];
        partial[blockIdx.x] = s;
    }
}

// r > 128: thread per position (the old scheme)
__global__ void mc_sampled_wide_k(long nnz, const std::int32_t* __restrict__ rowidx,
                                  const std::int32_t* __restrict__ colof, const double* __restrict__ ust,
                                  const double* __restrict__ vt, long r, const double* __restrict__ obs,
                                  double* resid, double* partial) {
    double ss = 0.0;
    for (long p = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; p < nnz;
         p += static_cast<long>(gridDim.x) * blockDim.x) {
        const double* a = ust + static_cast<long>(rowidx[p]) * r;
        const double* b = vt + static_cast<long>(colof[p]) * r;
        double s0 = 0.0, s1 = 0.0;
        long c = 0;
        for (; c + 1 < r; c += 2) {
            s0 += a[c] * b[c];
            s1 += a[c + 1] * b[c + 1];
        }
        if (c < r) s0 += a[c] * b[c];
        const double res = obs[p] - (s0 + s1);
        resid[p] = res;
        ss += res * res;
    }
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += sh[w];
        partial[blockIdx.x] = s;
    }
}

__global__ void row_major_scaled_k(const double* X, long ld, long rows, long cols, const double* s, double* out) {
    const long total = rows * cols;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const long i = idx / cols, c = idx % cols;
        out[idx] = X[i + c * ld] * (s ? s[c] : 1.0);
    }
}

__global__ void vec_axpy_k(long n, double* y, const double* x, double a) {
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long>(gridDim.x) * blockDim.x)
        y[i] += a * x[i];
}

__global__ void vec_scale_k(long n, double* y, const double* x, double a) {
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long>(gridDim.x) * blockDim.x)
        y[i] = a * x[i];
}

double sum_partials(Context& ctx, const double* part, Index count) {
    DBuf<double> out(ctx, 1);
    reduce_partials(ctx, part, count, out.get());
    double h = 0;
    ctx.read(out.get(), &h, 1);
    return h;
}

// One K7 launch (alm_tma_k, or alm_fused_k when a panel cannot be TMA-mapped or
// BLWS_K7=cpasync). eonly: store E = shrink(D - a + Y/mu, lambda/mu) alone (Yout,
// W, partial, bad untouched). Returns the number of partials written.
long alm_launch(Context& ctx, bool eonly, Index rows, Index m, Index r, const DMat& us, View v, const double* D,
                const double* Y, double* Yout, double* W, double* E, Index ld, double mu, double mu_next,
                double lambda_mu, double* part, int* bad) {
    using namespace gemm_detail;
    static const bool use_tma = [] {
        const char* e = std::getenv("BLWS_K7");
        return !(e && std::string(e) == "cpasync");
    }();
    static bool cfg = false;
    constexpr int smem = smem_bytes<false, true>();
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(alm_fused_k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        BLWS_CUDA(cudaFuncSetAttribute(alm_fused_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        BLWS_CUDA(cudaFuncSetAttribute(alm_tma_k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, k7::SMEM));
        BLWS_CUDA(cudaFuncSetAttribute(alm_tma_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, k7::SMEM));
        cfg = true;
    }
    CUtensorMap tmu, tmv, tmd, tmy;
    if (use_tma && r > 0 && tma_map_2d(&tmu, us.data(), rows, r, us.ld, k7::BK) &&
        tma_map_2d(&tmv, v.p, m, r, v.ld, k7::BK) && tma_map_2d(&tmd, D, rows, m, ld, k7::BN) &&
        tma_map_2d(&tmy, Y, rows, m, ld, k7::BN)) {
        const long tiles = ceil_div(rows, k7::BM) * ceil_div(m, k7::BN);
        const unsigned ctas = static_cast<unsigned>(std::min<long>(2L * ctx.sm_count(), tiles));
        const long nparts = tiles * k7::CONS;
        if (eonly)
            alm_tma_k<true><<<ctas, k7::THREADS, k7::SMEM, ctx.stream()>>>(tmu, tmv, tmd, tmy, rows, m, r, Yout, W, E,
                                                                           ld, mu, mu_next, lambda_mu, part, bad);
        else
            alm_tma_k<false><<<ctas, k7::THREADS, k7::SMEM, ctx.stream()>>>(tmu, tmv, tmd, tmy, rows, m, r, Yout, W, E,
                                                                            ld, mu, mu_next, lambda_mu, part, bad);
        ctx.note_launch();
        ctx.check_launch("alm_tma_k");
        return nparts;
    }
    const dim3 grid(static_cast<unsigned>(ceil_div(rows, BM)), static_cast<unsigned>(ceil_div(m, BN)));
    if (eonly)
        alm_fused_k<true><<<grid, THREADS, smem, ctx.stream()>>>(us.data(), us.ld, v.p, v.ld, rows, m, r, D, Y, Yout, W,
                                                                 E, ld, mu, mu_next, lambda_mu, part, bad);
    else
        alm_fused_k<false><<<grid, THREADS, smem, ctx.stream()>>>(us.data(), us.ld, v.p, v.ld, rows, m, r, D, Y, Yout,
                                                                  W, E, ld, mu, mu_next, lambda_mu, part, bad);
    ctx.note_launch();
    ctx.check_launch("alm_fused_k");
    return static_cast<long>(grid.x) * grid.y;
}

long alm_partials_max(Index rows, Index m) {
    using namespace gemm_detail;
    return std::max<long>(ceil_div(rows, BM) * ceil_div(m, BN), ceil_div(rows, k7::BM) * ceil_div(m, k7::BN) * k7::CONS);
}

double frob(Context& ctx, View x) {
    DBuf<double> s(ctx, 1);
    sumsq(ctx, x, s.get());
    double h = 0;
    ctx.read(s.get(), &h, 1);
    return std::sqrt(h);
}

}  // namespace

// ============================================================ K7 microbenchmark
namespace {
__global__ void hash_fill_k(double* x, long rows, long cols, long ld, unsigned long long seed, double scale) {
    const long total = rows * cols;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        unsigned long long z = seed + 0x9e3779b97f4a7c15ull * static_cast<unsigned long long>(idx + 1);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        x[idx % rows + (idx / rows) * ld] = scale * (static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0);
    }
}
}  // namespace

// Average device microseconds of one K7 launch (one ALM iteration's fused
// reconstruction + update) on an m x m problem with rank r, seeded inputs;
// eonly: the end-of-solve E pass. out[1] = the partials' sum (a checksum).
double alm_microbench(Context& ctx, Index m, Index r, int reps, bool eonly, double* checksum) {
    const Index ld = std::max<Index>(2, round_up(m, 2));
    DMat D(ctx, m, m, false), Y0(ctx, m, m, false), Y1(ctx, m, m, false), W(ctx, m, m, false);
    DMat us(ctx, m, r, false), v(ctx, m, r, false);
    const unsigned g = gridn(m * m, 8192);
    hash_fill_k<<<g, kT, 0, ctx.stream()>>>(D.data(), m, m, ld, 1, 1.0);
    hash_fill_k<<<g, kT, 0, ctx.stream()>>>(Y0.data(), m, m, ld, 2, 0.01);
    hash_fill_k<<<gridn(m * r), kT, 0, ctx.stream()>>>(us.data(), m, r, us.ld, 3, 1.0 / std::sqrt(double(r)));
    hash_fill_k<<<gridn(m * r), kT, 0, ctx.stream()>>>(v.data(), m, r, v.ld, 4, 1.0);
    ctx.note_launch(4);
    DBuf<double> part(ctx, static_cast<size_t>(alm_partials_max(m, m)));
    DBuf<int> bad(ctx, 1);
    cudaEvent_t e0, e1;
    BLWS_CUDA(cudaEventCreate(&e0));
    BLWS_CUDA(cudaEventCreate(&e1));
    float total = 0;
    long nparts = 0;
    for (int it = -1; it < reps; ++it) {
        BLWS_CUDA(cudaEventRecord(e0, ctx.stream()));
        nparts = alm_launch(ctx, eonly, m, m, r, us, v.view(), D.data(), Y0.data(), Y1.data(), W.data(), Y1.data(), ld,
                            0.5, 0.6, 0.3, part.get(), bad.get());
        BLWS_CUDA(cudaEventRecord(e1, ctx.stream()));
        BLWS_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        BLWS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (it >= 0) total += ms;
    }
    BLWS_CUDA(cudaEventDestroy(e0));
    BLWS_CUDA(cudaEventDestroy(e1));
    if (checksum) *checksum = eonly ? frob(ctx, Y1.view()) : sum_partials(ctx, part.get(), nparts);
    return 1e3 * total / std::max(reps, 1);
}

// ============================================================ rpca_adm
// Row-sharded form: with `shard`, this rank holds rows [row0, row0 +
// rows) of the m x m problem (D, Y, E, W and A row panels). The operator and the
// SVT are sharded (U local rows, V replicated); the ALM update is row-local; the
// scalars the loop branches on (||D||_F, max|D|, ||R||_F, the non-finite flags,
// the final counts and norms) are allreduced, so every rank takes the same path.
SolverStats rpca_adm(Context& ctx, Index m, const double* d_in, Index ldd, double lambda_in, SvdBackend& backend,
                     const RpcaOptions& opts, const double* truth, double* a_out, double* e_out, const RowShard* shard,
                     Index rows_in) {
    const auto t0 = std::chrono::steady_clock::now();
    std::optional<RegionGuard> phase(std::in_place, ctx, 8);  // set-up, then (9) the epilogue
    SolverStats stats;
    const bool sharded = shard != nullptr;
    if (sharded && (shard->m_total != m || rows_in < 1 || shard->row0 < 0 || shard->row0 + rows_in > m))
        throw std::invalid_argument("rpca_adm: bad row shard");
    const Index rows = sharded ? rows_in : m;
    const bool reduce = sharded && ctx.has_comm();
    DBuf<double> red(ctx, 2);
    // sum over the ranks of a device scalar (read back)
    auto total = [&](double* dev, Index count, double* host) {
        if (reduce) ctx.allreduce_sum(dev, static_cast<size_t>(count));
        ctx.read(dev, host, count);
    };
    const Index ld = std::max<Index>(2, round_up(rows, 2));
    DMat D(ctx, rows, m, false);
    copy(ctx, D.view(), View{const_cast<double*>(d_in), rows, m, ldd});
    {
        DBuf<int> bad0(ctx, 1);
        nonfinite_count(ctx, D.view(), bad0.get());
        int hb = 0;
        BLWS_CUDA(cudaMemcpyAsync(&hb, bad0.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx.stream()));
        ctx.sync();
        double hbad = hb ? 1.0 : 0.0;
        ctx.write(red.get(), &hbad, 1);
        total(red.get(), 1, &hbad);
        if (hbad > 0.0) throw std::invalid_argument("rpca_adm: D has non-finite entries");
    }
    const double lambda = lambda_in > 0.0 ? lambda_in : 1.0 / std::sqrt(static_cast<double>(m));
    double norm_d_fro = 0.0;
    sumsq(ctx, D.view(), red.get());
    total(red.get(), 1, &norm_d_fro);
    norm_d_fro = std::sqrt(norm_d_fro);
    if (norm_d_fro == 0.0) {
        if (a_out) fill(ctx, View{a_out, rows, m, ldd}, 0.0);
        if (e_out) fill(ctx, View{e_out, rows, m, ldd}, 0.0);
        stats.converged = true;
        stats.e_l0 = 0;
        return stats;
    }
    // Y ping-pong (K7 reads one, writes the other); E exists only as the zero
    // initial iterate until the end, where it is recomputed into the free Y buffer
    DMat Wm(ctx, rows, m, false), Ybuf[2] = {DMat(ctx, rows, m, false), DMat(ctx, rows, m, true)};
    int ycur = 0;
    copy(ctx, Wm.view(), D.view());
    DenseOperator op(ctx, rows, m, Wm.data(), Wm.ld);
    if (sharded) op.set_row_shard(m, shard->row0);
    const double norm2_d = spectral_norm(op);
    double mu = 1.25 / norm2_d;
    const double mu_max = mu * opts.mu_max_factor;
    double dmax = 0;
    {
        const unsigned blocks = gridn(rows * m, 1024);
        DBuf<double> part(ctx, blocks);
        maxabs_partial_k<<<blocks, kT, 0, ctx.stream()>>>(D.data(), rows, m, ld, part.get());
        ctx.note_launch();
        std::vector<double> h(blocks);
        ctx.read(part.get(), h.data(), blocks);
        for (double x : h) dmax = std::max(dmax, x);
        if (reduce) {
            ctx.write(red.get(), &dmax, 1);
            ctx.allreduce_max(red.get(), 1);
            ctx.read(red.get(), &dmax, 1);
        }
    }
    const double dual_scale = std::max(norm2_d, dmax / lambda);
    scale_into_k<<<gridn(rows * m), kT, 0, ctx.stream()>>>(D.data(), Ybuf[0].data(), rows, m, ld, dual_scale);
    ctx.note_launch();

    RankPredictor predictor;
    predictor.r = opts.initial_rank;
    predictor.increment = opts.rank_increment;
    predictor.max_rank = m;
    stats.matvec_init = op.application_count();
    std::int64_t mark = stats.matvec_init;
    Index last_rank = 0;
    DBuf<int> bad(ctx, 1);
    // first W = D - E + Y/mu (later ones come out of the fused kernel)
    zero(ctx, bad.get(), sizeof(int));
    form_w_k<<<gridn(rows * m), kT, 0, ctx.stream()>>>(D.data(), Ybuf[1].data() /* E0 = 0 */, Ybuf[0].data(),
                                                        Wm.data(), rows, m, ld, mu, bad.get());
    ctx.note_launch();
    DBuf<double> part(ctx, static_cast<size_t>(alm_partials_max(rows, m)));
    long nparts = 0;
    DMat us;                         // U diag(s) of the last prox (kept for the E pass)
    double mu_last = mu;             // mu of the last K7 launch
    SvtResult prox;
    phase.reset();
    for (Index it = 1; it <= opts.max_iter; ++it) {
        int hbad = 0;
        BLWS_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx.stream()));
        ctx.sync();
        if (reduce) {
            double hb = hbad ? 1.0 : 0.0;
            ctx.write(red.get(), &hb, 1);
            total(red.get(), 1, &hb);
            hbad = hb > 0.0;
        }
        if (hbad) throw std::invalid_argument("DenseOperator: non-finite entries");
        prox = svt(op, 1.0 / mu, backend, predictor);
        last_rank = prox.achieved_rank;
        const Index r = prox.achieved_rank;
        us = DMat(ctx, rows, std::max<Index>(r, 1), false);
        if (r > 0) scale_columns(ctx, us.view().left(r), prox.trip.u(), prox.sigma_dev.get());
        const double mu_next = std::min(opts.rho * mu, mu_max);
        zero(ctx, bad.get(), sizeof(int));
        nparts = alm_launch(ctx, false, rows, m, r, us, prox.trip.v(), D.data(), Ybuf[ycur].data(),
                            Ybuf[1 - ycur].data(), Wm.data(), nullptr, ld, mu, mu_next, lambda / mu, part.get(),
                            bad.get());
        ycur = 1 - ycur;
        mu_last = mu;
        mu = mu_next;
        stats.matvec_history.push_back(op.application_count() - mark);
        mark = op.application_count();
        double rsq = 0.0;
        reduce_partials(ctx, part.get(), nparts, red.get());
        total(red.get(), 1, &rsq);
        const double feas = std::sqrt(rsq) / norm_d_fro;
        stats.residual_history.push_back(feas);
        stats.iterations = it;
        if (feas <= opts.tol_outer) {
            stats.converged = true;
            break;
        }
    }
    phase.emplace(ctx, 9);
    // A = U diag(s) V^T of the last prox; E, e_l0, rel_err
    const Index r = prox.achieved_rank;
    // E of the last iteration: the K7 tile recomputed from that iteration's
    // inputs (U diag(s), V, D, the Y it read, its mu), bitwise the values the
    // iteration formed, stored into the Y buffer it wrote (not needed any more)
    DMat& E = Ybuf[ycur];
    if (stats.iterations > 0)
        alm_launch(ctx, true, rows, m, r, us, prox.trip.v(), D.data(), Ybuf[1 - ycur].data(), nullptr, nullptr,
                   E.data(), ld, mu_last, mu, lambda / mu_last, nullptr, nullptr);
    else
        fill(ctx, E.view(), 0.0);
    DMat A(ctx, rows, m, false);
    if (r > 0) {
        DMat us(ctx, rows, r, false);
        scale_columns(ctx, us.view(), prox.trip.u(), prox.sigma_dev.get());
        gemm(ctx, false, true, rows, m, r, 1.0, us.data(), us.ld, prox.trip.v().p, prox.trip.uv.ld, 0.0, A.data(),
             A.ld);
    } else {
        fill(ctx, A.view(), 0.0);
    }
    {
        DBuf<unsigned long long> cnt(ctx, 2);
        zero(ctx, cnt.get(), 2 * sizeof(unsigned long long));
        e_counts_k<<<gridn(rows * m, 1024), kT, 0, ctx.stream()>>>(E.data(), rows, m, ld, 1e-8 * dmax, cnt.get());
        ctx.note_launch();
        unsigned long long h[2];
        BLWS_CUDA(cudaMemcpyAsync(h, cnt.get(), sizeof(h), cudaMemcpyDeviceToHost, ctx.stream()));
        ctx.sync();
        double hc[2] = {static_cast<double>(h[0]), static_cast<double>(h[1])};  // exact below 2^53
        if (reduce) {
            ctx.write(red.get(), hc, 2);
            total(red.get(), 2, hc);
        }
        stats.e_l0 = static_cast<std::int64_t>(hc[0]);
        stats.e_nnz = static_cast<std::int64_t>(hc[1]);
    }
    if (truth) {
        DMat diff(ctx, rows, m, false);
        copy(ctx, diff.view(), A.view());
        axpy(ctx, diff.view(), View{const_cast<double*>(truth), rows, m, ldd}, -1.0);
        double nd[2];
        sumsq(ctx, diff.view(), red.get());
        sumsq(ctx, View{const_cast<double*>(truth), rows, m, ldd}, red.get() + 1);
        total(red.get(), 2, nd);
        stats.rel_err = std::sqrt(nd[0]) / std::sqrt(nd[1]);
    }
    if (a_out) copy(ctx, View{a_out, rows, m, ldd}, A.view());
    if (e_out) copy(ctx, View{e_out, rows, m, ldd}, E.view());
    ctx.sync();
    stats.rank_hat = last_rank;
    stats.matvec_count = op.application_count();
    stats.predicted_ranks = predictor.history;
    stats.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return stats;
}

// ============================================================ mc_svt
// Row-sharded form: the observed rows [row0, row0 + rows) live here as a local
// CSC; the SpMM / SpMV Wᵀ halves are allreduced by the operator, K9 is
// row-local, and the scalars (nnz, ||P_Ω D||_F, the residual norm, the error
// norms) are summed over the ranks.
McSolution mc_svt(Context& ctx, Index m, Index n, Index nnz, const std::int64_t* colptr, const std::int32_t* rowidx,
                  const double* vals, double tau_in, double delta_in, SvdBackend& backend, const McOptions& opts,
                  const double* truth_ml, const double* truth_mr, Index r_true, const RowShard* shard, Index rows_in) {
    const auto t0 = std::chrono::steady_clock::now();
    std::optional<RegionGuard> phase(std::in_place, ctx, 8);  // set-up, then (9) the epilogue
    const bool sharded = shard != nullptr;
    if (sharded && (shard->m_total != m || rows_in < 1 || shard->row0 < 0 || shard->row0 + rows_in > m))
        throw std::invalid_argument("mc_svt: bad row shard");
    const Index rows = sharded ? rows_in : m;
    const bool reduce = sharded && ctx.has_comm();
    DBuf<double> red(ctx, 2);
    auto total = [&](double* host, Index count) {  // host values summed over the ranks
        if (!reduce) return;
        ctx.write(red.get(), host, count);
        ctx.allreduce_sum(red.get(), static_cast<size_t>(count));
        ctx.read(red.get(), host, count);
    };
    double head[2] = {static_cast<double>(nnz), 0.0};  // nnz, non-finite count (exact below 2^53)
    for (Index i = 0; i < nnz; ++i)
        if (!std::isfinite(vals[i])) head[1] += 1.0;
    total(head, 2);
    const double nnz_all = head[0];
    if (nnz_all == 0.0) throw std::invalid_argument("mc_svt: empty observation set");
    if (head[1] > 0.0) throw std::invalid_argument("mc_svt: non-finite observations");
    const double tau = tau_in > 0.0 ? tau_in : 5.0 * static_cast<double>(m);
    const double delta = delta_in > 0.0 ? delta_in : 1.2 * static_cast<double>(m) * static_cast<double>(n) / nnz_all;
    SparseOperator op(ctx, rows, n, nnz, colptr, rowidx, vals);
    if (sharded) op.set_row_shard(m, shard->row0);
    const double norm2_pd = spectral_norm(op);
    const double k0 = std::ceil(tau / (delta * norm2_pd));
    const size_t nb = static_cast<size_t>(std::max<Index>(nnz, 1));
    DBuf<double> obs(ctx, nb), y(ctx, nb), resid(ctx, nb);
    if (nnz > 0)
        BLWS_CUDA(cudaMemcpyAsync(obs.get(), op.val_csc(), sizeof(double) * nnz, cudaMemcpyDeviceToDevice,
                                  ctx.stream()));
    double obs_norm = 0;
    {
        DBuf<double> s1(ctx, 1);
        zero(ctx, s1.get(), sizeof(double));
        if (nnz > 0) sumsq(ctx, View{obs.get(), nnz, 1, nnz}, s1.get());
        ctx.read(s1.get(), &obs_norm, 1);
        total(&obs_norm, 1);
        obs_norm = std::sqrt(obs_norm);
    }
    if (nnz > 0) {
        vec_scale_k<<<gridn(nnz), kT, 0, ctx.stream()>>>(nnz, y.get(), obs.get(), k0 * delta);
        ctx.note_launch();
    }

    RankPredictor predictor;
    predictor.r = opts.initial_rank;
    predictor.increment = opts.rank_increment;
    predictor.max_rank = std::min(m, n);
    McSolution sol;
    SolverStats& stats = sol.stats;
    stats.matvec_init = op.application_count();
    std::int64_t mark = stats.matvec_init;
    const unsigned blocks = gridn(std::max<Index>(nnz, 1), 2048);
    DBuf<double> part(ctx, blocks);
    phase.reset();
    for (Index it = 1; it <= opts.max_iter; ++it) {
        ctx.region_begin(7);
        op.assign_values_device(y.get());
        ctx.region_end(7, 0.0, 0.0);
        SvtResult prox = svt(op, tau, backend, predictor);
        ctx.region_begin(7);
        stats.rank_hat = prox.achieved_rank;
        const Index r = prox.achieved_rank;
        DBuf<double> ust(ctx, static_cast<size_t>(std::max<Index>(rows * r, 1))),
            vt(ctx, static_cast<size_t>(std::max<Index>(n * r, 1)));
        if (r > 0) {
            row_major_scaled_k<<<gridn(rows * r), kT, 0, ctx.stream()>>>(prox.trip.u().p, prox.trip.uv.ld, rows, r,
                                                                         prox.sigma_dev.get(), ust.get());
            row_major_scaled_k<<<gridn(n * r), kT, 0, ctx.stream()>>>(prox.trip.v().p, prox.trip.uv.ld, n, r, nullptr,
                                                                      vt.get());
            ctx.note_launch(2);
        }
        if (nnz == 0)
            zero(ctx, part.get(), sizeof(double) * blocks);
        else if (r <= 32)
            mc_sampled_k<1><<<blocks, kT, 0, ctx.stream()>>>(nnz, op.rowidx_csc(), op.colof_csc(), ust.get(), vt.get(),
                                                             r, obs.get(), resid.get(), part.get());
        else if (r <= 64)
            mc_sampled_k<2><<<blocks, kT, 0, ctx.stream()>>>(nnz, op.rowidx_csc(), op.colof_csc(), ust.get(), vt.get(),
                                                             r, obs.get(), resid.get(), part.get());
        else if (r <= 128)
            mc_sampled_k<4><<<blocks, kT, 0, ctx.stream()>>>(nnz, op.rowidx_csc(), op.colof_csc(), ust.get(), vt.get(),
                                                             r, obs.get(), resid.get(), part.get());
        else
            mc_sampled_wide_k<<<blocks, kT, 0, ctx.stream()>>>(nnz, op.rowidx_csc(), op.colof_csc(), ust.get(),
                                                               vt.get(), r, obs.get(), resid.get(), part.get());
        ctx.note_launch();
        ctx.check_launch("mc_sampled_k");
        sol.uv = std::move(prox.trip);
        stats.matvec_history.push_back(op.application_count() - mark);
        mark = op.application_count();
        reduce_partials(ctx, part.get(), blocks, red.get());
        double rsq = 0.0;
        if (reduce) ctx.allreduce_sum(red.get(), 1);
        ctx.read(red.get(), &rsq, 1);
        const double rel = std::sqrt(rsq) / obs_norm;
        stats.residual_history.push_back(rel);
        stats.iterations = it;
        if (rel <= opts.tol_outer) {
            ctx.region_end(7, 0.0, 0.0);
            stats.converged = true;
            break;
        }
        if (nnz > 0) {
            vec_axpy_k<<<gridn(nnz), kT, 0, ctx.stream()>>>(nnz, y.get(), resid.get(), delta);
            ctx.note_launch();
        }
        ctx.region_end(7, 0.0, 0.0);
    }
    phase.emplace(ctx, 9);
    stats.matvec_count = op.application_count();
    stats.predicted_ranks = predictor.history;
    if (truth_ml && truth_mr && r_true > 0) {
        // ||U S V^T - ML MR^T||_F / ||ML MR^T||_F via one GEMM with K = rank + r_true
        // (this rank's rows; the squares are summed over the ranks)
        const Index r = sol.uv.rank();
        DMat left(ctx, rows, r + r_true, false), right(ctx, n, r + r_true, false);
        if (r > 0) {
            DBuf<double> sd(ctx, static_cast<size_t>(r));
            ctx.write(sd.get(), sol.uv.sigma.data(), r);
            scale_columns(ctx, left.view().left(r), sol.uv.u(), sd.get());
            copy(ctx, right.view().left(r), sol.uv.v());
        }
        upload(ctx, left.view().cols_range(r, r_true), truth_ml, rows);
        copy(ctx, left.view().cols_range(r, r_true), left.view().cols_range(r, r_true), -1.0);
        upload(ctx, right.view().cols_range(r, r_true), truth_mr, n);
        DMat full(ctx, rows, n, false);
        gemm(ctx, false, true, rows, n, r + r_true, 1.0, left.data(), left.ld, right.data(), right.ld, 0.0, full.data(),
             full.ld);
        double nd[2];
        sumsq(ctx, full.view(), red.get());
        gemm(ctx, false, true, rows, n, r_true, -1.0, left.data() + r * left.ld, left.ld, right.data() + r * right.ld,
             right.ld, 0.0, full.data(), full.ld);
        sumsq(ctx, full.view(), red.get() + 1);
        ctx.read(red.get(), nd, 2);
        total(nd, 2);
        stats.rel_err = std::sqrt(nd[0]) / std::sqrt(nd[1]);
    }
    stats.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return sol;
}

}  // namespace blws
