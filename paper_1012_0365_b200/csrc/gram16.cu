// K2 Gram G = X^T X of a panel of width b <= 112 (the CholQR passes, rows of
// order 10^3 - 10^4): one 16 x 16 tile of G's upper triangle per CL-CTA
// cluster. The cluster splits the rows (k-steps of 4 rows interleaved over its
// CL x 8 warps); every warp accumulates the tile's four 8 x 8 DMMA fragments
// over its k-steps, the CTA sums its warps in shared memory, the CTAs store
// their partial tiles into rank 0's shared memory (DSMEM) and rank 0 sums them
// in rank order and writes the tile and its mirror. The reduction moves 2 KB
// per CTA instead of a split-K workspace of S x b^2 doubles, there is no second
// launch, and the summation order is fixed (bitwise reproducible). G comes out
// exactly symmetric.
//
// Why tiles over clusters: the split-K GEMM for 4000 x 100 spends ~16 us in
// the GEMM plus ~4.5 us in the slice reduce; a 100 x 100 partial per row slab
// (round 2's first one-launch Gram) moved 80 KB per slab through the
// reduction. Here each CTA reads 32 columns x rows / CL of X from L2 (X is
// re-read by the 7 tiles of each column) and does 0.26 MFLOP at C2's shape.
#include <cooperative_groups.h>

#include "ops.cuh"

namespace cg = cooperative_groups;

namespace blws {
namespace {


__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <int CL, int kGW, int kGU>
__global__ void __launch_bounds__(kGW * 32) gram16_k(const double* __restrict__ x, long ld, long rows, int b, double* g,
                                               long ldg) {
    __shared__ double red[kGW][256];
    __shared__ double part[CL][256];  // rank 0's: every rank's partial tile
    cg::cluster_group cl = cg::this_cluster();
    const int rank = static_cast<int>(cl.block_rank());
    // DSMEM may only be written once the target CTA runs: arrive now, wait
    // just before the remote store (the wait is free by then)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    // tile -> (ti, tj), ti <= tj, row-major over the upper triangle of T x T tiles
    const int T = (b + 15) / 16;
    int ti = 0, rem = static_cast<int>(blockIdx.x) / CL;
    while (rem >= T - ti) {
        rem -= T - ti;
        ++ti;
    }
    const int tj = ti + rem;
    const bool diag = ti == tj;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g8 = lane >> 2, t4 = lane & 3;
    // the four fragment columns of X this lane reads (A: rows of the tile, B: its columns)
    const int ca0 = 16 * ti + g8, ca1 = ca0 + 8, cb0 = 16 * tj + g8, cb1 = cb0 + 8;
    const double* pa0 = x + static_cast<long>(min(ca0, b - 1)) * ld;
    const double* pa1 = x + static_cast<long>(min(ca1, b - 1)) * ld;
    const double* pb0 = x + static_cast<long>(min(cb0, b - 1)) * ld;
    const double* pb1 = x + static_cast<long>(min(cb1, b - 1)) * ld;
    const bool oa0 = ca0 < b, oa1 = ca1 < b, ob0 = cb0 < b, ob1 = cb1 < b;
    double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    const long ksteps = (rows + 3) / 4;
    const long stride = static_cast<long>(CL) * kGW;
    for (long s0 = static_cast<long>(rank) * kGW + wid; s0 < ksteps; s0 += kGU * stride) {
        double a0[kGU], a1[kGU], b0[kGU], b1[kGU];
#pragma unroll
        for (int u = 0; u < kGU; ++u) {
            const long k = 4 * (s0 + u * stride) + t4;
            const bool ok = k < rows;
            const long kk = ok ? k : 0;
            a0[u] = ok && oa0 ? __ldg(pa0 + kk) : 0.0;
            a1[u] = ok && oa1 ? __ldg(pa1 + kk) : 0.0;
            if (!diag) {
                b0[u] = ok && ob0 ? __ldg(pb0 + kk) : 0.0;
                b1[u] = ok && ob1 ? __ldg(pb1 + kk) : 0.0;
            } else {
                b0[u] = a0[u];
                b1[u] = a1[u];
            }
        }
#pragma unroll
        for (int u = 0; u < kGU; ++u) {
            dmma(acc[0], a0[u], b0[u]);
            dmma(acc[1], a0[u], b1[u]);
            dmma(acc[2], a1[u], b0[u]);
            dmma(acc[3], a1[u], b1[u]);
        }
    }
    // position p = (f * 32 + lane) * 2 + e holds fragment f = 2 fi + fj, element (g8, 2 t4 + e)
#pragma unroll
    for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int e = 0; e < 2; ++e) red[wid][(f * 32 + lane) * 2 + e] = acc[f][e];
    __syncthreads();
    const int p = threadIdx.x;
    double s = 0.0;
    if (p < 256) {
#pragma unroll
        for (int w = 0; w < kGW; ++w) s += red[w][p];
    }
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    if (p < 256) {
        double* dst = cl.map_shared_rank(&part[0][0], 0);
        dst[rank * 256 + p] = s;
    }
    cl.sync();
    if (rank != 0 || p >= 256) return;
    double tot = 0.0;
#pragma unroll
    for (int r = 0; r < CL; ++r) tot += part[r][p];
    const int f = p >> 6, l = (p >> 1) & 31, e = p & 1;
    const int i = 16 * ti + 8 * (f >> 1) + (l >> 2), j = 16 * tj + 8 * (f & 1) + 2 * (l & 3) + e;
    if (i < b && j < b && (!diag || i <= j)) {
        g[i + static_cast<long>(j) * ldg] = tot;
        g[j + static_cast<long>(i) * ldg] = tot;
    }
}

template <int CL, int NW, int U>
void launch_gram16(Context& ctx, View x, double* g, long ldg) {
    const int b = static_cast<int>(x.cols);
    const int T = (b + 15) / 16;
    const int tiles = T * (T + 1) / 2;
    cudaLaunchConfig_t config = {};
    config.gridDim = dim3(static_cast<unsigned>(tiles * CL), 1, 1);
    config.blockDim = dim3(32 * NW, 1, 1);
    config.dynamicSmemBytes = 0;
    config.stream = ctx.stream();
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    config.attrs = attr;
    config.numAttrs = 1;
    BLWS_CUDA(cudaLaunchKernelEx(&config, gram16_k<CL, NW, U>, static_cast<const double*>(x.p), static_cast<long>(x.ld),
                                 static_cast<long>(x.rows), b, g, ldg));
    ctx.note_launch();
    ctx.check_launch("gram16_k");
}

}  // namespace

bool gram16_fits(Index rows, Index b) { return b >= 1 && b <= 112 && rows >= 1; }

void gram16(Context& ctx, View x, double* g, Index ldg) {
    launch_gram16<8, 8, 4>(ctx, x, g, ldg);
}

}  // namespace blws
