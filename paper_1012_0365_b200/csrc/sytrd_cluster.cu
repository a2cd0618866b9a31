// Householder tridiagonalisation of the projected T over a thread-block
// cluster (K4, stage 1), LAPACK dsytd2 (lower) semantics.
//
// A single CTA is instruction/latency bound (~1 ms at order 200, one SM of
// 148 busy). Here the packed lower triangle is distributed by columns
// (round-robin) over CL CTAs of one cluster and the per-step vectors move
// through distributed shared memory:
//   1. the owner of column k forms v, tau, beta and pushes v into every CTA
//      (DSMEM stores);                                        cluster barrier
//   2. each CTA forms its partial p = A(own columns) v: rows by threads (the
//      L(i, j) v_j part, deterministic order) and columns by warps (the
//      L(:, j)^T v part);                                     cluster barrier
//   3. every CTA sums the CL partials (DSMEM loads, same order everywhere ->
//      identical p), forms w = tau p - K v and updates its own columns.
// v and the partials are double-buffered by step parity, so two barriers per
// step suffice. Opt-in (BLWS_SYTRD=cluster): slower than sytrd_k at the
// orders BLWS produces, see sytrd_cluster() below. Output layout equals the single-CTA sytrd_k (packed lower
// with reflectors, d, e, tau) so ormtr_k is shared.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "ops.cuh"

namespace cg = cooperative_groups;

namespace blws {
namespace {

constexpr int kCT = 512;

__device__ __forceinline__ int gloff(int j, int n) { return j * n - ((j * (j - 1)) >> 1); }  // global packed col start

template <int CL>
struct Local {
    // CTA c owns columns j = c, c + CL, ...; local column t = (j - c) / CL of length n - j
    __device__ static int off(int t, int c, int n) { return t * n - c * t - CL * ((t * (t - 1)) >> 1); }
};

// GM: the own columns stay in the global packed output `lp` (L2-resident, used
// in place) instead of shared memory -- orders whose 1/CL share of the triangle
// does not fit a CTA (n > ~920 at CL = 16; C3's transient b ~ 528 gives 1056).
template <int CL, bool GM>
__global__ void __launch_bounds__(kCT) sytrd_cluster_k(const double* __restrict__ tin, long ld, int n, double* lp,
                                                       double* d, double* e, double* tau) {
    cg::cluster_group cluster = cg::this_cluster();
    const int c = static_cast<int>(cluster.block_rank());
    if (cluster.num_blocks() != CL) {
        if (threadIdx.x == 0) tau[n - 1] = -1.0;  // geometry error marker (checked by the host)
        return;
    }
    extern __shared__ __align__(16) double sm[];
    double* vbuf = sm;            // 2 x n   (double-buffered v)
    double* pp = vbuf + 2 * n;    // 2 x n   (double-buffered partial p)
    double* pf = pp + 2 * n;      // n       (full p, then w)
    double* red = pf + n;         // 64
    double* cols = red + 64;      // own packed columns (shared-memory variant)
    // own local column t: rows j..n-1 of global column j = c + t CL
    auto colp = [&](int t) -> double* {
        return GM ? lp + gloff(c + t * CL, n) : cols + Local<CL>::off(t, c, n);
    };
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int ncols = (n - c + CL - 1) / CL;  // local column count

    // load own columns (lower triangle, symmetrised)
    for (int t = wid; t < ncols; t += nw) {
        const int j = c + t * CL;
        double* col = colp(t);
        for (int i = j + lane; i < n; i += 32) col[i - j] = 0.5 * (tin[i + static_cast<long>(j) * ld] + tin[j + static_cast<long>(i) * ld]);
    }
    cluster.sync();

    for (int k = 0; k < n - 2; ++k) {
        const int w = n - k - 1;
        const int par = k & 1;
        double* v = vbuf + par * n;   // v[i] for trailing row index i (0..w-1)
        double* ppk = pp + par * n;
        const int owner = k % CL;
        __shared__ double s_tau, s_beta;
        if (c == owner) {
            __syncthreads();  // column k was updated by other warps of this CTA in step k-1
            const int tk = k / CL;
            double* x = colp(tk) + 1;  // rows k+1..n-1 of column k
            double s = 0.0;
            for (int i = 1 + threadIdx.x; i < w; i += blockDim.x) s += x[i] * x[i];
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) red[wid] = s;
            __syncthreads();
            double sigma2 = 0.0;
            for (int q = 0; q < nw; ++q) sigma2 += red[q];
            const double alpha = x[0];
            double tk_ = 0.0, beta = alpha, scl = 0.0;
            if (sigma2 > 0.0) {
                beta = -copysign(sqrt(alpha * alpha + sigma2), alpha);
                tk_ = (beta - alpha) / beta;
                scl = 1.0 / (alpha - beta);
            }
            // push v into every CTA's buffer (DSMEM), keep the reflector in column k
            for (int r = 0; r < CL; ++r) {
                double* dst = cluster.map_shared_rank(v, r);
                for (int i = threadIdx.x; i < w; i += blockDim.x) dst[i] = (tk_ == 0.0) ? 0.0 : (i == 0 ? 1.0 : x[i] * scl);
                if (threadIdx.x == 0) {
                    double* dt = cluster.map_shared_rank(&s_tau, r);
                    double* db = cluster.map_shared_rank(&s_beta, r);
                    *dt = tk_;
                    *db = beta;
                }
            }
            if (threadIdx.x == 0) {
                d[k] = colp(tk)[0];
                e[k] = beta;
                tau[k] = tk_;
            }
            __syncthreads();
            for (int i = threadIdx.x; i < w; i += blockDim.x) x[i] = (tk_ == 0.0) ? 0.0 : (i == 0 ? 1.0 : x[i] * scl);
        }
        cluster.sync();  // (1) v, tau visible everywhere
        const double tk_ = s_tau;
        if (tk_ == 0.0) {
            cluster.sync();  // keep the barrier count uniform
            continue;
        }
        // (2) partial p over own columns j > k: rows by threads (sum_j L(i, j) v_j, j <= i)
        //     plus, per own column j, its strictly-lower dot with v (added at row j)
        const int t0 = (k + 1 - c + CL - 1) / CL;  // first own local column with j >= k+1
        for (int ii = threadIdx.x; ii < w; ii += blockDim.x) {
            const int i = k + 1 + ii;
            double s = 0.0;
            for (int t = t0; t < ncols; ++t) {
                const int j = c + t * CL;
                if (j > i) break;
                s = fma(colp(t)[i - j], v[j - k - 1], s);
            }
            ppk[ii] = s;
        }
        __syncthreads();
        for (int t = t0 + wid; t < ncols; t += nw) {
            const int j = c + t * CL;
            const double* col = colp(t);
            double s = 0.0;
            for (int i = j + 1 + lane; i < n; i += 32) s = fma(col[i - j], v[i - k - 1], s);
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) ppk[j - k - 1] += s;
        }
        cluster.sync();  // (2) partials visible everywhere
        // (3) full p (same summation order in every CTA), K, w
        double pv = 0.0;
        for (int ii = threadIdx.x; ii < w; ii += blockDim.x) {
            double s = 0.0;
            for (int r = 0; r < CL; ++r) s += cluster.map_shared_rank(ppk, r)[ii];
            s *= tk_;
            pf[ii] = s;
            pv = fma(s, v[ii], pv);
        }
        for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
        if (lane == 0) red[32 + wid] = pv;
        __syncthreads();
        double tot = 0.0;
        for (int q = 0; q < nw; ++q) tot += red[32 + q];
        const double K = 0.5 * tk_ * tot;
        for (int ii = threadIdx.x; ii < w; ii += blockDim.x) pf[ii] -= K * v[ii];
        __syncthreads();
        // rank-2 update of own columns: L(i, j) -= v_i w_j + w_i v_j, i >= j > k
        for (int t = t0 + wid; t < ncols; t += nw) {
            const int j = c + t * CL;
            double* col = colp(t);
            const double vj = v[j - k - 1], wj = pf[j - k - 1];
            for (int i = j + lane; i < n; i += 32) col[i - j] -= fma(v[i - k - 1], wj, pf[i - k - 1] * vj);
        }
        // no trailing barrier: the next step writes the other parity buffers
    }
    cluster.sync();
    // tail: d[n-2], d[n-1], e[n-2]; write own columns to the global packed layout
    if (n >= 2 && c == (n - 2) % CL && threadIdx.x == 0) {
        const double* col = colp((n - 2) / CL);
        d[n - 2] = col[0];
        e[n - 2] = col[1];
        tau[n - 2] = 0.0;
    }
    if (c == (n - 1) % CL && threadIdx.x == 0) {
        d[n - 1] = colp((n - 1) / CL)[0];
        tau[n - 1] = 0.0;
    }
    if (!GM) {
        for (int t = wid; t < ncols; t += nw) {
            const int j = c + t * CL;
            const double* col = colp(t);
            double* g = lp + gloff(j, n);
            for (int i = lane; i < n - j; i += 32) g[i] = col[i];
        }
    }
}

template <int CL, bool GM = false>
size_t smem_bytes(int n) {
    // largest per-CTA column share is CTA 0's
    const long ncols = (n + CL - 1) / CL;
    long elems = 0;
    if (!GM)
        for (long t = 0; t < ncols; ++t) elems += n - t * CL;
    return static_cast<size_t>((5L * n + 64 + elems) * 8);
}

template <int CL, bool GM = false>
void launch(Context& ctx, View t, int n, double* lp, double* d, double* e, double* tau) {
    const size_t bytes = smem_bytes<CL, GM>(n);
    static bool cfg = false;
    if (!cfg) {
        BLWS_CUDA(cudaFuncSetAttribute(sytrd_cluster_k<CL, GM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       220 * 1024));
        if (CL > 8)
            BLWS_CUDA(cudaFuncSetAttribute(sytrd_cluster_k<CL, GM>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cfg = true;
    }
    cudaLaunchConfig_t config = {};
    config.gridDim = dim3(CL, 1, 1);
    config.blockDim = dim3(kCT, 1, 1);
    config.dynamicSmemBytes = bytes;
    config.stream = ctx.stream();
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    config.attrs = attr;
    config.numAttrs = 1;
    BLWS_CUDA(cudaLaunchKernelEx(&config, sytrd_cluster_k<CL, GM>, static_cast<const double*>(t.p), static_cast<long>(t.ld),
                                 n, lp, d, e, tau));
    ctx.note_launch();
    ctx.check_launch("sytrd_cluster_k");
}

// A 16-CTA cluster is a non-portable size: ask the occupancy calculator once
// whether this device can place one.
bool cluster16_ok() {
    static int ok = -1;
    if (ok < 0) {
        ok = 0;
        if (cudaFuncSetAttribute(sytrd_cluster_k<16, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                cudaSuccess &&
            cudaFuncSetAttribute(sytrd_cluster_k<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024) ==
                cudaSuccess) {
            cudaLaunchConfig_t config = {};
            config.gridDim = dim3(16, 1, 1);
            config.blockDim = dim3(kCT, 1, 1);
            config.dynamicSmemBytes = 220 * 1024;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 16;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            config.attrs = attr;
            config.numAttrs = 1;
            int clusters = 0;
            if (cudaOccupancyMaxActiveClusters(&clusters, sytrd_cluster_k<16, false>, &config) == cudaSuccess)
                ok = clusters > 0 ? 1 : 0;
        }
        cudaGetLastError();  // a refusal above is not a launch error
    }
    return ok == 1;
}

}  // namespace

bool sytrd_cluster(Context& ctx, View t, double* lp, double* d, double* e, double* tau, bool auto_pick) {
    const int n = static_cast<int>(t.rows);
    if (n < 64) return false;
    // Measured on B200 (order 208): 1.16 ms vs 0.95 ms for the single-CTA sytrd_k
    // -- two cluster barriers (~400 cyc each) plus DSMEM broadcast / all-reduce
    // (~20 B/cyc) per column cost more than the extra SMs save while the
    // triangle fits one CTA (sytrd_fused, n <= 224): opt-in there
    // (BLWS_SYTRD=cluster). Above that (C3's T of order 230-300 and a transient
    // 1056, C5's ~810) the alternative is the one-CTA global-memory sytrd_k, so
    // the cluster path is picked automatically (auto_pick); orders whose
    // 1/16 share does not fit shared memory keep their columns in L2 (GM).
    const char* env = std::getenv("BLWS_SYTRD");
    const bool forced = env && std::string(env) == "cluster";
    if (!forced && !auto_pick) return false;
    if (smem_bytes<8>(n) <= 220u * 1024u) {
        launch<8>(ctx, t, n, lp, d, e, tau);
        return true;
    }
    if (!cluster16_ok()) return false;
    if (smem_bytes<16>(n) <= 220u * 1024u) {
        launch<16>(ctx, t, n, lp, d, e, tau);
        return true;
    }
    if (smem_bytes<16, true>(n) <= 220u * 1024u) {
        launch<16, true>(ctx, t, n, lp, d, e, tau);
        return true;
    }
    return false;
}

}  // namespace blws
