// Per-phase cycle accounting of sytrd_fused_k (thread 0's view) on a random
// symmetric T of order 200. Build: nvcc -DSYTRD_PROBE ... (see sytrd_probe.sh)
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_1012_0365_b200/csrc/sytrd_fused.cu"

namespace blws {
// the library's Context is not linked here (sytrd_fused() is unused): stub
void Context::check_launch(const char*) {}
}  // namespace blws

int main() {
    const int n = 200;
    std::vector<double> t(n * n);
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i <= j; ++i) t[i + j * n] = t[j + i * n] = nd(g);
    double *dt, *lp, *d, *e, *tau;
    cudaMalloc(&dt, sizeof(double) * n * n);
    cudaMalloc(&lp, sizeof(double) * n * (n + 1) / 2);
    cudaMalloc(&d, sizeof(double) * n);
    cudaMalloc(&e, sizeof(double) * n);
    cudaMalloc(&tau, sizeof(double) * n);
    cudaMemcpy(dt, t.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    const size_t bytes = blws::fused_smem<7, false>(n);
    cudaFuncSetAttribute(blws::sytrd_fused_k<7, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int rep = 0; rep < 3; ++rep) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(g_sytrd_phase, z, sizeof(z));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        blws::sytrd_fused_k<7, false><<<1, blws::kFT, bytes>>>(dt, n, n, lp, d, e, tau);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long h[8];
        cudaMemcpyFromSymbol(h, g_sytrd_phase, sizeof(h));
        unsigned long long tot = 0;
        for (int i = 0; i < 8; ++i) tot += h[i];
        printf("rep %d: %.1f us (%s), cycles total %llu\n", rep, ms * 1e3, cudaGetErrorString(cudaGetLastError()), tot);
        const char* names[8] = {"load+prologue", "sweep+reduce", "sync A wait", "P1", "sync B wait", "P2",
                                "P3", "sync D wait"};
        for (int i = 0; i < 8; ++i)
            printf("  %-14s %10llu cycles (%5.1f%%), %.0f per step\n", names[i], h[i], 100.0 * h[i] / tot,
                   h[i] / 198.0);
        unsigned sw[256];
        cudaMemcpyFromSymbol(sw, g_sytrd_sweep, sizeof(sw));
        printf("  sweep cycles at k = 0,10,...: ");
        for (int k = 0; k < 198; k += 10) printf("%u ", sw[k]);
        printf("\n");
    }
    return 0;
}
