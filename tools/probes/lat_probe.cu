// Dependent-chain latencies on one warp (clock64 deltas): DFMA, DADD, DMUL,
// 64-bit SHFL, LDS.64, MUFU.RSQ64H + Newton, and a 512-thread __syncthreads.
#include <cstdio>

__global__ void lat_k(double* out, long long* cyc, double seed) {
    __shared__ double s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = seed + i;
    __syncthreads();
    double x = seed + threadIdx.x;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) x = fma(x, 0.999, 1e-3);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0);
    // DADD chain
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) x = x + 1e-3;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = (t1 - t0);
    // SHFL chain (double)
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15));
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = (t1 - t0);
    // LDS chain
    int idx = threadIdx.x & 7;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) {
        const double v = s[idx];
        idx = (static_cast<int>(v) & 7) + 8 * (i & 3);
    }
    t1 = clock64();
    x += idx;
    if (threadIdx.x == 0) cyc[3] = (t1 - t0);
    // rsqrt approx chain
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        double y;
        asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
        x = y + 1.0;
    }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[4] = (t1 - t0);
    // syncthreads chain
    t0 = clock64();
    for (int i = 0; i < 64; ++i) {
        __syncthreads();
    }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[5] = (t1 - t0);
    // DMUL
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) x = x * 0.9999;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[6] = (t1 - t0);
    out[threadIdx.x] = x;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 512 * 8);
    cudaMalloc(&cyc, 8 * 8);
    for (int threads : {32, 512}) {
        for (int rep = 0; rep < 2; ++rep) lat_k<<<1, threads>>>(out, cyc, 1.5);
        long long h[8];
        cudaMemcpy(h, cyc, 7 * 8, cudaMemcpyDeviceToHost);
        printf("threads %d: dfma %.1f  dadd %.1f  shfl64 %.1f  lds-chain %.1f  rsqrt+dadd %.1f  bar %.1f  dmul %.1f cycles\n",
               threads, h[0] / 64.0, h[1] / 64.0, h[2] / 64.0, h[3] / 64.0, h[4] / 16.0, h[5] / 64.0, h[6] / 64.0);
    }
    return 0;
}
