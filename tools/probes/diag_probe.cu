// Standalone probe: cycles per pivot step of a warp-level 32x32 Cholesky in registers.
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void k(double* out, double* buf_g) {
    __shared__ double rowbuf[32];
    const int lane = threadIdx.x & 31;
    double a[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) a[j] = (j == lane ? 40.0 : 0.01 * (j + lane));
    long long c0 = clock64();
    for (int kk = 0; kk < 32; ++kk) {
        double mykk = 0.0;
#pragma unroll
        for (int j = 0; j < 32; ++j) mykk = (j == kk) ? a[j] : mykk;
        const double piv = __shfl_sync(0xffffffffu, mykk, kk);
        double rs;
        if (V == 1) rs = 1.0 / 6.3;  // no rsqrt
        else rs = rsqrt(piv);
        const bool me = lane == kk;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const double scaled = (j == kk) ? piv * rs : ((j > kk) ? a[j] * rs : a[j]);
            a[j] = me ? scaled : a[j];
        }
        double rk[32];
        if (V == 2) {
#pragma unroll
            for (int j = 0; j < 32; ++j) rk[j] = __shfl_sync(0xffffffffu, a[j], kk);
        } else {
            if (me) {
#pragma unroll
                for (int j = 0; j < 32; ++j) rowbuf[j] = a[j];
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 32; ++j) rk[j] = rowbuf[j];
        }
        double rki = 0.0;
#pragma unroll
        for (int j = 0; j < 32; ++j) rki = (j == lane) ? rk[j] : rki;
        const double f = lane > kk ? -rki : 0.0;
        if (V != 3) {
#pragma unroll
            for (int j = 0; j < 32; ++j) a[j] = fma((j >= lane) ? f : 0.0, rk[j], a[j]);
        }
        __syncwarp();
    }
    long long c1 = clock64();
    double s = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) s += a[j];
    buf_g[lane] = s;
    if (lane == 0) out[V] = (c1 - c0) / 32.0;
}
__global__ void empty_loop(double* out) {
    long long c0 = clock64();
    double x = 1.0;
    for (int i = 0; i < 32; ++i) { x = rsqrt(x + 1.0); }
    long long c1 = clock64();
    if (threadIdx.x == 0) { out[5] = (c1 - c0) / 32.0; out[6] = x; }
}
int main() {
    double *o, *b;
    cudaMalloc(&o, 64); cudaMalloc(&b, 256 * 8);
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<1, 32>>>(o, b); k<1><<<1, 32>>>(o, b); k<2><<<1, 32>>>(o, b); k<3><<<1, 32>>>(o, b);
        empty_loop<<<1, 32>>>(o);
        cudaDeviceSynchronize();
    }
    double h[8];
    cudaMemcpy(h, o, 64, cudaMemcpyDeviceToHost);
    printf("cycles/step: full %.0f | no-rsqrt %.0f | shfl-broadcast %.0f | no-update %.0f | rsqrt-chain %.0f\n",
           h[0], h[1], h[2], h[3], h[5]);
    return 0;
}
