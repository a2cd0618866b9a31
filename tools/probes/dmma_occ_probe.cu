// DMMA (mma.sync m8n8k4 f64) throughput vs warps per SM and independent
// accumulator chains per warp: is the tall-skinny GEMM's 2 warps / SMSP enough?
#include <cstdio>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int CH>
__global__ void peak_k(double* sink, int iters) {
    double acc[CH][2];
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) dmma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) sink[0] = s;
}

template <int CH>
void run(int warps_per_sm) {
    double* sink;
    cudaMalloc(&sink, 8);
    int sms = 148;
    const int threads = 32 * warps_per_sm;  // one CTA per SM
    const int iters = 20000 * 8 / CH;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        peak_k<CH><<<sms, threads>>>(sink, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double flops = double(sms) * warps_per_sm * iters * CH * 512.0;
    printf("warps/SM %2d chains %2d: %6.2f TFLOP/s\n", warps_per_sm, CH, flops / (best * 1e-3) / 1e12);
    cudaFree(sink);
}

// GEMM-like feeding: per k-step 2 A and 13 B fragments from shared memory
// (the ts kernel's layout, LD = 20 for B, 68 for A), 26 DMMAs
__global__ void lds_fed_k(double* sink, int iters) {
    __shared__ double As[16 * 68], Bs[104 * 20];
    for (int i = threadIdx.x; i < 16 * 68; i += blockDim.x) As[i] = 1.0 + i * 1e-9;
    for (int i = threadIdx.x; i < 104 * 20; i += blockDim.x) Bs[i] = 1.0 - i * 1e-9;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & 3, g = lane >> 2, t = lane & 3;
    double acc[2][13][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 13; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 16; kk += 4) {
            double af[2];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) af[mi] = As[(kk + t) * 68 + warp * 16 + mi * 8 + g];
#pragma unroll
            for (int ni = 0; ni < 13; ++ni) {
                const double bf = Bs[(ni * 8 + g) * 20 + kk + t];
                dmma(acc[0][ni], af[0], bf);
                dmma(acc[1][ni], af[1], bf);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 13; ++b) s += acc[a][b][0] + acc[a][b][1];
    if (s == 12345.678) sink[0] = s;
}

void run_lds(int warps_per_sm) {
    double* sink;
    cudaMalloc(&sink, 8);
    const int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        lds_fed_k<<<148, 32 * warps_per_sm>>>(sink, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double flops = 148.0 * warps_per_sm * iters * 4 * 26 * 512.0;
    printf("LDS-fed warps/SM %2d: %6.2f TFLOP/s (%s)\n", warps_per_sm, flops / (best * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(sink);
}

int main() {
    for (int w : {4, 8, 16}) run_lds(w);
    for (int w : {4, 8, 16, 32}) {
        run<4>(w);
        run<8>(w);
        if (w < 32) {
            run<16>(w);
            run<26>(w);
        }
    }
    return 0;
}
