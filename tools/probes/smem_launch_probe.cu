// Launch cost of a one-CTA kernel vs its dynamic shared memory size and block
// size (event-timed; the CholQR factor kernel is one CTA with ~135 KB).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void touch_k(double* out, int n) {
    extern __shared__ double sm[];
    for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = i;
    __syncthreads();
    if (threadIdx.x == 0) out[0] = sm[n / 2];
}
__global__ void copy_k(double* a, const double* b, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = b[i];
}

int main() {
    double *d, *a, *b;
    printf("malloc: %s\n", cudaGetErrorString(cudaMalloc(&d, 8)));
    cudaMalloc(&a, 1 << 24);
    cudaMalloc(&b, 1 << 24);
    cudaFuncSetAttribute(touch_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int kb : {0, 16, 48, 100, 135, 200}) {
        for (int threads : {256, 512, 1024}) {
            for (int interleave = 0; interleave < 2; ++interleave) {
                const int n = kb * 1024 / 8;
                float tot = 0;
                for (int r = 0; r < 50; ++r) {
                    if (interleave) copy_k<<<148, 256>>>(a, b, 10000);
                    cudaEventRecord(e0);
                    touch_k<<<1, threads, kb > 0 ? kb * 1024 : 1024>>>(d, n > 0 ? n : 1);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (r > 5) tot += ms;
                }
                { cudaError_t er = cudaGetLastError(); if (er != cudaSuccess) printf("err %s\n", cudaGetErrorString(er)); }
                printf("smem %3d KB threads %4d interleaved-copy %d: %.2f us\n", kb, threads, interleave, tot / 44 * 1e3);
            }
        }
    }
    // back-to-back launches in one event bracket
    for (int kb : {0, 135}) {
        cudaEventRecord(e0);
        for (int r = 0; r < 100; ++r) {
            copy_k<<<148, 256>>>(a, b, 10000);
            touch_k<<<1, 512, kb > 0 ? kb * 1024 : 1024>>>(d, kb * 128 > 0 ? kb * 128 : 1);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("100x (copy + touch %d KB): %.2f us per pair\n", kb, ms * 10);
    }
    return 0;
}
