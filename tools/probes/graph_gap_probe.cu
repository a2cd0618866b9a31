// Per-kernel cost of a dependent chain of small kernels in a CUDA graph, with
// and without programmatic dependent launch (PDL): the launch gaps of the
// ~100-kernel blws_svd graph.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tiny_k(double* x, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1.0;
    if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int pdl = 0; pdl < 2; ++pdl) {
        for (int blocks : {1, 148}) {
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int i = 0; i < 100; ++i) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(blocks);
                cfg.blockDim = dim3(128);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl ? 1 : 0;
                cudaLaunchKernelEx(&cfg, tiny_k, d, pdl);
            }
            cudaStreamEndCapture(s, &g);
            if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
            cudaEventRecord(a, s);
            for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("pdl %d blocks %3d: %.2f us per kernel (%s)\n", pdl, blocks, ms * 1e3 / 2000,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
