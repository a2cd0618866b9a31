// cost of cooperative_groups grid.sync() vs grid size (256-thread blocks)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k(int iters, double* sink) {
    cg::grid_group g = cg::this_grid();
    double x = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        x = x * 1.0000001 + 1.0;
        g.sync();
    }
    if (x == 12345.0) sink[0] = x;
}

int main() {
    double* sink;
    cudaMalloc(&sink, 8);
    for (int blocks : {74, 148, 296}) {
        int iters = 2000;
        void* args[] = {&iters, &sink};
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaLaunchCooperativeKernel((void*)k, blocks, 256, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k, blocks, 256, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("blocks %3d: grid.sync %.2f us (%s)\n", blocks, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
