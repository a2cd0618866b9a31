#!/bin/bash
# build the per-phase probe of the cooperative Lanczos kernels (links the in-tree library)
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -DCOOP_PROBE \
    -diag-suppress 177 -I ../../include coop_probe.cu -o coop_probe \
    -L ../../paper_1012_0365_b200/_lib -lblws_cuda -Xlinker -rpath -Xlinker '$ORIGIN/../../paper_1012_0365_b200/_lib'
