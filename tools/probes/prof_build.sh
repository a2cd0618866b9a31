#!/bin/bash
# Builds an instrumented copy of libblws_cuda.so (phase clocks, -D$1) into
# tools/probes/prof_lib/ for A/B runs through BLWS_LIB_PATH. Not a product build.
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
OUT=$ROOT/tools/probes/prof_lib
mkdir -p $OUT/obj
DEF=${1:-BLWS_CHOLQR_PROF}
for f in $ROOT/paper_1012_0365_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I $ROOT/include -D$DEF -c $f -o $OUT/obj/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $OUT/obj/*.o -o $OUT/libblws_cuda.so \
  -lcudart_static -lrt -ldl -lpthread
echo $OUT/libblws_cuda.so
