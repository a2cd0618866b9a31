#!/bin/bash
# A/B variant of libblws_cuda.so: the product objects (build/obj) with the
# listed sources recompiled under extra defines, linked into
# tools/probes/var_<name>/libblws_cuda.so (select with BLWS_LIB_PATH).
# Not a product build.
#   usage: tools/probes/variant_build.sh <name> "<-DX=1 ...>" src1.cu [src2.cu ...]
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
NAME=$1; DEFS=$2; shift 2
OUT=$ROOT/tools/probes/var_$NAME
mkdir -p $OUT/obj
cp $ROOT/build/obj/*.o $OUT/obj/
for s in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I $ROOT/include $DEFS -c $ROOT/paper_1012_0365_b200/csrc/$s -o $OUT/obj/$(basename $s .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $OUT/obj/*.o -o $OUT/libblws_cuda.so \
  -lcudart_static -lrt -ldl -lpthread
rm -rf $OUT/obj
echo $OUT/libblws_cuda.so
