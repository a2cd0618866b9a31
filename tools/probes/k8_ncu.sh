#!/bin/bash
# ncu --set full of one K8 launch at C4 scale, gather and tiled (after the plain run exits 0)
O=gpurun_out
for v in gather tiled; do
  BLWS_K8=$v timeout 600 python tools/probes/solver_kernels.py C4 > $O/k8plain_$v.log 2>&1 && \
  BLWS_K8=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr_spmm -s 300 -c 1 -f -o $O/k8_$v python tools/probes/solver_kernels.py C4 > $O/k8ncu_$v.log 2>&1
  ncu -i $O/k8_$v.ncu-rep --page details > $O/k8_${v}_details.txt 2>&1
done
