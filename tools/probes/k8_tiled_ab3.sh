#!/bin/bash
O=gpurun_out
BLWS_K8=gather timeout 600 python tools/probes/k8_tiled_check.py /tmp/k8_gather.npz > $O/k8_check_gather.log 2>&1; tail -1 $O/k8_check_gather.log
BLWS_K8=tiled timeout 600 python tools/probes/k8_tiled_check.py /tmp/k8_tiled.npz /tmp/k8_gather.npz > $O/k8_check_tiled.log 2>&1; tail -2 $O/k8_check_tiled.log
for v in gather tiled gather tiled; do
  echo "== $v"; BLWS_K8=$v timeout 900 python tools/solve_configs.py C4 --no-oracle 2>&1 | tail -1 | cut -c1-120
done
M=gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
for v in tiled; do
  BLWS_K8=$v timeout 900 ncu --metrics $M --clock-control none -k regex:csr_spmm -s 200 -c 12 --csv --log-file $O/k8ab_$v.csv python tools/probes/solver_kernels.py C4 > /dev/null 2>&1
  echo "== $v"; python tools/ncu_metrics_csv.py $O/k8ab_$v.csv | tail -3
done
