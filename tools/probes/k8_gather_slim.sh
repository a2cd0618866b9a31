#!/bin/bash
# K8 gather kernel after the instruction diet: bitwise check against the (unchanged) tiled
# kernel, sparse / MC GPU tests, the C4 solve, per-launch ncu metrics
O=gpurun_out
BLWS_K8=gather timeout 600 python tools/probes/k8_tiled_check.py /tmp/k8_gather.npz > $O/k8_check_gather.log 2>&1; tail -1 $O/k8_check_gather.log
BLWS_K8=tiled timeout 600 python tools/probes/k8_tiled_check.py /tmp/k8_tiled.npz /tmp/k8_gather.npz > $O/k8_check_tiled.log 2>&1; tail -2 $O/k8_check_tiled.log
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py tests/test_gpu_variants.py tests/test_gpu_configs.py -q -k "sparse or mc or c4 or k8 or variant" 2>&1 | tail -3
for i in 1 2 3; do timeout 900 python tools/solve_configs.py C4 --no-oracle 2>&1 | tail -1 | cut -c1-130; done
M=gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:csr_spmm -s 200 -c 12 --csv --log-file $O/k8slim.csv python tools/probes/solver_kernels.py C4 > /dev/null 2>&1
python tools/ncu_metrics_csv.py $O/k8slim.csv | tail -3
python bench.py 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['parity']['status'], d['solves']['C4']['solve_s'], d['solves']['C3']['solve_s'])"
