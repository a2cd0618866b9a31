#!/bin/bash
O=gpurun_out
BLWS_K8=gather timeout 600 python tools/probes/k8_tiled_check.py /tmp/k8_gather.npz > $O/k8_check_gather.log 2>&1; tail -2 $O/k8_check_gather.log
BLWS_K8=tiled timeout 600 python tools/probes/k8_tiled_check.py /tmp/k8_tiled.npz /tmp/k8_gather.npz > $O/k8_check_tiled.log 2>&1; tail -3 $O/k8_check_tiled.log
timeout 1200 python -m pytest tests/test_gpu_variants.py -q -k "K8 or k8" 2>&1 | tail -5
BLWS_K8=tiled timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -q -k "sparse or mc" 2>&1 | tail -3
