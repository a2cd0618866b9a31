cd $GRAFT_REPO_ROOT
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "evd" > gpurun_out/i_tests.log 2>&1
timeout 300 python tools/probes/evd_sizes.py 200 230 300 810 1056 > gpurun_out/i_evd.log 2>&1
timeout 300 python tools/probes/solver_regions.py 2000 100 0.1 > gpurun_out/i_c3_regions.log 2>&1
