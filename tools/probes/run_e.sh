cd $GRAFT_REPO_ROOT
set -x
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_dist.py -x -q > gpurun_out/l_tests.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"alm_" -c 30 --csv --log-file gpurun_out/l_c3_k7.csv python tools/probes/solver_kernels.py C3 > gpurun_out/l_k7.log 2>&1
BLWS_K7=cpasync timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"alm_" -c 30 --csv --log-file gpurun_out/l_c3_k7_old.csv python tools/probes/solver_kernels.py C3 > gpurun_out/l_k7_old.log 2>&1
timeout 300 python tools/solve_configs.py C1 C3 --no-oracle > gpurun_out/l_solve.log 2>&1
