cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_solvers.py -x -q -k "k7" > gpurun_out/y_tests0.log 2>&1
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_dist.py -x -q > gpurun_out/y_tests.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"alm_" -c 26 --csv --log-file gpurun_out/y_k7.csv python tools/probes/solver_kernels.py C3 > gpurun_out/y_k7.log 2>&1
