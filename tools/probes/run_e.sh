cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "sparse" > gpurun_out/w_tests.log 2>&1
timeout 600 python tools/probes/solver_regions.py 10000 50 0.1 --mc > gpurun_out/w_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:"csr_spmm|mc_sampled" -c 40 --csv --log-file gpurun_out/w_c4_kernels.csv python tools/probes/solver_kernels.py C4 > gpurun_out/w_k.log 2>&1
