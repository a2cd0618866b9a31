cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "mc or sparse" > gpurun_out/k9_tests.log 2>&1
timeout 600 python tools/probes/solver_regions.py 10000 50 0.1 --mc > gpurun_out/k9_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:"mc_sampled" -c 10 --csv --log-file gpurun_out/k9.csv python tools/probes/solver_kernels.py C4 > gpurun_out/k9_k.log 2>&1
