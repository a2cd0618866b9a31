# r01e: bench, launch lists, solver configs and region breakdowns, solver-kernel counters
cd $GRAFT_REPO_ROOT
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/e5_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e5_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/e5_bench.json 2> gpurun_out/e5_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01e_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/e5_e2.log 2>&1
BLWS_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01e_c2_call_launches.csv python tools/c2_once.py > gpurun_out/e5_e3.log 2>&1
timeout 900 python tools/solve_configs.py C1 C3 C4 --baseline > gpurun_out/r01e_solve_configs.jsonl 2> gpurun_out/e5_solve.err
timeout 900 python tools/solve_configs.py C5 --no-oracle >> gpurun_out/r01e_solve_configs.jsonl 2>> gpurun_out/e5_solve.err
for c in "500 25 0.05" "2000 100 0.1" "40000 400 0.05"; do timeout 900 python tools/probes/solver_regions.py $c; done > gpurun_out/r01e_solver_regions.txt 2>&1
timeout 600 python tools/probes/solver_regions.py 10000 50 0.1 --mc >> gpurun_out/r01e_solver_regions.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"alm_|lanczos_rows" -c 40 --csv --log-file gpurun_out/r01e_c3_kernels.csv python tools/probes/solver_kernels.py C3 > gpurun_out/e5_k3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:"csr_spmm|mc_sampled|csr_spmv" -c 60 --csv --log-file gpurun_out/r01e_c4_kernels.csv python tools/probes/solver_kernels.py C4 > gpurun_out/e5_k4.log 2>&1
ls -la gpurun_out/
