# r01g: the committed end-of-round state: GPU tests, smoke, bench (with solve leg), K9 counters
cd $GRAFT_REPO_ROOT
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g7_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g7_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r01g_bench.json 2> gpurun_out/g7_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:"mc_sampled|csr_spmm" -c 40 --launch-skip 0 --csv --log-file gpurun_out/r01g_c4_kernels.csv python tools/probes/solver_kernels.py C4 > gpurun_out/g7_k4.log 2>&1
