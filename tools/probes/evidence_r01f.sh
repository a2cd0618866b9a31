# r01f (final of round 1): tests, smoke, bench with the solve-time leg, launch lists, K7 counters
cd $GRAFT_REPO_ROOT
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f6_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f6_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r01f_bench.json 2> gpurun_out/f6_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01f_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-solves > gpurun_out/f6_e2.log 2>&1
BLWS_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01f_c2_call_launches.csv python tools/c2_once.py > gpurun_out/f6_e3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"alm_" -c 26 --csv --log-file gpurun_out/r01f_c3_k7.csv python tools/probes/solver_kernels.py C3 > gpurun_out/f6_k7.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01f_reference.json 2> gpurun_out/f6_ref.err
ls -la gpurun_out/
