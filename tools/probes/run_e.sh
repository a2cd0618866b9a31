cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_tests.log 2>&1
BLWS_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c2_call.csv python tools/c2_once.py > gpurun_out/r2_e3.log 2>&1
timeout 900 python bench.py --no-solves > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
