# r01d: GPU tests, smoke, bench, launch list and a K1 full capture of the TMA GEMM build
cd $GRAFT_REPO_ROOT
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/d_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/d_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/d_bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01d_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/d_e2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -o gpurun_out/k1_r01d python tools/k1_profile.py > gpurun_out/d_e1.log 2>&1
BLWS_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01d_c2_call_launches.csv python tools/c2_once.py > gpurun_out/d_e3.log 2>&1
ls -la gpurun_out/
