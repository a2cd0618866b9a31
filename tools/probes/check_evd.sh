# EVD kernels: parity tests and one eager C2 call's launch list
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ev_tests.log 2>&1
BLWS_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_c2.csv python tools/c2_once.py > gpurun_out/ev_e3.log 2>&1
