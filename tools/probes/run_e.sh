cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v_tests.log 2>&1
timeout 600 python tools/probes/solver_regions.py 10000 50 0.1 --mc > gpurun_out/v_c4.log 2>&1
