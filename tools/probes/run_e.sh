cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "mc or sparse or lanczos or spectral" > gpurun_out/s_tests1.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s_tests.log 2>&1
