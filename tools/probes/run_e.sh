cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err
