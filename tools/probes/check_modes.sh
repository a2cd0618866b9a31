# sharded-mode and torchrun launches of bench.py (one GPU): stdout must be one JSON line
cd $GRAFT_REPO_ROOT
env | grep -i nccl > gpurun_out/l_env.txt
timeout 600 python bench.py --mode sharded --steps 5 --warmup 3 --no-cpu --no-solves > gpurun_out/l_sharded.json 2> gpurun_out/l_sharded.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --no-solves > gpurun_out/l_torchrun.json 2> gpurun_out/l_torchrun.err
