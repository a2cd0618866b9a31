cd $GRAFT_REPO_ROOT
set -x
ncu --set full --import-source on --clock-control none --profile-from-start off -o gpurun_out/k1_r01c python tools/k1_profile.py > gpurun_out/e1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/e2.log 2>&1
BLWS_GRAPHS=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c_c2_call_launches.csv python tools/c2_once.py > gpurun_out/e3.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:"alm_fused|lanczos_rows" -c 30 --csv --log-file gpurun_out/r01c_c3_kernels.csv python tools/solve_configs.py C3 --no-oracle > gpurun_out/e4.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:"csr_spmm|mc_sampled" -c 40 --csv --log-file gpurun_out/r01c_c4_kernels.csv python tools/solve_configs.py C4 > gpurun_out/e5.log 2>&1
ls -la gpurun_out/
