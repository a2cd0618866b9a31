#!/bin/bash
# Roofline evidence for the r02 profiles (run on the GPU box; each ncu run only
# after the same command ran clean without it). Launch lists with duration,
# DRAM and L2 bytes per kernel; summaries by tools/ncu_metrics_csv.py.
set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
O=gpurun_out
python tools/k1_profile.py > /dev/null 2>&1
ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/r02_k1.csv python tools/k1_profile.py > $O/r02_k1.log 2>&1
ncu --metrics $M --clock-control none -k regex:sytrd_fused -c 2 --csv --log-file $O/r02_k4.csv python tools/c2_once.py 2 > $O/r02_k4.log 2>&1
python tools/solve_configs.py C3 --no-oracle > $O/r02_c3_plain.log 2>&1
ncu --metrics $M --clock-control none -k regex:alm_ -s 40 -c 6 --csv --log-file $O/r02_k7.csv python tools/solve_configs.py C3 --no-oracle > $O/r02_k7.log 2>&1
ncu --metrics $M --clock-control none -k "regex:csr_spmm_k|mc_sampled_k" -s 200 -c 24 --csv --log-file $O/r02_k89.csv python tools/solve_configs.py C4 > $O/r02_k89.log 2>&1
for f in k1 k4 k7 k89; do echo "== $f"; python tools/ncu_metrics_csv.py $O/r02_$f.csv; done
BLWS_GRAPHS=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_c2_call.csv python tools/c2_once.py 2 > /dev/null 2>&1
python tools/launches.py $O/r02_c2_call.csv > $O/r02_c2_call.txt
cat $O/r02_c2_call.txt
