# K9 row-blocked vs flat: C4 solve time (plain runs), then launch metrics of both kernels (ncu)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
O=gpurun_out
for v in seg flat seg; do
  if [ $v = flat ]; then export BLWS_K9=flat; else unset BLWS_K9; fi
  echo "== $v"; python tools/solve_configs.py C4 --no-oracle 2>&1 | tail -1
done > $O/k9_ab.log
python tools/probes/solver_kernels.py C4 > $O/k9_plain.log 2>&1 &&
ncu --metrics $M --clock-control none -k "regex:mc_sampled|csr_spmm_k|seg_build" -s 200 -c 12 --csv --log-file $O/k9_seg.csv python tools/probes/solver_kernels.py C4 > $O/k9_ncu.log 2>&1
BLWS_K9=flat ncu --metrics $M --clock-control none -k "regex:mc_sampled" -s 20 -c 3 --csv --log-file $O/k9_flat.csv python tools/probes/solver_kernels.py C4 > $O/k9_ncu2.log 2>&1
python tools/ncu_metrics_csv.py $O/k9_seg.csv >> $O/k9_ab.log
python tools/ncu_metrics_csv.py $O/k9_flat.csv >> $O/k9_ab.log
