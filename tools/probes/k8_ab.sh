M=gpu__time_duration.sum,lts__t_bytes.sum
python tools/probes/solver_kernels.py C4 > gpurun_out/sk.log 2>&1
for v in base k8u4 k8u16 k8u32; do
  if [ $v = base ]; then unset BLWS_LIB_PATH; else export BLWS_LIB_PATH=$PWD/tools/probes/var_$v/libblws_cuda.so; fi
  ncu --metrics $M --clock-control none -k regex:csr_spmm_k -s 100 -c 6 --csv --log-file gpurun_out/k8_$v.csv python tools/probes/solver_kernels.py C4 > /dev/null 2>&1
  echo "== $v"; python tools/ncu_metrics_csv.py gpurun_out/k8_$v.csv | tail -1
done
