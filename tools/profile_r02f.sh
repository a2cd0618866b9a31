#!/bin/bash
# r02f evidence (GPU box): full GPU suite, bench line, C2 call launch list, K7
# ncu capture (C3), each ncu run after the same command ran clean without it.
O=gpurun_out
python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; tail -3 $O/gputest.log
python bench.py > $O/bench.json 2> $O/bench.err
BLWS_GRAPHS=0 python tools/c2_once.py 2 > $O/c2plain.log 2>&1 && \
  BLWS_GRAPHS=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02f_c2_call.csv python tools/c2_once.py 2 > /dev/null 2>&1
python tools/launches.py $O/r02f_c2_call.csv > $O/r02f_c2_call.txt
python tools/k7_micro.py C3 > $O/k7plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:alm_tma_k -s 2 -c 1 -o $O/r02f_k7_c3 python tools/k7_micro.py C3 > $O/k7ncu.log 2>&1
