#!/bin/bash
# r02g evidence (GPU box): full GPU suite, bench line, C2 call launch list, the
# C5-scale sharded call and its region split, each ncu run after the same
# command ran clean without it.
O=gpurun_out
python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; tail -3 $O/gputest.log
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --mode sharded --steps 3 --warmup 1 > $O/sharded_c5_n1.json 2> $O/sharded.err
python tools/probes/c5_call_regions.py > $O/c5_call_regions.log 2>&1
BLWS_GRAPHS=0 python tools/c2_once.py 2 > $O/c2plain.log 2>&1 && \
  BLWS_GRAPHS=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02g_c2_call.csv python tools/c2_once.py 2 > /dev/null 2>&1
python tools/launches.py $O/r02g_c2_call.csv > $O/r02g_c2_call.txt
