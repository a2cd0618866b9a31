#!/bin/bash
# r02i evidence (GPU box, rebuilt from a clean checkout): full GPU suite, smoke,
# bench line, reference arm.
O=gpurun_out
python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; tail -3 $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err; cat $O/bench.json
python bench.py --impl reference --steps 3 --warmup 1 > $O/ref.json 2> $O/ref.err; cat $O/ref.json
# C2 call launch list (eager), after the same command ran clean without ncu
BLWS_GRAPHS=0 python tools/c2_once.py 2 > $O/c2plain.log 2>&1 && \
  BLWS_GRAPHS=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02i_c2_call.csv python tools/c2_once.py 2 > /dev/null 2>&1
python tools/launches.py $O/r02i_c2_call.csv > $O/r02i_c2_call.txt
python bench.py --mode sharded --steps 3 --warmup 1 > $O/sharded_c5_n1.json 2> $O/sharded.err; cut -c1-300 $O/sharded_c5_n1.json
