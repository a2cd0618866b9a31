#!/bin/bash
# r02i evidence (GPU box, rebuilt from a clean checkout): full GPU suite, smoke,
# bench line, reference arm.
O=gpurun_out
python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; tail -3 $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err; cat $O/bench.json
python bench.py --impl reference --steps 3 --warmup 1 > $O/ref.json 2> $O/ref.err; cat $O/ref.json
