#!/bin/bash
# A/B of GEMM tile configurations (libraries in build/ab/): bench value and K1 group time
cd "$GRAFT_REPO_ROOT"
for lib in "$@"; do
  for sk in 1 0; do
    BLWS_LIB_PATH=$PWD/build/ab/$lib BLWS_STREAMK=$sk python bench.py --no-cpu 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib streamk=$sk', round(d['value'],1), 'calls/s; K1', round(1e3*d['roofline']['avg_launch_ms'],1), 'us', round(d['roofline']['achieved'],2), 'TF/s')"
  done
done
