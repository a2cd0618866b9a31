#!/bin/bash
# bench value / e2e / K1 time for alternative library builds in build/ab/ (BLWS_LIB_PATH)
cd "$GRAFT_REPO_ROOT"
for lib in "$@"; do
  for rep in 1 2; do
    BLWS_LIB_PATH=$PWD/build/ab/$lib python bench.py --no-cpu 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), round(d['e2e']['value'],1), 'K1', round(1e3*d['roofline']['avg_launch_ms'],1), round(d['roofline']['frac'],3))"
  done
done
