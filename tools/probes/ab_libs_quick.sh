#!/bin/bash
# bench value / K1 time for library builds in build/ab/ (BLWS_LIB_PATH), alternating,
# without the cpu / solve legs; extra env per lib as lib:VAR=val
cd "$GRAFT_REPO_ROOT"
for rep in 1 2 3; do
  for spec in "$@"; do
    lib=${spec%%:*}; envs=""; [ "$spec" != "$lib" ] && envs=${spec#*:}
    env $envs BLWS_LIB_PATH=$PWD/build/ab/$lib python bench.py --no-cpu --no-solves 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$spec', round(d['value'],1), 'K1', round(1e3*d['roofline']['avg_launch_ms'],1), round(d['roofline']['frac'],3), 'ms', round(d['ms_per_step'],4))"
  done
done
