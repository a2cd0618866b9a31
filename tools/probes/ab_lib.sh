cd $GRAFT_REPO_ROOT
for i in 1 2; do
for lib in new old; do
  if [ $lib = old ]; then export BLWS_LIB_PATH=$PWD/build/ab/libold.so; else unset BLWS_LIB_PATH; fi
  python bench.py --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), round(d['e2e']['value'],1))"
done; done
for lib in new old; do
  if [ $lib = old ]; then export BLWS_LIB_PATH=$PWD/build/ab/libold.so; else unset BLWS_LIB_PATH; fi
  echo $lib; python tools/probes/solver_regions.py 2>&1 | tail -8
done
