# A/B of library builds on config 4 (BatchPlan.fill wall / event microseconds)
for i in 1 2; do
  for lib in "$@"; do
    echo -n "$lib "; ZF_LIB=$lib python tools/bench_configs.py c4 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('wall %.1f us  event %.1f us' % (d['batched_seconds']*1e6, d['batched_event_seconds']*1e6))"
  done
done
