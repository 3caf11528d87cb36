# every BASELINE config through bench (kernel + step time), short runs, each bounded
for c in 1 2 3 4 5; do
  timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.err
  echo "cfg $c rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/cfg$c.json').readline())
c=d['config']; print('  W %.3g m %d kernel_ms %.3f step_ms %.3f mode %s rank %s' % (c['W'], c['m'], d['count_only']['kernel_ms'], d['ms_per_step'], c['mode'], c['ranking']))" 2>&1 | tail -1; tail -2 gpurun_out/cfg$c.err
done
