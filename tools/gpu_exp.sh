for e in "$@"; do
  BF_EXPERIMENT=$e timeout 100 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --mode total > gpurun_out/exp_$e.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/exp_$e.json').readline())
print('exp $e total-mode kernel_ms %.3f' % d['count_only']['kernel_ms'])"
done
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --mode total > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/exp_launches.csv | head -5
