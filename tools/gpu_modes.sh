# kernel time per mode / orientation on config $1 (default 2)
cfg=${1:-2}
for mode in total vertex edge; do for orient in high low; do
  timeout 120 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --mode $mode --orient $orient > gpurun_out/modes_${cfg}_${mode}_${orient}.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/modes_${cfg}_${mode}_${orient}.json').readline())
print('cfg $cfg $mode $orient kernel_ms %.3f step_ms %.3f W %d' % (d['count_only']['kernel_ms'], d['ms_per_step'], d['config']['W']))"
done; done
