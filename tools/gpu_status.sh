# DESIGN.md 8b table: every config (default mode) + c2/c3 modes, bounded
bash tools/gpu_configs.sh
for mode in total edge; do
  for c in 2 3; do
    timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --mode $mode > gpurun_out/st_${c}_${mode}.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/st_${c}_${mode}.json').readline())
print('cfg $c $mode kernel_ms %.3f step_ms %.3f' % (d['count_only']['kernel_ms'], d['ms_per_step']))"
  done
done
