for e in 0 1 2 3; do
  BF_EXPERIMENT=$e timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/exp_$e.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/exp_$e.json').readline())
print('exp $e kernel_ms %.3f' % d['count_only']['kernel_ms'])"
done
