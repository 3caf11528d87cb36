for v in "" cap16 sm8 sm24; do
  lib=libbf.so; [ -n "$v" ] && lib=libbf_$v.so
  echo "== $lib"; BF_LIB=$lib timeout 200 python tools/step_breakdown.py 2 2>&1 | tail -1
  for c in 3 4; do
  BF_LIB=$lib timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c$c kernel_ms %.3f' % d['count_only']['kernel_ms'])"
  done
done
