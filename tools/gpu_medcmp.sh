for v in "" wur3 wur1 wp32 mur1; do
  lib=libbf.so; [ -n "$v" ] && lib=libbf_$v.so
  echo "== $lib"; BF_LIB=$lib timeout 200 python tools/step_breakdown.py 2 2>&1 | tail -1
  BF_LIB=$lib timeout 300 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c3 kernel_ms %.3f' % d['count_only']['kernel_ms'])"
done
