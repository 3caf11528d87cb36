# kernel times of libbf_<variant>.so builds (tuning), c2 vertex + total
for v in "$@"; do for mode in vertex total; do
  BF_LIB=libbf_$v.so timeout 100 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --mode $mode 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v $mode kernel_ms %.3f step_ms %.3f' % (d['count_only']['kernel_ms'], d['ms_per_step']))"
done; done
