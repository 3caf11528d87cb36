# kernel time of libbf_<variant>.so builds on one config (vertex): gpu_variants_cfg.sh <config> <variants...>
c=$1; shift
for v in "$@"; do
  BF_LIB=libbf_$v.so timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v cfg $c kernel_ms %.3f step_ms %.3f' % (d['count_only']['kernel_ms'], d['ms_per_step']))"
done
