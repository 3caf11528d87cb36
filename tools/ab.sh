# A/B on one box: bench (kernel + step) for each built variant, interleaved, R rounds
# usage: bash tools/ab.sh <tag> <config> <rounds> <variant...>
tag=$1; cfg=$2; rounds=$3; shift 3
for r in $(seq 1 $rounds); do
  for v in "$@"; do
    BF_LIB=libbf_$v.so timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_$v.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/${tag}_$v.json').readline())
print('$v', 'kernel %.3f step %.3f count %.3f' % (d['count_only']['kernel_ms'], d['ms_per_step'], d['phases_ms']['t_count']))"
  done
done
