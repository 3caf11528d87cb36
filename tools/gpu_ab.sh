# parity (GPU parity suite) of each variant build, then interleaved A/B on c2 (2 rounds),
# c4 vertex and c3 edge (1 round each)
# usage: bash tools/gpu_ab.sh <tag> <variant...>
tag=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  BF_LIB=libbf_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${tag}_parity_$v.log 2>&1
  echo "$v parity rc=$? $(tail -1 gpurun_out/${tag}_parity_$v.log)"
done
bash tools/ab.sh ${tag} 2 2 "$@"
bash tools/ab.sh ${tag}c4 4 1 "$@"
for v in "$@"; do
  BF_LIB=libbf_$v.so timeout 600 python bench.py --config 3 --mode edge --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${tag}c3_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/${tag}c3_$v.json').readline())
print('c3 $v', 'kernel %.3f step %.3f count %.3f' % (d['count_only']['kernel_ms'], d['ms_per_step'], d['phases_ms']['t_count']), d['parity']['status'])"
done
