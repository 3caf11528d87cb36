# parity + A/B of two variant builds on c2, c4, c3 (edge), c5
tag=$1; A=$2; B=$3
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
bash tools/ab.sh ${tag} 2 1 $A $B
bash tools/ab.sh ${tag}c4 4 1 $A $B
for v in $A $B; do
  BF_LIB=libbf_$v.so timeout 600 python bench.py --config 3 --mode edge --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${tag}c3_$v.json 2>/dev/null
  BF_LIB=libbf_$v.so timeout 900 python bench.py --config 5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}c5_$v.json 2>/dev/null
  for c in c3 c5; do python -c "
import json; d=json.loads(open('gpurun_out/${tag}${c}_$v.json').readline())
print('$c $v', 'kernel %.3f step %.3f count %.3f' % (d['count_only']['kernel_ms'], d['ms_per_step'], d['phases_ms']['t_count']), d['parity']['status'])"; done
done
