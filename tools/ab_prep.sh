# A/B of preprocessing variants: step / t_prep on c4, c2 and c3 (edge), interleaved, parity status shown
# usage: bash tools/ab_prep.sh <tag> <variant...>
tag=$1; shift
mkdir -p gpurun_out
run() {  # cfg mode steps variant
  BF_LIB=libbf_$4.so timeout 600 python bench.py --config $1 --mode $2 --steps $3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c$1_$4.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/${tag}_c$1_$4.json').readline())
print('c$1 $4', 'step %.3f prep %.3f count %.3f' % (d['ms_per_step'], d['phases_ms']['t_prep_and_destroy'], d['phases_ms']['t_count']), d['parity']['status'])"
}
for r in 1 2; do for v in "$@"; do run 4 vertex 5 $v; done; done
for r in 1 2; do for v in "$@"; do run 2 vertex 10 $v; done; done
for v in "$@"; do run 3 edge 3 $v; done
