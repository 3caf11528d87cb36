# final capture of a round on one B200: GPU tests, default bench line, c2 launch list + ncu --set full,
# c4 / c3 bench lines + c4 launch list, hub twin-position A/B on c5 and c3
tag=${1:-r02f}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/${tag}_gpu_tests.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches_c2_rc=$?
bash tools/ncu_kernel.sh ${tag}_ncu_c2 "k_(big|small)" 3 3 --config 2
ncu -i gpurun_out/${tag}_ncu_c2.ncu-rep --page raw --csv > gpurun_out/${tag}_ncu_c2_raw.csv 2>/dev/null
for c in 4 3; do
  m=vertex; [ $c = 3 ] && m=edge
  timeout 900 python bench.py --config $c --mode $m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_c${c}.json 2> gpurun_out/${tag}_bench_c${c}.err; echo bench_c${c}_rc=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c4.csv \
  python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches_c4_rc=$?
for r in 1 2; do for v in nohub ""; do
  lib=libbf.so; [ -n "$v" ] && lib=libbf_$v.so
  BF_LIB=$lib timeout 600 python bench.py --config 5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ab_c5_${v:-hub}.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/${tag}_ab_c5_${v:-hub}.json').readline())
print('c5 ${v:-hub}', 'step %.3f prep %.3f count %.3f' % (d['ms_per_step'], d['phases_ms']['t_prep_and_destroy'], d['phases_ms']['t_count']))"
done; done
timeout 900 python bench.py --config 5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/${tag}_bench_c5.json 2> gpurun_out/${tag}_bench_c5.err; echo bench_c5_rc=$?
du -sh gpurun_out
