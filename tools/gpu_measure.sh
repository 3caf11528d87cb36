# the round's measurement on one B200: GPU tests, default bench line, launch lists and
# ncu --set full captures of the wedge kernels (c2 vertex, c4 vertex, c3 edge, c5 vertex),
# bench lines of the other configs, and the debug-build triage
tag=${1:-r02}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/${tag}_gpu_tests.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches_c2_rc=$?
bash tools/ncu_kernel.sh ${tag}_ncu_c2 "k_(big|small)" 3 3 --config 2
for c in 3 4 5; do
  m=vertex; [ $c = 3 ] && m=edge
  timeout 900 python bench.py --config $c --mode $m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_c${c}.json 2> gpurun_out/${tag}_bench_c${c}.err; echo bench_c${c}_rc=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c4.csv \
  python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches_c4_rc=$?
bash tools/ncu_kernel.sh ${tag}_ncu_c4 "k_(big|small|split_walk|split_fin)" 5 5 --config 4
bash tools/ncu_kernel.sh ${tag}_ncu_c3 "k_(big|small)" 3 3 --config 3 --mode edge
bash tools/ncu_kernel.sh ${tag}_ncu_c5 "k_(big|small)" 3 3 --config 5
# keep gpurun_out small (it must come back under 64 MiB): raw-page CSVs of every capture, the
# c2 report itself only
for r in gpurun_out/${tag}_ncu_c*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
  case $r in *_ncu_c2.ncu-rep) ;; *) rm -f $r ;; esac
done
du -sh gpurun_out
BF_LIB=libbf_debug.so timeout 2400 python tools/dbg_triage.py > gpurun_out/${tag}_debug_triage.log 2>&1; echo triage_rc=$?; tail -1 gpurun_out/${tag}_debug_triage.log
