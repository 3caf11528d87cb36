# the round's measurement: default bench line, launch list, ncu --set full of the wedge kernels (1 GPU)
tag=${1:-r01}
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench_rc=$?
tail -c 1500 gpurun_out/${tag}_bench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches_rc=$?
bash tools/ncu_tiers.sh ${tag}_full
