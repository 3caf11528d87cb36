# round-2 baseline on one B200: every config through bench (short), step breakdowns,
# c4 launch list and ncu --set full of c4's wedge kernels
tag=${1:-r02a}
mkdir -p gpurun_out
for c in 2 3 4; do
  timeout 400 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_cfg$c.json 2> gpurun_out/${tag}_cfg$c.err
  echo "cfg $c rc=$?"
done
timeout 300 python tools/step_breakdown.py 4 > gpurun_out/${tag}_steps_c4.txt 2>&1; echo steps_rc=$?
timeout 400 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c4plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c4.csv \
  python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_(big|small|split)" -s 4 -c 4 -o gpurun_out/${tag}_c4full \
  python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c4ncu.log 2>&1; echo ncu_rc=$?
