# launch list of one bench config (1 GPU): bash tools/gpu_launches.sh <tag> <bench args...>
tag=$1; shift
timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > /dev/null 2>&1; echo launches_rc=$?
python tools/launch_summary.py gpurun_out/${tag}_launches.csv | head -30
