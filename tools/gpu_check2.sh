tag=${1:-chk}
timeout 240 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -2 gpurun_out/${tag}_tests.log
for mode in total vertex edge; do
  timeout 100 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --mode $mode > gpurun_out/${tag}_$mode.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/${tag}_$mode.json').readline())
print('$mode kernel_ms %.3f step_ms %.3f' % (d['count_only']['kernel_ms'], d['ms_per_step']))"
done
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/${tag}_launches.csv | head -8
BF_LIB=libbf_prof.so timeout 100 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep "bf_prof" | tail -4
