# fast loop: debug triage (subset), 3-mode kernel times, launch list, phase profile (c2)
tag=${1:-q}
BF_LIB=libbf_debug.so timeout 330 python tools/dbg_triage.py > gpurun_out/${tag}_triage.log 2>&1; echo triage_ok=$(grep -c "^ok" gpurun_out/${tag}_triage.log) bad=$(grep -vc "^ok" gpurun_out/${tag}_triage.log)
for mode in total vertex; do
  timeout 100 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --mode $mode > gpurun_out/${tag}_$mode.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/${tag}_$mode.json').readline())
print('$mode kernel_ms %.3f step_ms %.3f' % (d['count_only']['kernel_ms'], d['ms_per_step']))"
done
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/${tag}_launches.csv | sed -n 2,4p
BF_LIB=libbf_prof.so timeout 100 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep "bf_prof" | tail -3
