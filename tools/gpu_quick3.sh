# triage + GPU tests + kernel/step times on the given configs
tag=${1:-q}; shift
BF_LIB=libbf_debug.so timeout 330 python tools/dbg_triage.py > gpurun_out/${tag}_triage.log 2>&1; echo triage_ok=$(grep -c "^ok" gpurun_out/${tag}_triage.log) bad=$(grep -vc "^ok" gpurun_out/${tag}_triage.log)
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_cfg$c.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/${tag}_cfg$c.json').readline())
print('cfg $c kernel_ms %.3f step_ms %.3f' % (d['count_only']['kernel_ms'], d['ms_per_step']))"
done
