# usage: bash tools/gpu_quick.sh <tag> [bench args]  -- GPU parity tests then a short bench (1 GPU)
tag=${1:-q}; shift
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo tests_rc=$?; tail -15 gpurun_out/${tag}_gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/${tag}_bench.json').readline())
print('value %.3e ms/step %.3f kernel_ms %.3f frac %.4f e2e %.3e' % (d['value'], d['ms_per_step'], d['count_only']['kernel_ms'], d['roofline']['frac'], d['e2e']['value']))
" ; tail -3 gpurun_out/${tag}_bench.err
