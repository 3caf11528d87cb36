# quick check: GPU tests (optional) + short bench lines for the given configs
# usage: bash tools/gpu_quick.sh <tag> <tests:0|1> <configs...>
tag=$1; tests=$2; shift 2
mkdir -p gpurun_out
if [ "$tests" = "1" ]; then timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/${tag}_pytest.log; fi
for c in "$@"; do
  timeout 400 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_cfg$c.json 2> gpurun_out/${tag}_cfg$c.err
  echo "cfg $c rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/${tag}_cfg$c.json').readline())
c=d['config']; print('  W %.3g m %d kernel_ms %.3f step_ms %.3f mode %s rank %s' % (c['W'], c['m'], d['count_only']['kernel_ms'], d['ms_per_step'], c['mode'], c['ranking']))" 2>&1 | tail -1; tail -2 gpurun_out/${tag}_cfg$c.err
done
if [ -n "$BENCH_FULL" ]; then
  timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench_rc=$?
  tail -c 3000 gpurun_out/${tag}_bench.json
fi
