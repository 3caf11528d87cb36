# parity of the hub twin-position path, then its effect on the c4 / c3 / c2 steps
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hub_pos or forced_paths or random_graphs" > gpurun_out/hub_parity.log 2>&1; echo parity_rc=$?; tail -3 gpurun_out/hub_parity.log
BF_LIB=libbf_debug.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hub_pos" > gpurun_out/hub_parity_debug.log 2>&1; echo parity_debug_rc=$?; tail -3 gpurun_out/hub_parity_debug.log
run() {
  timeout 600 python bench.py --config $1 --mode $2 --steps $3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/hub_c$1.json 2>gpurun_out/hub_c$1.err
  python -c "
import json; d=json.loads(open('gpurun_out/hub_c$1.json').readline())
print('c$1', 'step %.3f prep %.3f count %.3f' % (d['ms_per_step'], d['phases_ms']['t_prep_and_destroy'], d['phases_ms']['t_count']), d['parity']['status'])"
}
run 4 vertex 5; run 4 vertex 5; run 3 edge 3; run 2 vertex 10; run 2 vertex 10; run 5 vertex 2
