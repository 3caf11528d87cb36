# c4 iteration: parity subset, c4 + c2 bench lines, c4 launch list
tag=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "forced or configs_scaled or virtual or random_graphs" > gpurun_out/${tag}_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/${tag}_pytest.log
bash tools/gpu_quick.sh $tag 0 4 2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c4.csv \
  python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches_rc=$?
python tools/launch_summary.py gpurun_out/${tag}_launches_c4.csv | head -14
