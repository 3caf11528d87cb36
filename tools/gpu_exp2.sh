for e in "$@"; do
  BF_EXPERIMENT=$e timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp_l$e.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --mode total > /dev/null 2>&1; echo "== exp $e"; python tools/launch_summary.py gpurun_out/exp_l$e.csv | sed -n 2,4p
done
