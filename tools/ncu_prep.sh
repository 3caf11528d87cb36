# ncu --set full of the preprocessing kernels of one c2 step (after a plain run exits 0);
# the report is summarised on the box (raw csv) and not brought back (size)
tag=$1; shift
timeout 120 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none \
  -k "regex:k_(pos|hi|validate_degree|slot_keys|wslot|rs_downsweep|rs_upsweep|tile_scan|tile_reduce)" -s 0 -c 40 -o /tmp/${tag} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${tag}_ncu.log 2>&1
echo ncu_rc=$?
python tools/ncu_summary.py /tmp/${tag}.ncu-rep > gpurun_out/${tag}_summary.json 2>&1
ncu -i /tmp/${tag}.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>&1
ls -la gpurun_out/ | tail -5
