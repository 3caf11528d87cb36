# ncu --set full (with source) of the 64-bit slot-sort passes of one c2 step:
# the 8 k_rs_downsweep<u64> launches (U half 5, V half 3) and their upsweeps
tag=$1; shift
timeout 120 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_rs_(down|up)sweep<unsigned long" -s 0 -c 16 \
  -o gpurun_out/${tag} python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${tag}_ncu.log 2>&1
echo ncu_rc=$?
