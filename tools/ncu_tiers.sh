tag=$1; shift
timeout 120 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_(big|small)" -s 3 -c 3 -o gpurun_out/${tag} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${tag}_ncu.log 2>&1
echo ncu_rc=$?
