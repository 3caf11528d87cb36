# usage: bash tools/ncu_full.sh <tag> <bench args...>   (1 GPU; plain run first, then ncu on the wedge kernel)
tag=$1; shift
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_count -s 1 -c 1 -o gpurun_out/${tag} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${tag}_ncu.log 2>&1
echo ncu_rc=$?
