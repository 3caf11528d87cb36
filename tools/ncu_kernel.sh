# usage: bash tools/ncu_kernel.sh <tag> <kernel regex> <skip> <count> <bench args...>
# plain run first, then ncu --set full of the matching launches (1 GPU)
tag=$1; re=$2; skip=$3; cnt=$4; shift 4
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${re}" -s $skip -c $cnt -o gpurun_out/${tag} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${tag}_ncu.log 2>&1
echo ncu_rc=$?
