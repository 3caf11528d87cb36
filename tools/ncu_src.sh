# source-level hot spots of the c2 wedge kernels: ncu --set full with source,
# then the per-line CSV (tools/src_lines.py) of each kernel
# usage: bash tools/ncu_src.sh <tag> [bench args...]
tag=$1; shift
mkdir -p gpurun_out
bash tools/ncu_kernel.sh $tag "k_big|k_small" 0 3 "$@"
for id in 0 1 2; do
  ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source cuda,sass --launch-skip $id --launch-count 1 > gpurun_out/${tag}_src$id.csv 2> gpurun_out/${tag}_src$id.err
  python tools/src_lines.py gpurun_out/${tag}_src$id.csv 45 > gpurun_out/${tag}_lines$id.txt 2>&1
  head -3 gpurun_out/${tag}_lines$id.txt
done
ls -la gpurun_out
