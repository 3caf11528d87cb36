# parity of the working tree's default build, then an A/B of two variant builds on c2 and c4
# usage: bash tools/gpu_ab_check.sh <tag> <varA> <varB>
tag=$1; A=$2; B=$3
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_fullsize.py -x -q -k "exact and (2 or 4)" 2>&1 | tail -2
bash tools/ab.sh ${tag} 2 2 $A $B
bash tools/ab.sh ${tag}c4 4 1 $A $B
timeout 300 python tools/step_breakdown.py 2 2>&1 | tail -3
