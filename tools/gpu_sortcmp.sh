# parity tests on the default build, then step breakdowns of sort variants
tag=$1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/${tag}_tests.log
for v in "" os3 os4w1 os16 classic cballot; do
  lib=libbf.so; [ -n "$v" ] && lib=libbf_$v.so
  echo "== $lib"; BF_LIB=$lib timeout 200 python tools/step_breakdown.py 2 2>&1 | tail -2
done
