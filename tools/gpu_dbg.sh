tag=${1:-dbg}
mkdir -p gpurun_out
BF_LIB=libbf_debug.so timeout 300 python tools/dbg_k4033.py > gpurun_out/${tag}_dbg.log 2>&1; echo dbg_rc=$?; head -30 gpurun_out/${tag}_dbg.log
BF_LIB=libbf_debug.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo tests_rc=$?; grep -E "BF_CHECK|passed|failed|FAILED" gpurun_out/${tag}_gpu_tests.log | head -20
