# triage (debug lib) + GPU parity + per-mode kernel times on config 2; every step time-bounded
tag=${1:-chk}
BF_LIB=libbf_debug.so timeout 240 python tools/dbg_triage.py > gpurun_out/${tag}_triage.log 2>&1; echo triage_ok=$(grep -c "^ok" gpurun_out/${tag}_triage.log); grep -v "^ok" gpurun_out/${tag}_triage.log | cut -c1-300 | head -5
timeout 240 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; tail -3 gpurun_out/${tag}_tests.log
timeout 200 bash tools/gpu_modes.sh 2 2>&1 | grep cfg
