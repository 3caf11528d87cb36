# round measurement: smoke, all GPU tests, default bench line, launch list, ncu --set full of the wedge kernels
tag=${1:-r01}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/${tag}_gpu_tests.log
bash tools/gpu_measure.sh ${tag}
