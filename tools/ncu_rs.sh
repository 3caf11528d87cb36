tag=$1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_rs_downsweep" -s 10 -c 2 -o /tmp/${tag} python tools/step_breakdown.py 2 > gpurun_out/${tag}_ncu.log 2>&1; echo rc=$?
python tools/ncu_summary.py /tmp/${tag}.ncu-rep > gpurun_out/${tag}_summary.json 2>&1
ncu -i /tmp/${tag}.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>&1
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_source.csv 2>&1
ls -la gpurun_out | grep $tag
