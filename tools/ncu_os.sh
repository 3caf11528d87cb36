tag=$1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv python tools/step_breakdown.py 2 > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_rs_(onesweep|hist)" -s 2 -c 3 -o /tmp/${tag} python tools/step_breakdown.py 2 > gpurun_out/${tag}_ncu.log 2>&1; echo rc=$?
python tools/ncu_summary.py /tmp/${tag}.ncu-rep > gpurun_out/${tag}_summary.json 2>&1
ncu -i /tmp/${tag}.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>&1
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_source.csv 2>&1
ls -la gpurun_out | grep $tag
