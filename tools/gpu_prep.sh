# c2 launch list (prep breakdown) + per-rank shares
tag=$1
mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c2.csv \
  python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches_rc=$?
python tools/launch_summary.py gpurun_out/${tag}_launches_c2.csv | head -40
timeout 900 python tools/rank_shares.py 2 3 4 5 > gpurun_out/${tag}_shares.log 2>&1; echo shares_rc=$?; cat gpurun_out/${tag}_shares.log | cut -c1-400
