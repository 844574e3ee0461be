# ncu launch list of the default bench command, skipping the weight-generation launches
O=gpurun_out/final_r2b; mkdir -p $O
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 600 -c 1500 --csv --log-file $O/ncu_launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-cupti --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu-launch rc=$?"
