#!/bin/bash
# warp-stall breakdown (per issued instruction) of the decode kernels, for the next round
O=gpurun_out/${TAG:-stalls}; mkdir -p $O
M='regex:smsp__average_warps_issue_stalled_.*_per_issue_active\.ratio|smsp__warps_active\.avg\.pct_of_peak_sustained_active|gpu__time_duration\.sum|dram__throughput\.avg\.pct_of_peak_sustained_elapsed'
timeout 900 ncu --profile-from-start off --metrics "$M" --clock-control none --csv -k regex:"attn_decode|gemm_tm" -c 6 \
   --log-file $O/stalls_c6.csv python bench.py --config c6 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-cupti --profile > $O/c6.out 2>&1
timeout 900 ncu --profile-from-start off --metrics "$M" --clock-control none --csv -k regex:"attn_decode|gemm_tm" -c 6 \
   --log-file $O/stalls_c5.csv python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-cupti --profile > $O/c5.out 2>&1
