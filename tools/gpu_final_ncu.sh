#!/bin/bash
O=gpurun_out/${TAG:-fncu}; mkdir -p $O
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:"gemm_tm_kernel|attn_decode|ws_reduce|layernorm|attn_merge" -c 14 -o $O/prof_c5_decode -f \
   python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-cupti --profile > $O/prof_c5.out 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/ncu_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-cupti --profile \
   > $O/ncu_launches_c5.out 2>&1
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
