#!/bin/bash
# ncu --set full of one LLaMA decode layer (c6 b=64, c7 b=1) + launch lists, summarised on
# the box (the .ncu-rep files exceed gpurun's copy-back limit), for roofline.traffic
O=gpurun_out/${TAG:-ncul}; mkdir -p $O; R=/tmp/ncul; mkdir -p $R
for c in c6 c7; do
  timeout 1200 ncu --profile-from-start off --set full --clock-control none \
     -k regex:"gemm_tm_kernel|gemv_int4|attn_decode|ws_reduce|layernorm|rope|swiglu|attn_merge" -c 16 -o $R/prof_${c}_decode -f \
     python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-cupti --profile > $O/prof_$c.out 2>&1
  python tools/ncu_summary.py full $R/prof_${c}_decode.ncu-rep > $O/ncu_full_summary_$c.json 2> $O/sum_$c.err
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file $R/ncu_launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-cupti --profile \
     > $O/ncu_launches_$c.out 2>&1
  python tools/ncu_summary.py launches $R/ncu_launches_$c.csv > $O/ncu_launches_summary_$c.json 2>> $O/sum_$c.err
done
ls -la $R >> $O/files.txt
