#!/bin/bash
# Full sweep of every config with the current code + the c5 ncu evidence.
O=gpurun_out/${TAG:-sweep4}; mkdir -p $O
for c in c5 c2 c1 c3 c6 c7; do
  timeout 1200 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 1200 python bench.py --config c3 --kv-fmt int4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3_kv4.json 2> $O/bench_c3_kv4.err
timeout 1500 python bench.py --config c4 --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config c5 --wfmt fp16 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c5_fp16.json 2> $O/bench_c5_fp16.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_c5_reference.json 2> $O/bench_c5_reference.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/ncu_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-cupti --profile \
   > $O/ncu_launches_c5.out 2>&1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:"gemm_tm_kernel|attn_decode|ws_reduce|layernorm" -c 14 -o $O/prof_c5_decode -f \
   python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-cupti --profile > $O/prof_c5.out 2>&1
ls -la $O
