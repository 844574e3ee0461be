#!/bin/bash
O=gpurun_out/${TAG:-red5}; mkdir -p $O
for v in 0 1; do
  echo "== late=$v" >> $O/kbench.log
  PIPO_RED_LATE=$v KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_out c5_fc1 c5_fc2 c3_qkv c6_fc1 c6_fc2 >> $O/kbench.log 2>&1
  PIPO_RED_LATE=$v timeout 300 python tools/ktrace.py c5_out c5_qkv > $O/ktrace_late$v.log 2>&1
done
echo "== late=1 cpt=2" >> $O/kbench.log
PIPO_RED_LATE=1 PIPO_RED_CPT=2 KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_out c5_fc1 c5_fc2 c3_qkv c6_fc1 c6_fc2 >> $O/kbench.log 2>&1
for v in 0 1; do
  echo "== device-tier c5 late=$v" >> $O/kbench.log
  PIPO_RED_LATE=$v timeout 600 python bench.py --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/bench_dev_late$v.json 2> $O/eb$v
done
