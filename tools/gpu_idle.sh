#!/bin/bash
O=gpurun_out/${TAG:-idle}; mkdir -p $O
for idle in 0 100 1000 5000; do
  echo "== idle_us=$idle" >> $O/idle.log
  PIPO_BENCH_IDLE_US=$idle KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_fc2 >> $O/idle.log 2>&1
done
