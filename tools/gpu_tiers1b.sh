#!/bin/bash
# the paper's offloading-overhead table for LLaMA3.2-1B on B200
O=gpurun_out/${TAG:-tiers1b}; mkdir -p $O
for w in device host disk; do for kv in device host; do
  timeout 900 python bench.py --config c8 --weight-tier $w --kv-tier $kv --steps 10 --no-cpu-baseline > $O/c8_${w}_${kv}.json 2> $O/e_${w}_${kv}
done; done
