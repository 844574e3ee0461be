#!/bin/bash
# the paper's offloading-overhead table for LLaMA3.1-8B int4 on B200:
# weight location x cache location, b=1, P=512
O=gpurun_out/${TAG:-tiers}; mkdir -p $O
for w in device host disk; do for kv in device host; do
  timeout 900 python bench.py --config c7 --weight-tier $w --kv-tier $kv --steps 10 --no-cpu-baseline > $O/c7_${w}_${kv}.json 2> $O/e_${w}_${kv}
done; done
