#!/bin/bash
O=gpurun_out/${TAG:-gqa}; mkdir -p $O
for w in -1 1 2 4 8; do
  PIPO_ATTN_WAVES=$w timeout 900 python bench.py --config c6 --weight-tier device --steps 5 --no-cpu-baseline --no-e2e --no-cupti > $O/c6_w$w.json 2> $O/e$w
done
