#!/bin/bash
O=gpurun_out/${TAG:-c4}; mkdir -p $O
for c in 0 8 4; do
  timeout 1200 python bench.py --config c4 --chunk-mb $c --steps 5 --no-cpu-baseline --no-e2e --no-cupti > $O/c4_chunk$c.json 2> $O/e$c
done
