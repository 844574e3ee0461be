#!/bin/bash
O=gpurun_out/${TAG:-chunk}; mkdir -p $O
for c in 0 64 8 2; do
  timeout 900 python bench.py --chunk-mb $c --steps 5 --no-cpu-baseline --no-e2e --no-cupti > $O/bench_c5_chunk$c.json 2> $O/e$c
done
