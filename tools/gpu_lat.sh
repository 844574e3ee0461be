#!/bin/bash
# the paper's latency table on B200: LLaMA3.1-8B int4, b=1, host-streamed
O=gpurun_out/${TAG:-lat}; mkdir -p $O
for p in 512 1024 1536 2048; do
  timeout 900 python bench.py --config c7 --prompt $p --steps 10 --no-cpu-baseline > $O/c7_P$p.json 2> $O/e$p
done
