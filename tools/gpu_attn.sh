#!/bin/bash
O=gpurun_out/${TAG:-attnw}; mkdir -p $O
for w in 0 1 2 4 8 16; do
  echo "== waves=$w" >> $O/abench.log
  PIPO_ATTN_WAVES=$w timeout 300 python tools/abench.py >> $O/abench.log 2>&1
done
