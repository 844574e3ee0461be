#!/bin/bash
O=gpurun_out/${TAG:-knobs}; mkdir -p $O
for d in 128 129 130 132 133 136 144 150 158; do
  echo "== dbg=$d" >> $O/knobs.log
  PIPO_REDUCE=1 PIPO_WS_DEBUG=$d KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_fc2 2>&1 | grep -E "mma_end|epi_end|c5_" >> $O/knobs.log
done
