#!/bin/bash
O=gpurun_out/${TAG:-knobs2}; mkdir -p $O
for cfg in 0 1 3; do for d in 128 158; do
  echo "== cfg=$cfg dbg=$d" >> $O/knobs.log
  PIPO_TM_CFG=$cfg PIPO_REDUCE=1 PIPO_WS_DEBUG=$d KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_fc2 2>&1 | grep -E "mma_end|c5_" >> $O/knobs.log
done; done
for cfg in 0 1; do
  echo "== waits cfg=$cfg" >> $O/knobs.log
  PIPO_TM_CFG=$cfg PIPO_REDUCE=1 PIPO_WS_DEBUG=32 KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv 2>&1 >> $O/knobs.log
done
