#!/bin/bash
O=gpurun_out/${TAG:-knobs3}; mkdir -p $O
for d in 159 158 156 157; do
  echo "== dbg=$d" >> $O/knobs.log
  PIPO_REDUCE=1 PIPO_WS_DEBUG=$d KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv >> $O/knobs.log 2>&1
done
for d in 32 62 63; do
  echo "== waits dbg=$d" >> $O/knobs.log
  PIPO_REDUCE=1 PIPO_WS_DEBUG=$d KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv >> $O/knobs.log 2>&1
done
