#!/bin/bash
O=gpurun_out/${TAG:-stamps}; mkdir -p $O
for f in 0 1; do for d in 128; do
  echo "== fixup=$f dbg=$d" >> $O/stamps.log
  PIPO_TM_FIXUP=$f PIPO_WS_DEBUG=$d KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_fc2 >> $O/stamps.log 2>&1
done; done
