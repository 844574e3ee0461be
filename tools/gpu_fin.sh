#!/bin/bash
O=gpurun_out/${TAG:-fin}; mkdir -p $O
for d in 128 4224 8320 16512 28800; do
echo "== dbg=$d" >> $O/fin.log
PIPO_TM_FIXUP=1 PIPO_WS_DEBUG=$d KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_out 2>&1 | grep -v tm-stamp | head -4 >> $O/fin.log
done
