#!/bin/bash
O=gpurun_out/${TAG:-red4}; mkdir -p $O
for v in 1 2 4; do
  echo "== cpt=$v" >> $O/kbench.log
  PIPO_RED_CPT=$v KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_out c5_fc1 c5_fc2 c2_qkv c3_qkv c6_qkv c6_fc1 c6_fc2 >> $O/kbench.log 2>&1
done
echo "== main kernel only (dbg 64)" >> $O/kbench.log
PIPO_WS_DEBUG=64 KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_out c5_fc1 c5_fc2 c2_qkv c3_qkv >> $O/kbench.log 2>&1
for v in 2 4; do
  PIPO_RED_CPT=$v timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "tm_fixup or tm_configs" > $O/tests_cpt$v.log 2>&1; echo rc=$? >> $O/tests_cpt$v.log
done
