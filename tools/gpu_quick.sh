#!/bin/bash
# quick GPU check: kernel parity tests + isolated tm-kernel timing with/without the in-kernel fixup
O=gpurun_out/${TAG:-quick}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
for f in ${FIXES:-0 1}; do
  echo "== fixup=$f" >> $O/kbench.log
  PIPO_TM_FIXUP=$f KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_out c5_fc1 c5_fc2 c2_qkv c2_fc2 c3_qkv >> $O/kbench.log 2>&1
done
