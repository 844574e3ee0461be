#!/bin/bash
O=gpurun_out/${TAG:-pipe}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "tm_configs or linear_vs_oracle" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for c in 0 6 0 6; do
  echo "== cfg=$c" >> $O/kbench.log
  PIPO_TM_CFG=$c KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_out c5_fc1 c5_fc2 c3_qkv >> $O/kbench.log 2>&1
done
echo "== cfg=6 stamps" >> $O/kbench.log
PIPO_TM_CFG=6 PIPO_REDUCE=1 PIPO_WS_DEBUG=128 KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv 2>&1 | grep -E "mma_end|c5_" >> $O/kbench.log
