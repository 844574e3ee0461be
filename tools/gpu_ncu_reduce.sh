#!/bin/bash
O=gpurun_out/${TAG:-ncured}; mkdir -p $O
KBENCH_PATHS=tm timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ws_reduce_kernel|gemm_tm_kernel" -s 20 -c 4 \
  -o $O/red -f python tools/kbench.py c5_qkv > $O/ncu.out 2>&1
ls -la $O
