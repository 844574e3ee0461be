#!/bin/bash
O=gpurun_out/${TAG:-ncutp}; mkdir -p $O
TP_CFGS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tp_kernel" -s 3 -c 1 \
  -o $O/tp -f python tools/tpbench.py pre_c5_qkv > $O/ncu.out 2>&1
ls -la $O
