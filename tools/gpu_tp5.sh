#!/bin/bash
O=gpurun_out/${TAG:-tp5}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "prefill_configs" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
TP_CFGS=0,5,7,8,10,11 timeout 900 python tools/tpbench.py > $O/tpbench.log 2>&1
