#!/bin/bash
O=gpurun_out/${TAG:-tp4}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -m gpu -q -x -k "prefill" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
TP_CFGS=0,5 timeout 900 python tools/tpbench.py > $O/tpbench.log 2>&1
