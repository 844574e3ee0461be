#!/bin/bash
O=gpurun_out/${TAG:-gemv}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
KBENCH_PATHS=gemv,tm timeout 300 python tools/kbench.py c7_qkv c7_fc1 c1_fc1 > $O/k.log 2>&1
timeout 900 python bench.py --config c7 --weight-tier device --no-cpu-baseline > $O/c7_dev.json 2> $O/e1
timeout 900 python bench.py --config c7 --no-cpu-baseline > $O/c7.json 2> $O/e2
timeout 900 python bench.py --config c1 --no-cpu-baseline > $O/c1.json 2> $O/e3
