#!/bin/bash
O=gpurun_out/${TAG:-red3}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -m gpu -q -x > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_out c5_fc1 c5_fc2 c2_qkv c2_fc2 c3_qkv > $O/kbench.log 2>&1
timeout 900 python bench.py --weight-tier device --no-cpu-baseline --no-e2e > $O/bench_c5_dev.json 2> $O/e1
