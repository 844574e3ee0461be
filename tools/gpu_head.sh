#!/bin/bash
O=gpurun_out/${TAG:-head}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -m gpu -q -x > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
KBENCH_PATHS=gemm_mma KBENCH_WFMT=0 timeout 300 python tools/kbench.py c5_head c6_head c5_qkv c2_qkv > $O/kbench_fp16.log 2>&1
timeout 600 python bench.py --config c6 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c6_dev.json 2> $O/e6
timeout 900 python bench.py --wfmt fp16 --no-cpu-baseline --no-cupti > $O/c5_fp16.json 2> $O/e5
