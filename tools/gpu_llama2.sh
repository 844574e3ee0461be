#!/bin/bash
O=gpurun_out/${TAG:-llama2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_llama.py tests/test_gpu_kernels.py -m gpu -q -x > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 900 python bench.py --config c6 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c6.json 2> $O/bench_c6.err
timeout 900 python bench.py --config c6 --steps 5 --warmup 3 --no-cpu-baseline --weight-tier device --no-e2e > $O/bench_c6_dev.json 2> $O/bench_c6_dev.err
ls -la $O
