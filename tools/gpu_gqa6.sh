#!/bin/bash
O=gpurun_out/${TAG:-gqa6}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_llama.py tests/test_gpu_fullsize.py -m gpu -q -x -k "llama or gqa or c6" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 600 python bench.py --config c6 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c6_dev.json 2> $O/e1
timeout 600 python bench.py --config c6 --no-cpu-baseline > $O/c6.json 2> $O/e2
timeout 600 python bench.py --config c7 --no-cpu-baseline > $O/c7.json 2> $O/e3
timeout 600 python bench.py --config c7 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c7_dev.json 2> $O/e4
timeout 600 python bench.py --config c8 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c8_dev.json 2> $O/e5
