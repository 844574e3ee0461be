#!/bin/bash
O=gpurun_out/${TAG:-conn}; mkdir -p $O
timeout 900 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-cupti > $O/base.json 2> $O/e0
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 900 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-cupti > $O/conn32.json 2> $O/e1
CUDA_DEVICE_MAX_CONNECTIONS=1 timeout 900 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-cupti > $O/conn1.json 2> $O/e2
timeout 900 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-cupti --no-timeline > $O/notl.json 2> $O/e3
