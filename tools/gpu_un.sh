#!/bin/bash
O=gpurun_out/${TAG:-un}; mkdir -p $O
timeout 900 python bench.py --config c2 --no-cpu-baseline > $O/c2.json 2> $O/e1
timeout 900 python bench.py --no-cpu-baseline > $O/c5.json 2> $O/e2
timeout 600 python -m pytest tests/test_abi_cpu.py tests/test_gpu_pipeline.py -q -x -m gpu > $O/t.log 2>&1; echo rc=$? >> $O/t.log
