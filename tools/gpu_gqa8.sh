#!/bin/bash
O=gpurun_out/${TAG:-gqa8}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_llama.py -m gpu -q -x > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for i in 1 2; do
timeout 600 python bench.py --config c6 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c6_dev_$i.json 2> $O/e6_$i
done
