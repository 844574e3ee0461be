#!/bin/bash
O=gpurun_out/${TAG:-gqa7}; mkdir -p $O
PIPO_GQA_TILE=32 timeout 900 python -m pytest tests/test_gpu_llama.py -m gpu -q -x > $O/tests_t32.log 2>&1; echo rc=$? >> $O/tests_t32.log
for t in 64 32; do
  PIPO_GQA_TILE=$t timeout 600 python bench.py --config c6 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c6_dev_t$t.json 2> $O/e6_$t
  PIPO_GQA_TILE=$t timeout 600 python bench.py --config c7 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c7_dev_t$t.json 2> $O/e7_$t
  PIPO_GQA_TILE=$t timeout 600 python bench.py --config c8 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c8_dev_t$t.json 2> $O/e8_$t
done
PIPO_GQA_TILE=32 timeout 600 python bench.py --config c6 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c6_dev_t32b.json 2> $O/e6b
