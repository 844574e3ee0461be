#!/bin/bash
O=gpurun_out/${TAG:-gqa4}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_llama.py -m gpu -q -x > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for sp in 0 1 2 3; do
  PIPO_ATTN_V2=2 PIPO_GQA_SPLITS=$sp timeout 600 python bench.py --config c6 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c6_dev_v2_s$sp.json 2> $O/e_$sp
done
PIPO_ATTN_V2=1 timeout 600 python bench.py --config c6 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c6_dev_v1.json 2> $O/e_v1
PIPO_ATTN_V2=2 timeout 600 python bench.py --config c7 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c7_dev_v2.json 2> $O/e_c7v2
timeout 600 python bench.py --config c7 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c7_dev_v0.json 2> $O/e_c7v0
